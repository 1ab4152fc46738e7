timeout 900 python scripts/bench_model.py --kv bf16 --batch 32 > gpurun_out/m_bf16_32.log 2>&1; echo rc $?; tail -3 gpurun_out/m_bf16_32.log
timeout 900 python scripts/bench_model.py --kv nsn1b --batch 32 > gpurun_out/m_1b_32.log 2>&1; echo rc $?; tail -3 gpurun_out/m_1b_32.log
timeout 900 python scripts/bench_model.py --kv bf16 --batch 64 > gpurun_out/m_bf16_64.log 2>&1; echo rc $?; tail -3 gpurun_out/m_bf16_64.log
timeout 1500 python scripts/bench_model.py --kv nsn1b --batch 256 > gpurun_out/m_1b_256.log 2>&1; echo rc $?; tail -3 gpurun_out/m_1b_256.log
