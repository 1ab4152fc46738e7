timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc $?; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode_full.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
tail -3 gpurun_out/gpu_tests.log
timeout 600 python scripts/bench_encode.py > gpurun_out/enc2.log 2>&1; echo enc rc $?
cat gpurun_out/enc2.log | tail -3
ncu --set full --clock-control none --import-source on -k regex:encode_chunks -s 2 -c 1 -o gpurun_out/prof_enc2 python scripts/bench_encode.py --batch 8 --steps 1 --modes 2 > /dev/null 2>&1; echo ncu rc $?
