set -x
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc $?
tail -4 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode_full.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
tail -30 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench2.log 2>&1; echo bench rc $?
tail -3 gpurun_out/bench2.log
