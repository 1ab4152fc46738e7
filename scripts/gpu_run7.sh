timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode_full.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
tail -4 gpurun_out/gpu_tests.log
