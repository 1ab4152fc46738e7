timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/b.log 2>&1; echo bench rc $?
python -c "import json;d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]);print('c2',d['value'],d['ms_per_step'],d['roofline'])"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attend_kernel|combine_kernel" -c 4 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo launches rc $?
