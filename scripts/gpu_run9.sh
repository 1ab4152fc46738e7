timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode_full.py -x -q -m gpu -s > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
grep -E "worst|passed|failed|Error" gpurun_out/gpu_tests.log | tail -14
for cfg in c2 c2_1b; do
for pr in precise fast; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config $cfg --precision $pr > gpurun_out/b.log 2>&1; echo bench rc $?
python -c "import json;d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]);print('ws $cfg $pr',d['value'],d['ms_per_step'],d['roofline']['frac'])"
NSNKV_DECODE_KERNEL=grouped timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config $cfg --precision $pr > gpurun_out/b.log 2>&1; echo bench rc $?
python -c "import json;d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]);print('grouped $cfg $pr',d['value'],d['ms_per_step'],d['roofline']['frac'])"
done; done
ncu --set full --clock-control none --import-source on -k regex:attend_ws -s 3 -c 1 -o gpurun_out/prof_ws1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/profws.log 2>&1; echo rc $?
