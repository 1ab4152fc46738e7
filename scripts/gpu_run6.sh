timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode_full.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
tail -4 gpurun_out/gpu_tests.log
for cfg in c2 c2_1b; do
for ff in "" "--fast-fp16"; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --config $cfg $ff > gpurun_out/b.log 2>&1; echo bench rc $?
python -c "import json;d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]);print('$cfg $ff',d['value'],d['ms_per_step'],d['roofline']['frac'])"
done; done
ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 3 -c 1 -o gpurun_out/prof_attend4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof4.log 2>&1; echo rc $?
