timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode_full.py tests/test_gpu_cache_semantics.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
tail -2 gpurun_out/gpu_tests.log
for cfg in c2 c2_1b; do
for pr in precise fast; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras --config $cfg --precision $pr > gpurun_out/b.log 2>&1; echo bench rc $?
python -c "import json;d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]);print('$cfg $pr',d['value'],d['ms_per_step'],d['roofline']['frac'])"
done; done
