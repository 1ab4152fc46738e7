timeout 900 python bench.py > gpurun_out/bench10.log 2>&1; echo bench rc $?
tail -1 gpurun_out/bench10.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['e2e'],d['serving_step'],d['encode'],d['cpu_baseline'])"
timeout 1200 python bench.py --config c4 --no-cpu-baseline --no-extras --steps 5 --warmup 3 > gpurun_out/bench10_c4.log 2>&1; echo c4 rc $?
tail -1 gpurun_out/bench10_c4.log | cut -c1-400
