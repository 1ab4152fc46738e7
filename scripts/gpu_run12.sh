timeout 600 python -m pytest tests/test_gpu_cache_semantics.py -x -q -m gpu > gpurun_out/gpu_sem.log 2>&1; echo sem rc $?
tail -5 gpurun_out/gpu_sem.log
for tool in memcheck racecheck synccheck; do
timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1; echo $tool rc $?
tail -4 gpurun_out/sanitize_$tool.log
done
