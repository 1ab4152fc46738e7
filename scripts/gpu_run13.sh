timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_racecheck.log 2>&1; echo racecheck rc $?
tail -2 gpurun_out/sanitize_racecheck.log
timeout 600 python -m pytest tests/ -x -q -m gpu > gpurun_out/gpu_all.log 2>&1; echo gpu tests rc $?
tail -2 gpurun_out/gpu_all.log
