# v2 decode: parity tests, then one ncu --set full capture per precision mode
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v2.txt 2>&1; echo tests rc $?
tail -2 gpurun_out/pytest_v2.txt
for p in fast precise; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:attend2_kernel -s 3 -c 1 -o gpurun_out/prof_v2_$p python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --precision $p > /dev/null 2>&1; echo ncu $p rc $?
done
