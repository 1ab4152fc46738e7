# ncu --set full of the v3 decode kernel (fast, precise) on the C2 bench workload
for p in fast precise; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:attend3_kernel -s 3 -c 1 -o gpurun_out/prof_v3_$p python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --precision $p > /dev/null 2>&1; echo ncu $p rc $?
done
