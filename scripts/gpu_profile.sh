# ncu evidence for the default bench command (profiles/), decode kernel v3:
#  1. per-launch device times of every launch of the bench command (all kernels)
#  2. one --set full capture of the dominant kernel (attend3_kernel), fast and precise
#  3. DRAM bytes per launch of the decode launches (traffic vs algorithmic)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo launches rc $?
for p in fast precise; do
ncu --set full --clock-control none --import-source on -k regex:attend3_kernel -s 3 -c 1 -o gpurun_out/prof_v3_final_$p python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras --precision $p > /dev/null 2>&1; echo full $p rc $?
done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"attend3|combine" -s 6 -c 4 --csv --log-file gpurun_out/traffic_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo traffic rc $?
