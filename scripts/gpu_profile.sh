# ncu evidence for the default bench command (profiles/):
#  1. per-launch device times of the decode launches (attend + combine)
#  2. one --set full capture of the dominant kernel (attend_kernel)
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attend_kernel|combine_kernel" -c 20 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo launches rc $?
ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 3 -c 1 -o gpurun_out/prof_attend_final python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo full rc $?
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"attend_kernel|combine_kernel" -s 6 -c 2 --csv --log-file gpurun_out/traffic_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1; echo traffic rc $?
