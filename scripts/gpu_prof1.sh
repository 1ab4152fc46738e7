ncu --set full --clock-control none --import-source on -k regex:attend_kernel -s 3 -c 1 -o gpurun_out/prof_attend1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof1.log 2>&1; echo rc $?
ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/launches1.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo rc $?
tail -5 gpurun_out/prof1.log
