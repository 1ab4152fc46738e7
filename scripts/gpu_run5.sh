timeout 600 python scripts/bench_encode.py > gpurun_out/enc1.log 2>&1; echo enc rc $?
cat gpurun_out/enc1.log | tail -3
ncu --set full --clock-control none --import-source on -k regex:encode_chunks -s 2 -c 1 -o gpurun_out/prof_enc1 python scripts/bench_encode.py --batch 8 --steps 1 --modes 2 > /dev/null 2>&1; echo ncu rc $?
ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo rc $?
timeout 900 python bench.py > gpurun_out/bench5.log 2>&1; echo bench rc $?
tail -1 gpurun_out/bench5.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench5_ref.log 2>&1; echo ref rc $?
tail -1 gpurun_out/bench5_ref.log
nproc; lscpu | grep "Model name"
