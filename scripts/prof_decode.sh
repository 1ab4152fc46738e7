# ncu --set full of the decode kernel on a bench workload; exports the raw
# metrics and the SASS source page (per-instruction counts, wavefronts, stall
# samples) as CSV.  usage: bash scripts/prof_decode.sh TAG PRECISION [CONFIG]
tag=$1; prec=$2; cfg=${3:-c2}
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:attend3_kernel -s 3 -c 1 -o gpurun_out/prof_$tag -f \
  python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-extras --precision $prec > /dev/null 2>&1
echo "ncu rc $?"
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv
ncu -i gpurun_out/prof_$tag.ncu-rep --page details --csv > gpurun_out/prof_${tag}_details.csv
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_src.csv
rm -f gpurun_out/prof_$tag.ncu-rep
