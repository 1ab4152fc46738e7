# ncu --set full of the decode kernel on the C2 bench workload; exports the
# raw metrics and the SASS source page (per-instruction counts, wavefronts,
# stall samples) as CSV.  usage: bash scripts/prof_decode.sh TAG KERNEL(v3|v4) PRECISION [CONFIG]
tag=$1; kern=$2; prec=$3; cfg=${4:-c2}
rx=$([ "$kern" = v3 ] && echo attend3_kernel || echo attend4_kernel)
NSNKV_DECODE_KERNEL=$kern timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:$rx -s 3 -c 1 -o gpurun_out/prof_$tag -f \
  python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-extras --precision $prec > /dev/null 2>&1
echo "ncu rc $?"
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv
ncu -i gpurun_out/prof_$tag.ncu-rep --page details --csv > gpurun_out/prof_${tag}_details.csv
ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${tag}_src.csv
rm -f gpurun_out/prof_$tag.ncu-rep
