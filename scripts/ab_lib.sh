# A/B a decode experiment library against the product library on the C2
# workloads (kernel ms from bench.py CUDA events).
# usage (GPU box): bash scripts/ab_lib.sh paper_2505_18231_b200/libexp_X.so [steps]
exp=$1; steps=${2:-50}
for cfg in "c2" "c2_1b"; do
  for lib in "" "$exp"; do
    r=$(env ${lib:+NSNKV_LIB=$lib} python bench.py --config $cfg --steps $steps --warmup 5 --no-cpu-baseline --no-extras 2>/dev/null \
        | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['roofline']['kernel_ms'], r['roofline']['frac'])")
    echo "$cfg ${lib:-product} kernel_ms/frac: $r"
  done
done
