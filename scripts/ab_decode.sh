# A/B of decode kernels / precisions on the C2 (2-bit and 1-bit) bench workloads.
# usage (on the GPU box): bash scripts/ab_decode.sh [steps]
steps=${1:-50}
for kern in ${KERNELS:-v3}; do
  for cfg in "c2 vfast" "c2 precise" "c2_1b precise"; do
    set -- $cfg
    r=$(NSNKV_DECODE_KERNEL=$kern python bench.py --config $1 --precision $2 --steps $steps --warmup 5 \
        --no-cpu-baseline --no-extras 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['roofline']['kernel_ms'], r['roofline']['frac'])")
    echo "$kern $1 $2 kernel_ms/frac: $r"
  done
done
