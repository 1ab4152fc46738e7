# A/B of decode library builds on the C2 bench: bash scripts/ab_decode.sh LIB_A LIB_B [reps] [extra bench args]
A=$1; B=$2; N=${3:-2}; shift 3 2>/dev/null
for i in $(seq $N); do
  for L in $A $B; do
    echo -n "$(basename $L) "
    NSNKV_LIB=$L timeout 60 python bench.py --no-cpu-baseline --no-extras --steps 30 "$@" 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*' | head -1
  done
done
