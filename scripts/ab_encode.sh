# A/B of encode library builds on C3: bash scripts/ab_encode.sh LIB...
for L in "$@"; do
  echo -n "$(basename $L) "
  NSNKV_LIB=$L timeout 200 python scripts/bench_encode.py 2>&1 | tail -2 | grep -o '"bit_mode": [12]\|"ms": [0-9.]*' | tr '\n' ' '
  echo
done
