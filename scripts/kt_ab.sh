# A/B per-kernel times: bash scripts/kt_ab.sh LIB_A LIB_B (paths relative to the repo root); CASES overrides
# the default configs (one "B H N d alpha causal [gen rho]" per line)
CASES=${CASES:-"4 12 8192 64 1.5 0
8 12 1024 64 1.5 1
1 16 32768 128 1.5 1"}
for L in "$@"; do
  echo LIB=$L
  while read -r a; do
    [ -n "$a" ] && ENTMAX_ATTN_LIB=$PWD/$L python scripts/kernel_times.py $a
  done <<< "$CASES"
done
