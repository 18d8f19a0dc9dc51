# Level kernels' occupancy: PO_LEVEL_MINB=argmax,aggregate,leaf_stats.
for cfg in "2 1000000 6" "3 10000000 4" "4 20000000 3"; do
  for v in 1,1,1 6,4,4 8,6,6 4,8,8; do
    out=$(PO_LEVEL_MINB=$v timeout 60 python tools/time_calls.py $cfg 60 2>&1 | tail -2)
    echo "== C$cfg minb=$v: $(echo "$out" | grep -oE 'call [0-9]+: [0-9.]+ ms') $(echo "$out" | sed 's| [|] |\n|g' | grep -E 'k_argmax |k_aggregate|k_leaf_stats' | sed 's/.*top: //' | tr '\n' ' ')"
  done
done
