# String-rank merge sort (cub) vs the radix refinement rounds (PO_MERGE_RANK=0).
for cfg in "2 1000000 6" "3 10000000 4" "5 3000000 3"; do
  for v in PO_MERGE_RANK=1 PO_MERGE_RANK=0; do
    echo "== C$cfg $v: $(env $v timeout 200 python tools/time_calls.py $cfg 2>&1 | tail -1)"
    echo "   $(env $v timeout 200 python tools/time_calls.py $cfg 12 2>&1 | tail -1)"
  done
done
