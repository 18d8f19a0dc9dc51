# Hand-written stable merge sort (csrc/msort.cuh) vs cub::DeviceMergeSort
# (PO_MSORT=cub) on the small-job string sorts.
for cfg in "2 1000000 6" "3 10000000 4" "5 3000000 3"; do
  for v in PO_MSORT=hand PO_MSORT=cub; do
    out=$(env $v timeout 60 python tools/time_calls.py $cfg 60 2>&1 | tail -2)
    echo "== C$cfg $v: $(echo "$out" | grep -oE 'call [0-9]+: [0-9.]+ ms') $(echo "$out" | sed 's| [|] |\n|g' | grep -E 'merge_sort|msort' | sed 's/.*top: //' | tr '\n' ' ')"
  done
done
