# k_hash_probe vs PO_PROBE_SHAPE (0: (min blocks 1, 4 words/step), 1: (5,4),
# 2: (6,4), 3: (4,8), 4: (5,8), 5: (6,8)) and k_verify_cells vs
# PO_VERIFY_MINB (0: 1, 1: 4, 2: 5, 3: 6, 4: 8), swept together (index i).
for cfg in "2 1000000 4" "3 10000000 3" "4 20000000 3" "5 3000000 3"; do
  for v in 0 1 2 3 4 5; do
    out=$(PO_PROBE_SHAPE=$v PO_VERIFY_MINB=$v timeout 60 python tools/time_calls.py $cfg 40 2>&1 | tail -2)
    echo "== C$cfg shape=$v: $(echo "$out" | grep -oE 'call [0-9]+: [0-9.]+ ms') $(echo "$out" | sed 's| [|] |\n|g' | grep -E 'hash_probe|verify_cells' | sed 's/.*(k_/k_/; s/<[0-9, ]*>)//' | tr '\n' ' ')"
  done
done
