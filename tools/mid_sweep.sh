# k_hash_probe / k_verify_cells vs PO_MID_CELL (8-lane groups for cells of
# [mid, 1024) bytes; 1024 = off).
for cfg in "2 1000000 4" "3 10000000 3" "4 20000000 3" "5 3000000 3"; do
  for v in 1024 256 128 64 32 0; do
    echo "== C$cfg mid=$v: $(PO_MID_CELL=$v timeout 60 python tools/time_calls.py $cfg 40 2>&1 | tail -2 | tr '\n' ' ' | grep -oE 'call [0-9]+: [0-9.]+ ms|(k_hash_probe|k_verify_cells)[^,]*' | tr '\n' ' ')"
  done
done
