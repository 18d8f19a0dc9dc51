# warp-cooperative hashing / verification threshold (PO_LONG_CELL bytes) on C2 and a C5 prefix
for L in 1000000000 1024 512 256; do
  echo "long_min $L"
  PO_LONG_CELL=$L python tools/time_calls.py 2 1000000 4 4 2>&1 | tail -1
  PO_LONG_CELL=$L python tools/time_calls.py 5 3000000 3 4 2>&1 | tail -1
done
