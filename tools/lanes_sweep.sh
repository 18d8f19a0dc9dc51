# dictionary kernel experiments on C2 and a C5 prefix: split (default) vs fused
for K in split fused; do
  echo "kernel $K"
  PO_DICT_KERNEL=$K python tools/time_calls.py 2 1000000 4 6 2>&1 | tail -1
  PO_DICT_KERNEL=$K python tools/time_calls.py 5 1000000 3 6 2>&1 | tail -1
done
