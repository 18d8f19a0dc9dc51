# Hand-written radix vs CUB on C2/C3/C4-20M (profile scopes), then the ncu
# launch list of one C3 call each (kernel durations without launch gaps).
timeout 300 python -m pytest tests/test_gpu_radix.py -x -q 2>&1 | tail -1
for cfg in "2 1000000 6" "3 10000000 4" "4 20000000 3"; do
  for v in ${RADIX_VARIANTS:-PO_RADIX_TILE=256x20 PO_RADIX_TILE=384x12 PO_RADIX=cub}; do
    echo "== C$cfg $v: $(env $v timeout 200 python tools/time_calls.py $cfg 60 2>&1 | tail -2 | tr '\n' ' ' | grep -oE 'call [0-9]+: [0-9.]+ ms|(radix_sort|cub_radix_sort|k_radix_pass|k_radix_hist)[^,]*' | tr '\n' ' ')"
  done
done
if [ -n "$RADIX_NCU" ]; then
  for v in PO_RADIX=hand PO_RADIX=cub; do
    env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/radix_ncu_${v#PO_RADIX=}.csv python tools/time_calls.py 3 10000000 2 > /dev/null 2>&1
    python tools/ncu_sum.py gpurun_out/radix_ncu_${v#PO_RADIX=}.csv radix RadixSort
  done
fi
