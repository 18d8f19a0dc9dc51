# Tile shape of the radix pass below 3M keys (PO_RADIX_SMALL) on C2 and a
# C3 1.5M-row prefix: median wall ms of 15 ggr() calls, then the radix
# scope of a profiled call.
for shape in 256x20 256x12 256x8 256x4 512x8; do
  for cfg in "2 1000000" "3 1500000"; do
    echo "== $shape C$cfg"
    PO_RADIX_SMALL=$shape python tools/time_calls.py $cfg 18 | tail -15 | \
      awk '{print $3}' | sort -n | awk '{a[NR]=$1} END {print "median ms", a[int((NR+1)/2)]}'
    PO_RADIX_SMALL=$shape python tools/time_calls.py $cfg 3 30 | grep -o "k_radix_pass [0-9]*x [0-9.]*\|scope:radix_sort [0-9]*x [0-9.]*" | tail -2
  done
done
