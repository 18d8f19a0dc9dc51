# e2e A/B on one box: bench.py twice per setting, alternating.
for i in 1 2; do
  for v in PO_EARLY_FALLBACK=1 PO_EARLY_FALLBACK=0 PO_MSORT=cub; do
    env $v timeout 600 python bench.py --steps 20 --no-cpu > gpurun_out/ab.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$v', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3))"
  done
done
