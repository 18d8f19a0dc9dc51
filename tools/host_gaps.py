"""Device idle gaps inside one ggr() call, charged to the launch that ends
each gap (profile mode: events around every launch): python
tools/host_gaps.py <cfg> <rows> [reps] [top]."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE, cuda_lib

cfg_id, rows = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
t = gen.generate(cfg_id, n_rows=rows)
n, m = t.row_count(), t.field_count()
fd = [[t.require_field(x) for x in g] for g in gen.fds(cfg_id)]
dv = t.view(PO_LOC_DEVICE, arena=torch.from_numpy(t.arena).cuda(),
            offsets=torch.from_numpy(t.offsets.view(np.int64)).cuda())
r_ = torch.empty(n, dtype=torch.int64, device="cuda")
o_ = torch.empty(n * m, dtype=torch.int32, device="cuda")
lib = cuda_lib()
walls = []
for i in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    po.ggr_into(dv, fd, po.GgrConfig(), 0, 0, PO_LOC_DEVICE, r_, o_, 0)
    torch.cuda.synchronize()
    walls.append((time.perf_counter() - t0) * 1e3)
print("unprofiled wall ms:", " ".join(f"{w:.3f}" for w in walls))
lib.profile_enable(1)
lib.profile_report()
for i in range(reps):
    torch.cuda.synchronize()
    po.ggr_into(dv, fd, po.GgrConfig(), 0, 0, PO_LOC_DEVICE, r_, o_, 0)
    torch.cuda.synchronize()
rep = lib.profile_report(raw=True)
lib.profile_enable(0)
gaps = {k[4:]: v for k, v in rep.items() if k.startswith("gap:")}
tot = sum(v[1] for v in gaps.values()) / reps
cnt = sum(v[0] for v in gaps.values()) / reps
print(f"per call: {cnt:.0f} gaps, {tot:.3f} ms idle between launches")
for k, v in sorted(gaps.items(), key=lambda x: -x[1][1])[:top]:
    print(f"  before {k:40s} {v[0] / reps:6.1f}x {v[1] / reps * 1e3:8.1f} us")
host = {k[5:]: v for k, v in rep.items() if k.startswith("host:")}
print("host sections (wall, overlaps device work):")
for k, v in sorted(host.items(), key=lambda x: -x[1][1]):
    print(f"  {k:40s} {v[0] / reps:6.1f}x {v[1] / reps * 1e3:8.1f} us")
kern = {k: v for k, v in rep.items() if not k.startswith(("host:", "gap:"))}
print("scopes:", ", ".join(f"{k} {v[0] / reps:.0f}x {v[1] / reps * 1e3:.1f}us"
                          for k, v in sorted(kern.items(), key=lambda x: -x[1][1])[:12]))
