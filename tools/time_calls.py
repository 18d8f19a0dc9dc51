"""Wall time of repeated device-resident ggr() calls on C<cfg> (first rows)."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE

cfg_id, rows, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
t = gen.generate(cfg_id, n_rows=rows)
n, m = t.row_count(), t.field_count()
fd = [[t.require_field(x) for x in g] for g in gen.fds(cfg_id)]
dv = t.view(PO_LOC_DEVICE, arena=torch.from_numpy(t.arena).cuda(),
            offsets=torch.from_numpy(t.offsets.view(np.int64)).cuda())
r_ = torch.empty(n, dtype=torch.int64, device="cuda")
o_ = torch.empty(n * m, dtype=torch.int32, device="cuda")
from paper_2403_05821_b200._abi import cuda_lib
lib = cuda_lib()
prof = len(sys.argv) > 4
if prof:
    lib.profile_enable(1)
for i in range(reps):
    if prof:
        lib.profile_report()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    phc, st = po.ggr_into(dv, fd, po.GgrConfig(), 0, 0, PO_LOC_DEVICE, r_, o_, 0)
    torch.cuda.synchronize()
    print(f"call {i}: {(time.perf_counter() - t0) * 1e3:.1f} ms (wall_ms {st.wall_ms:.1f}) "
          f"free {torch.cuda.mem_get_info()[0] / 1e9:.1f} GB", flush=True)
    if prof:
        rep = {k: v for k, v in lib.profile_report().items() if not k.startswith(("gap:", "host:"))}
        top = sorted(rep.items(), key=lambda x: -x[1][1])[:int(sys.argv[4]) if sys.argv[4].isdigit() else 4]
        busy = rep.pop("busy:", (0, 0.0))[1]
        print("   busy %.3f ms; top: %s" % (busy,
              " | ".join(f"{k} {v[0]}x {v[1]:.3f}" for k, v in top)), flush=True)
