"""Repeat ggr() on a generated config through host and device buffers and
check every result is identical (race hunting)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE, PO_LOC_HOST

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 200000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
t = gen.generate(cfg_id, n_rows=rows)
n, m = t.row_count(), t.field_count()
fd = [[t.require_field(x) for x in g] for g in gen.fds(cfg_id)]
cfg = po.GgrConfig()
d_arena = torch.from_numpy(t.arena).cuda(); d_offs = torch.from_numpy(t.offsets.view(np.int64)).cuda()
dv = t.view(PO_LOC_DEVICE, arena=d_arena, offsets=d_offs)
pinned = len(sys.argv) > 4 and sys.argv[4] == "pinned"
if pinned:
    h_arena = torch.from_numpy(t.arena).pin_memory(); h_offs = torch.from_numpy(t.offsets.view(np.int64)).pin_memory()
    hv = t.view(PO_LOC_HOST, arena=h_arena, offsets=h_offs)
else:
    hv = t.view(PO_LOC_HOST)
ref = None
for i in range(reps):
    for name, v, loc in (("device", dv, PO_LOC_DEVICE), ("host", hv, PO_LOC_HOST)):
        if loc == PO_LOC_DEVICE:
            r_ = torch.empty(n, dtype=torch.int64, device='cuda'); o_ = torch.empty(n*m, dtype=torch.int32, device='cuda')
        else:
            if pinned:
                r_ = torch.empty(n, dtype=torch.int64).pin_memory(); o_ = torch.empty(n*m, dtype=torch.int32).pin_memory()
            else:
                r_ = np.empty(n, np.uint64); o_ = np.empty(n*m, np.int32)
        t0 = time.perf_counter()
        try:
            phc, st = po.ggr_into(v, fd, cfg, 0, 0, loc, r_, o_, torch.cuda.current_stream().cuda_stream)
        except Exception as e:
            print(i, name, "ERROR", e, flush=True); continue
        ms = (time.perf_counter() - t0) * 1e3
        rr = r_.cpu().numpy() if (loc == PO_LOC_DEVICE or pinned) else r_
        key = (phc, st.recursive_calls, st.candidates_examined, st.max_depth, hash(rr.tobytes()))
        if ref is None: ref = key
        print(i, name, f"{ms:.1f} ms", key[:4], "SAME" if key == ref else "DIFF", flush=True)
