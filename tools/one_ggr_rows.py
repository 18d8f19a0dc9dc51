"""One or more device-resident ggr() calls on the first ROWS rows of C<cfg> (ncu captures).
    python tools/one_ggr_rows.py CFG ROWS [REPS]"""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE
cfg_id, rows = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
t = gen.generate(cfg_id, n_rows=rows); n, m = t.row_count(), t.field_count()
fd = [[t.require_field(x) for x in g] for g in gen.fds(cfg_id)]
d_arena = torch.from_numpy(t.arena).cuda(); d_offs = torch.from_numpy(t.offsets.view(np.int64)).cuda()
dv = t.view(PO_LOC_DEVICE, arena=d_arena, offsets=d_offs)
r_ = torch.empty(n, dtype=torch.int64, device='cuda'); o_ = torch.empty(n*m, dtype=torch.int32, device='cuda')
for _ in range(reps):
    phc, st = po.ggr_into(dv, fd, po.GgrConfig(), 0, 0, PO_LOC_DEVICE, r_, o_, 0)
torch.cuda.synchronize()
print("phc", phc, st)
