"""k_dict_insert time on column subsets of C2 (hot-spot hypothesis)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE, cuda_lib
lib = cuda_lib()
for cols in ([0,1,2,3,4,5], [0,1,2,5], [3,4], [0,1], [5], [2]):
    t = gen.generate(2, columns=cols); n, m = t.row_count(), t.field_count()
    d_arena = torch.from_numpy(t.arena).cuda(); d_offs = torch.from_numpy(t.offsets.view(np.int64)).cuda()
    v = t.view(PO_LOC_DEVICE, arena=d_arena, offsets=d_offs)
    card = np.zeros(m, np.uint64); tot = np.zeros(m, np.uint64)
    for _ in range(2): lib.check(lib.compute_stats(v.ref(), 0, 0, card.ctypes.data, tot.ctypes.data, 0))
    lib.profile_enable(1); lib.profile_report()
    for _ in range(3): lib.check(lib.compute_stats(v.ref(), 0, 0, card.ctypes.data, tot.ctypes.data, 0))
    torch.cuda.synchronize(); rep = lib.profile_report(); lib.profile_enable(0)
    d = rep.get('k_dict_insert', (1, 0)); print(cols, f"{t.cell_bytes/1e6:.0f}MB", "dict %.3f ms" % (d[1]/d[0]), "card", card.tolist(), flush=True)
