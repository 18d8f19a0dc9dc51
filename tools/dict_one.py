"""compute_stats (dictionary encode) on a C2 column subset, for ncu."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE, cuda_lib
lib = cuda_lib()
cols = [int(x) for x in sys.argv[1].split(',')]
t = gen.generate(2, columns=cols); n, m = t.row_count(), t.field_count()
d_arena = torch.from_numpy(t.arena).cuda(); d_offs = torch.from_numpy(t.offsets.view(np.int64)).cuda()
v = t.view(PO_LOC_DEVICE, arena=d_arena, offsets=d_offs)
card = np.zeros(m, np.uint64); tot = np.zeros(m, np.uint64)
lib.check(lib.compute_stats(v.ref(), 0, 0, card.ctypes.data, tot.ctypes.data, 0))
print(card)
