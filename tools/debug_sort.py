"""Repeated whole-table fixed-order sorts (po_sort_rows_fixed_order) with
permutation validity checks."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch, ctypes as C
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE, PO_LOC_HOST, cuda_lib
rows = int(sys.argv[1]); reps = int(sys.argv[2]); pinned = sys.argv[3] == "pinned"
lib = cuda_lib()
t = gen.generate(2, n_rows=rows); n, m = t.row_count(), t.field_count()
if pinned:
    h_arena = torch.from_numpy(t.arena).pin_memory(); h_offs = torch.from_numpy(t.offsets.view(np.int64)).pin_memory()
    v = t.view(PO_LOC_HOST, arena=h_arena, offsets=h_offs)
else:
    d_arena = torch.from_numpy(t.arena).cuda(); d_offs = torch.from_numpy(t.offsets.view(np.int64)).cuda()
    v = t.view(PO_LOC_DEVICE, arena=d_arena, offsets=d_offs)
order = np.array([1, 0, 2, 3, 4, 5], dtype=np.int32)
out = np.empty(n, np.uint64)
bad_runs = 0
for i in range(reps):
    lib.check(lib.sort_rows_fixed_order(v.ref(), order.ctypes.data, PO_LOC_HOST, out.ctypes.data, 0))
    ok = np.array_equal(np.sort(out), np.arange(n, dtype=np.uint64))
    if not ok: bad_runs += 1
print("rows", rows, "pinned", pinned, "bad runs", bad_runs, "of", reps, flush=True)
