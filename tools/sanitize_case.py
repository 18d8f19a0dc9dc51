"""Small solves for compute-sanitizer (tests/test_gpu_sanitizer.py): C1 rows
through po_ggr (host table: streamed dictionary; device table: resident),
po_phc, po_sort_rows_fixed_order, the sharded solver on 2 in-process ranks,
and — with PO_DEBUG_HASH_BITS=3 set by the caller — forced 64-bit hash
collisions on every path of the dictionary (claim races, byte verification,
the collision fix-up)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_05821_b200 as po  # noqa: E402
from paper_2403_05821_b200 import gen  # noqa: E402
from paper_2403_05821_b200._abi import PO_LOC_DEVICE  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
t = gen.generate(1, n_rows=rows)
r = po.ggr(t, None, po.GgrConfig())
assert po.phc(r.schedule, t) == r.phc_score
po.ggr(t, None, po.exact_config())
po.sort_rows_fixed_order(t, [3, 2, 1, 0])
c3 = gen.generate(3, n_rows=rows)
po.ggr(c3, gen.fds(3), po.GgrConfig())
n, m = t.row_count(), t.field_count()
d_arena = torch.from_numpy(t.arena).cuda()
d_offs = torch.from_numpy(t.offsets.view(np.int64)).cuda()
dv = t.view(PO_LOC_DEVICE, arena=d_arena, offsets=d_offs)
d_rows = torch.empty(n, dtype=torch.int64, device="cuda")
d_ord = torch.empty(n * m, dtype=torch.int32, device="cuda")
phc, _ = po.ggr_into(dv, [], po.GgrConfig(), 0, 0, PO_LOC_DEVICE, d_rows, d_ord, 0)
assert phc == r.phc_score
torch.cuda.synchronize()
print("sanitize case ok", r.phc_score)
