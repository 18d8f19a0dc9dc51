"""Per-kernel profile of one replay (unbounded cache) over the rendered C2
prompts (device-resident), plus the refine rounds (PO_DEBUG_TIMING=1)."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE, cuda_lib

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
tok = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lib = cuda_lib()
t = gen.generate(2, n_rows=rows)
res = po.ggr(t, None, po.GgrConfig())
arena, off = po.render_prompts_arena(res.schedule, t, b"You are a shopping assistant.", b"Helpful?")
d_a = torch.from_numpy(arena.copy()).cuda()
d_o = torch.from_numpy(off.view(np.int64)).cuda()
n = rows
outs = [np.zeros(n, np.uint64) for _ in range(4)]
tot = np.zeros(3, np.uint64)
call = lambda: lib.check(lib.replay_unbounded(n, d_a.data_ptr(), d_o.data_ptr(), PO_LOC_DEVICE, tok, 0,
                                              *(o.ctypes.data for o in outs), tot.ctypes.data, 0))
call()
lib.profile_enable(1)
lib.profile_report()
call()
torch.cuda.synchronize()
prof = lib.profile_report()
print("total kernel ms", sum(v[1] for v in prof.values()))
for k, (c, ms) in sorted(prof.items(), key=lambda x: -x[1][1])[:15]:
    print(f"  {k:30s} {ms:8.3f} ms {c:5d}")
