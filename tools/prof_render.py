"""Per-kernel profile of one device-resident render of the C2 ggr schedule."""
import ctypes as C
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE, cuda_lib

lib = cuda_lib()
t = gen.generate(2)
n = t.row_count()
dv = t.view(PO_LOC_DEVICE, arena=torch.from_numpy(t.arena).cuda(),
            offsets=torch.from_numpy(t.offsets.view(np.int64)).cuda())
sch = po.ggr(t, None, po.GgrConfig()).schedule
d_rows = torch.from_numpy(sch.row_ids.view(np.int64)).cuda()
d_soff = torch.from_numpy(sch.order_offsets.view(np.int64)).cuda()
d_flds = torch.from_numpy(sch.order_fields).cuda()
sp, q = np.frombuffer(b"You are a shopping assistant.", np.uint8), np.frombuffer(b"Helpful?", np.uint8)
out_off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
total = C.c_uint64(0)
args = (dv.ref(), n, d_rows.data_ptr(), d_soff.data_ptr(), d_flds.data_ptr(), PO_LOC_DEVICE,
        sp.ctypes.data, sp.size, q.ctypes.data, q.size, PO_LOC_DEVICE, out_off.data_ptr())
lib.check(lib.render_prompts(*args, None, 0, C.byref(total), 0))
out = torch.empty(int(total.value), dtype=torch.uint8, device="cuda")
call = lambda: lib.check(lib.render_prompts(*args, out.data_ptr(), out.numel(), C.byref(total), 0))
call()
torch.cuda.synchronize()
t0 = time.perf_counter()
call()
torch.cuda.synchronize()
print("wall ms", (time.perf_counter() - t0) * 1e3)
lib.profile_enable(1)
lib.profile_report()
call()
torch.cuda.synchronize()
prof = lib.profile_report()
print("kernel ms", sum(v[1] for v in prof.values()))
for k, (c, ms) in sorted(prof.items(), key=lambda x: -x[1][1])[:8]:
    print(f"  {k:28s} {ms:8.3f} ms {c:4d}")
