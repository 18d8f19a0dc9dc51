"""Replays bench.py's call sequence with validity checks after every call."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE, PO_LOC_HOST, cuda_lib

mode = sys.argv[1] if len(sys.argv) > 1 else "prof"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1000000
lib = cuda_lib()
t = gen.generate(2, n_rows=rows)
n, m = t.row_count(), t.field_count()
cfg = po.GgrConfig()
sp = torch.cuda.current_stream().cuda_stream
d_arena = torch.from_numpy(t.arena).cuda(); d_offs = torch.from_numpy(t.offsets.view(np.int64)).cuda()
dv = t.view(PO_LOC_DEVICE, arena=d_arena, offsets=d_offs)
d_rows = torch.empty(n, dtype=torch.int64, device="cuda"); d_orders = torch.empty(n * m, dtype=torch.int32, device="cuda")
h_arena = torch.from_numpy(t.arena).pin_memory(); h_offs = torch.from_numpy(t.offsets.view(np.int64)).pin_memory()
hv = t.view(PO_LOC_HOST, arena=h_arena, offsets=h_offs)
h_rows = torch.empty(n, dtype=torch.int64).pin_memory(); h_orders = torch.empty(n * m, dtype=torch.int32).pin_memory()
ref = None
def run(tag, dev):
    global ref
    try:
        if dev:
            phc, st = po.ggr_into(dv, [], cfg, 0, 0, PO_LOC_DEVICE, d_rows, d_orders, sp)
            rr = d_rows.cpu().numpy()
        else:
            phc, st = po.ggr_into(hv, [], cfg, 0, 0, PO_LOC_HOST, h_rows, h_orders, sp)
            rr = h_rows.numpy()
    except Exception as e:
        print(tag, "ERROR", e, flush=True); return
    key = (phc, hash(rr.tobytes()))
    if ref is None: ref = key
    print(tag, "SAME" if key == ref else f"DIFF {phc}", flush=True)

for i in range(4): run(f"dev{i}", True)
if mode in ("prof", "profdev"):
    lib.profile_enable(1); lib.profile_report()
    for i in range(3): run(f"prof{i}", mode == "profdev" or True)
    torch.cuda.synchronize(); print(list(lib.profile_report().items())[:3]); lib.profile_enable(0)
nh = int(sys.argv[3]) if len(sys.argv) > 3 else 6
for i in range(nh): run(f"host{i}", False)
for i in range(3): run(f"dev_after{i}", True)
