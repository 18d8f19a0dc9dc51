"""Call-time distribution of repeated device-resident ggr() calls, optionally
with nvidia-smi polling the GPU every 20 ms in the background (as bench.py's
clock sampler does).  python tools/stall_probe.py CFG ROWS CALLS [smi]"""
import subprocess
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE

cfg, rows, calls = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
smi = len(sys.argv) > 4 and sys.argv[4] == "smi"
t = gen.generate(cfg, n_rows=rows)
n, m = t.row_count(), t.field_count()
fd = [[t.require_field(x) for x in g] for g in gen.fds(cfg)]
dv = t.view(PO_LOC_DEVICE, arena=torch.from_numpy(t.arena).cuda(),
            offsets=torch.from_numpy(t.offsets.view(np.int64)).cuda())
r_ = torch.empty(n, dtype=torch.int64, device="cuda")
o_ = torch.empty(n * m, dtype=torch.int32, device="cuda")
proc = None
if smi:
    proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv", "-lms", "20"],
                            stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    time.sleep(1)
try:
    from cuda.bindings import runtime as rt
except ImportError:
    from cuda import cudart as rt
_, pool = rt.cudaDeviceGetDefaultMemPool(0)


def reserved():
    _, v = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
    return int(v) / 1e9


ts, rs = [], []
for i in range(calls):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    po.ggr_into(dv, fd, po.GgrConfig(), 0, 0, PO_LOC_DEVICE, r_, o_, 0)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
    rs.append(reserved())
if proc:
    proc.terminate()
print(" ".join(f"{x:.1f}" for x in ts[1:]))
print("reserved GB:", " ".join(f"{x:.2f}" for x in rs))
