import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200._abi import PO_LOC_DEVICE
try:
    from cuda.bindings import runtime as rt
except ImportError:
    from cuda import cudart as rt
cfg, rows = int(sys.argv[1]), int(sys.argv[2])
t = gen.generate(cfg, n_rows=rows)
n, m = t.row_count(), t.field_count()
fd = [[t.require_field(x) for x in g] for g in gen.fds(cfg)]
dv = t.view(PO_LOC_DEVICE, arena=torch.from_numpy(t.arena).cuda(),
            offsets=torch.from_numpy(t.offsets.view(np.int64)).cuda())
r_ = torch.empty(n, dtype=torch.int64, device="cuda")
o_ = torch.empty(n * m, dtype=torch.int32, device="cuda")
err, pool = rt.cudaDeviceGetDefaultMemPool(0)
def attr(a):
    e, v = rt.cudaMemPoolGetAttribute(pool, a)
    return int(v) if not hasattr(v, 'value') else int(v.value) if hasattr(v,'value') else v
A = rt.cudaMemPoolAttr
for i in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    po.ggr_into(dv, fd, po.GgrConfig(), 0, 0, PO_LOC_DEVICE, r_, o_, 0)
    torch.cuda.synchronize()
    print(f"call {i}: {(time.perf_counter()-t0)*1e3:.1f} ms reserved {attr(A.cudaMemPoolAttrReservedMemCurrent)/1e9:.2f} GB high {attr(A.cudaMemPoolAttrReservedMemHigh)/1e9:.2f} GB used {attr(A.cudaMemPoolAttrUsedMemCurrent)/1e9:.2f} thr {attr(A.cudaMemPoolAttrReleaseThreshold)}", flush=True)
