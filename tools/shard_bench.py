"""Sharded solve with N thread-ranks on ONE GPU (in-process transport), each
rank holding rows_per_rank rows of config C<cfg>: total wall time per call
and the per-phase host timing (PO_DEBUG_TIMING=1). GPU work of the ranks
serialises on the one device, so time/N approximates the per-rank cost on
dedicated GPUs (transfers over NVLink excluded).

    python tools/shard_bench.py N [rows_per_rank] [cfg] [reps]
"""
import sys
import threading
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_05821_b200 as po  # noqa: E402
from paper_2403_05821_b200 import gen  # noqa: E402
from paper_2403_05821_b200._abi import PO_LOC_DEVICE  # noqa: E402
from paper_2403_05821_b200.dist import ggr_sharded_into, local_comms  # noqa: E402

N = int(sys.argv[1])
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
cfg_id = int(sys.argv[3]) if len(sys.argv) > 3 else 2
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
comms = local_comms(N)
views, keep = [], []
for r in range(N):
    t = gen.generate(cfg_id, n_rows=rows, row_begin=r * rows)
    a = torch.from_numpy(t.arena).cuda()
    o = torch.from_numpy(t.offsets.view(np.int64)).cuda()
    keep.append((a, o))
    views.append(t.view(PO_LOC_DEVICE, arena=a, offsets=o))
fds = [[gen.field_names(cfg_id).index(x.encode()) for x in g] for g in gen.fds(cfg_id)]
out = [None] * N
streams = [torch.cuda.Stream() for _ in range(N)]


def work(r):
    out[r] = ggr_sharded_into(comms[r], views[r], fds, po.GgrConfig(), 0, 0,
                              streams[r].cuda_stream, out_location=None)


from paper_2403_05821_b200._abi import cuda_lib  # noqa: E402
lib = cuda_lib()
for it in range(reps):
    if it == reps - 1:
        lib.profile_enable(1)
        lib.profile_report()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    th = [threading.Thread(target=work, args=(r,)) for r in range(N)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    print(f"N={N} rows/rank={rows}: {ms:.2f} ms per call ({ms / N:.2f} ms per rank), "
          f"phc={out[0][4]}, stats={out[0][5]}", flush=True)

prof = lib.profile_report()
lib.profile_enable(0)
tot = sum(v[1] for v in prof.values())
print(f"kernel time of the last call, all ranks: {tot:.2f} ms ({tot / N:.2f} ms per rank)")
for k, (c, ms) in sorted(prof.items(), key=lambda x: -x[1][1])[:22]:
    print(f"  {k:34s} {ms:8.3f} ms  {c:5d} launches")
