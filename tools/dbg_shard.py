"""Repeated sharded solves on thread ranks (determinism check):
    python tools/dbg_shard.py CFG ROWS N REPS"""
import sys, threading
sys.path.insert(0, '.')
import paper_2403_05821_b200 as po
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200.dist import ggr_sharded, local_comms, shard_range
cfg, rows, N, reps = (int(x) for x in sys.argv[1:5])
t = gen.generate(cfg, n_rows=rows)
ref = po.ggr(t, gen.fds(cfg), po.GgrConfig())
comms = local_comms(N)
for rep in range(reps):
    res = [None] * N
    def w(r):
        lo, hi = shard_range(t.row_count(), N, r)
        res[r] = ggr_sharded(comms[r], t.row_slice(lo, hi), gen.fds(cfg), po.GgrConfig())
    th = [threading.Thread(target=w, args=(r,)) for r in range(N)]
    [x.start() for x in th]; [x.join() for x in th]
    print(rep, [r.stats.candidates_examined for r in res], res[0].phc_score == ref.phc_score,
          ref.stats.candidates_examined, flush=True)
