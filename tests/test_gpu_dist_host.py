"""The row-sharded solver (po_ggr_sharded, csrc/shard.cu) across PROCESSES:
world size 2 and 3 over torch.distributed with the gloo backend, through the
host-staged transport (po_comm_init_host / dist.host_comm), every rank a
separate process on the one GPU of the test box (NCCL cannot put two ranks
on one GPU; its wrapper issues the same collective sequence). The slices in
rank order must equal po.ggr on the whole table: row ids, field orders, PHC
and counters."""
import os
import socket
import sys
import traceback
from pathlib import Path

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tables():
    import random
    import paper_2403_05821_b200 as po
    from paper_2403_05821_b200 import gen
    sys.path.insert(0, str(ROOT / "tests"))
    from tables import ALPHABETS, random_table
    out = [("C1", gen.generate(1, n_rows=6000), None, po.GgrConfig()),
           ("C3_fd", gen.generate(3, n_rows=20000), gen.fds(3), po.GgrConfig()),
           ("C2_exact", gen.generate(2, n_rows=3000), None, po.exact_config())]
    rng = random.Random(5)
    for k in range(3):
        t = random_table(rng, 40, 4, ALPHABETS[rng.choice(list(ALPHABETS))], max_len=4, min_len=0,
                         min_rows=10)
        out.append((f"random{k}", t, None, rng.choice([po.GgrConfig(), po.exact_config()])))
    return out


def _worker(rank, world, port, result_dir):
    try:
        sys.path.insert(0, str(ROOT))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import numpy as np
        import paper_2403_05821_b200 as po
        from paper_2403_05821_b200.dist import ggr_sharded, host_comm, shard_range
        comm = host_comm()
        lines = []
        for name, t, fds, cfg in _tables():
            lo, hi = shard_range(t.row_count(), world, rank)
            part = t.row_slice(lo, hi)
            r = ggr_sharded(comm, part, fds, cfg)
            got = [None] * world
            dist.all_gather_object(got, (r.slice_offset, r.row_ids.tolist(),
                                         r.field_orders.reshape(-1).tolist(), r.phc_score,
                                         (r.stats.recursive_calls, r.stats.candidates_examined,
                                          r.stats.max_depth)))
            if rank == 0:
                whole = po.ggr(t, fds, cfg)
                rows = [x for g in sorted(got) for x in g[1]]
                orders = [x for g in sorted(got) for x in g[2]]
                st = whole.stats
                ok = (rows == whole.schedule.row_ids.tolist()
                      and orders == whole.schedule.order_fields.tolist()
                      and all(g[3] == whole.phc_score for g in got)
                      and all(g[4] == (st.recursive_calls, st.candidates_examined, st.max_depth)
                              for g in got))
                lines.append(f"{name} {'ok' if ok else 'MISMATCH'} phc={whole.phc_score}")
        comm.close()
        dist.destroy_process_group()
        if rank == 0:
            Path(result_dir, "result.txt").write_text("\n".join(lines) + "\n")
    except Exception:
        Path(result_dir, f"error{rank}.txt").write_text(traceback.format_exc())
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_ggr_across_processes_gloo(tmp_path, world):
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    errs = list(tmp_path.glob("error*.txt"))
    assert not errs, errs[0].read_text()
    res = (tmp_path / "result.txt").read_text()
    print(res)
    assert "MISMATCH" not in res and res.count(" ok ") == len(_tables())
