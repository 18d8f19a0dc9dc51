"""World-size-2 gloo tests (CPU) of the multi-process path: the row-range
sharded PHC with the one-entry boundary exchange equals the single-process
PHC. The local scorer is the oracle restatement (test infrastructure) so the
distributed logic is exercised without a GPU; on B200 the same function runs
with po.phc and NCCL."""
import os
import random
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_05821_b200.dist import shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, seeds, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import oracle
    from paper_2403_05821_b200 import RequestSchedule
    from paper_2403_05821_b200.dist import sharded_phc
    from tables import ALPHABETS, random_table
    P = oracle("port")
    out = []
    for seed in seeds:
        rng = random.Random(seed)
        t = random_table(rng, 40, 4, ALPHABETS["ab"], max_len=2)
        n, m = t.row_count(), t.field_count()
        entries = [(r, rng.sample(range(m), rng.randint(0, m))) for r in rng.sample(range(n), n)]
        s = RequestSchedule.from_entries(entries)
        got = sharded_phc(s, t, local_phc=P.phc)
        out.append((seed, got, P.phc(s, t)))
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_phc_matches_single_process(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    seeds = list(range(12))
    procs = [ctx.Process(target=_worker, args=(r, world, port, seeds, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for seed, got, want in res:
        assert got == want, seed


def test_shard_range_covers_exactly():
    for n in (0, 1, 7, 100, 101):
        for w in (1, 2, 3, 8):
            ranges = [shard_range(n, w, r) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(w - 1))


def _id_worker(rank, world, port, q):
    import numpy as np
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2403_05821_b200.dist import share_id
    uid = np.arange(128, dtype=np.uint8) if rank == 0 else np.zeros(128, dtype=np.uint8)
    got = share_id(uid, world)
    q.put((rank, got.tobytes()))
    dist.destroy_process_group()


def test_comm_id_broadcast_gloo():
    """The NCCL unique id reaches every rank intact (nccl_comm's side channel)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0] == got[1] == bytes(range(128))


def test_row_slices_reassemble_table():
    """Rank shards (Table.row_slice over shard_range) cover the table exactly."""
    import random
    from tables import ALPHABETS, random_table
    rng = random.Random(5)
    for _ in range(20):
        t = random_table(rng, 40, 4, ALPHABETS["esc"], max_len=3)
        for w in (1, 2, 3, 5):
            cells = []
            for r in range(w):
                sh = t.row_slice(*shard_range(t.row_count(), w, r))
                cells += [sh.row(i) for i in range(sh.row_count())]
            assert cells == [t.row(i) for i in range(t.row_count())]
