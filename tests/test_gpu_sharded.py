"""Row-sharded GGR against the single-GPU solver.

The sharded solve runs as N ranks on one GPU: N host threads, each with its
own CUDA stream and its contiguous range of rows, over the in-process
communicator (po_comm_init_local). The concatenated slices must equal
po.ggr on the whole table bit for bit: row permutation, field orders, PHC
and the three solver counters. This exercises the global dictionary
(sample sort + exact owner dedup), the replicated tables built from
exchanged contributions, the raw-rank tie-break, single-column leaves, the
distributed leaf sort and the whole-table fallback competition with the
same code that runs over NCCL on 2/4/8 GPUs. The NCCL transport itself is
covered at world size 1 (the box has one GPU)."""
import random
import threading

import numpy as np
import pytest
import torch

import paper_2403_05821_b200 as po
from golden_cases import load_cases
from paper_2403_05821_b200 import gen
from paper_2403_05821_b200.dist import ggr_sharded, local_comms, nccl_comm, shard_range
from tables import ALPHABETS, random_table

pytestmark = pytest.mark.gpu


def run_sharded(t, world, fds=None, cfg=None, tok=None, sc=po.SegmentScoring.value_only,
                bounds=None, comms=None):
    n = t.row_count()
    if bounds is None:
        bounds = [shard_range(n, world, r) for r in range(world)]
    comms = comms or local_comms(world)
    res, errs = [None] * world, [None] * world

    def work(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            shard = t.row_slice(*bounds[r])
            res[r] = ggr_sharded(comms[r], shard, fds, cfg, tok, sc, stream=st.cuda_stream)
        except Exception as e:  # surfaced below
            errs[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=600)
    for e in errs:
        if e is not None:
            raise e
    return res


def assert_same(t, res, ref):
    n, m = t.row_count(), t.field_count()
    off = 0
    rows, orders = [], []
    for r in res:
        assert r.slice_offset == off
        off += len(r.row_ids)
        rows.append(r.row_ids)
        orders.append(r.field_orders.reshape(-1, m) if m else np.zeros((len(r.row_ids), 0), np.int32))
        assert r.phc_score == ref.phc_score
        assert (r.stats.recursive_calls, r.stats.candidates_examined, r.stats.max_depth) == \
            (ref.stats.recursive_calls, ref.stats.candidates_examined, ref.stats.max_depth)
    assert off == n
    got_rows = np.concatenate(rows) if rows else np.zeros(0, np.uint64)
    assert got_rows.tolist() == ref.schedule.row_ids.tolist()
    if m and n:
        want = ref.schedule.order_fields.reshape(n, m)
        assert np.array_equal(np.concatenate(orders), want)


def check(t, world, fds=None, cfg=None, tok=None, sc=po.SegmentScoring.value_only, bounds=None):
    cfg = cfg or po.GgrConfig()
    ref = po.ggr(t, fds, cfg, tok or po.char_tokenizer(), sc)
    res = run_sharded(t, world, fds, cfg, tok, sc, bounds)
    assert_same(t, res, ref)
    return ref


@pytest.mark.parametrize("world", [2, 3])
def test_golden_cases_sharded(world):
    for name, t, fds, cfg, tok, sc, exp in load_cases()[:60]:
        check(t, world, fds, cfg, tok, sc)


@pytest.mark.parametrize("alpha", sorted(ALPHABETS))
@pytest.mark.parametrize("world", [2, 4])
def test_random_tables_sharded(alpha, world):
    rng = random.Random(1000 + world)
    for _ in range(12):
        t = random_table(rng, rng.randint(1, 80), rng.randint(1, 4), ALPHABETS[alpha],
                         max_len=rng.randint(1, 4))
        cfg = rng.choice([po.GgrConfig(), po.exact_config(),
                          po.GgrConfig(hitcount_stop_threshold=0)])
        check(t, world, None, cfg)


def test_uneven_and_empty_shards():
    rng = random.Random(7)
    t = random_table(rng, 50, 3, ALPHABETS["ab"], max_len=3, min_rows=50)
    for bounds in ([(0, 0), (0, 50)], [(0, 50), (50, 50)], [(0, 1), (1, 1), (1, 49), (49, 50)],
                   [(0, 10), (10, 10), (10, 50)]):
        check(t, len(bounds), None, po.exact_config(), bounds=bounds)


def test_tiny_tables_sharded():
    for rows in ([], [[b"a"]], [[b"a", b"b"]], [[b"x"], [b"x"]]):
        t = po.Table([b"f0", b"f1"][:len(rows[0]) if rows else 2], rows)
        check(t, 3, None, po.exact_config())
    t0 = po.Table([], [[] for _ in range(5)])  # no fields: rows in order
    check(t0, 2)


def test_ties_and_single_column_leaves():
    # equal scores across values force the raw-byte tie-break; 1-2 column
    # tables end in single-column leaves sorted by raw bytes
    rng = random.Random(3)
    for _ in range(10):
        vals = [bytes([rng.choice(b"\"\\\n a\x01\x7f\xc3")]) * rng.randint(1, 3) for _ in range(6)]
        rows = [[rng.choice(vals), rng.choice(vals)] for _ in range(60)]
        t = po.Table([b"x", b"y"], rows)
        check(t, 3, None, po.exact_config())
        check(t, 2, None, po.GgrConfig(hitcount_stop_threshold=0))


@pytest.mark.parametrize("tok,sc", [(po.word_tokenizer(), po.SegmentScoring.value_only),
                                    (po.char_tokenizer(), po.SegmentScoring.full_fragment),
                                    (po.word_tokenizer(), po.SegmentScoring.full_fragment)])
def test_c1_tokenizers_sharded(tok, sc):
    t = gen.generate(1, n_rows=4_000)
    check(t, 3, None, po.GgrConfig(), tok, sc)


@pytest.mark.parametrize("cfg_id,rows,world", [(1, 10_000, 4), (2, 30_000, 2), (2, 30_000, 4),
                                               (3, 30_000, 3), (4, 20_000, 4), (5, 2_000, 2),
                                               (3, 40_000, 8), (4, 40_000, 8)])
def test_config_prefix_sharded(cfg_id, rows, world):
    t = gen.generate(cfg_id, n_rows=rows)
    check(t, world, gen.fds(cfg_id))


def test_fd_groups_sharded():
    rng = random.Random(11)
    for _ in range(6):
        names = [b"a", b"b", b"c", b"d"]
        t = po.Table(names, [[bytes([rng.choice(b"xy")]) * rng.randint(1, 2) for _ in range(4)]
                             for _ in range(60)])
        fds = po.FunctionalDependencySet([[names[0], names[1]], [names[2], names[3]]])
        check(t, 2, fds, po.exact_config())


def test_c2_full_sharded_4():
    t = gen.generate(2)
    check(t, 4)


def test_nccl_transport_world1():
    comm = nccl_comm(rank=0, world=1)
    t = gen.generate(1, n_rows=3_000)
    ref = po.ggr(t, None, po.GgrConfig())
    res = run_sharded(t, 1, comms=[comm])
    assert_same(t, res, ref)
    comm.close()


def test_sharded_hash_collisions(monkeypatch):
    # 3-bit hashes: the local dictionaries must separate colliding values on
    # their bytes; the global dictionary compares bytes at the owners anyway
    monkeypatch.setenv("PO_DEBUG_HASH_BITS", "3")
    rng = random.Random(17)
    for _ in range(15):
        t = random_table(rng, 50, 4, ALPHABETS["all"], max_len=5, min_len=0)
        check(t, rng.choice([2, 3]), None, rng.choice([po.GgrConfig(), po.exact_config()]))


def test_c2_full_sharded_8():
    # the bench's largest world size, one full C2 table split 8 ways
    t = gen.generate(2)
    check(t, 8)
