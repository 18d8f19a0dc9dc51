"""GPU parity: the CUDA path (libprefixopt_cuda.so through the C ABI) must be
bit-exact with the reference — row permutation, per-row field orders, PHC and
the three SolveStats counters — on the reference-generated golden vectors and,
differentially, against the oracle restatement on seeded random tables."""
import os
import random

import numpy as np
import pytest

import paper_2403_05821_b200 as po
from golden_cases import check_result, load_cases, same_result
from oracle.pyoracle import available, oracle
from tables import (ALPHABETS, distinct_first_table, fd_covered_table, group_per_field_table,
                    random_table, skewed_table)

pytestmark = pytest.mark.gpu
CASES = load_cases()
TOKS = [po.char_tokenizer(), po.word_tokenizer()]
SCS = [po.SegmentScoring.value_only, po.SegmentScoring.full_fragment]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_ggr_matches_reference_golden(case):
    name, t, fds, cfg, tok, sc, exp = case
    check_result(po.ggr(t, fds, cfg, tok, sc), exp, name)


def test_quickstart_known_answer():
    case = next(c for c in CASES if c[0] == "movie_reviews_quickstart")
    assert po.ggr(*case[1:6]).phc_score == 254072


def test_structured_families_closed_form():
    # test_solver_greedy.cpp:109-124
    for n in (2, 4, 7, 10):
        t = distinct_first_table(n, 3)
        r = po.ggr(t, None, po.exact_config())
        assert r.phc_score == 2 * (n - 1)
        assert po.phc(r.schedule, t) == r.phc_score
    for x in (2, 3):
        assert po.ggr(group_per_field_table(x, 3), None, po.exact_config()).phc_score == 3 * (x - 1)


def test_random_tables_vs_oracle():
    rng = random.Random(1234)
    P = oracle("port")
    for trial in range(400):
        alpha = ALPHABETS[rng.choice(list(ALPHABETS))]
        t = random_table(rng, 12, 5, alpha, max_len=4, min_len=0, min_rows=0)
        m = t.field_count()
        fds = None
        if m >= 2 and rng.random() < 0.35:
            fds = [[f"f{i}" for i in rng.sample(range(m), rng.randint(2, m))]]
        cfg = rng.choice([po.GgrConfig(), po.exact_config(), po.GgrConfig(1, 1, 0),
                          po.GgrConfig(0, 0, 3), po.GgrConfig(2, 1, 1, True, po.StatsScoreVariant(rng.randint(0, 2)))])
        tok, sc = rng.choice(TOKS), rng.choice(SCS)
        a = po.ggr(t, fds, cfg, tok, sc)
        b = P.ggr(t, fds, cfg, tok, sc)
        assert same_result(a, b), (trial, t.row_count(), m, cfg, tok.name, sc, fds)


def test_fd_covered_tables_vs_oracle():
    rng = random.Random(53)
    P = oracle("port")
    for _ in range(60):
        t = fd_covered_table(rng, 10, 4)
        fds = [t.field_names]
        assert same_result(po.ggr(t, fds, po.exact_config()), P.ggr(t, fds, po.exact_config()))


@pytest.mark.parametrize("cfg", [po.GgrConfig(), po.exact_config(),
                                 po.GgrConfig(hitcount_stop_threshold=50)])
def test_skewed_medium_tables_vs_oracle(cfg):
    rng = random.Random(99)
    P = oracle("port")
    for n in (300, 2000):
        t = skewed_table(rng, n, [3, 40, 200, n], [6, 12, 20, 10])
        for tok in TOKS:
            a = po.ggr(t, [["col1", "col2"]], cfg, tok)
            b = P.ggr(t, [["col1", "col2"]], cfg, tok)
            assert same_result(a, b), (n, cfg, tok.name)


def test_hash_collisions_are_resolved_on_bytes(monkeypatch):
    # force 3-bit hashes: every column has colliding distinct values, so the
    # dictionary must separate them by byte comparison
    monkeypatch.setenv("PO_DEBUG_HASH_BITS", "3")
    rng = random.Random(5)
    P = oracle("port")
    for trial in range(40):
        t = random_table(rng, 30, 4, ALPHABETS["all"], max_len=5, min_len=0)
        cfg = rng.choice([po.GgrConfig(), po.exact_config()])
        assert same_result(po.ggr(t, None, cfg), P.ggr(t, None, cfg)), trial


@pytest.mark.parametrize("bits", ["3", "64"])
def test_long_values_collisions_resolved_on_bytes(monkeypatch, bits):
    # cells of 60-300 bytes (cooperative byte verification) that differ only
    # in a byte near the end or in length, under forced hash collisions
    monkeypatch.setenv("PO_DEBUG_HASH_BITS", bits)
    rng = random.Random(11)
    P = oracle("port")
    for trial in range(12):
        n = rng.choice([33, 100, 700])
        base = [bytes(rng.choice(b"abc \"\n") for _ in range(rng.randint(60, 300)))
                for _ in range(3)]
        vals = []
        for b in base:
            k = rng.randrange(len(b))
            vals += [b, b[:k] + b"z" + b[k + 1:], b + b"x", b[:-1]]
        rows = [[rng.choice(vals), rng.choice(vals[:4]), bytes([97 + rng.randrange(3)])]
                for _ in range(n)]
        t = po.Table(["a", "b", "c"], rows)
        cfg = rng.choice([po.GgrConfig(), po.exact_config()])
        assert same_result(po.ggr(t, None, cfg), P.ggr(t, None, cfg)), (trial, bits)
        st = po.compute_stats(t)
        card, _ = P.compute_stats(t)
        assert [f.cardinality for f in st.fields] == card.tolist()


@pytest.mark.parametrize("env", [{"PO_RANK_UNIQUE": "1"}, {"PO_MERGE_RANK": "0"},
                                 {"PO_MERGE_RANK": "0", "PO_MERGE_ROUND0_MAX": "0"}])
def test_alternate_sort_paths_vs_oracle(monkeypatch, env):
    # PO_RANK_UNIQUE=1 ranks unique columns too (no tie-break pass);
    # PO_MERGE_RANK=0 sorts small string jobs by refinement rounds instead of
    # the one-pass merge sort (and PO_MERGE_ROUND0_MAX=0 with radix round 0)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = random.Random(21)
    P = oracle("port")
    for trial in range(60):
        t = random_table(rng, 14, 4, ALPHABETS[rng.choice(list(ALPHABETS))], max_len=4, min_len=0)
        cfg = rng.choice([po.GgrConfig(), po.exact_config(), po.GgrConfig(0, 0, 0)])
        assert same_result(po.ggr(t, None, cfg), P.ggr(t, None, cfg)), trial
        m = t.field_count()
        order = list(range(m))
        rng.shuffle(order)
        assert (po.sort_rows_fixed_order(t, order).row_ids.tolist()
                == P.sort_rows_fixed_order(t, order).tolist())


def test_trim_device_cache_then_solve_again():
    # idle cached blocks go back to the driver; the next call allocates anew
    from paper_2403_05821_b200._abi import cuda_lib
    rng = random.Random(8)
    P = oracle("port")
    t = skewed_table(rng, 3000, [3, 40, 200, 3000], [6, 12, 20, 10])
    first = po.ggr(t, None, po.GgrConfig())
    cuda_lib().trim_device_cache()
    cuda_lib().trim_device_cache()  # nothing idle left: a no-op
    again = po.ggr(t, None, po.GgrConfig())
    assert same_result(first, again)
    assert same_result(again, P.ggr(t, None, po.GgrConfig()))


def test_phc_hit_random_schedules_vs_oracle():
    rng = random.Random(42)
    P = oracle("port")
    for trial in range(200):
        t = random_table(rng, 8, 4, ALPHABETS["esc"], max_len=3, min_len=0)
        n, m = t.row_count(), t.field_count()
        entries = [(r, rng.sample(range(m), rng.randint(0, m))) for r in rng.sample(range(n), n)]
        s = po.RequestSchedule.from_entries(entries)
        for tok in TOKS:
            for sc in SCS:
                assert po.phc(s, t, tok, sc) == P.phc(s, t, tok, sc)
        if n:
            r = rng.randrange(n)
            prev = P.phc(po.RequestSchedule.from_entries(entries[max(r - 1, 0):r + 1]), t) if r else 0
            assert po.hit(s, r, t) == prev


def test_sort_rows_fixed_order_and_stats_vs_oracle():
    rng = random.Random(3)
    P = oracle("port")
    for trial in range(150):
        t = random_table(rng, 10, 4, ALPHABETS[rng.choice(list(ALPHABETS))], max_len=4, min_len=0)
        m = t.field_count()
        order = list(range(m))
        rng.shuffle(order)
        s = po.sort_rows_fixed_order(t, order)
        assert s.row_ids.tolist() == P.sort_rows_fixed_order(t, order).tolist()
        for tok in TOKS:
            for sc in SCS:
                st = po.compute_stats(t, tok, sc)
                card, tot = P.compute_stats(t, tok, sc)
                assert [f.cardinality for f in st.fields] == card.tolist()
                n = t.row_count()
                assert [f.avg_len for f in st.fields] == [float(x) / n for x in tot.tolist()]


def _unique_column_table(rng, n, m_low, prefix_len):
    """A column with one distinct value per row (shared prefixes, bytes that
    JSON escaping reorders) next to low-cardinality columns."""
    alpha = ALPHABETS["esc"] + b"\x7f\xc3"
    uniq = set()
    while len(uniq) < n:
        uniq.add(b"p" * rng.randint(0, prefix_len)
                 + bytes(rng.choice(alpha) for _ in range(rng.randint(0, 4))))
    uniq = list(uniq)
    rng.shuffle(uniq)
    rows = [[bytes([97 + rng.randrange(3)]) * rng.randint(1, 2) for _ in range(m_low)] + [u]
            for u in uniq]
    k = rng.randrange(m_low + 1)
    rows = [r[:k] + [r[-1]] + r[k:-1] for r in rows]
    return po.Table([f"f{i}" for i in range(m_low + 1)], rows), k


@pytest.mark.parametrize("short_max,long_budget", [(None, None), ("0", None), ("0", "0"),
                                                   ("4", "0")])
def test_unique_columns_tie_break_on_bytes(monkeypatch, short_max, long_budget):
    # unique columns are left unranked by the solver; every sort that reaches
    # one orders its tied runs by the column's escaped bytes instead: short
    # runs by direct ranking, long runs by prefix keys + counting or by a sort
    if short_max is not None:
        monkeypatch.setenv("PO_SHORT_RUN_MAX", short_max)
    if long_budget is not None:
        monkeypatch.setenv("PO_LONG_RUN_BUDGET", long_budget)
    rng = random.Random(77)
    P = oracle("port")
    for trial in range(40):
        n = rng.choice([2, 3, 17, 200, 1500])
        t, k = _unique_column_table(rng, n, rng.randint(1, 3), rng.choice([0, 3, 40]))
        m = t.field_count()
        order = list(range(m))
        rng.shuffle(order)
        assert (po.sort_rows_fixed_order(t, order).row_ids.tolist()
                == P.sort_rows_fixed_order(t, order).tolist()), (trial, n, order)
        for cfg in (po.GgrConfig(0, 0, 0), po.GgrConfig(1, 1, 0), po.GgrConfig()):
            assert same_result(po.ggr(t, None, cfg), P.ggr(t, None, cfg)), (trial, n, cfg)


def test_error_behaviour():
    t = po.Table(["A", "B"], [["1", "2"]])
    with pytest.raises(po.SchemaError):
        po.sort_rows_fixed_order(t, [0])
    with pytest.raises(po.SchemaError):
        po.sort_rows_fixed_order(t, [0, 0])
    s = po.RequestSchedule.from_entries([(0, [0])])
    with pytest.raises(po.DomainError):
        po.hit(s, 1, t)
    bad = po.RequestSchedule.from_entries([(0, [0]), (5, [0])])
    with pytest.raises(IndexError):
        po.phc(bad, t)
    with pytest.raises(po.SchemaError):
        po.ggr(t, [["A", "nope"]], po.GgrConfig())
    # unknown FD names are ignored when use_fds is false (ggr.hpp:155)
    po.ggr(t, [["A", "nope"]], po.GgrConfig(use_fds=False))


def test_degenerate_tables():
    assert po.ggr(po.Table(["a"], []), None).schedule.size() == 0
    r = po.ggr(po.Table(["a", "b"], [["1", "2"]]), None)
    assert r.phc_score == 0 and r.schedule.entries[0].field_order == [0, 1]
    r = po.ggr(po.Table([], [[], [], []]), None)
    assert r.schedule.row_ids.tolist() == [0, 1, 2]


def test_launches_counted():
    before = po._abi.cuda_lib().kernel_launch_count()
    po.ggr(distinct_first_table(5, 3), None)
    assert po._abi.cuda_lib().kernel_launch_count() > before


def test_all_empty_cells_null_arena():
    # every cell "": the C++ drop-in passes an empty vector's data() (null);
    # the reference returns a valid schedule with PHC 0
    t = po.Table(["a", "b", "c"], [["", "", ""]] * 7)
    P = oracle("port")
    for cfg in (po.GgrConfig(), po.exact_config()):
        assert same_result(po.ggr(t, None, cfg), P.ggr(t, None, cfg))
    view = t.view(arena=0)
    rows = np.empty(7, np.uint64)
    orders = np.empty(21, np.int32)
    phc, st = po.api.ggr_into(view, [], po.GgrConfig(), po.char_tokenizer().kind, 0,
                              po._abi.PO_LOC_HOST, rows, orders)
    ref = P.ggr(t, None, po.GgrConfig())
    assert phc == ref.phc_score == 0
    assert rows.tolist() == ref.schedule.row_ids.tolist()


def test_fd_groups_sharing_members_vs_reference():
    # groups that share two members: the reference emits a partner once per
    # group holding it and counts its length as often (ggr.hpp:154-164,
    # 252-255, 280-282), so field orders get longer than the schema
    rng = random.Random(77)
    R = oracle("reference") if available("reference") else oracle("port")
    shapes = [[["f0", "f1", "f2"], ["f0", "f1"]], [["f0", "f1"], ["f0", "f1"]],
              [["f0", "f1", "f2"], ["f1", "f2", "f3"]], [["f1", "f0"], ["f0", "f1", "f2"], ["f2", "f1"]]]
    seen_long = False
    for trial in range(160):
        alpha = ALPHABETS[rng.choice(list(ALPHABETS))]
        t = random_table(rng, 40, 5, alpha, max_len=3, min_len=0, min_rows=2)
        m = t.field_count()
        fds = [g for g in rng.choice(shapes) if all(int(x[1:]) < m for x in g)]
        cfg = rng.choice([po.GgrConfig(), po.exact_config(), po.GgrConfig(1, 1, 0),
                          po.GgrConfig(2, 2, 0, True, po.StatsScoreVariant(rng.randint(0, 2)))])
        tok, sc = rng.choice(TOKS), rng.choice(SCS)
        a = po.ggr(t, fds, cfg, tok, sc)
        b = R.ggr(t, fds, cfg, tok, sc)
        assert same_result(a, b), (trial, fds, cfg)
        assert a.schedule.order_offsets.tolist() == b.schedule.order_offsets.tolist()
        assert po.phc(a.schedule, t, tok, sc) == a.phc_score
        seen_long |= a.schedule.order_fields.size > t.row_count() * m
    assert seen_long  # some schedule did carry repeated partners
