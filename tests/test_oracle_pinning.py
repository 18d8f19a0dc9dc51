"""CPU: pin the oracle restatement (oracle/ggr_oracle.cpp) against the
reference — the committed reference-generated golden vectors always, and the
reference library itself (oracle/_ref) when it is built in this container."""
import random

import pytest

from golden_cases import check_result, load_cases, same_result
from oracle.pyoracle import available, oracle
from paper_2403_05821_b200 import GgrConfig, SegmentScoring, char_tokenizer, exact_config, word_tokenizer
from tables import ALPHABETS, random_table

CASES = load_cases()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_oracle_matches_reference_golden(case):
    name, t, fds, cfg, tok, sc, exp = case
    check_result(oracle("port").ggr(t, fds, cfg, tok, sc), exp, name)


def test_quickstart_known_answer():
    # demos/quickstart.cpp on movie_reviews.csv, threshold 0: ggr PHC 254,072
    case = next(c for c in CASES if c[0] == "movie_reviews_quickstart")
    assert case[-1]["phc"] == 254072
    assert oracle("port").ggr(*case[1:6]).phc_score == 254072


@pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built here")
def test_oracle_matches_reference_random():
    P, R = oracle("port"), oracle("reference")
    rng = random.Random(7)
    for trial in range(600):
        alpha = ALPHABETS[rng.choice(list(ALPHABETS))]
        t = random_table(rng, 10, 4, alpha, max_len=4, min_len=0)
        m = t.field_count()
        fds = None
        if m >= 2 and rng.random() < 0.4:
            fds = [[f"f{i}" for i in rng.sample(range(m), rng.randint(2, m))]]
        cfg = rng.choice([GgrConfig(), exact_config(), GgrConfig(1, 1, 0), GgrConfig(0, 0, 3)])
        tok = rng.choice([char_tokenizer(), word_tokenizer()])
        sc = rng.choice([SegmentScoring.value_only, SegmentScoring.full_fragment])
        assert same_result(P.ggr(t, fds, cfg, tok, sc), R.ggr(t, fds, cfg, tok, sc)), trial


@pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built here")
def test_oracle_phc_sort_stats_match_reference():
    P, R = oracle("port"), oracle("reference")
    rng = random.Random(11)
    for trial in range(200):
        t = random_table(rng, 8, 4, ALPHABETS["esc"], max_len=3, min_len=0)
        n, m = t.row_count(), t.field_count()
        order = list(range(m))
        rng.shuffle(order)
        assert P.sort_rows_fixed_order(t, order).tolist() == R.sort_rows_fixed_order(t, order).tolist()
        for tok in (char_tokenizer(), word_tokenizer()):
            for sc in (SegmentScoring.value_only, SegmentScoring.full_fragment):
                pc, pt = P.compute_stats(t, tok, sc)
                rc, rt = R.compute_stats(t, tok, sc)
                assert pc.tolist() == rc.tolist() and pt.tolist() == rt.tolist()
                entries = [(r, rng.sample(range(m), rng.randint(0, m))) for r in rng.sample(range(n), n)]
                assert P.phc(entries, t, tok, sc) == R.phc(entries, t, tok, sc)


# ---- functional dependencies (fd.hpp:56-141) ------------------------------
import random as _random

from fd_cases import known_fd_cases
from tables import ALPHABETS as _ALPHA, random_table as _rt


@pytest.mark.parametrize("kind", ["port", "reference"])
def test_fd_oracle_known_answers(kind):
    if kind == "reference" and not available("reference"):
        pytest.skip("oracle/_ref not built")
    for name, check in known_fd_cases():
        check(oracle(kind))


def test_fd_port_matches_reference():
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    rng = _random.Random(20240101)
    P, R = oracle("port"), oracle("reference")
    for _ in range(400):
        t = _rt(rng, 14, 5, _ALPHA["ab"], max_len=2)
        assert P.discover_fds(t, 100) == R.discover_fds(t, 100)
        names = [t.field_name(f) for f in range(t.field_count())]
        rng.shuffle(names)
        cut = rng.randint(0, len(names))
        groups = [g for g in (names[:cut], names[cut:]) if g]
        assert P.validate_fds(t, groups) == R.validate_fds(t, groups)


# ---- prompt rendering + dedup (objective.hpp:102-131, cost.hpp:171-186) ----
def _random_schedule(rng, t):
    from paper_2403_05821_b200 import RequestSchedule
    n, m = t.row_count(), t.field_count()
    ent = [(rng.randrange(n), rng.sample(range(m), rng.randint(0, m)))
           for _ in range(rng.randint(0, 25))]
    return RequestSchedule.from_entries(ent)


def test_render_dedup_port_matches_reference():
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    rng = _random.Random(99)
    P, R = oracle("port"), oracle("reference")
    for _ in range(150):
        t = _rt(rng, 15, 4, _ALPHA["all"], max_len=4)
        s = _random_schedule(rng, t)
        sp = bytes(rng.randrange(256) for _ in range(rng.randint(0, 4)))
        q = b"Which?" if rng.random() < 0.5 else b""
        a = P.render_prompts(s, t, sp, q)
        assert a == R.render_prompts(s, t, sp, q)
        dup = a + a[: rng.randint(0, len(a))]
        rng.shuffle(dup)
        assert P.dedup(dup) == R.dedup(dup)


def test_render_known_answer():
    # render_body / render_prompt format (objective.hpp:102-131)
    from paper_2403_05821_b200 import RequestSchedule, Table
    t = Table([b"title", b"q\"t"], [[b"Dune", b"a\nb"]])
    s = RequestSchedule.from_entries([(0, [1, 0]), (0, [])])
    want = [b'SYS\nQ\n{"q\\"t": "a\\nb", "title": "Dune"}', b"SYS\nQ\n{}"]
    for kind in ("port",) + (("reference",) if available("reference") else ()):
        assert oracle(kind).render_prompts(s, t, b"SYS", b"Q") == want


# ---- prefix-cache replay, eviction none (cache_sim.hpp:223-285) -----------
def test_simulate_port_matches_reference():
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    from paper_2403_05821_b200 import CacheConfig, char_tokenizer, word_tokenizer
    rng = _random.Random(8)
    P, R = oracle("port"), oracle("reference")
    for _ in range(200):
        alpha = rng.choice([b"ab", b"ab  \n", b"a b\tc\x0b", bytes(range(256))])
        ps = [bytes(rng.choice(alpha) for _ in range(rng.randint(0, 14)))
              for _ in range(rng.randint(1, 25))]
        for tok in (char_tokenizer(), word_tokenizer()):
            cfg = CacheConfig(min_cacheable_prefix_tokens=rng.choice([0, 1, 3, 6]))
            assert P.simulate(ps, cfg, tok) == R.simulate(ps, cfg, tok)


def test_simulate_known_answers():
    # test_cache_sim.cpp:51-60: k identical prompts hit (k-1)/k of their tokens
    from paper_2403_05821_b200 import word_tokenizer
    for kind in ("port",) + (("reference",) if available("reference") else ()):
        for k in (2, 3, 5, 8):
            rep = oracle(kind).simulate([b"the same prompt body"] * k, None, word_tokenizer())
            assert rep.phr == (k - 1) / k
            assert rep.requests[0].hit_tokens == 0
            assert all(r.hit_tokens == r.input_tokens for r in rep.requests[1:])


# ---- CSV ingest (table.hpp:114-215) ----------------------------------------
def test_csv_port_matches_reference():
    if not available("reference"):
        pytest.skip("oracle/_ref not built")
    from csv_util import SOUPS, outcome, to_csv
    rng = _random.Random(31)
    P, R = oracle("port"), oracle("reference")
    for _ in range(1500):
        alpha = rng.choice(SOUPS)
        d = bytes(rng.choice(alpha) for _ in range(rng.randint(0, 50)))
        assert outcome(P.load_csv, d) == outcome(R.load_csv, d)
    for _ in range(100):
        t = _rt(rng, 12, 4, _ALPHA["esc"], max_len=5, min_len=0)
        d = to_csv(t, rng.choice([b"\n", b"\r\n", b"\r"]))
        assert outcome(P.load_csv, d) == outcome(R.load_csv, d)
