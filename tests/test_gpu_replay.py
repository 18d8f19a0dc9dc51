"""Prefix-cache replay with an unbounded cache on the GPU (csrc/replay.cu)
against the reference's own simulate() (oracle/_ref, cache_sim.hpp:223-285)
and the reference unit tests' answers (test_cache_sim.cpp)."""
import random

import pytest

import paper_2403_05821_b200 as po
from oracle.pyoracle import available, oracle
from paper_2403_05821_b200 import gen
from tables import ALPHABETS, random_table

pytestmark = pytest.mark.gpu

TOKS = [po.char_tokenizer(), po.word_tokenizer()]


def _ref():
    return oracle("reference" if available("reference") else "port")


def test_identical_prompts_known_answer():
    for tok in TOKS:
        for k in (2, 3, 5, 8):
            rep = po.simulate([b"the same prompt body"] * k, None, tok)
            assert rep.phr == (k - 1) / k
            assert rep.requests[0].hit_tokens == 0
            assert all(r.hit_tokens == r.input_tokens for r in rep.requests[1:])


@pytest.mark.parametrize("tok", TOKS, ids=["char", "word"])
def test_random_prompts_vs_reference(tok):
    rng = random.Random(12)
    R = _ref()
    for _ in range(150):
        alpha = rng.choice([b"ab", b"ab  \n", b"a b\tc\x0b", bytes(range(256)), b"xy "])
        base = [bytes(rng.choice(alpha) for _ in range(rng.randint(0, 40))) for _ in range(8)]
        ps = [rng.choice(base)[: rng.randint(0, 40)] + bytes(rng.choice(alpha) for _ in range(rng.randint(0, 6)))
              for _ in range(rng.randint(1, 60))]
        cfg = po.CacheConfig(min_cacheable_prefix_tokens=rng.choice([0, 1, 4, 10]))
        assert po.simulate(ps, cfg, tok) == R.simulate(ps, cfg, tok)


@pytest.mark.parametrize("tok", TOKS, ids=["char", "word"])
def test_schedule_prompts_vs_reference(tok):
    # test_cache_sim.cpp:99-113 shape: rendered prompts of random schedules
    rng = random.Random(21)
    R = _ref()
    for _ in range(30):
        t = random_table(rng, 12, 3, ALPHABETS["esc"], max_len=6)
        n, m = t.row_count(), t.field_count()
        rows = rng.sample(range(n), n)
        s = po.RequestSchedule.from_entries([(r, rng.sample(range(m), rng.randint(0, m))) for r in rows])
        got = po.phr_for_schedule(s, t, b"System:", b"Q?", None, tok)
        assert got == R.simulate(po.render_prompts(s, t, b"System:", b"Q?"), None, tok)


def test_ggr_schedule_c1_phr():
    # the pipeline after ggr (run.hpp:450-463): PHR of the reordered schedule
    # vs the original order, exact against the reference simulator
    t = gen.generate(1, n_rows=3_000)
    res = po.ggr(t, None, po.GgrConfig())
    orig = po.original_order_schedule(t)
    R = _ref()
    for sched in (res.schedule, orig):
        prompts = po.render_prompts(sched, t, b"You are a critic.", b"Rate it:")
        for tok in TOKS:
            assert po.simulate(prompts, None, tok) == R.simulate(prompts, None, tok)
    # unbounded cache: total hits depend on the prompt set, not its order
    # (every prompt's tokens end up in the trie exactly once)
    got = po.phr_for_schedule(res.schedule, t, b"You are a critic.", b"Rate it:")
    assert got == R.simulate(po.render_prompts(res.schedule, t, b"You are a critic.", b"Rate it:"))


def test_errors():
    with pytest.raises(po.DomainError):
        po.simulate([], None)
    with pytest.raises(po.SchemaError):
        po.simulate([b"a"], po.CacheConfig(eviction="lru"))
    t = po.Table([b"a"], [[b"x"], [b"y"]])
    with pytest.raises(po.SchemaError):
        po.phr_for_schedule(po.RequestSchedule.from_entries([(0, [0]), (0, [0])]), t)
