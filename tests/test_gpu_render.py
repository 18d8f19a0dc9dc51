"""Prompt rendering and byte-exact dedup on the GPU (csrc/render.cu) against
the compiled reference's render_prompt / dedup (objective.hpp:102-131,
cost.hpp:171-186) and the CPU restatement."""
import random

import pytest

import paper_2403_05821_b200 as po
from oracle.pyoracle import available, oracle
from paper_2403_05821_b200 import gen
from tables import ALPHABETS, random_table

pytestmark = pytest.mark.gpu


def _ref():
    return oracle("reference" if available("reference") else "port")


@pytest.mark.parametrize("alpha", sorted(ALPHABETS))
def test_render_random_schedules(alpha):
    rng = random.Random(31)
    R = _ref()
    for _ in range(40):
        t = random_table(rng, 30, 5, ALPHABETS[alpha], max_len=rng.randint(1, 40))
        n, m = t.row_count(), t.field_count()
        s = po.RequestSchedule.from_entries(
            [(rng.randrange(n), rng.sample(range(m), rng.randint(0, m))) for _ in range(50)])
        sp = bytes(rng.randrange(256) for _ in range(rng.randint(0, 80)))
        q = b"Is the review positive?" if rng.random() < 0.5 else b""
        got = po.render_prompts(s, t, sp, q)
        assert got == R.render_prompts(s, t, sp, q)
        dup = got + [got[rng.randrange(len(got))] for _ in range(20)]
        rng.shuffle(dup)
        assert po.dedup(dup) == R.dedup(dup)


def test_render_out_of_range():
    t = po.Table([b"a"], [[b"x"]])
    s = po.RequestSchedule.from_entries([(3, [0])])
    with pytest.raises(IndexError):
        po.render_prompts(s, t)


def test_render_dedup_ggr_schedule_c1():
    # the pipeline step after ggr (run.hpp:457-466) on a C1 prefix with 20% duplicate rows
    t = gen.generate(1, n_rows=4_000)
    res = po.ggr(t, None, po.GgrConfig())
    P = oracle("port")
    got = po.render_prompts(res.schedule, t, b"You are a movie critic.", b"Summarise:")
    assert got == P.render_prompts(res.schedule, t, b"You are a movie critic.", b"Summarise:")
    d = po.dedup(got)
    assert d == P.dedup(got)
    assert [d.uniques[i] for i in d.expansion_map] == got


def test_dedup_edge_cases():
    for prompts in ([], [b""], [b"", b""], [b"a", b"b", b"a", b"", b"b"], [bytes([0]) * 70] * 3):
        assert po.dedup(prompts) == oracle("port").dedup(prompts)


def test_dedup_and_fd_with_hash_collisions(monkeypatch):
    monkeypatch.setenv("PO_DEBUG_HASH_BITS", "3")
    rng = random.Random(23)
    P = oracle("port")
    for _ in range(20):
        ps = [bytes(rng.randrange(256) for _ in range(rng.randint(0, 6))) for _ in range(60)]
        ps += [rng.choice(ps) for _ in range(30)]
        assert po.dedup(ps) == P.dedup(ps)
        t = random_table(rng, 40, 4, ALPHABETS["all"], max_len=4, min_len=0)
        assert po.discover_fds(t, 1000) == P.discover_fds(t, 1000)
