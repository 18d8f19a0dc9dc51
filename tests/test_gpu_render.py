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


@pytest.mark.parametrize("dense", [True, False])
def test_render_long_cells_and_prompts(dense):
    # cells up to ~9 KB (many 128-byte copy steps, staging-buffer flushes
    # mid-cell), escapes inside long runs of plain bytes, a system prompt
    # longer than the 4 KB staging buffer, odd field names; dense schedules
    # take the storage-order length pass, sparse ones the per-request pass
    rng = random.Random(57 + dense)
    R = _ref()
    for trial in range(6):
        n, m = rng.randint(20, 60), rng.randint(1, 6)
        rows = []
        for _ in range(n):
            row = []
            for _ in range(m):
                ln = rng.choice([0, 1, 3, 7, 64, 127, 128, 129, 500, 4093, 9000])
                plain = rng.random() < 0.6
                alpha = b"abcdefghij" if plain else ALPHABETS["all" if rng.random() < 0.5 else "esc"]
                row.append(bytes(rng.choice(alpha) for _ in range(ln)))
            rows.append(row)
        names = [f"f{i}\"{'x' * rng.randint(0, 9)}\\" if rng.random() < 0.3 else f"col{i}" for i in range(m)]
        t = po.Table(names, rows)
        if dense:
            ent = [(r, rng.sample(range(m), m)) for r in range(n)] + \
                  [(rng.randrange(n), rng.sample(range(m), rng.randint(0, m))) for _ in range(10)]
        else:
            ent = [(rng.randrange(n), rng.sample(range(m), rng.randint(0, m))) for _ in range(3)]
        s = po.RequestSchedule.from_entries(ent)
        sp = bytes(rng.randrange(256) for _ in range(rng.choice([0, 5, 5000])))
        q = b"Q?" if trial % 2 else b""
        assert po.render_prompts(s, t, sp, q) == R.render_prompts(s, t, sp, q)


@pytest.mark.parametrize("shift", [0, 3, 13])
def test_render_into_device_buffer(shift):
    # device destination (the bytes are written in place, at any alignment);
    # the bytes around the destination stay untouched
    import ctypes as C

    import numpy as np
    import torch

    from paper_2403_05821_b200._abi import PO_LOC_DEVICE, cuda_lib

    lib = cuda_lib()
    t = gen.generate(2, n_rows=3000)
    n = t.row_count()
    res = po.ggr(t, None, po.GgrConfig())
    want = _ref().render_prompts(res.schedule, t, b"You are a shopping assistant.", b"Helpful?")
    dv = t.view(PO_LOC_DEVICE, arena=torch.from_numpy(t.arena).cuda(),
                offsets=torch.from_numpy(t.offsets.view(np.int64)).cuda())
    sch = res.schedule
    d_rows = torch.from_numpy(sch.row_ids.view(np.int64)).cuda()
    d_soff = torch.from_numpy(sch.order_offsets.view(np.int64)).cuda()
    d_flds = torch.from_numpy(sch.order_fields).cuda()
    sp, q = np.frombuffer(b"You are a shopping assistant.", np.uint8), np.frombuffer(b"Helpful?", np.uint8)
    out_off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    total = C.c_uint64(0)
    args = (dv.ref(), n, d_rows.data_ptr(), d_soff.data_ptr(), d_flds.data_ptr(), PO_LOC_DEVICE,
            sp.ctypes.data, sp.size, q.ctypes.data, q.size, PO_LOC_DEVICE, out_off.data_ptr())
    lib.check(lib.render_prompts(*args, None, 0, C.byref(total), 0))
    tot = int(total.value)
    out = torch.full((tot + shift + 32,), 0xA5, dtype=torch.uint8, device="cuda")
    lib.check(lib.render_prompts(*args, out.data_ptr() + shift, tot, C.byref(total), 0))
    torch.cuda.synchronize()
    h = out.cpu().numpy().tobytes()
    assert h[:shift] == b"\xa5" * shift and h[shift + tot:] == b"\xa5" * 32
    off = out_off.cpu().numpy()
    body = h[shift:shift + tot]
    assert [body[off[i]:off[i + 1]] for i in range(n)] == want
