"""Throughput of the §8f components on the bench table (C2 1M x 6 unless
--rows), device-resident like bench.py's `value` (inputs and outputs in HBM,
wall time of the synchronous C-ABI call): FD validation (po_fd_compare over
the validate_fds pairs) and discovery (all field pairs), prompt rendering of
the ggr() schedule (po_render_prompts) and byte-exact dedup of the prompts
(po_dedup). The reference implementation (oracle/_ref) runs beside it on a
bounded row sample, one thread. One JSON line per component.

    python tools/bench_next.py [--rows N] [--cpu-rows N] [--reps K]
"""
import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_05821_b200 as po  # noqa: E402
from paper_2403_05821_b200 import gen  # noqa: E402
from paper_2403_05821_b200._abi import PO_LOC_DEVICE, cuda_lib  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--cpu-rows", type=int, default=50_000)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    from oracle.pyoracle import available, oracle
    ref = oracle("reference" if available("reference") else "port")
    lib = cuda_lib()
    t = gen.generate(2, n_rows=a.rows)
    n, m = t.row_count(), t.field_count()
    names = t.field_names
    d_arena = torch.from_numpy(t.arena).cuda()
    d_offs = torch.from_numpy(t.offsets.view(np.int64)).cuda()
    dv = t.view(PO_LOC_DEVICE, arena=d_arena, offsets=d_offs)
    small = gen.generate(2, n_rows=a.cpu_rows)
    sp, q = b"You are a shopping assistant.", b"Is this review helpful?"

    def line(name, secs, cpu_secs, extra):
        print(json.dumps({"component": name, "rows": n, "gpu_ms": secs * 1e3,
                          "gpu_rows_per_s": n / secs, "cpu_reference_rows_per_s": a.cpu_rows / cpu_secs,
                          "cpu_sample_rows": a.cpu_rows, "cpu_cores": 1, "cpu_kind": ref.kind,
                          "residency": "device (inputs and outputs in HBM)", **extra}), flush=True)

    def fd_call(pa, pb):
        k = len(pa)
        A, B = np.array(pa, np.int32), np.array(pb, np.int32)
        fd, sa, sb = (np.zeros(k, np.uint64) for _ in range(3))
        lib.check(lib.fd_compare(dv.ref(), k, A.ctypes.data, B.ctypes.data, fd.ctypes.data,
                                 sa.ctypes.data, sb.ctypes.data, 0))
        return fd

    s, _ = timed(lambda: fd_call([0, 2], [1, 3]), a.reps)
    c, _ = timed(lambda: ref.validate_fds(small, [[names[0], names[1]], [names[2], names[3]]]), 1)
    line("validate_fds (fd.hpp:66-109)", s, c, {"pairs": 2})
    pairs = [(i, j) for i in range(m) for j in range(i + 1, m)]
    s, _ = timed(lambda: fd_call([p[0] for p in pairs], [p[1] for p in pairs]), a.reps)
    c, _ = timed(lambda: ref.discover_fds(small, a.cpu_rows), 1)
    line("discover_fds (fd.hpp:114-141)", s, c, {"pairs": len(pairs)})

    res = po.ggr(t, None, po.GgrConfig())
    sch = res.schedule
    d_rows = torch.from_numpy(sch.row_ids.view(np.int64)).cuda()
    d_soff = torch.from_numpy(sch.order_offsets.view(np.int64)).cuda()
    d_flds = torch.from_numpy(sch.order_fields).cuda()
    spa, qa = np.frombuffer(sp, np.uint8), np.frombuffer(q, np.uint8)
    out_off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    total = C.c_uint64(0)
    args = (dv.ref(), n, d_rows.data_ptr(), d_soff.data_ptr(), d_flds.data_ptr(), PO_LOC_DEVICE,
            spa.ctypes.data, len(sp), qa.ctypes.data, len(q), PO_LOC_DEVICE, out_off.data_ptr())
    lib.check(lib.render_prompts(*args, None, 0, C.byref(total), 0))
    out = torch.empty(int(total.value), dtype=torch.uint8, device="cuda")
    s, _ = timed(lambda: lib.check(lib.render_prompts(*args, out.data_ptr(), out.numel(),
                                                      C.byref(total), 0)), a.reps)
    rs = po.ggr(small, None, po.GgrConfig()).schedule
    c, cp = timed(lambda: ref.render_prompts(rs, small, sp, q), 1)
    line("render_prompt x n (objective.hpp:102-131)", s, c,
         {"bytes_out": int(total.value), "gpu_GBps_out": int(total.value) / s / 1e9})

    ex = np.zeros(n, np.uint64)
    uf = np.zeros(n, np.uint64)
    nu = C.c_uint64(0)
    s, _ = timed(lambda: lib.check(lib.dedup(n, out.data_ptr(), out_off.data_ptr(), PO_LOC_DEVICE,
                                             ex.ctypes.data, uf.ctypes.data, C.byref(nu), 0)),
                 a.reps)
    c, _ = timed(lambda: ref.dedup(cp), 1)
    line("dedup (cost.hpp:171-186)", s, c,
         {"unique": int(nu.value), "bytes_in": int(total.value),
          "gpu_GBps_in": int(total.value) / s / 1e9, "outputs": "expansion map to host"})

    # prefix-cache replay, unbounded cache, over the same prompts
    for tk, name in ((po.char_tokenizer(), "char"), (po.word_tokenizer(), "word")):
        outs = [np.zeros(n, np.uint64) for _ in range(4)]
        tot = np.zeros(3, np.uint64)
        s, _ = timed(lambda: lib.check(lib.replay_unbounded(
            n, out.data_ptr(), out_off.data_ptr(), PO_LOC_DEVICE, tk.kind, 0,
            *(o.ctypes.data for o in outs), tot.ctypes.data, 0)), a.reps)
        c, rep = timed(lambda: ref.simulate(cp, po.CacheConfig(), tk), 1)
        line(f"simulate eviction=none, {name} tokens (cache_sim.hpp:223-285)", s, c,
             {"phr": float(tot[1]) / float(tot[0]), "input_tokens": int(tot[0]),
              "bytes_in": int(total.value), "gpu_GBps_in": int(total.value) / s / 1e9,
              "outputs": "per-request arrays to host"})

    # CSV ingest: the table written as CSV, text resident in HBM
    sys.path.insert(0, str(ROOT / "tests"))
    from csv_util import to_csv
    text = to_csv(t)
    d_text = torch.from_numpy(np.frombuffer(text, np.uint8).copy()).cuda()
    small_text = to_csv(small)

    def csv_call():
        h = C.c_void_p(0)
        lib.check(lib.load_csv(d_text.data_ptr(), len(text), PO_LOC_DEVICE, C.byref(h), 0))
        lib.csv_free(h)

    s, _ = timed(csv_call, a.reps)
    c, _ = timed(lambda: ref.load_csv(small_text), 1)
    line("load_csv (table.hpp:114-215)", s, c,
         {"bytes_in": len(text), "gpu_GBps_in": len(text) / s / 1e9,
          "outputs": "parsed table in HBM (handle)"})


if __name__ == "__main__":
    main()
