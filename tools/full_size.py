"""Full-size BASELINE tables through ggr() on one B200 (evidence runs).

    python tools/full_size.py CFG [ROWS] [--paths device,host] [--reps 2]

For config C<CFG> (all its rows unless ROWS is given): generate the table on
the host, then for each path
  device  arena + offsets uploaded to HBM once, po_ggr on device buffers
          (timed with CUDA events on the call's stream, after a warm-up call)
  host    po_ggr on the host table (row chunks streamed through the
          dictionary pass while the previous chunk is encoded)
print one JSON line: time, rows/s, cell GB/s, the schedule digests in the
form of tests/golden/full_digests.json, PHC, counters, and checks
  perm    row ids form a permutation, every field order a permutation of the
          schema
  phc_recomputed  PHC of the emitted schedule recomputed by po_phc (a separate
          entry point: equality-only dictionary + k_phc) == the solver's
  det     every call returned the same digest
When tests/golden/full_digests.json holds a reference digest for the same
(config, rows) it is compared too ("reference": true/false)."""
import hashlib
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2403_05821_b200 as po  # noqa: E402
from paper_2403_05821_b200 import gen  # noqa: E402
from paper_2403_05821_b200._abi import PO_LOC_DEVICE  # noqa: E402

GOLD = Path(__file__).resolve().parent.parent / "tests" / "golden" / "full_digests.json"


def digests(rows, orders, n, m):
    offs = np.arange(n + 1, dtype=np.uint64) * np.uint64(m)
    return {
        "rows_sha256": hashlib.sha256(np.ascontiguousarray(rows).astype("<u8").tobytes()).hexdigest(),
        "offsets_sha256": hashlib.sha256(offs.astype("<u8").tobytes()).hexdigest(),
        "fields_sha256": hashlib.sha256(np.ascontiguousarray(orders).astype("<i4").tobytes()).hexdigest(),
    }


def checks(t, rows, orders, n, m, phc):
    perm = bool(np.array_equal(np.sort(rows), np.arange(n, dtype=rows.dtype)))
    o = orders.reshape(n, m)
    perm_f = bool(np.array_equal(np.sort(o, axis=1), np.broadcast_to(np.arange(m, dtype=o.dtype), (n, m))))
    sched = po.RequestSchedule.full(rows, o)
    t0 = time.time()
    phc2 = po.phc(sched, t)
    return {"perm": perm and perm_f, "phc_recomputed": phc2 == phc,
            "phc_recompute_s": round(time.time() - t0, 2)}


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    opts = dict(a[2:].split("=", 1) for a in sys.argv[1:] if a.startswith("--") and "=" in a)
    cfg = int(args[0])
    rows = int(args[1]) if len(args) > 1 else None
    paths = opts.get("paths", "device,host").split(",")
    reps = int(opts.get("reps", "2"))
    t0 = time.time()
    t = gen.generate(cfg, n_rows=rows)
    n, m = t.row_count(), t.field_count()
    gen_s = time.time() - t0
    fds = gen.fds(cfg)
    fd_idx = [[t.require_field(x) for x in g] for g in fds]
    gold = None
    if GOLD.exists():
        for v in json.loads(GOLD.read_text()).values():
            if v["config"] == cfg and v["rows"] == n:
                gold = v
    base = {"workload": gen.CONFIGS[cfg].name, "rows": n, "fields": m, "cell_bytes": int(t.cell_bytes),
            "generate_s": round(gen_s, 1)}
    for path in paths:
        res, seen = None, set()
        if path == "device":
            po._abi.cuda_lib().trim_device_cache()
            torch.cuda.empty_cache()
            s = torch.cuda.current_stream()
            d_arena = torch.from_numpy(t.arena).to("cuda")
            d_offs = torch.from_numpy(t.offsets.view(np.int64)).to("cuda")
            dv = t.view(PO_LOC_DEVICE, arena=d_arena, offsets=d_offs)
            d_rows = torch.empty(n, dtype=torch.int64, device="cuda")
            d_ord = torch.empty(n * m, dtype=torch.int32, device="cuda")
            times = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(s)
                phc, st = po.ggr_into(dv, fd_idx, po.GgrConfig(), 0, 0, PO_LOC_DEVICE, d_rows, d_ord,
                                      s.cuda_stream)
                e1.record(s)
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
                h_rows, h_ord = d_rows.cpu().numpy().view(np.uint64), d_ord.cpu().numpy()
                seen.add(json.dumps(digests(h_rows, h_ord, n, m), sort_keys=True))
            ms = min(times[1:] or times)
            del d_arena, d_offs, dv, d_rows, d_ord
            torch.cuda.empty_cache()
        else:
            times = []
            for _ in range(reps):
                t1 = time.time()
                r = po.ggr(t, fds, po.GgrConfig())
                times.append((time.time() - t1) * 1e3)
                phc, st = r.phc_score, r.stats
                h_rows, h_ord = r.schedule.row_ids, r.schedule.order_fields
                seen.add(json.dumps(digests(h_rows, h_ord, n, m), sort_keys=True))
            ms = min(times[1:] or times)
        d = json.loads(next(iter(seen)))
        line = dict(base)
        line.update({"path": path, "ms": round(ms, 2), "ms_all": [round(x, 2) for x in times],
                     "rows_per_s": n / (ms / 1e3), "cell_GBps": t.cell_bytes / (ms / 1e3) / 1e9,
                     "phc": int(phc), "recursive_calls": st.recursive_calls,
                     "candidates_examined": st.candidates_examined, "max_depth": st.max_depth,
                     "det": len(seen) == 1, **d})
        line.update(checks(t, h_rows, h_ord, n, m, int(phc)))
        if gold is not None:
            line["reference"] = all(gold[k] == line[k] for k in
                                    ("rows_sha256", "offsets_sha256", "fields_sha256", "phc",
                                     "recursive_calls", "candidates_examined", "max_depth"))
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
