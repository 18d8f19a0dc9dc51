"""Golden digests of the REFERENCE on the large BASELINE tables (test
infrastructure; run in the build container, which has /root/reference and
62 GB of RAM):

    python tests/golden/make_full_digests.py [name ...]

For each case the unmodified reference (oracle/_ref/libggr_ref.so, built by
`make -C oracle ref` from /root/reference) runs prefixopt::ggr on the
deterministic synthetic table paper_2403_05821_b200.gen.generate(cfg, rows)
and the result is stored as SHA-256 digests of the row permutation (u64 LE),
the CSR field-order offsets (u64 LE) and fields (i32 LE), plus PHC and the
three SolveStats counters -> tests/golden/full_digests.json. The GPU test
tests/test_gpu_full_size.py regenerates the same tables on the B200 box and
checks po.ggr against these digests. Sizes: C3 in full (10M rows, ~270 s,
~23 GB RSS); C4 and C5 as the largest row prefixes this host holds with the
reference's ~3-5x RSS overhead."""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.pyoracle import oracle  # noqa: E402
from paper_2403_05821_b200 import GgrConfig, gen  # noqa: E402

CASES = {
    "C3_full": (3, None),
    "C4_prefix_8M": (4, 8_000_000),
    "C5_prefix_1200K": (5, 1_200_000),
}
OUT = Path(__file__).resolve().parent / "full_digests.json"


def digest(res) -> dict:
    s = res.schedule
    return {
        "rows_sha256": hashlib.sha256(s.row_ids.astype("<u8").tobytes()).hexdigest(),
        "offsets_sha256": hashlib.sha256(s.order_offsets.astype("<u8").tobytes()).hexdigest(),
        "fields_sha256": hashlib.sha256(s.order_fields.astype("<i4").tobytes()).hexdigest(),
        "n_entries": int(s.size()),
        "phc": int(res.phc_score),
        "recursive_calls": int(res.stats.recursive_calls),
        "candidates_examined": int(res.stats.candidates_examined),
        "max_depth": int(res.stats.max_depth),
    }


def main(names):
    out = json.loads(OUT.read_text()) if OUT.exists() else {}
    for name in names:
        cfg, rows = CASES[name]
        t0 = time.time()
        t = gen.generate(cfg, n_rows=rows)
        res = oracle("reference").ggr(t, gen.fds(cfg), GgrConfig())
        d = digest(res)
        d.update({"config": cfg, "rows": int(t.row_count()), "cell_bytes": int(t.cell_bytes),
                  "workload": gen.CONFIGS[cfg].name, "reference_wall_s": res.stats.wall_ms / 1e3})
        out[name] = d
        OUT.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
        print(name, d, f"{time.time() - t0:.0f}s", flush=True)
        del t, res


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
