"""Generate tests/golden/*.json from the REFERENCE implementation.

Runs the unmodified reference headers (oracle/_ref/libggr_ref.so, built by
`make -C oracle ref` from /root/reference) on small deterministic tables and
stores inputs + outputs, so the GPU box (which has no /root/reference) can
check against reference-produced vectors. Re-run in the build container:

    make -C oracle ref && python tests/golden/make_golden.py
"""
from __future__ import annotations

import csv
import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE.parent))

from oracle.pyoracle import oracle  # noqa: E402
from paper_2403_05821_b200 import (GgrConfig, SegmentScoring, Table, char_tokenizer,  # noqa: E402
                                   exact_config, word_tokenizer)
from tables import (ALPHABETS, distinct_first_table, fd_covered_table,  # noqa: E402
                    group_per_field_table, random_table)

REF_CSV = Path("/root/reference/proj/demos/data/movie_reviews.csv")


def enc(b: bytes) -> str:
    return b.decode("latin-1")


def table_json(t: Table) -> dict:
    return {"fields": [enc(f) for f in t.field_names],
            "rows": [[enc(c) for c in t.row(r)] for r in range(t.row_count())]}


def cfg_json(c: GgrConfig) -> dict:
    return {"row": c.row_recursion_depth, "col": c.column_recursion_depth,
            "thr": c.hitcount_stop_threshold, "use_fds": bool(c.use_fds),
            "variant": int(c.stats_variant)}


def case(ref, name, t, fds, cfg, tok, scoring):
    r = ref.ggr(t, fds, cfg, tok, scoring)
    return {
        "name": name, "table": table_json(t), "fds": fds, "cfg": cfg_json(cfg),
        "tok": tok.name, "scoring": int(scoring),
        "expect": {"phc": r.phc_score, "rows": r.schedule.row_ids.tolist(),
                   "orders": r.schedule.order_fields.tolist(),
                   "calls": r.stats.recursive_calls, "cands": r.stats.candidates_examined,
                   "depth": r.stats.max_depth},
    }


def main():
    ref = oracle("reference")
    cases = []
    # Demo data: quickstart settings (demos/quickstart.cpp:35-56), threshold 0.
    with open(REF_CSV, newline="") as f:
        rows = list(csv.reader(f))
    movies = Table(rows[0], rows[1:])
    fds = [["movie_title", "movie_info"]]
    cases.append(case(ref, "movie_reviews_quickstart", movies, fds,
                      GgrConfig(hitcount_stop_threshold=0), char_tokenizer(),
                      SegmentScoring.value_only))
    for sc in (SegmentScoring.value_only, SegmentScoring.full_fragment):
        for tok in (char_tokenizer(), word_tokenizer()):
            for cfg in (GgrConfig(), exact_config()):
                cases.append(case(ref, f"movie_reviews_{tok.name}_{int(sc)}", movies, fds, cfg,
                                  tok, sc))
    # Structured families (test_solver_greedy.cpp:109-137).
    for n in (2, 4, 7, 10):
        cases.append(case(ref, f"distinct_first_{n}", distinct_first_table(n, 3), None,
                          exact_config(), char_tokenizer(), SegmentScoring.value_only))
    for x in (2, 3):
        for cfg in (exact_config(), GgrConfig()):
            cases.append(case(ref, f"group_per_field_{x}", group_per_field_table(x, 3), None, cfg,
                              char_tokenizer(), SegmentScoring.value_only))
    # Random tables over several byte classes.
    rng = random.Random(20241017)
    for i in range(160):
        alpha = ALPHABETS[["ab", "esc", "all", "ws"][i % 4]]
        t = random_table(rng, 9, 4, alpha, max_len=4, min_len=0)
        m = t.field_count()
        f = None
        if m >= 2 and i % 3 == 0:
            f = [[f"f{k}" for k in rng.sample(range(m), rng.randint(2, m))]]
        cfg = [exact_config(), GgrConfig(), GgrConfig(1, 1, 0), GgrConfig(0, 0, 2)][i % 4]
        tok = [char_tokenizer(), word_tokenizer()][(i // 4) % 2]
        sc = [SegmentScoring.value_only, SegmentScoring.full_fragment][(i // 8) % 2]
        cases.append(case(ref, f"random_{i}", t, f, cfg, tok, sc))
    for i in range(20):
        t = fd_covered_table(rng, 8, 4)
        cases.append(case(ref, f"fd_covered_{i}", t, [[enc(x) for x in t.field_names]],
                          exact_config(), char_tokenizer(), SegmentScoring.value_only))
    out = HERE / "ggr_reference_cases.json"
    out.write_text(json.dumps({"generator": "tests/golden/make_golden.py",
                               "source": "oracle/_ref (reference prefixopt::ggr)",
                               "cases": cases}, separators=(",", ":")))
    print(f"wrote {len(cases)} cases to {out}")


if __name__ == "__main__":
    main()
