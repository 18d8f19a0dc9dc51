"""Loader for tests/golden/ggr_reference_cases.json (reference-produced)."""
from __future__ import annotations

import json
from pathlib import Path

from paper_2403_05821_b200 import (GgrConfig, SegmentScoring, StatsScoreVariant, Table,
                                   tokenizer_by_name)

GOLDEN = Path(__file__).resolve().parent / "golden" / "ggr_reference_cases.json"


def load_cases():
    data = json.loads(GOLDEN.read_text())
    out = []
    for c in data["cases"]:
        t = Table([f.encode("latin-1") for f in c["table"]["fields"]],
                  [[x.encode("latin-1") for x in row] for row in c["table"]["rows"]])
        g = c["cfg"]
        cfg = GgrConfig(g["row"], g["col"], g["thr"], g["use_fds"], StatsScoreVariant(g["variant"]))
        fds = [[x.encode("latin-1") for x in grp] for grp in c["fds"]] if c["fds"] else None
        out.append((c["name"], t, fds, cfg, tokenizer_by_name(c["tok"]),
                    SegmentScoring(c["scoring"]), c["expect"]))
    return out


def check_result(res, exp, name=""):
    assert res.phc_score == exp["phc"], name
    assert res.schedule.row_ids.tolist() == exp["rows"], name
    assert res.schedule.order_fields.tolist() == exp["orders"], name
    assert res.stats.recursive_calls == exp["calls"], name
    assert res.stats.candidates_examined == exp["cands"], name
    assert res.stats.max_depth == exp["depth"], name


def same_result(a, b):
    return (a.phc_score == b.phc_score
            and a.schedule.row_ids.tolist() == b.schedule.row_ids.tolist()
            and a.schedule.order_fields.tolist() == b.schedule.order_fields.tolist()
            and (a.stats.recursive_calls, a.stats.candidates_examined, a.stats.max_depth)
            == (b.stats.recursive_calls, b.stats.candidates_examined, b.stats.max_depth))
