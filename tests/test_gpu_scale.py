"""GPU parity at BASELINE-config shapes.

* row-prefix samples of C1..C5 (sizes the CPU oracle finishes in seconds):
  bit-exact against the oracle restatement (permutation, field orders, PHC,
  counters);
* full C2 (1M rows, the bench workload): size-independent properties — the
  schedule is a permutation with full field permutations, the reported PHC
  equals an independent recomputation through po_phc (CSR path), the run is
  deterministic, and the whole-table fixed-order sort is a permutation whose
  adjacent rows are in fragment-key order."""
import numpy as np
import pytest

import paper_2403_05821_b200 as po
from golden_cases import same_result
from oracle.pyoracle import oracle
from paper_2403_05821_b200 import gen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg_id,rows", [(1, 10_000), (2, 30_000), (3, 30_000), (4, 30_000),
                                         (5, 2_000)])
def test_config_prefix_matches_oracle(cfg_id, rows):
    t = gen.generate(cfg_id, n_rows=rows)
    fds = gen.fds(cfg_id)
    a = po.ggr(t, fds, po.GgrConfig())
    b = oracle("port").ggr(t, fds, po.GgrConfig())
    assert same_result(a, b), (cfg_id, a.phc_score, b.phc_score, a.stats, b.stats)


@pytest.mark.parametrize("tok,sc", [(po.word_tokenizer(), po.SegmentScoring.value_only),
                                    (po.char_tokenizer(), po.SegmentScoring.full_fragment),
                                    (po.word_tokenizer(), po.SegmentScoring.full_fragment)])
def test_c1_tokenizers_and_scoring(tok, sc):
    t = gen.generate(1, n_rows=5_000)
    for cfg in (po.GgrConfig(), po.GgrConfig(hitcount_stop_threshold=0)):
        assert same_result(po.ggr(t, None, cfg, tok, sc), oracle("port").ggr(t, None, cfg, tok, sc))


def test_c1_exact_config():
    t = gen.generate(1, n_rows=3_000)
    assert same_result(po.ggr(t, None, po.exact_config()),
                       oracle("port").ggr(t, None, po.exact_config()))


@pytest.fixture(scope="module")
def c2_full():
    return gen.generate(2)


def _fragment_key(t, r, order):
    return b"".join(po.fragment_text(t.field_name(f), t.cell(r, f)) for f in order)


def test_c2_full_properties(c2_full):
    t = c2_full
    n, m = t.row_count(), t.field_count()
    r1 = po.ggr(t, None, po.GgrConfig())
    rows = r1.schedule.row_ids
    assert np.array_equal(np.sort(rows), np.arange(n, dtype=np.uint64))
    orders = r1.schedule.order_fields.reshape(n, m)
    assert np.array_equal(np.sort(orders, axis=1), np.tile(np.arange(m, dtype=np.int32), (n, 1)))
    # PHC of the emitted schedule recomputed through the CSR po_phc path
    assert po.phc(r1.schedule, t) == r1.phc_score
    r2 = po.ggr(t, None, po.GgrConfig())
    assert same_result(r1, r2)


def test_c2_full_fixed_order_sort(c2_full):
    t = c2_full
    n = t.row_count()
    order = [1, 0, 2, 3, 4, 5]
    s = po.sort_rows_fixed_order(t, order)
    rows = s.row_ids
    assert np.array_equal(np.sort(rows), np.arange(n, dtype=np.uint64))
    rng = np.random.default_rng(0)
    for i in rng.integers(1, n, size=3000):
        a, b = int(rows[i - 1]), int(rows[i])
        ka, kb = _fragment_key(t, a, order), _fragment_key(t, b, order)
        assert ka < kb or (ka == kb and a < b)


_DEBUG_SCRIPT = r"""
import sys
sys.path.insert(0, 'tests')
import paper_2403_05821_b200 as po
from golden_cases import load_cases
from paper_2403_05821_b200 import gen
for name, t, fds, cfg, tok, sc, exp in load_cases():
    po.ggr(t, fds, cfg, tok, sc)
for cid, rows in [(1, 20000), (2, 50000), (3, 20000), (4, 20000), (5, 3000)]:
    po.ggr(gen.generate(cid, n_rows=rows), gen.fds(cid), po.GgrConfig())
    po.ggr(gen.generate(cid, n_rows=rows), None, po.GgrConfig(hitcount_stop_threshold=0))
print("done")
"""


def test_internal_debug_checks_clean():
    """PO_DEBUG_CHECKS cross-checks device invariants inside ggr(): every
    node's row count, leaf-sort permutation validity, and the prefix-group
    fallback PHC against the PHC of the materialised fixed-order sort."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, PO_DEBUG_CHECKS="1")
    r = subprocess.run([sys.executable, "-c", _DEBUG_SCRIPT], cwd=root, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "done" in r.stdout
    assert "[po debug]" not in r.stderr, r.stderr[-2000:]
