"""Bit-exact against the REFERENCE ITSELF (oracle/_ref: the unmodified
prefixopt headers compiled from /root/reference) at the bench's full size:
C2 1M x 6 in full, and large row prefixes of C3 (FD), C4 and C5 — same row
permutation, field orders, PHC and solver counters. Each reference run takes
10-30 s on one core."""
import pytest

import paper_2403_05821_b200 as po
from golden_cases import same_result
from oracle.pyoracle import available, oracle
from paper_2403_05821_b200 import gen

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not available("reference"),
                                                  reason="oracle/_ref not built")]


@pytest.mark.parametrize("cfg_id,rows", [(2, None), (3, 1_500_000), (4, 1_000_000), (5, 150_000)])
def test_matches_reference(cfg_id, rows):
    t = gen.generate(cfg_id, n_rows=rows)
    fds = gen.fds(cfg_id)
    a = po.ggr(t, fds, po.GgrConfig())
    b = oracle("reference").ggr(t, fds, po.GgrConfig())
    assert same_result(a, b), (cfg_id, a.phc_score, b.phc_score, a.stats, b.stats)
