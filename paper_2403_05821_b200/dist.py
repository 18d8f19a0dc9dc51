"""Multi-GPU pieces over torch.distributed (NCCL between B200s; gloo in the
CPU tests). One process per GPU.

Implemented: the row-range-sharded PHC with the one-entry boundary exchange
(SURVEY.md §8e step 7): a schedule split into contiguous request ranges is
scored per rank, the first request of every range against the last request
of the previous range (sent point-to-point), and the per-rank sums are
all-reduced. The sum is taken modulo 2^64 exactly like the reference's u64
accumulation (objective.hpp:96-98). The sharded GGR itself (global
dictionary exchange, per-level histogram merges) is not built yet; see
DESIGN.md §7.
"""
from __future__ import annotations

from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from .api import RequestSchedule, SegmentScoring, char_tokenizer, phc as device_phc

_MASK64 = (1 << 64) - 1


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) range of n items for rank."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _entry_tensor(s: RequestSchedule, i: int) -> torch.Tensor:
    o = s.order_offsets
    fields = s.order_fields[int(o[i]):int(o[i + 1])]
    return torch.tensor([int(s.row_ids[i])] + [int(f) for f in fields], dtype=torch.int64)


def _slice(s: RequestSchedule, lo: int, hi: int) -> RequestSchedule:
    o = s.order_offsets
    offs = o[lo:hi + 1] - o[lo]
    return RequestSchedule(s.row_ids[lo:hi], offs, s.order_fields[int(o[lo]):int(o[hi])])


def _prepend(entry: torch.Tensor, s: RequestSchedule) -> RequestSchedule:
    e = entry.tolist()
    rows = np.concatenate([np.array([e[0]], np.uint64), s.row_ids])
    offs = np.concatenate([np.array([0], np.uint64), s.order_offsets + np.uint64(len(e) - 1)])
    flds = np.concatenate([np.array(e[1:], np.int32), s.order_fields])
    return RequestSchedule(rows, offs, flds)


def sharded_phc(sched: RequestSchedule, table, tok=None,
                scoring: SegmentScoring = SegmentScoring.value_only, group=None,
                local_phc: Callable | None = None, device: str | torch.device = "cpu") -> int:
    """PHC of `sched` with its requests range-partitioned over the ranks of
    `group`. Every rank passes the full schedule (or a view with the same
    length) and scores only its own range plus the boundary pair."""
    tok = tok or char_tokenizer()
    local_phc = local_phc or device_phc
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = sched.size()
    lo, hi = shard_range(n, world, rank)
    local = _slice(sched, lo, hi)
    # boundary exchange: last entry of range r -> rank r+1 (length first)
    if rank + 1 < world:
        last = _entry_tensor(sched, hi - 1) if hi > lo else torch.zeros(0, dtype=torch.int64)
        ln = torch.tensor([last.numel()], dtype=torch.int64, device=device)
        dist.send(ln, rank + 1, group=group)
        if last.numel():
            dist.send(last.to(device), rank + 1, group=group)
    if rank > 0:
        ln = torch.zeros(1, dtype=torch.int64, device=device)
        dist.recv(ln, rank - 1, group=group)
        if int(ln.item()):
            prev = torch.zeros(int(ln.item()), dtype=torch.int64, device=device)
            dist.recv(prev, rank - 1, group=group)
            if hi > lo:
                local = _prepend(prev.cpu(), local)
    part = int(local_phc(local, table, tok, scoring)) if local.size() > 1 else 0
    # modulo-2^64 sum through int64 two's complement
    as_i64 = part - (1 << 64) if part >= (1 << 63) else part
    t = torch.tensor([as_i64], dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    return int(t.item()) & _MASK64
