"""Multi-GPU pieces: one rank per GPU.

* `ggr_sharded` — the row-sharded GGR solve (csrc/shard.cu through
  po_ggr_sharded): every rank passes a contiguous range of the table's rows
  and gets back one contiguous slice of the schedule; the slices in rank
  order are bit-identical to ggr() on the whole table. Collectives run over a
  `ShardComm`: NCCL between B200s (`nccl_comm`, one process per GPU, the
  unique id shipped over torch.distributed), host-staged collectives over any
  torch.distributed backend (`host_comm`, e.g. gloo: processes sharing a
  GPU) or an in-process thread group
  (`local_comms`, several ranks on one GPU — how the parity tests exercise
  the sharded path on a 1-GPU box).
* `sharded_phc` — the row-range-sharded PHC over torch.distributed with the
  one-entry boundary exchange, whose host logic the
  gloo tests cover on CPU.
"""
from __future__ import annotations

from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from ._abi import PO_LOC_DEVICE, PO_LOC_HOST, FdView, cuda_lib, po_solve_stats
from .api import (GgrConfig, RequestSchedule, SegmentScoring, SolveStats, _fd_indices, _view,
                  char_tokenizer, phc as device_phc)
import ctypes as C
from dataclasses import dataclass

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


# ---------------------------------------------------------------------------
# row-sharded GGR
# ---------------------------------------------------------------------------
class ShardComm:
    """A rank's communicator handle (po_comm)."""

    def __init__(self, handle: int, rank: int, world: int):
        self.handle, self.rank, self.world = handle, rank, world

    def close(self) -> None:
        if self.handle:
            cuda_lib().comm_destroy(self.handle)
            self.handle = 0

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def local_comms(world: int) -> list:
    """`world` communicators of one in-process group (one host thread per rank)."""
    lib = cuda_lib()
    arr = (C.c_void_p * world)()
    lib.check(lib.comm_init_local(world, arr))
    return [ShardComm(arr[r], r, world) for r in range(world)]


def share_id(uid: np.ndarray, world: int, group=None) -> np.ndarray:
    """Rank 0's 128-byte communicator id on every rank (torch.distributed)."""
    if world <= 1:
        return uid
    obj = [uid.tobytes()]
    dist.broadcast_object_list(obj, src=0, group=group)
    return np.frombuffer(obj[0], dtype=np.uint8).copy()


def nccl_comm(rank: int | None = None, world: int | None = None, group=None) -> ShardComm:
    """NCCL communicator over the ranks of an initialised torch.distributed
    group (the 128-byte NCCL id is broadcast from rank 0 through it)."""
    lib = cuda_lib()
    rank = dist.get_rank(group) if rank is None else rank
    world = dist.get_world_size(group) if world is None else world
    uid = np.zeros(128, dtype=np.uint8)
    if rank == 0:
        lib.check(lib.comm_unique_id(uid.ctypes.data))
    uid = share_id(uid, world, group)
    h = C.c_void_p(0)
    lib.check(lib.comm_init_nccl(uid.ctypes.data, world, rank, C.byref(h)))
    return ShardComm(h.value, rank, world)


# host-staged transport: po_host_collectives implemented with torch.distributed
_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)
_ALLGATHERV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64))
_ALLTOALLV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p,
                         C.POINTER(C.c_uint64))


class _HostCollectives(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgather", _ALLGATHER), ("allgatherv", _ALLGATHERV),
                ("alltoallv", _ALLTOALLV)]


def _host_bytes(ptr: int, n: int) -> torch.Tensor:
    return torch.from_numpy(np.ctypeslib.as_array((C.c_uint8 * max(n, 1)).from_address(ptr))[:n].copy())


def _gather_padded(mine: torch.Tensor, world: int, group) -> list:
    """Every rank's byte tensor (different sizes allowed), via equal-size
    all_gather (the gloo backend has no variable-size collectives)."""
    n = torch.tensor([mine.numel()], dtype=torch.int64)
    ns = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    mx = max(int(x.item()) for x in ns)
    pad = torch.zeros(max(mx, 1), dtype=torch.uint8)
    pad[:mine.numel()] = mine
    outs = [torch.zeros(max(mx, 1), dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return [o[:int(k.item())] for o, k in zip(outs, ns)]


def host_comm(group=None) -> ShardComm:
    """Communicator over the ranks of an initialised torch.distributed group
    of ANY backend (gloo on CPU included) through po_comm_init_host: device
    buffers are staged through host memory and exchanged with
    torch.distributed collectives. Slower than NCCL; it lets the sharded
    solver run across processes where NCCL cannot (several ranks on one GPU)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)

    def allgather(ctx, send, recv, nbytes):
        try:
            parts = _gather_padded(_host_bytes(send, nbytes), world, group)
            out = torch.cat(parts).numpy()
            C.memmove(recv, out.ctypes.data, out.nbytes)
            return 0
        except Exception:  # pragma: no cover - reported as PO_ERR_ERROR
            return 1

    def allgatherv(ctx, send, recv, recv_bytes):
        try:
            parts = _gather_padded(_host_bytes(send, int(recv_bytes[rank])), world, group)
            out = torch.cat(parts).numpy()
            if out.nbytes:
                C.memmove(recv, out.ctypes.data, out.nbytes)
            return 0
        except Exception:  # pragma: no cover
            return 1

    def alltoallv(ctx, send, send_bytes, recv, recv_bytes):
        try:
            sb = [int(send_bytes[r]) for r in range(world)]
            mine = _host_bytes(send, sum(sb))
            counts = _gather_padded(torch.tensor(sb, dtype=torch.int64).view(torch.uint8), world, group)
            datas = _gather_padded(mine, world, group)
            pieces = []
            for r in range(world):
                c = counts[r].view(torch.int64).tolist()
                off = sum(c[:rank])
                pieces.append(datas[r][off:off + c[rank]])
                assert c[rank] == int(recv_bytes[r])
            out = torch.cat(pieces).numpy()
            if out.nbytes:
                C.memmove(recv, out.ctypes.data, out.nbytes)
            return 0
        except Exception:  # pragma: no cover
            return 1

    ops = _HostCollectives(None, _ALLGATHER(allgather), _ALLGATHERV(allgatherv),
                           _ALLTOALLV(alltoallv))
    lib = cuda_lib()
    h = C.c_void_p(0)
    lib.check(lib.comm_init_host(C.byref(ops), world, rank, C.byref(h)))
    comm = ShardComm(h.value, rank, world)
    comm._keep = ops  # the callbacks must outlive the communicator
    return comm


@dataclass
class ShardResult:
    slice_offset: int          # position of this slice in the whole schedule
    row_ids: np.ndarray        # u64 global row ids, one per request of the slice
    field_orders: np.ndarray   # i32 [count, m]
    phc_score: int             # PHC of the WHOLE schedule (same on every rank)
    stats: SolveStats


def ggr_sharded_into(comm: ShardComm, view, fd_groups: list, cfg: GgrConfig, tok_kind: int,
                     scoring: int, stream: int = 0, out_location: int | None = PO_LOC_HOST):
    """po_ggr_sharded on a prepared view of this rank's rows. Returns
    (slice_offset, count, rows, orders, phc, stats); rows/orders are host
    arrays (out_location HOST), device tensors (DEVICE) or None (None: the
    slice stays on the device and is freed)."""
    lib = cuda_lib()
    fdv = FdView(fd_groups)
    sl = C.c_void_p(0)
    score = C.c_uint64(0)
    st = po_solve_stats()
    c = cfg.abi()
    lib.check(lib.ggr_sharded(comm.handle, view.ref(), fdv.ref(), C.byref(c), tok_kind, scoring,
                              C.byref(sl), C.byref(score), C.byref(st), stream))
    try:
        off, cnt = C.c_uint64(0), C.c_uint64(0)
        lib.check(lib.slice_info(sl, C.byref(off), C.byref(cnt)))
        n, m = int(cnt.value), int(view.view.n_fields)
        rows = orders = None
        if out_location == PO_LOC_HOST:
            rows = np.empty(max(n, 1), dtype=np.uint64)
            orders = np.empty(max(n * m, 1), dtype=np.int32)
            lib.check(lib.slice_copy(sl, PO_LOC_HOST, rows.ctypes.data, orders.ctypes.data, stream))
            rows, orders = rows[:n], orders[:n * m].reshape(n, m)
        elif out_location == PO_LOC_DEVICE:
            rows = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
            orders = torch.empty(max(n * m, 1), dtype=torch.int32, device="cuda")
            lib.check(lib.slice_copy(sl, PO_LOC_DEVICE, rows.data_ptr(), orders.data_ptr(), stream))
            rows, orders = rows[:n], orders[:n * m].view(n, m)
    finally:
        lib.slice_free(sl)
    return (int(off.value), n, rows, orders, int(score.value),
            SolveStats(st.recursive_calls, st.candidates_examined, st.max_depth, st.wall_ms))


def ggr_sharded(comm: ShardComm, t, fds=None, cfg: GgrConfig | None = None, tok=None,
                scoring: SegmentScoring = SegmentScoring.value_only,
                stream: int = 0) -> ShardResult:
    """Row-sharded prefixopt::ggr (ggr.hpp:367-394): `t` is this rank's
    contiguous range of rows (rank order = row order). Collective."""
    cfg = cfg or GgrConfig()
    tok = tok or char_tokenizer()
    view = _view(t, tok, scoring)
    off, n, rows, orders, phc_score, st = ggr_sharded_into(
        comm, view, _fd_indices(t, fds, cfg), cfg, tok.kind, int(scoring), stream)
    return ShardResult(off, rows, orders, phc_score, st)
