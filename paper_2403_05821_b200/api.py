"""Host-side mirror of the reference's hot-path API (namespace prefixopt).

Same names, argument meaning and error behaviour as the C++ reference:
  ggr                           ggr.hpp:367-394
  phc / hit                     objective.hpp:70-99
  sort_rows_fixed_order         objective.hpp:154-171
  compute_stats                 stats.hpp:25-45
  fixed_order_by_hitcount_stats ggr.hpp:59-84
  fixed_order_by_stats          objective.hpp:176-188
Every call that touches table data goes through the CUDA library
(include/prefixopt_cuda.h); if it is not built, ExtensionMissing is raised.
The double-precision field ranking is host math in the reference too and is
evaluated by the same library's host code.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from ._abi import (PO_LOC_DEVICE, PO_LOC_HOST, FdView, TableView, _ptr, cuda_lib,
                   po_ggr_config, po_solve_stats)
from .errors import DomainError, SchemaError, SizeError
from .table import Table, _to_bytes


# --------------------------------------------------------------------------
# enums and small types
# --------------------------------------------------------------------------
class SegmentScoring(enum.IntEnum):
    """scoring.hpp:20."""
    value_only = 0
    full_fragment = 1


def scoring_by_name(name: str) -> SegmentScoring:
    if name == "value":
        return SegmentScoring.value_only
    if name == "fragment":
        return SegmentScoring.full_fragment
    raise SchemaError(f"unknown scoring mode: {name} (expected 'value' or 'fragment')")


class StatsScoreVariant(enum.IntEnum):
    """ggr.hpp:25-29."""
    cardinality_weighted_squared = 0
    squared_length = 1
    length_frequency = 2


def stats_variant_by_name(name: str) -> StatsScoreVariant:
    table = {"weighted": 0, "squared": 1, "length-freq": 2}
    if name not in table:
        raise SchemaError(f"unknown stats variant: {name} "
                          "(expected 'weighted', 'squared' or 'length-freq')")
    return StatsScoreVariant(table[name])


_WS = frozenset(b" \t\n\r\f\v")


class Tokenizer:
    """Tokenizer (tokenizer.hpp:18-30). Subclasses overriding count() are
    'custom': their per-cell lengths are computed here and passed through the
    ABI (po_table.cell_lens); char and word run on the GPU."""
    kind = 2
    name = "custom"

    def count(self, text: bytes) -> int:  # pragma: no cover - abstract
        raise NotImplementedError


class CharTokenizer(Tokenizer):
    kind = 0
    name = "char"

    def count(self, text: bytes) -> int:
        return len(text)


class WordTokenizer(Tokenizer):
    kind = 1
    name = "word"

    def count(self, text: bytes) -> int:
        n, inword = 0, False
        for b in text:
            sp = b in _WS
            if not sp and not inword:
                n += 1
            inword = not sp
        return n


_CHAR, _WORD = CharTokenizer(), WordTokenizer()


def char_tokenizer() -> Tokenizer:
    return _CHAR


def word_tokenizer() -> Tokenizer:
    return _WORD


def tokenizer_by_name(name: str) -> Tokenizer:
    if name == "char":
        return _CHAR
    if name == "word":
        return _WORD
    raise SchemaError(f"unknown tokenizer: {name} (expected 'char' or 'word')")


def json_escape(s: bytes) -> bytes:
    """json_escape (scoring.hpp:33-57)."""
    out = bytearray()
    named = {0x22: b'\\"', 0x5C: b"\\\\", 0x08: b"\\b", 0x0C: b"\\f", 0x0A: b"\\n",
             0x0D: b"\\r", 0x09: b"\\t"}
    for b in _to_bytes(s):
        if b in named:
            out += named[b]
        elif b < 0x20:
            out += b"\\u00%02x" % b
        else:
            out.append(b)
    return bytes(out)


def fragment_text(field_name: bytes, value: bytes) -> bytes:
    """fragment_text (scoring.hpp:62-69)."""
    return b'"' + json_escape(field_name) + b'": "' + json_escape(value) + b'", '


def segment_len(field_name: bytes, value: bytes, tok: Tokenizer,
                scoring: SegmentScoring = SegmentScoring.value_only) -> int:
    """segment_len (scoring.hpp:72-76)."""
    if scoring == SegmentScoring.value_only:
        return tok.count(_to_bytes(value))
    return tok.count(fragment_text(_to_bytes(field_name), _to_bytes(value)))


@dataclass
class GgrConfig:
    """GgrConfig (ggr.hpp:48-54)."""
    row_recursion_depth: int = 4
    column_recursion_depth: int = 2
    hitcount_stop_threshold: int = 100000
    use_fds: bool = True
    stats_variant: StatsScoreVariant = StatsScoreVariant.cardinality_weighted_squared

    def abi(self) -> po_ggr_config:
        return po_ggr_config(self.row_recursion_depth, self.column_recursion_depth,
                             self.hitcount_stop_threshold, int(bool(self.use_fds)),
                             int(self.stats_variant))


def exact_config() -> GgrConfig:
    """No early stopping (test_solver_greedy.cpp:18-24)."""
    return GgrConfig(1 << 20, 1 << 20, 0)


@dataclass
class FunctionalDependencySet:
    """FunctionalDependencySet (fd.hpp:21-26)."""
    groups: list = field(default_factory=list)
    validated: bool = False

    def empty(self) -> bool:
        return not self.groups


@dataclass
class ScheduleEntry:
    row_id: int
    field_order: list


class RequestSchedule:
    """RequestSchedule (objective.hpp:21-32) in CSR form: row_ids[i] is
    request i, rendered with order_fields[order_offsets[i]:order_offsets[i+1]]."""

    def __init__(self, row_ids, order_offsets, order_fields):
        self.row_ids = np.ascontiguousarray(row_ids, dtype=np.uint64)
        self.order_offsets = np.ascontiguousarray(order_offsets, dtype=np.uint64)
        self.order_fields = np.ascontiguousarray(order_fields, dtype=np.int32)

    @classmethod
    def from_entries(cls, entries) -> "RequestSchedule":
        rows, offs, flds = [], [0], []
        for e in entries:
            r, fo = (e.row_id, e.field_order) if isinstance(e, ScheduleEntry) else e
            rows.append(int(r))
            flds.extend(int(f) for f in fo)
            offs.append(len(flds))
        return cls(np.array(rows, dtype=np.uint64), np.array(offs, dtype=np.uint64),
                   np.array(flds, dtype=np.int32))

    @classmethod
    def full(cls, row_ids: np.ndarray, field_orders: np.ndarray) -> "RequestSchedule":
        n, m = field_orders.shape
        return cls(row_ids, np.arange(n + 1, dtype=np.uint64) * m, field_orders.reshape(-1))

    def size(self) -> int:
        return int(self.row_ids.shape[0])

    __len__ = size

    @property
    def entries(self) -> list:
        o = self.order_offsets
        return [ScheduleEntry(int(self.row_ids[i]), self.order_fields[o[i]:o[i + 1]].tolist())
                for i in range(self.size())]


@dataclass
class SolveStats:
    """SolveStats (solve_result.hpp:9-14)."""
    recursive_calls: int = 0
    candidates_examined: int = 0
    max_depth: int = 0
    wall_ms: float = 0.0


@dataclass
class SolveResult:
    """SolveResult (solve_result.hpp:16-21)."""
    phc_score: int
    schedule: RequestSchedule
    stats: SolveStats
    optimal: bool = True


@dataclass
class FieldStats:
    name: bytes
    cardinality: int
    avg_len: float


@dataclass
class ColumnStats:
    """ColumnStats (stats.hpp:14-23)."""
    fields: list
    total_rows: int


# --------------------------------------------------------------------------
# marshalling
# --------------------------------------------------------------------------
def _cell_lens(t: Table, tok: Tokenizer, scoring: SegmentScoring):
    """Per-cell lengths for a custom tokenizer (the only host-side length
    computation; char/word lengths are computed on the GPU)."""
    if tok.kind != 2:
        return None
    n, m = t.row_count(), t.field_count()
    out = np.empty(n * m, dtype=np.uint64)
    for r in range(n):
        for f in range(m):
            out[r * m + f] = segment_len(t.field_name(f), t.cell(r, f), tok, scoring)
    return out


def _view(t: Table, tok: Tokenizer, scoring: SegmentScoring) -> TableView:
    return t.view(cell_lens=_cell_lens(t, tok, scoring))


def _fd_indices(t: Table, fds, cfg: GgrConfig) -> list:
    """Resolve FD names (ggr.hpp:154-164): only when use_fds, unknown names
    raise SchemaError via require_field."""
    if not cfg.use_fds or fds is None:
        return []
    groups = fds.groups if isinstance(fds, FunctionalDependencySet) else fds
    return [[t.require_field(nm) if not isinstance(nm, int) else nm for nm in g] for g in groups]


# --------------------------------------------------------------------------
# entry points
# --------------------------------------------------------------------------
def ggr(t: Table, fds=None, cfg: GgrConfig | None = None, tok: Tokenizer = _CHAR,
        scoring: SegmentScoring = SegmentScoring.value_only, stream: int = 0) -> SolveResult:
    """prefixopt::ggr (ggr.hpp:367-394) on the GPU."""
    cfg = cfg or GgrConfig()
    lib = cuda_lib()
    fdv = FdView(_fd_indices(t, fds, cfg))
    view = _view(t, tok, scoring)
    score = C.c_uint64(0)
    st = po_solve_stats()
    c = cfg.abi()
    # schedule handle with CSR field orders (FD groups sharing members make
    # some orders longer than the schema, ggr.hpp:280-282)
    h = C.c_void_p(0)
    lib.check(lib.ggr_schedule(view.ref(), fdv.ref(), C.byref(c), tok.kind, int(scoring),
                               C.byref(h), C.byref(score), C.byref(st), stream))
    try:
        ne, tot = C.c_uint64(0), C.c_uint64(0)
        lib.check(lib.schedule_info(h, C.byref(ne), C.byref(tot)))
        n, total = int(ne.value), int(tot.value)
        rows = np.empty(max(n, 1), dtype=np.uint64)
        offs = np.empty(n + 1, dtype=np.uint64)
        fields = np.empty(max(total, 1), dtype=np.int32)
        lib.check(lib.schedule_copy(h, PO_LOC_HOST, rows.ctypes.data, offs.ctypes.data,
                                    fields.ctypes.data, stream))
    finally:
        lib.schedule_free(h)
    sched = RequestSchedule(rows[:n], offs, fields[:total])
    return SolveResult(int(score.value), sched,
                       SolveStats(st.recursive_calls, st.candidates_examined, st.max_depth,
                                  st.wall_ms))


def _sched_args(s: RequestSchedule):
    return s.size(), s.row_ids.ctypes.data, s.order_offsets.ctypes.data, \
        (s.order_fields if s.order_fields.size else np.zeros(1, np.int32)).ctypes.data


def phc(s: RequestSchedule, t: Table, tok: Tokenizer = _CHAR,
        scoring: SegmentScoring = SegmentScoring.value_only, stream: int = 0) -> int:
    """prefixopt::phc (objective.hpp:94-99) on the GPU."""
    lib = cuda_lib()
    if not isinstance(s, RequestSchedule):
        s = RequestSchedule.from_entries(s)
    view = _view(t, tok, scoring)
    out = C.c_uint64(0)
    n, rp, op, fp = _sched_args(s)
    lib.check(lib.phc(view.ref(), tok.kind, int(scoring), n, rp, op, fp, PO_LOC_HOST,
                      C.byref(out), stream))
    return int(out.value)


def hit(s: RequestSchedule, r: int, t: Table, tok: Tokenizer = _CHAR,
        scoring: SegmentScoring = SegmentScoring.value_only, stream: int = 0) -> int:
    """prefixopt::hit (objective.hpp:70-91) on the GPU."""
    lib = cuda_lib()
    if not isinstance(s, RequestSchedule):
        s = RequestSchedule.from_entries(s)
    view = _view(t, tok, scoring)
    out = C.c_uint64(0)
    n, rp, op, fp = _sched_args(s)
    lib.check(lib.hit(view.ref(), tok.kind, int(scoring), n, rp, op, fp, PO_LOC_HOST, r,
                      C.byref(out), stream))
    return int(out.value)


def sort_rows_fixed_order(t: Table, field_order: Sequence[int], stream: int = 0) -> RequestSchedule:
    """prefixopt::sort_rows_fixed_order (objective.hpp:154-171) on the GPU."""
    lib = cuda_lib()
    fo = np.array(list(field_order) or [0], dtype=np.int32)
    m = t.field_count()
    if len(field_order) != m:  # validate_field_permutation (objective.hpp:140-142)
        raise SchemaError("field order must name every field exactly once")
    n = t.row_count()
    rows = np.empty(max(n, 1), dtype=np.uint64)
    view = t.view()
    lib.check(lib.sort_rows_fixed_order(view.ref(), fo.ctypes.data, PO_LOC_HOST,
                                        rows.ctypes.data, stream))
    orders = np.tile(fo[:m], (n, 1)) if n else np.zeros((0, m), np.int32)
    return RequestSchedule.full(rows[:n], orders)


def compute_stats(t: Table, tok: Tokenizer = _CHAR,
                  scoring: SegmentScoring = SegmentScoring.value_only, stream: int = 0) -> ColumnStats:
    """prefixopt::compute_stats (stats.hpp:25-45) on the GPU."""
    lib = cuda_lib()
    m, n = t.field_count(), t.row_count()
    card = np.zeros(max(m, 1), dtype=np.uint64)
    tot = np.zeros(max(m, 1), dtype=np.uint64)
    view = _view(t, tok, scoring)
    lib.check(lib.compute_stats(view.ref(), tok.kind, int(scoring), card.ctypes.data,
                                tot.ctypes.data, stream))
    fields = [FieldStats(t.field_name(f), int(card[f]), (float(tot[f]) / n) if n else 0.0)
              for f in range(m)]
    return ColumnStats(fields, n)


def _stats_arrays(stats: ColumnStats):
    m = len(stats.fields)
    card = np.array([fs.cardinality for fs in stats.fields] or [0], dtype=np.uint64)
    avg = np.array([fs.avg_len for fs in stats.fields] or [0.0], dtype=np.float64)
    return m, card, avg


def fixed_order_by_hitcount_stats(stats: ColumnStats, variant: StatsScoreVariant =
                                  StatsScoreVariant.cardinality_weighted_squared) -> list:
    """prefixopt::fixed_order_by_hitcount_stats (ggr.hpp:59-84)."""
    lib = cuda_lib()
    m, card, avg = _stats_arrays(stats)
    out = np.zeros(max(m, 1), dtype=np.int32)
    lib.check(lib.fixed_order_by_hitcount_stats(m, stats.total_rows, card.ctypes.data,
                                                avg.ctypes.data, int(variant), out.ctypes.data))
    return out[:m].tolist()


def fixed_order_by_stats(stats: ColumnStats) -> list:
    """prefixopt::fixed_order_by_stats (objective.hpp:176-188)."""
    lib = cuda_lib()
    m, card, avg = _stats_arrays(stats)
    out = np.zeros(max(m, 1), dtype=np.int32)
    lib.check(lib.fixed_order_by_stats(m, stats.total_rows, card.ctypes.data, avg.ctypes.data,
                                       out.ctypes.data))
    return out[:m].tolist()


def original_order_schedule(t: Table) -> RequestSchedule:
    """objective.hpp:55-62."""
    n, m = t.row_count(), t.field_count()
    return RequestSchedule.full(np.arange(n, dtype=np.uint64),
                                np.tile(np.arange(m, dtype=np.int32), (n, 1)))


@dataclass
class HitCountResult:
    score: float
    fields: list


def hitcount(t: Table, field_name, value, fds=None, tok: Tokenizer = _CHAR,
             scoring: SegmentScoring = SegmentScoring.value_only) -> HitCountResult:
    """prefixopt::hitcount (ggr.hpp:95-133). Not on the solver path (the
    solver never calls it); a single-value host
    computation kept for API compatibility."""
    c = t.require_field(field_name)
    fname = _to_bytes(field_name)
    inferred: list[int] = []
    groups = (fds.groups if isinstance(fds, FunctionalDependencySet) else fds) or []
    for g in groups:
        g = [_to_bytes(x) for x in g]
        if fname not in g:
            continue
        for nm in g:
            o = t.require_field(nm)
            if o != c:
                inferred.append(o)
        break
    inferred.sort()
    value = _to_bytes(value)
    count = 0
    inferred_total = 0
    for r in range(t.row_count()):
        if t.cell(r, c) != value:
            continue
        count += 1
        for o in inferred:
            inferred_total += segment_len(t.field_name(o), t.cell(r, o), tok, scoring)
    if count == 0:
        raise DomainError(f"hitcount: value does not occur in field {fname.decode('utf-8', 'replace')}")
    ln = float(segment_len(fname, value, tok, scoring))
    tot = ln * ln + float(inferred_total) / count
    return HitCountResult(tot * float(count - 1), [fname] + [t.field_name(o) for o in inferred])


# --------------------------------------------------------------------------
# functional dependencies (fd.hpp:28-141): signatures compared on the GPU
# --------------------------------------------------------------------------
@dataclass
class FdWitness:
    row_a: int
    row_b: int
    agree_field: object
    differ_field: object


@dataclass
class FdGroupReport:
    group: list
    satisfied: bool = False
    witness: FdWitness | None = None


@dataclass
class FdValidationReport:
    groups: list = field(default_factory=list)

    def all_satisfied(self) -> bool:
        return all(g.satisfied for g in self.groups)


def _fd_compare(t: Table, pa: list, pb: list):
    """po_fd_compare: first differing row of each pair's partition signatures
    (fd.hpp:56-64) and both signatures there."""
    n = t.row_count()
    k = len(pa)
    first = np.full(max(k, 1), n, dtype=np.uint64)
    sa = np.zeros(max(k, 1), dtype=np.uint64)
    sb = np.zeros(max(k, 1), dtype=np.uint64)
    if k:
        lib = cuda_lib()
        a = np.asarray(pa, dtype=np.int32)
        b = np.asarray(pb, dtype=np.int32)
        view = t.view()
        lib.check(lib.fd_compare(view.ref(), k, a.ctypes.data, b.ctypes.data, first.ctypes.data,
                                 sa.ctypes.data, sb.ctypes.data, 0))
    return first[:k], sa[:k], sb[:k]


def validate_fds(t: Table, fds) -> FdValidationReport:
    """prefixopt::validate_fds (fd.hpp:66-109)."""
    groups = fds.groups if isinstance(fds, FunctionalDependencySet) else (fds or [])
    claimed = set()
    for g in groups:
        for nm in g:
            t.require_field(nm)
            key = nm if isinstance(nm, bytes) else str(nm).encode()
            if key in claimed:
                raise SchemaError(f"field appears in more than one FD group: {key.decode('utf-8', 'replace')}")
            claimed.add(key)
    n = t.row_count()
    pa, pb, first_pair = [], [], []
    for g in groups:
        first_pair.append(len(pa))
        if len(g) >= 2 and n >= 2:
            for k in range(1, len(g)):
                pa.append(t.require_field(g[0]))
                pb.append(t.require_field(g[k]))
    diff, sa, sb = _fd_compare(t, pa, pb)
    rep = FdValidationReport()
    for gi, g in enumerate(groups):
        gr = FdGroupReport(list(g), True, None)
        if len(g) >= 2 and n >= 2:
            for k in range(1, len(g)):
                q = first_pair[gi] + k - 1
                r = int(diff[q])
                if r >= n:
                    continue
                gr.satisfied = False
                base_earlier = int(sa[q]) != r
                gr.witness = FdWitness(int(sa[q]) if base_earlier else int(sb[q]), r,
                                       g[0] if base_earlier else g[k],
                                       g[k] if base_earlier else g[0])
                break
        rep.groups.append(gr)
    return rep


def discover_fds(t: Table, max_rows: int = 10000) -> FunctionalDependencySet:
    """prefixopt::discover_fds (fd.hpp:114-141)."""
    n, m = t.row_count(), t.field_count()
    if n > max_rows:
        raise SizeError(f"discover_fds: table has {n} rows, cap is {max_rows}")
    pairs = [(i, j) for i in range(m) for j in range(i + 1, m)]
    diff, _, _ = _fd_compare(t, [p[0] for p in pairs], [p[1] for p in pairs])
    same = {p: int(d) >= n for p, d in zip(pairs, diff)}
    classes: list = []  # (first field, members)
    for f in range(m):
        for c in classes:
            if same[(c[0], f)]:
                c[1].append(t.field_name(f))
                break
        else:
            classes.append((f, [t.field_name(f)]))
    return FunctionalDependencySet([c[1] for c in classes if len(c[1]) >= 2], True)


# --------------------------------------------------------------------------
# prompt rendering and byte-exact dedup (objective.hpp:102-131, cost.hpp:171-186)
# --------------------------------------------------------------------------
def render_prompts_arena(s: RequestSchedule, t: Table, system_prompt: bytes = b"",
                         question: bytes = b"", stream: int = 0):
    """render_prompt of every entry on the GPU: (bytes arena, u64 offsets)."""
    lib = cuda_lib()
    view = t.view()
    n = s.size()
    _, rows_p, offs_p, flds_p = _sched_args(s)
    sp = _to_bytes(system_prompt)
    q = _to_bytes(question)
    sp_a = np.frombuffer(sp or b"\0", dtype=np.uint8)
    q_a = np.frombuffer(q or b"\0", dtype=np.uint8)
    out_off = np.zeros(n + 1, dtype=np.uint64)
    total = C.c_uint64(0)
    args = (view.ref(), n, rows_p, offs_p, flds_p, PO_LOC_HOST, sp_a.ctypes.data,
            len(sp), q_a.ctypes.data, len(q), PO_LOC_HOST, out_off.ctypes.data)
    lib.check(lib.render_prompts(*args, None, 0, C.byref(total), stream))
    arena = np.empty(max(int(total.value), 1), dtype=np.uint8)
    lib.check(lib.render_prompts(*args, arena.ctypes.data, arena.size, C.byref(total), stream))
    return arena[:int(total.value)], out_off


def render_prompts(s: RequestSchedule, t: Table, system_prompt: bytes = b"",
                   question: bytes = b"") -> list:
    """[render_prompt(e, t, system_prompt, question) for e in s] (objective.hpp:118-131)."""
    arena, off = render_prompts_arena(s, t, system_prompt, question)
    buf = arena.tobytes()
    return [buf[int(off[i]):int(off[i + 1])] for i in range(s.size())]


@dataclass
class DedupResult:
    uniques: list            # first-occurrence order
    expansion_map: list      # original index -> unique index


def dedup(prompts) -> DedupResult:
    """prefixopt::dedup (cost.hpp:171-186), byte-exact, on the GPU dictionary."""
    lib = cuda_lib()
    items = [_to_bytes(p) for p in prompts]
    n = len(items)
    offs = np.zeros(n + 1, dtype=np.uint64)
    if n:
        np.cumsum([len(x) for x in items], out=offs[1:])
    arena = np.frombuffer(b"".join(items) or b"\0", dtype=np.uint8)
    ex = np.zeros(max(n, 1), dtype=np.uint64)
    uf = np.zeros(max(n, 1), dtype=np.uint64)
    nu = C.c_uint64(0)
    lib.check(lib.dedup(n, arena.ctypes.data, offs.ctypes.data, PO_LOC_HOST, ex.ctypes.data,
                        uf.ctypes.data, C.byref(nu), 0))
    return DedupResult([items[int(i)] for i in uf[:int(nu.value)]], [int(x) for x in ex[:n]])


# --------------------------------------------------------------------------
# prefix-cache replay, unbounded cache (cache_sim.hpp:29-299)
# --------------------------------------------------------------------------
@dataclass
class CacheConfig:
    capacity_tokens: int = 0            # 0 = unbounded; ignored under eviction none
    eviction: str = "none"              # "none" | "lru"
    min_cacheable_prefix_tokens: int = 0


@dataclass
class RequestSim:
    input_tokens: int = 0
    hit_tokens: int = 0
    miss_tokens: int = 0
    written_tokens: int = 0
    uncacheable: bool = False


@dataclass
class SimReport:
    requests: list = field(default_factory=list)
    total_input: int = 0
    total_hit: int = 0
    total_miss: int = 0
    evicted_tokens: int = 0
    phr: float = 0.0


def _strings_arena(items):
    n = len(items)
    offs = np.zeros(n + 1, dtype=np.uint64)
    if n:
        np.cumsum([len(x) for x in items], out=offs[1:])
    return np.frombuffer(b"".join(items) or b"\0", dtype=np.uint8), offs


def simulate(prompts, cfg: CacheConfig | None = None, tok: Tokenizer = _CHAR) -> SimReport:
    """prefixopt::simulate (cache_sim.hpp:223-285) for eviction none on the
    GPU: raw hit = longest token prefix shared with any earlier prompt."""
    cfg = cfg or CacheConfig()
    items = [_to_bytes(p) for p in prompts]
    if not items:
        raise DomainError("simulate: prompt list is empty")
    if cfg.eviction not in ("none", "lru"):
        raise SchemaError(f"unknown eviction policy: {cfg.eviction} (expected 'none' or 'lru')")
    if cfg.eviction == "lru":
        if cfg.capacity_tokens == 0:
            raise SchemaError("simulate: lru eviction needs a finite capacity "
                              "(capacity 0 means unbounded, use eviction none)")
        raise SchemaError("simulate: lru eviction replays strictly sequentially; only eviction "
                          "none runs on the GPU")
    if tok.kind not in (0, 1):
        raise SchemaError("simulate: char or word tokenizer")
    lib = cuda_lib()
    n = len(items)
    arena, offs = _strings_arena(items)
    out = [np.zeros(n, dtype=np.uint64) for _ in range(4)]
    tot = np.zeros(3, dtype=np.uint64)
    lib.check(lib.replay_unbounded(n, arena.ctypes.data, offs.ctypes.data, PO_LOC_HOST, tok.kind,
                                   int(cfg.min_cacheable_prefix_tokens), *(o.ctypes.data for o in out),
                                   tot.ctypes.data, 0))
    reqs = [RequestSim(int(a), int(b), int(c), int(d)) for a, b, c, d in zip(*out)]
    ti, th, tm = (int(x) for x in tot)
    return SimReport(reqs, ti, th, tm, 0, th / ti if ti else 0.0)


def validate_schedule(s: RequestSchedule, t: Table) -> None:
    """prefixopt::validate_schedule (objective.hpp:34-52)."""
    n, m = t.row_count(), t.field_count()
    seen = set()
    for e in s.entries:
        r, order = e.row_id, e.field_order
        if r >= n:
            raise SchemaError(f"schedule references row {r} outside table of {n} rows")
        if r in seen:
            raise SchemaError(f"schedule lists row {r} twice")
        seen.add(r)
        if any(f < 0 or f >= m for f in order):
            raise SchemaError(f"schedule entry for row {r} names a field outside the schema")
        if len(set(order)) != len(order):
            raise SchemaError(f"schedule entry for row {r} repeats a field")


def phr_for_schedule(s: RequestSchedule, t: Table, system_prompt: bytes = b"",
                     question: bytes = b"", cfg: CacheConfig | None = None,
                     tok: Tokenizer = _CHAR) -> SimReport:
    """prefixopt::phr_for_schedule (cache_sim.hpp:290-299): render every entry
    (GPU) and replay (GPU, eviction none)."""
    validate_schedule(s, t)
    return simulate(render_prompts(s, t, system_prompt, question), cfg, tok)


# --------------------------------------------------------------------------
# CSV ingest (table.hpp:114-215)
# --------------------------------------------------------------------------
def load_csv(source) -> Table:
    """prefixopt::load_csv on the GPU: `source` is the CSV text (bytes) or a
    path. Same table and same errors as the reference."""
    if isinstance(source, (bytes, bytearray, memoryview)):
        data = bytes(source)
    else:
        with open(source, "rb") as fh:
            data = fh.read()
    lib = cuda_lib()
    buf = np.frombuffer(data or b"\0", dtype=np.uint8)
    h = C.c_void_p(0)
    lib.check(lib.load_csv(buf.ctypes.data, len(data), PO_LOC_HOST, C.byref(h), 0))
    try:
        rows, fields = C.c_uint64(0), C.c_uint32(0)
        ab, nb = C.c_uint64(0), C.c_uint64(0)
        lib.check(lib.csv_info(h, C.byref(rows), C.byref(fields), C.byref(ab), C.byref(nb)))
        n, m = int(rows.value), int(fields.value)
        arena = np.empty(max(int(ab.value), 1), dtype=np.uint8)
        offs = np.empty(n * m + 1, dtype=np.uint64)
        names = np.empty(max(int(nb.value), 1), dtype=np.uint8)
        noff = np.empty(m + 1, dtype=np.uint64)
        lib.check(lib.csv_copy(h, PO_LOC_HOST, arena.ctypes.data, offs.ctypes.data,
                               names.ctypes.data, noff.ctypes.data, 0))
    finally:
        lib.csv_free(h)
    nb_ = names.tobytes()
    field_names = [nb_[int(noff[f]):int(noff[f + 1])] for f in range(m)]
    return Table.from_arena(field_names, arena, offs, n)


def load_jsonl(source) -> Table:
    """prefixopt::load_jsonl (table.hpp:225-269): `source` is the JSONL text
    (bytes) or a path. Parsed on the host behind the C ABI (po_load_jsonl) with
    the reference's JSON library; same table and same errors as the reference."""
    if isinstance(source, (bytes, bytearray, memoryview)):
        data = bytes(source)
    else:
        with open(source, "rb") as fh:
            data = fh.read()
    lib = cuda_lib()
    buf = np.frombuffer(data or b"\0", dtype=np.uint8)
    h = C.c_void_p(0)
    lib.check(lib.load_jsonl(buf.ctypes.data, len(data), C.byref(h)))
    try:
        rows, fields = C.c_uint64(0), C.c_uint32(0)
        ab, nb = C.c_uint64(0), C.c_uint64(0)
        lib.check(lib.jsonl_info(h, C.byref(rows), C.byref(fields), C.byref(ab), C.byref(nb)))
        n, m = int(rows.value), int(fields.value)
        arena = np.empty(max(int(ab.value), 1), dtype=np.uint8)
        offs = np.empty(n * m + 1, dtype=np.uint64)
        names = np.empty(max(int(nb.value), 1), dtype=np.uint8)
        noff = np.empty(m + 1, dtype=np.uint64)
        lib.check(lib.jsonl_copy(h, arena.ctypes.data, offs.ctypes.data, names.ctypes.data,
                                 noff.ctypes.data))
    finally:
        lib.jsonl_free(h)
    nb_ = names.tobytes()
    field_names = [nb_[int(noff[f]):int(noff[f + 1])] for f in range(m)]
    return Table.from_arena(field_names, arena, offs, n)


# low-level entry for callers holding device buffers (bench.py, multi-GPU)
def ggr_into(view: TableView, fd_groups: list, cfg: GgrConfig, tok_kind: int, scoring: int,
             out_location: int, out_rows, out_orders, stream: int = 0):
    """po_ggr with caller-owned (host or device) buffers. Returns (phc, SolveStats)."""
    lib = cuda_lib()
    fdv = FdView(fd_groups)
    score = C.c_uint64(0)
    st = po_solve_stats()
    c = cfg.abi()
    lib.check(lib.ggr(view.ref(), fdv.ref(), C.byref(c), tok_kind, scoring, out_location,
                      _ptr(out_rows), _ptr(out_orders), C.byref(score), C.byref(st), stream))
    return int(score.value), SolveStats(st.recursive_calls, st.candidates_examined,
                                        st.max_depth, st.wall_ms)


__all__ = [
    "Table", "SegmentScoring", "StatsScoreVariant", "Tokenizer", "CharTokenizer",
    "WordTokenizer", "char_tokenizer", "word_tokenizer", "tokenizer_by_name",
    "scoring_by_name", "stats_variant_by_name", "json_escape", "fragment_text", "segment_len",
    "GgrConfig", "exact_config", "FunctionalDependencySet", "ScheduleEntry", "RequestSchedule",
    "SolveStats", "SolveResult", "FieldStats", "ColumnStats", "ggr", "phc", "hit",
    "sort_rows_fixed_order", "compute_stats", "fixed_order_by_hitcount_stats",
    "fixed_order_by_stats", "original_order_schedule", "hitcount", "HitCountResult", "ggr_into",
    "PO_LOC_HOST", "PO_LOC_DEVICE", "FdWitness", "FdGroupReport", "FdValidationReport",
    "validate_fds", "discover_fds", "render_prompts", "render_prompts_arena", "DedupResult",
    "dedup", "CacheConfig", "RequestSim", "SimReport", "simulate", "validate_schedule",
    "phr_for_schedule", "load_csv", "load_jsonl",
]
