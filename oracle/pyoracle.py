"""ORACLE — TEST INFRASTRUCTURE ONLY.

Python bindings of the CPU checkers (oracle/oracle.h):
  kind="port"       oracle/libggr_oracle.so   the CPU restatement
  kind="reference"  oracle/_ref/libggr_ref.so the reference headers compiled
                                              from /root/reference
Used by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
--impl reference legs. The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2403_05821_b200._abi import FdView, _bind, po_ggr_config, po_solve_stats
from paper_2403_05821_b200.api import (GgrConfig, RequestSchedule, SegmentScoring, SolveResult,
                                       SolveStats, _cell_lens, _fd_indices)
from paper_2403_05821_b200.errors import raise_for

ORACLE_DIR = Path(__file__).resolve().parent
PATHS = {
    "port": ORACLE_DIR / "libggr_oracle.so",
    "reference": ORACLE_DIR / "_ref" / "libggr_ref.so",
}
PREFIX = {"port": "oracle_", "reference": "ref_"}


class OracleLib:
    def __init__(self, kind: str):
        path = PATHS[kind]
        if not path.exists():
            raise FileNotFoundError(
                f"{path} not built (make -C oracle{' ref' if kind == 'reference' else ''})")
        self.kind = kind
        self.path = path
        L = C.CDLL(str(path))
        p = PREFIX[kind]
        vp = C.c_void_p
        self._ggr = _bind(L, p + "ggr", C.c_int,
                          [vp, vp, vp, C.c_int32, C.c_int32, vp, vp, vp, C.c_uint64, vp, vp])
        self._phc = _bind(L, p + "phc", C.c_int, [vp, C.c_int32, C.c_int32, C.c_uint64, vp, vp, vp, vp])
        self._sort = _bind(L, p + "sort_rows_fixed_order", C.c_int, [vp, vp, vp])
        self._stats = _bind(L, p + "compute_stats", C.c_int, [vp, C.c_int32, C.c_int32, vp, vp])
        self._fohs = _bind(L, p + "fixed_order_by_hitcount_stats", C.c_int,
                           [C.c_uint32, C.c_uint64, vp, vp, C.c_int32, vp])
        self._vfd = _bind(L, p + "validate_fds", C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp])
        self._dfd = _bind(L, p + "discover_fds", C.c_int, [vp, C.c_uint64, vp])
        self._render = _bind(L, p + "render_prompts", C.c_int,
                             [vp, C.c_uint64, vp, vp, vp, vp, C.c_uint64, vp, C.c_uint64, vp, vp,
                              C.c_uint64, vp])
        self._dedup = _bind(L, p + "dedup", C.c_int, [C.c_uint64, vp, vp, vp, vp, vp])
        self._err = _bind(L, p + "last_error", C.c_char_p, [])

    def _check(self, code):
        if code:
            raise_for(code, (self._err() or b"").decode("utf-8", "replace"))

    # same call shapes as paper_2403_05821_b200.api
    def ggr(self, t, fds=None, cfg: GgrConfig | None = None, tok=None,
            scoring=SegmentScoring.value_only) -> SolveResult:
        from paper_2403_05821_b200.api import char_tokenizer
        cfg = cfg or GgrConfig()
        tok = tok or char_tokenizer()
        n, m = t.row_count(), t.field_count()
        groups = _fd_indices(t, fds, cfg)
        fdv = FdView(groups)
        view = t.view(cell_lens=_cell_lens(t, tok, scoring))
        # a row's order holds every field plus repeated FD partners (groups
        # sharing members, ggr.hpp:280-282): m + sum of group sizes bounds it
        cap = max(n * (m + sum(len(g) for g in groups)), 1)
        rows = np.empty(max(n, 1), dtype=np.uint64)
        offs = np.zeros(n + 1, dtype=np.uint64)
        fields = np.empty(cap, dtype=np.int32)
        score = C.c_uint64(0)
        st = po_solve_stats()
        c = cfg.abi()
        self._check(self._ggr(view.ref(), fdv.ref(), C.byref(c), tok.kind, int(scoring),
                              rows.ctypes.data, offs.ctypes.data, fields.ctypes.data, cap,
                              C.byref(score), C.byref(st)))
        sched = RequestSchedule(rows[:n], offs, fields[:int(offs[-1])])
        return SolveResult(int(score.value), sched,
                           SolveStats(st.recursive_calls, st.candidates_examined, st.max_depth,
                                      st.wall_ms))

    def phc(self, s, t, tok=None, scoring=SegmentScoring.value_only) -> int:
        from paper_2403_05821_b200.api import char_tokenizer
        tok = tok or char_tokenizer()
        if not isinstance(s, RequestSchedule):
            s = RequestSchedule.from_entries(s)
        view = t.view(cell_lens=_cell_lens(t, tok, scoring))
        out = C.c_uint64(0)
        flds = s.order_fields if s.order_fields.size else np.zeros(1, np.int32)
        self._check(self._phc(view.ref(), tok.kind, int(scoring), s.size(), s.row_ids.ctypes.data,
                              s.order_offsets.ctypes.data, flds.ctypes.data, C.byref(out)))
        return int(out.value)

    def sort_rows_fixed_order(self, t, field_order) -> np.ndarray:
        fo = np.array(list(field_order) or [0], dtype=np.int32)
        rows = np.empty(max(t.row_count(), 1), dtype=np.uint64)
        view = t.view()
        self._check(self._sort(view.ref(), fo.ctypes.data, rows.ctypes.data))
        return rows[:t.row_count()]

    def compute_stats(self, t, tok=None, scoring=SegmentScoring.value_only):
        from paper_2403_05821_b200.api import char_tokenizer
        tok = tok or char_tokenizer()
        m = t.field_count()
        card = np.zeros(max(m, 1), dtype=np.uint64)
        tot = np.zeros(max(m, 1), dtype=np.uint64)
        view = t.view(cell_lens=_cell_lens(t, tok, scoring))
        self._check(self._stats(view.ref(), tok.kind, int(scoring), card.ctypes.data,
                                tot.ctypes.data))
        return card[:m], tot[:m]

    def fixed_order_by_hitcount_stats(self, total_rows, card, avg, variant=0):
        m = len(card)
        c = np.array(list(card) or [0], dtype=np.uint64)
        a = np.array(list(avg) or [0.0], dtype=np.float64)
        out = np.zeros(max(m, 1), dtype=np.int32)
        self._check(self._fohs(m, total_rows, c.ctypes.data, a.ctypes.data, variant,
                               out.ctypes.data))
        return out[:m].tolist()


_LIBS: dict = {}


def oracle(kind: str = "port") -> OracleLib:
    if kind not in _LIBS:
        _LIBS[kind] = OracleLib(kind)
    return _LIBS[kind]


def available(kind: str) -> bool:
    return PATHS[kind].exists()


def _fd_oracle_methods():
    """validate_fds / discover_fds on the oracle libraries, with the same
    result types as paper_2403_05821_b200.api."""
    from paper_2403_05821_b200.api import (FdGroupReport, FdValidationReport, FdWitness,
                                           FunctionalDependencySet)

    def validate_fds(self, t, fds):
        groups = fds.groups if isinstance(fds, FunctionalDependencySet) else (fds or [])
        idx = [[t.require_field(nm) for nm in g] for g in groups]
        k = max(len(groups), 1)
        sat = np.zeros(k, np.uint8)
        hw = np.zeros(k, np.uint8)
        ra = np.zeros(k, np.uint64)
        rb = np.zeros(k, np.uint64)
        ag = np.zeros(k, np.int32)
        df = np.zeros(k, np.int32)
        view = t.view()
        self._check(self._vfd(view.ref(), FdView(idx).ref(), sat.ctypes.data, hw.ctypes.data,
                              ra.ctypes.data, rb.ctypes.data, ag.ctypes.data, df.ctypes.data))
        rep = FdValidationReport()
        for g, grp in enumerate(groups):
            w = None
            if hw[g]:
                pos = {f: i for i, f in enumerate(idx[g])}
                w = FdWitness(int(ra[g]), int(rb[g]), grp[pos[int(ag[g])]], grp[pos[int(df[g])]])
            rep.groups.append(FdGroupReport(list(grp), bool(sat[g]), w))
        return rep

    def discover_fds(self, t, max_rows=10000):
        m = t.field_count()
        out = np.zeros(max(m, 1), np.int32)
        view = t.view()
        self._check(self._dfd(view.ref(), max_rows, out.ctypes.data))
        ng = int(out[:m].max()) + 1 if m else 0
        groups = [[t.field_name(f) for f in range(m) if out[f] == g] for g in range(ng)]
        return FunctionalDependencySet(groups, True)

    OracleLib.validate_fds = validate_fds
    OracleLib.discover_fds = discover_fds


_fd_oracle_methods()


def _render_dedup_oracle_methods():
    from paper_2403_05821_b200.api import DedupResult, _sched_args
    from paper_2403_05821_b200.table import _to_bytes

    def render_prompts(self, s, t, system_prompt=b"", question=b""):
        view = t.view()
        n = s.size()
        _, rows_p, offs_p, flds_p = _sched_args(s)
        sp, q = _to_bytes(system_prompt), _to_bytes(question)
        sp_a = np.frombuffer(sp or b"\0", dtype=np.uint8)
        q_a = np.frombuffer(q or b"\0", dtype=np.uint8)
        out_off = np.zeros(n + 1, dtype=np.uint64)
        total = C.c_uint64(0)
        args = (view.ref(), n, rows_p, offs_p, flds_p,
                sp_a.ctypes.data, len(sp), q_a.ctypes.data, len(q), out_off.ctypes.data)
        self._check(self._render(*args, None, 0, C.byref(total)))
        arena = np.empty(max(int(total.value), 1), dtype=np.uint8)
        self._check(self._render(*args, arena.ctypes.data, arena.size, C.byref(total)))
        buf = arena.tobytes()
        return [buf[int(out_off[i]):int(out_off[i + 1])] for i in range(n)]

    def dedup(self, prompts):
        items = [_to_bytes(p) for p in prompts]
        n = len(items)
        offs = np.zeros(n + 1, dtype=np.uint64)
        if n:
            np.cumsum([len(x) for x in items], out=offs[1:])
        arena = np.frombuffer(b"".join(items) or b"\0", dtype=np.uint8)
        ex = np.zeros(max(n, 1), dtype=np.uint64)
        uf = np.zeros(max(n, 1), dtype=np.uint64)
        nu = C.c_uint64(0)
        self._check(self._dedup(n, arena.ctypes.data, offs.ctypes.data, ex.ctypes.data,
                                uf.ctypes.data, C.byref(nu)))
        return DedupResult([items[int(i)] for i in uf[:int(nu.value)]], [int(x) for x in ex[:n]])

    OracleLib.render_prompts = render_prompts
    OracleLib.dedup = dedup


_render_dedup_oracle_methods()


def _simulate_oracle_methods():
    """simulate (cache_sim.hpp:223-285): the reference itself through the
    shim (ref_simulate), and for kind="port" a brute-force restatement for
    eviction none: raw hit = max over earlier prompts of the common token
    prefix (what an unbounded trie returns)."""
    from paper_2403_05821_b200.api import CacheConfig, RequestSim, SimReport
    from paper_2403_05821_b200.errors import DomainError
    from paper_2403_05821_b200.table import _to_bytes

    WS = set(b" \t\n\r\f\v")

    def tokens(p, kind):  # tokenizer.hpp:33-73
        if kind == 0:
            return list(p)
        out, cur = [], bytearray()
        for c in p:
            if c in WS:
                if cur:
                    out.append(bytes(cur))
                    cur = bytearray()
            else:
                cur.append(c)
        if cur:
            out.append(bytes(cur))
        return out

    def simulate(self, prompts, cfg=None, tok=None):
        from paper_2403_05821_b200.api import char_tokenizer
        cfg = cfg or CacheConfig()
        tok = tok or char_tokenizer()
        items = [_to_bytes(p) for p in prompts]
        if not items:
            raise DomainError("simulate: prompt list is empty")
        if self.kind == "reference":
            n = len(items)
            offs = np.zeros(n + 1, np.uint64)
            np.cumsum([len(x) for x in items], out=offs[1:])
            arena = np.frombuffer(b"".join(items) or b"\0", np.uint8)
            outs = [np.zeros(n, np.uint64) for _ in range(4)]
            unc = np.zeros(n, np.uint8)
            tot = np.zeros(4, np.uint64)
            fn = _bind(C.CDLL(str(self.path)), "ref_simulate", C.c_int,
                       [C.c_uint64, C.c_void_p, C.c_void_p, C.c_int32, C.c_uint64, C.c_int32,
                        C.c_uint64] + [C.c_void_p] * 6)
            self._check(fn(n, arena.ctypes.data, offs.ctypes.data, tok.kind, cfg.capacity_tokens,
                           1 if cfg.eviction == "lru" else 0, cfg.min_cacheable_prefix_tokens,
                           *(o.ctypes.data for o in outs), unc.ctypes.data, tot.ctypes.data))
            reqs = [RequestSim(int(a), int(b), int(c), int(d), bool(u))
                    for a, b, c, d, u in zip(*outs, unc)]
            ti, th, tm, ev = (int(x) for x in tot)
            return SimReport(reqs, ti, th, tm, ev, th / ti if ti else 0.0)
        seqs = [tokens(p, tok.kind) for p in items]
        reqs = []
        for i, sq in enumerate(seqs):
            raw = 0
            for j in range(i):
                o = seqs[j]
                k = 0
                while k < len(sq) and k < len(o) and sq[k] == o[k]:
                    k += 1
                raw = max(raw, k)
            hit = raw if raw >= cfg.min_cacheable_prefix_tokens else 0
            reqs.append(RequestSim(len(sq), hit, len(sq) - hit, len(sq) - raw))
        ti = sum(r.input_tokens for r in reqs)
        th = sum(r.hit_tokens for r in reqs)
        return SimReport(reqs, ti, th, ti - th, 0, th / ti if ti else 0.0)

    OracleLib.simulate = simulate


_simulate_oracle_methods()


def _csv_oracle_methods():
    """load_csv (table.hpp:114-215): the reference itself through the shim;
    for kind="port" a restatement of detail::read_csv_record + load_csv."""
    from paper_2403_05821_b200.errors import SchemaError, StructuralError
    from paper_2403_05821_b200.table import Table

    def read_record(d, i, line):
        # table.hpp:117-178: returns (cells, i, line, blank, start_line) or None at EOF
        if i >= len(d):
            return None
        cells, cell = [], bytearray()
        quoted = any_quote = any_content = False
        start = line
        while True:
            if i >= len(d):
                if quoted:
                    raise StructuralError(
                        f"csv: unterminated quoted field starting near line {start}")
                cells.append(bytes(cell))
                return cells, i, line, (not any_quote and len(cells) == 1 and not cells[0]), start
            ch = d[i]
            i += 1
            if quoted:
                if ch == 0x22:
                    if i < len(d) and d[i] == 0x22:
                        cell.append(0x22)
                        i += 1
                    else:
                        quoted = False
                else:
                    if ch == 0x0A:
                        line += 1
                    cell.append(ch)
            elif ch == 0x22 and not cell and not any_content:
                quoted = any_quote = any_content = True
            elif ch == 0x2C:
                cells.append(bytes(cell))
                cell = bytearray()
                any_content = False
            elif ch == 0x0D or ch == 0x0A:
                if ch == 0x0D and i < len(d) and d[i] == 0x0A:
                    i += 1
                line += 1
                cells.append(bytes(cell))
                return cells, i, line, (not any_quote and len(cells) == 1 and not cells[0]), start
            else:
                cell.append(ch)
                any_content = True

    def ref_loader(self, symbol, data):
        fn = _bind(C.CDLL(str(self.path)), symbol, C.c_int, [C.c_void_p, C.c_uint64] + [C.c_void_p] * 8)
        buf = np.frombuffer(data or b"\0", np.uint8)
        rows, fields = C.c_uint64(0), C.c_uint32(0)
        ab, nb = C.c_uint64(0), C.c_uint64(0)
        args = (buf.ctypes.data, len(data), C.byref(rows), C.byref(fields), C.byref(ab),
                C.byref(nb))
        self._check(fn(*args, None, None, None, None))
        n, m = int(rows.value), int(fields.value)
        arena = np.zeros(max(int(ab.value), 1), np.uint8)
        offs = np.zeros(n * m + 1, np.uint64)
        names = np.zeros(max(int(nb.value), 1), np.uint8)
        noff = np.zeros(m + 1, np.uint64)
        self._check(fn(*args, arena.ctypes.data, offs.ctypes.data, names.ctypes.data,
                       noff.ctypes.data))
        nb_ = names.tobytes()
        return Table.from_arena([nb_[int(noff[f]):int(noff[f + 1])] for f in range(m)],
                                arena, offs, n)

    def load_jsonl(self, data):
        """load_jsonl (table.hpp:225-269): the reference itself only (its
        behaviour is nlohmann::json's parser and serializer; no restatement)."""
        if self.kind != "reference":
            raise NotImplementedError("load_jsonl has no port restatement; use the reference")
        return ref_loader(self, "ref_load_jsonl", bytes(data))

    def load_csv(self, data):
        data = bytes(data)
        if self.kind == "reference":
            return ref_loader(self, "ref_load_csv", data)
        first = read_record(data, 0, 1)
        if first is None:
            raise StructuralError("csv: missing header row")
        header, i, line, _, _ = first
        seen = set()
        for nm in header:
            if nm in seen:
                raise SchemaError(f"csv: duplicate header field: {nm.decode('latin-1')}")
            seen.add(nm)
        rows = []
        while True:
            rec = read_record(data, i, line)
            if rec is None:
                break
            cells, i, line, blank, start = rec
            if blank and i >= len(data):
                break
            if len(cells) != len(header):
                raise StructuralError(f"csv: line {start} has {len(cells)} cells, "
                                      f"expected {len(header)}")
            rows.append(cells)
        for k, nm in enumerate(header):
            if not nm:
                raise SchemaError(f"field {k} has an empty name")
        return Table(header, rows)

    OracleLib.load_csv = load_csv
    OracleLib.load_jsonl = load_jsonl


_csv_oracle_methods()
