"""Table: the immutable grid of byte-string cells the path reorders.

Mirrors prefixopt::Table (table.hpp:24-104): named fields, rows in ingestion
order (row ids never change), cells are opaque bytes. Storage is the
boundary's columnar-arena form instead of a vector of vectors: one byte arena
with cells in row-major order and n*m+1 u64 offsets, which is exactly what
the C ABI (po_table) consumes and what is copied to HBM.
"""
from __future__ import annotations

from typing import Iterable, Sequence

import numpy as np

from ._abi import PO_LOC_HOST, TableView
from .errors import SchemaError, StructuralError


def _to_bytes(x) -> bytes:
    if isinstance(x, bytes):
        return x
    if isinstance(x, (bytearray, memoryview)):
        return bytes(x)
    return str(x).encode("utf-8")


class Table:
    """prefixopt::Table (table.hpp:24-104)."""

    def __init__(self, field_names: Sequence, rows: Iterable[Sequence] = ()):
        names = [_to_bytes(n) for n in field_names]
        self._set_names(names)
        cells: list[bytes] = []
        n = 0
        for r, row in enumerate(rows):
            row = list(row)
            if len(row) != len(names):  # table.hpp:36-41
                raise StructuralError(
                    f"row {r} has {len(row)} cells, expected {len(names)}")
            cells.extend(_to_bytes(c) for c in row)
            n += 1
        lens = np.fromiter((len(c) for c in cells), dtype=np.uint64, count=len(cells))
        offsets = np.zeros(len(cells) + 1, dtype=np.uint64)
        np.cumsum(lens, out=offsets[1:])
        self._arena = np.frombuffer(b"".join(cells), dtype=np.uint8).copy() if cells else \
            np.zeros(0, dtype=np.uint8)
        self._offsets = offsets
        self._n = n

    def _set_names(self, names: list[bytes]) -> None:
        seen = set()
        for i, nm in enumerate(names):  # table.hpp:28-35
            if not nm:
                raise SchemaError(f"field {i} has an empty name")
            if nm in seen:
                raise SchemaError(f"duplicate field name: {nm.decode('utf-8', 'replace')}")
            seen.add(nm)
        self._names = names
        self._index = {nm: i for i, nm in enumerate(names)}

    @classmethod
    def from_arena(cls, field_names: Sequence, arena: np.ndarray, offsets: np.ndarray,
                   n_rows: int) -> "Table":
        """Wrap an existing row-major arena (generators, loaders)."""
        t = cls.__new__(cls)
        t._set_names([_to_bytes(n) for n in field_names])
        m = len(t._names)
        arena = np.ascontiguousarray(arena, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        if offsets.shape[0] != n_rows * m + 1:
            raise StructuralError(f"offsets has {offsets.shape[0]} entries, expected {n_rows * m + 1}")
        if n_rows * m and (offsets[0] != 0 or int(offsets[-1]) > arena.shape[0]
                           or np.any(offsets[1:] < offsets[:-1])):
            raise StructuralError("offsets are not a non-decreasing cover of the arena")
        t._arena, t._offsets, t._n = arena, offsets, int(n_rows)
        return t

    def row_slice(self, lo: int, hi: int) -> "Table":
        """Rows [lo, hi) as a table of their own (one rank's shard)."""
        m = len(self._names)
        lo, hi = max(0, lo), min(self._n, hi)
        hi = max(lo, hi)
        if m == 0:
            return Table.from_arena(self._names, np.zeros(0, np.uint8), np.zeros(1, np.uint64),
                                    hi - lo)
        a, b = int(self._offsets[lo * m]), int(self._offsets[hi * m])
        return Table.from_arena(self._names, self._arena[a:b], self._offsets[lo * m:hi * m + 1] - a,
                                hi - lo)

    # --- accessors (table.hpp:44-66) -------------------------------------
    def row_count(self) -> int:
        return self._n

    def field_count(self) -> int:
        return len(self._names)

    @property
    def field_names(self) -> list[bytes]:
        return list(self._names)

    def field_name(self, f: int) -> bytes:
        return self._names[f]

    def field_index(self, name) -> int:
        return self._index.get(_to_bytes(name), -1)

    def require_field(self, name) -> int:
        f = self.field_index(name)
        if f < 0:
            raise SchemaError(f"unknown field: {_to_bytes(name).decode('utf-8', 'replace')}")
        return f

    def cell(self, r: int, f: int) -> bytes:
        m = len(self._names)
        if not (0 <= r < self._n and 0 <= f < m):
            raise IndexError("cell index out of range")
        i = r * m + f
        return self._arena[int(self._offsets[i]):int(self._offsets[i + 1])].tobytes()

    def row(self, r: int) -> list[bytes]:
        return [self.cell(r, f) for f in range(len(self._names))]

    # --- boundary form ---------------------------------------------------
    @property
    def arena(self) -> np.ndarray:
        return self._arena

    @property
    def offsets(self) -> np.ndarray:
        return self._offsets

    @property
    def cell_bytes(self) -> int:
        return int(self._offsets[-1]) if self._offsets.shape[0] else 0

    def view(self, location: int = PO_LOC_HOST, arena=None, offsets=None, cell_lens=None) -> TableView:
        """ABI view. With location=PO_LOC_DEVICE pass device copies of arena
        and offsets (torch tensors or raw pointers)."""
        return TableView(self._names, self._n,
                         self._arena if arena is None else arena,
                         self._offsets if offsets is None else offsets,
                         location, cell_lens)
