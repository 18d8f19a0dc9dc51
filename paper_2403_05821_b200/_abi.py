"""ctypes mirror of include/prefixopt_cuda.h and the loaders for the shared
libraries that export it.

`cuda_lib()` loads the product library (libprefixopt_cuda.so, built in-tree
by __graft_entry__.build()). It raises ExtensionMissing when the library is
absent: there is no CPU fallback on the product path.

The CPU checkers live in oracle/ (oracle/pyoracle.py) and are not imported
from this package.
"""
from __future__ import annotations

import ctypes as C
import re
import os
from pathlib import Path

import numpy as np

from .errors import ExtensionMissing, raise_for

PKG_DIR = Path(__file__).resolve().parent
REPO_ROOT = PKG_DIR.parent
CUDA_LIB_PATH = PKG_DIR / "libprefixopt_cuda.so"

PO_LOC_HOST = 0
PO_LOC_DEVICE = 1

u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)


class po_table(C.Structure):
    _fields_ = [
        ("n_rows", C.c_uint64),
        ("n_fields", C.c_uint32),
        ("location", C.c_uint32),
        ("field_names", C.POINTER(C.c_char_p)),
        ("field_name_lens", u64p),
        ("arena", C.c_void_p),
        ("offsets", C.c_void_p),
        ("cell_lens", C.c_void_p),
    ]


class po_ggr_config(C.Structure):
    _fields_ = [
        ("row_recursion_depth", C.c_uint64),
        ("column_recursion_depth", C.c_uint64),
        ("hitcount_stop_threshold", C.c_uint64),
        ("use_fds", C.c_int32),
        ("stats_variant", C.c_int32),
    ]


class po_fd_groups(C.Structure):
    _fields_ = [
        ("n_groups", C.c_uint32),
        ("group_offsets", C.POINTER(C.c_uint32)),
        ("members", i32p),
    ]


class po_solve_stats(C.Structure):
    _fields_ = [
        ("recursive_calls", C.c_uint64),
        ("candidates_examined", C.c_uint64),
        ("max_depth", C.c_uint64),
        ("wall_ms", C.c_double),
    ]


def _ptr(x) -> int:
    """Address of a numpy array, a torch tensor or an int."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    raise TypeError(f"cannot take the address of {type(x)}")


class TableView:
    """Keeps the ctypes view of a table (and everything it points to) alive."""

    def __init__(self, field_names: list[bytes], n_rows: int, arena, offsets,
                 location: int = PO_LOC_HOST, cell_lens=None):
        self._names = [bytes(n) for n in field_names]
        m = len(self._names)
        self._name_arr = (C.c_char_p * max(m, 1))(*self._names)
        self._name_lens = np.array([len(n) for n in self._names] or [0], dtype=np.uint64)
        self._keep = (arena, offsets, cell_lens)
        self.view = po_table(
            n_rows=n_rows,
            n_fields=m,
            location=location,
            field_names=C.cast(self._name_arr, C.POINTER(C.c_char_p)),
            field_name_lens=self._name_lens.ctypes.data_as(u64p),
            arena=_ptr(arena),
            offsets=_ptr(offsets),
            cell_lens=_ptr(cell_lens),
        )

    def ref(self):
        return C.byref(self.view)


class FdView:
    def __init__(self, groups: list[list[int]]):
        offs = [0]
        mem: list[int] = []
        for g in groups:
            mem.extend(int(x) for x in g)
            offs.append(len(mem))
        self._offs = np.array(offs, dtype=np.uint32)
        self._mem = np.array(mem or [0], dtype=np.int32)
        self.view = po_fd_groups(
            n_groups=len(groups),
            group_offsets=self._offs.ctypes.data_as(C.POINTER(C.c_uint32)),
            members=self._mem.ctypes.data_as(i32p),
        )

    def ref(self):
        return C.byref(self.view)


def _bind(lib, name, restype, argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = argtypes
    return fn


class CudaLib:
    """The product library (include/prefixopt_cuda.h)."""

    def __init__(self, path: Path = CUDA_LIB_PATH):
        if not path.exists():
            raise ExtensionMissing(
                f"{path} is not built; run __graft_entry__.build() (no CPU fallback exists)")
        try:
            self.lib = C.CDLL(str(path), mode=C.RTLD_GLOBAL)
        except OSError as e:  # pragma: no cover - depends on the box
            raise ExtensionMissing(f"cannot load {path}: {e}") from e
        L = self.lib
        vp = C.c_void_p
        self.ggr = _bind(L, "po_ggr", C.c_int, [vp, vp, vp, C.c_int32, C.c_int32, C.c_uint32,
                                                 vp, vp, vp, vp, vp])
        self.phc = _bind(L, "po_phc", C.c_int, [vp, C.c_int32, C.c_int32, C.c_uint64, vp, vp,
                                                 vp, C.c_uint32, vp, vp])
        self.hit = _bind(L, "po_hit", C.c_int, [vp, C.c_int32, C.c_int32, C.c_uint64, vp, vp,
                                                 vp, C.c_uint32, C.c_uint64, vp, vp])
        self.sort_rows_fixed_order = _bind(L, "po_sort_rows_fixed_order", C.c_int,
                                           [vp, vp, C.c_uint32, vp, vp])
        self.compute_stats = _bind(L, "po_compute_stats", C.c_int,
                                   [vp, C.c_int32, C.c_int32, vp, vp, vp])
        self.fixed_order_by_hitcount_stats = _bind(
            L, "po_fixed_order_by_hitcount_stats", C.c_int,
            [C.c_uint32, C.c_uint64, vp, vp, C.c_int32, vp])
        self.fixed_order_by_stats = _bind(L, "po_fixed_order_by_stats", C.c_int,
                                          [C.c_uint32, C.c_uint64, vp, vp, vp])
        self.fd_compare = _bind(L, "po_fd_compare", C.c_int,
                                [vp, C.c_uint32, vp, vp, vp, vp, vp, vp])
        self.render_prompts = _bind(L, "po_render_prompts", C.c_int,
                                    [vp, C.c_uint64, vp, vp, vp, C.c_uint32, vp, C.c_uint64, vp,
                                     C.c_uint64, C.c_uint32, vp, vp, C.c_uint64, vp, vp])
        self.dedup = _bind(L, "po_dedup", C.c_int, [C.c_uint64, vp, vp, C.c_uint32, vp, vp, vp, vp])
        self.replay_unbounded = _bind(L, "po_replay_unbounded", C.c_int,
                                      [C.c_uint64, vp, vp, C.c_uint32, C.c_int32, C.c_uint64,
                                       vp, vp, vp, vp, vp, vp])
        self.load_csv = _bind(L, "po_load_csv", C.c_int, [vp, C.c_uint64, C.c_uint32,
                                                          C.POINTER(vp), vp])
        self.csv_info = _bind(L, "po_csv_info", C.c_int, [vp, vp, vp, vp, vp])
        self.csv_copy = _bind(L, "po_csv_copy", C.c_int, [vp, C.c_uint32, vp, vp, vp, vp, vp])
        self.csv_free = _bind(L, "po_csv_free", None, [vp])
        self.load_jsonl = _bind(L, "po_load_jsonl", C.c_int, [vp, C.c_uint64, vp])
        self.jsonl_info = _bind(L, "po_jsonl_info", C.c_int, [vp, vp, vp, vp, vp])
        self.jsonl_copy = _bind(L, "po_jsonl_copy", C.c_int, [vp, vp, vp, vp, vp])
        self.jsonl_free = _bind(L, "po_jsonl_free", None, [vp])
        # row-sharded solve
        self.comm_unique_id = _bind(L, "po_comm_unique_id", C.c_int, [vp])
        self.comm_init_nccl = _bind(L, "po_comm_init_nccl", C.c_int,
                                    [vp, C.c_int32, C.c_int32, C.POINTER(vp)])
        self.comm_init_local = _bind(L, "po_comm_init_local", C.c_int, [C.c_int32, vp])
        self.comm_destroy = _bind(L, "po_comm_destroy", C.c_int, [vp])
        self.ggr_schedule = _bind(L, "po_ggr_schedule", C.c_int,
                                  [vp, vp, vp, C.c_int32, C.c_int32, vp, vp, vp, vp])
        self.schedule_info = _bind(L, "po_schedule_info", C.c_int, [vp, vp, vp])
        self.schedule_copy = _bind(L, "po_schedule_copy", C.c_int, [vp, C.c_uint32, vp, vp, vp, vp])
        self.schedule_free = _bind(L, "po_schedule_free", None, [vp])
        self.debug_radix_sort = _bind(L, "po_debug_radix_sort", C.c_int,
                                      [vp, vp, C.c_uint64, C.c_int32, C.c_int32, vp, vp])
        self.debug_merge_sort = _bind(L, "po_debug_merge_sort", C.c_int,
                                      [vp, vp, vp, C.c_uint64, vp, vp, vp])
        self.comm_init_host = _bind(L, "po_comm_init_host", C.c_int,
                                    [vp, C.c_int32, C.c_int32, vp])
        self.ggr_sharded = _bind(L, "po_ggr_sharded", C.c_int,
                                 [vp, vp, vp, vp, C.c_int32, C.c_int32, C.POINTER(vp), vp, vp, vp])
        self.slice_info = _bind(L, "po_slice_info", C.c_int, [vp, vp, vp])
        self.slice_copy = _bind(L, "po_slice_copy", C.c_int, [vp, C.c_uint32, vp, vp, vp])
        self.slice_free = _bind(L, "po_slice_free", None, [vp])
        self.last_error = _bind(L, "po_last_error", C.c_char_p, [])
        self.build_info = _bind(L, "po_build_info", C.c_char_p, [])
        self.kernel_launch_count = _bind(L, "po_kernel_launch_count", C.c_uint64, [])
        self.trim_device_cache = _bind(L, "po_trim_device_cache", C.c_uint64, [])
        self.profile_enable = _bind(L, "po_profile_enable", None, [C.c_int])
        self._profile_report = _bind(L, "po_profile_report", C.c_uint64, [C.c_char_p, C.c_uint64])

    def profile_report(self, raw: bool = False) -> dict:
        """{kernel name: (launches, total ms)} since the last report. Template
        launches are reported under the kernel's name ("(k<6, 4>)" -> "k").
        "scope:<name>" entries wrap other launches (a sort, a library call);
        "busy:" is the device time under any launch (their union). raw=True
        keeps the names as recorded and adds the "gap:<launch>" (device idle
        before a launch) and "host:<section>" entries."""
        buf = C.create_string_buffer(1 << 16)
        self._profile_report(buf, len(buf))
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms = line.rsplit(" ", 2)
            if not raw:
                if name.startswith(("gap:", "host:")):
                    continue
                name = re.sub(r"^\((\w+)<.*>\)$", r"\1", name)
            c0, m0 = out.get(name, (0, 0.0))
            out[name] = (c0 + int(cnt), m0 + float(ms))
        return out

    def check(self, code: int) -> None:
        if code:
            raise_for(code, (self.last_error() or b"").decode("utf-8", "replace"))


_CUDA: CudaLib | None = None


def cuda_lib() -> CudaLib:
    global _CUDA
    if _CUDA is None:
        _CUDA = CudaLib()
    return _CUDA


def env_flag(name: str) -> bool:
    return os.environ.get(name, "") not in ("", "0", "false", "False")
