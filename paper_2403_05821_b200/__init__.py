"""B200-native GGR reorder + PHC (arXiv 2403.05821 hot path).

Host-side mirror of the reference `prefixopt` API over the CUDA C ABI in
include/prefixopt_cuda.h (library: paper_2403_05821_b200/libprefixopt_cuda.so).
"""
from .api import *  # noqa: F401,F403
from .api import __all__ as _api_all
from .errors import (DomainError, ExtensionMissing, IoError, PrefixoptError, SchemaError,
                     SizeError, StructuralError)
from .table import Table

__all__ = list(_api_all) + ["PrefixoptError", "SchemaError", "StructuralError", "DomainError",
                            "SizeError", "IoError", "ExtensionMissing", "Table"]
