"""Exception taxonomy of the reference (errors.hpp:10-42) plus the status-code
mapping of the C ABI (include/prefixopt_cuda.h)."""


class PrefixoptError(RuntimeError):
    """prefixopt::error (errors.hpp:10-13); also CUDA/driver failures."""


class SchemaError(PrefixoptError):
    """prefixopt::schema_error (errors.hpp:16-19)."""


class StructuralError(PrefixoptError):
    """prefixopt::structural_error (errors.hpp:22-25)."""


class DomainError(PrefixoptError):
    """prefixopt::domain_error (errors.hpp:28-31)."""


class SizeError(PrefixoptError):
    """prefixopt::size_error (errors.hpp:34-37)."""


class IoError(PrefixoptError):
    """prefixopt::io_error (errors.hpp:39-42)."""


class ExtensionMissing(PrefixoptError):
    """The CUDA library is not built/loadable. The product path never falls
    back to a CPU implementation; it raises this instead."""


PO_OK = 0
_CODE_TO_EXC = {
    1: PrefixoptError,
    2: SchemaError,
    3: StructuralError,
    4: DomainError,
    5: SizeError,
    6: IoError,
    7: IndexError,  # std::out_of_range from Table::cell (table.hpp:62-64)
    8: ValueError,  # ABI misuse
}


def raise_for(code: int, message: str) -> None:
    if code == PO_OK:
        return
    raise _CODE_TO_EXC.get(code, PrefixoptError)(message)
