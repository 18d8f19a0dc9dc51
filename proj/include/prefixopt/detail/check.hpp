#pragma once
// PO_ERR_* status of the C ABI (include/prefixopt_cuda.h) -> the reference's
// exception classes (errors.hpp:10-42).

#include <stdexcept>
#include <string>

#include "prefixopt_cuda.h"
#include "prefixopt/errors.hpp"

namespace prefixopt::detail {

inline void check(int code) {
  if (code == PO_OK) return;
  std::string msg = po_last_error();
  switch (code) {
    case PO_ERR_SCHEMA: throw schema_error(msg);
    case PO_ERR_STRUCTURAL: throw structural_error(msg);
    case PO_ERR_DOMAIN: throw domain_error(msg);
    case PO_ERR_SIZE: throw size_error(msg);
    case PO_ERR_IO: throw io_error(msg);
    case PO_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case PO_ERR_INVALID_ARG: throw std::invalid_argument(msg);
    default: throw error(msg);
  }
}

}  // namespace prefixopt::detail
