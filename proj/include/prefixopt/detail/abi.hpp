#pragma once
// Marshalling between the C++ API and the C ABI of libprefixopt_cuda.so
// (include/prefixopt_cuda.h). Link with -lprefixopt_cuda.

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "prefixopt_cuda.h"
#include "prefixopt/detail/check.hpp"
#include "prefixopt/errors.hpp"
#include "prefixopt/scoring.hpp"
#include "prefixopt/table.hpp"
#include "prefixopt/tokenizer.hpp"

namespace prefixopt::detail {

inline int tokenizer_kind(const Tokenizer& tok) {
  if (dynamic_cast<const CharTokenizer*>(&tok)) return PO_TOK_CHAR;
  if (dynamic_cast<const WordTokenizer*>(&tok)) return PO_TOK_WORD;
  return PO_TOK_CUSTOM;
}

// po_table view of a Table (host arena), with per-cell lengths for a custom
// tokenizer (segment_len, scoring.hpp:72-76).
struct TableAbi {
  po_table view{};
  int tok_kind = PO_TOK_CHAR;
  int scoring = PO_SCORE_VALUE;
  std::vector<std::uint64_t> lens;
  std::vector<const char*> name_ptrs;
  std::vector<std::uint64_t> name_lens;
  TableAbi(const Table& t, const Tokenizer& tok, SegmentScoring sc) {
    const Table::Arena& a = t.arena();
    tok_kind = tokenizer_kind(tok);
    scoring = sc == SegmentScoring::value_only ? PO_SCORE_VALUE : PO_SCORE_FRAGMENT;
    if (tok_kind == PO_TOK_CUSTOM) {
      lens.reserve(t.row_count() * t.field_count());
      for (std::size_t r = 0; r < t.row_count(); ++r)
        for (std::size_t f = 0; f < t.field_count(); ++f)
          lens.push_back(segment_len(t.field_name(f), t.cell(r, f), tok, sc));
    }
    for (const auto& nm : t.field_names()) {
      name_ptrs.push_back(nm.data());
      name_lens.push_back(nm.size());
    }
    view.n_rows = t.row_count();
    view.n_fields = static_cast<std::uint32_t>(t.field_count());
    view.location = PO_LOC_HOST;
    view.field_names = name_ptrs.data();
    view.field_name_lens = name_lens.data();
    view.arena = a.bytes.data();
    view.offsets = a.offsets.data();
    view.cell_lens = lens.empty() ? nullptr : lens.data();
  }
};

}  // namespace prefixopt::detail
