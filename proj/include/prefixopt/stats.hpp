#pragma once
// Column statistics (reference stats.hpp:14-45); compute_stats runs on the
// GPU (exact distinct counts from the dictionary encoding, length sums from
// the per-value segment lengths).

#include <cstddef>
#include <string>
#include <vector>

#include "prefixopt/detail/abi.hpp"
#include "prefixopt/scoring.hpp"
#include "prefixopt/table.hpp"
#include "prefixopt/tokenizer.hpp"

namespace prefixopt {

struct FieldStats {
  std::string name;
  std::size_t cardinality = 0;
  double avg_len = 0.0;
};

struct ColumnStats {
  std::vector<FieldStats> fields;
  std::size_t total_rows = 0;
};

inline ColumnStats compute_stats(const Table& t, const Tokenizer& tok,
                                 SegmentScoring scoring = SegmentScoring::value_only) {
  detail::TableAbi view(t, tok, scoring);
  const std::size_t m = t.field_count();
  std::vector<std::uint64_t> card(m ? m : 1), total(m ? m : 1);
  detail::check(po_compute_stats(&view.view, view.tok_kind, view.scoring, card.data(),
                                 total.data(), nullptr));
  ColumnStats s;
  s.total_rows = t.row_count();
  for (std::size_t f = 0; f < m; ++f)
    s.fields.push_back({t.field_name(f), static_cast<std::size_t>(card[f]),
                        t.row_count() ? static_cast<double>(total[f]) / t.row_count() : 0.0});
  return s;
}

}  // namespace prefixopt
