#pragma once
// Greedy Group Recursion (reference ggr.hpp) — drop-in front end of the
// B200 implementation. prefixopt::ggr() marshals the table once into the C
// ABI and the whole solve (dictionary encoding, level-synchronous recursion,
// leaf fallbacks, whole-table fallback competition, PHC) runs in
// libprefixopt_cuda.so. fixed_order_by_hitcount_stats is the same host
// IEEE-double ranking the library uses; hitcount() (not called by the
// solver) is a host computation kept for API compatibility.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <numeric>
#include <string>
#include <string_view>
#include <vector>

#include "prefixopt/detail/abi.hpp"
#include "prefixopt/errors.hpp"
#include "prefixopt/fd.hpp"
#include "prefixopt/objective.hpp"
#include "prefixopt/solve_result.hpp"
#include "prefixopt/stats.hpp"

namespace prefixopt {

enum class StatsScoreVariant {
  cardinality_weighted_squared,  // avg_len^2 * (n / cardinality - 1)
  squared_length,                // avg_len^2
  length_frequency,              // avg_len * n / cardinality
};

inline StatsScoreVariant stats_variant_by_name(std::string_view name) {
  if (name == "weighted") return StatsScoreVariant::cardinality_weighted_squared;
  if (name == "squared") return StatsScoreVariant::squared_length;
  if (name == "length-freq") return StatsScoreVariant::length_frequency;
  throw schema_error("unknown stats variant: " + std::string(name) +
                     " (expected 'weighted', 'squared' or 'length-freq')");
}

inline std::string_view stats_variant_name(StatsScoreVariant v) {
  switch (v) {
    case StatsScoreVariant::squared_length: return "squared";
    case StatsScoreVariant::length_frequency: return "length-freq";
    default: return "weighted";
  }
}

struct GgrConfig {
  std::size_t row_recursion_depth = 4;
  std::size_t column_recursion_depth = 2;
  std::uint64_t hitcount_stop_threshold = 100000;
  bool use_fds = true;
  StatsScoreVariant stats_variant = StatsScoreVariant::cardinality_weighted_squared;
};

inline std::vector<int> fixed_order_by_hitcount_stats(
    const ColumnStats& stats,
    StatsScoreVariant variant = StatsScoreVariant::cardinality_weighted_squared) {
  std::vector<std::uint64_t> card;
  std::vector<double> avg;
  detail::stats_arrays(stats, card, avg);
  std::vector<int> order(stats.fields.size() ? stats.fields.size() : 1);
  detail::check(po_fixed_order_by_hitcount_stats(
      static_cast<std::uint32_t>(stats.fields.size()), stats.total_rows, card.data(), avg.data(),
      static_cast<std::int32_t>(variant), order.data()));
  order.resize(stats.fields.size());
  return order;
}

struct HitCountResult {
  double score = 0.0;
  std::vector<std::string> fields;
};

inline HitCountResult hitcount(const Table& t, std::string_view field, std::string_view value,
                               const FunctionalDependencySet& fds, const Tokenizer& tok,
                               SegmentScoring scoring = SegmentScoring::value_only) {
  const int c = t.require_field(field);
  std::vector<int> inferred;
  for (const auto& g : fds.groups) {
    if (std::find(g.begin(), g.end(), field) == g.end()) continue;
    for (const auto& nm : g) {
      int o = t.require_field(nm);
      if (o != c) inferred.push_back(o);
    }
    break;  // first group holding the field
  }
  std::sort(inferred.begin(), inferred.end());
  std::uint64_t count = 0, inferred_total = 0;
  for (std::size_t r = 0; r < t.row_count(); ++r) {
    if (t.cell(r, c) != value) continue;
    ++count;
    for (int o : inferred) inferred_total += segment_len(t.field_name(o), t.cell(r, o), tok, scoring);
  }
  if (count == 0) throw domain_error("hitcount: value does not occur in field " + std::string(field));
  const double len = static_cast<double>(segment_len(field, value, tok, scoring));
  const double tot = len * len + static_cast<double>(inferred_total) / count;
  HitCountResult res;
  res.score = tot * static_cast<double>(count - 1);
  res.fields.emplace_back(field);
  for (int o : inferred) res.fields.push_back(t.field_name(o));
  return res;
}

// ggr (reference ggr.hpp:367-394) on the GPU.
inline SolveResult ggr(const Table& t, const FunctionalDependencySet& fds, const GgrConfig& cfg,
                       const Tokenizer& tok, SegmentScoring scoring = SegmentScoring::value_only) {
  const auto start = std::chrono::steady_clock::now();
  // FD names resolve only when FDs are used (ggr.hpp:155-158)
  std::vector<std::uint32_t> goff{0};
  std::vector<std::int32_t> members;
  if (cfg.use_fds)
    for (const auto& g : fds.groups) {
      for (const auto& nm : g) members.push_back(t.require_field(nm));
      goff.push_back(static_cast<std::uint32_t>(members.size()));
    }
  if (members.empty()) members.push_back(0);
  po_fd_groups fv{static_cast<std::uint32_t>(goff.size() - 1), goff.data(), members.data()};
  po_ggr_config c{cfg.row_recursion_depth, cfg.column_recursion_depth,
                  cfg.hitcount_stop_threshold, cfg.use_fds ? 1 : 0,
                  static_cast<std::int32_t>(cfg.stats_variant)};
  detail::TableAbi tv(t, tok, scoring);
  std::uint64_t score = 0;
  po_solve_stats st{};
  // the schedule handle carries CSR field orders: FD groups sharing members
  // make some orders longer than the schema (ggr.hpp:280-282)
  po_schedule* h = nullptr;
  detail::check(po_ggr_schedule(&tv.view, &fv, &c, tv.tok_kind, tv.scoring, &h, &score, &st,
                                nullptr));
  std::uint64_t n = 0, total = 0;
  po_schedule_info(h, &n, &total);
  std::vector<std::uint64_t> rows(n ? n : 1), offs(n + 1);
  std::vector<std::int32_t> fields(total ? total : 1);
  const int rc = po_schedule_copy(h, PO_LOC_HOST, rows.data(), offs.data(), fields.data(), nullptr);
  po_schedule_free(h);
  detail::check(rc);
  SolveResult res;
  res.phc_score = score;
  res.schedule.entries.reserve(n);
  for (std::size_t i = 0; i < n; ++i)
    res.schedule.entries.push_back(
        {rows[i], std::vector<int>(fields.begin() + offs[i], fields.begin() + offs[i + 1])});
  res.stats.recursive_calls = st.recursive_calls;
  res.stats.candidates_examined = st.candidates_examined;
  res.stats.max_depth = st.max_depth;
  res.stats.wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();
  return res;
}

}  // namespace prefixopt
