#pragma once
// GPU implementations of the steps around the reorder path in cmd_solve
// (run.hpp:390-466) and of CSV ingest, for C++ callers of the
// drop-in headers. They are offered under prefixopt::b200 next to the
// reference's own cost.hpp / cache_sim.hpp / table.hpp (which keep resolving
// to the reference tree): same inputs, outputs and exceptions as
//   prefixopt::render_prompt over a schedule  (objective.hpp:102-131)
//   prefixopt::dedup                          (cost.hpp:171-186)
//   prefixopt::simulate, EvictionPolicy::none (cache_sim.hpp:223-285)
//   prefixopt::load_csv                       (table.hpp:188-215)
// Per-request results of the replay are returned as plain vectors (the
// reference's RequestSim / SimReport live in cache_sim.hpp).

#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "prefixopt/detail/abi.hpp"
#include "prefixopt/objective.hpp"
#include "prefixopt/table.hpp"
#include "prefixopt/tokenizer.hpp"

namespace prefixopt::b200 {

// render_prompt(e, t, system_prompt, question) for every entry, in order.
inline std::vector<std::string> render_prompts(const RequestSchedule& s, const Table& t,
                                               std::string_view system_prompt,
                                               std::string_view question) {
  detail::TableAbi tv(t, char_tokenizer(), SegmentScoring::value_only);
  detail::ScheduleAbi sa(s);
  const std::uint64_t n = s.size();
  std::vector<std::uint64_t> off(n + 1, 0);
  std::uint64_t total = 0;
  auto call = [&](std::uint8_t* out, std::uint64_t cap) {
    detail::check(po_render_prompts(
        &tv.view, n, sa.rows.data(), sa.offsets.data(), sa.fields.data(), PO_LOC_HOST,
        reinterpret_cast<const std::uint8_t*>(system_prompt.data()), system_prompt.size(),
        reinterpret_cast<const std::uint8_t*>(question.data()), question.size(), PO_LOC_HOST,
        off.data(), out, cap, &total, nullptr));
  };
  call(nullptr, 0);
  std::string bytes(total, '\0');
  call(reinterpret_cast<std::uint8_t*>(bytes.data()), total);
  std::vector<std::string> out;
  out.reserve(n);
  for (std::uint64_t i = 0; i < n; ++i) out.push_back(bytes.substr(off[i], off[i + 1] - off[i]));
  return out;
}

struct DedupResult {
  std::vector<std::string> uniques;        // first-occurrence order
  std::vector<std::size_t> expansion_map;  // original index -> unique index
};

inline void pack_strings(const std::vector<std::string>& v, std::string& arena,
                         std::vector<std::uint64_t>& off) {
  off.assign(1, 0);
  for (const auto& x : v) {
    arena += x;
    off.push_back(arena.size());
  }
  if (arena.empty()) arena.push_back('\0');
}

// dedup (cost.hpp:171-186), byte-exact.
inline DedupResult dedup(const std::vector<std::string>& prompts) {
  std::string arena;
  std::vector<std::uint64_t> off;
  pack_strings(prompts, arena, off);
  const std::uint64_t n = prompts.size();
  std::vector<std::uint64_t> ex(n ? n : 1), uf(n ? n : 1);
  std::uint64_t nu = 0;
  detail::check(po_dedup(n, reinterpret_cast<const std::uint8_t*>(arena.data()), off.data(),
                         PO_LOC_HOST, ex.data(), uf.data(), &nu, nullptr));
  DedupResult r;
  for (std::uint64_t u = 0; u < nu; ++u) r.uniques.push_back(prompts[uf[u]]);
  r.expansion_map.assign(ex.begin(), ex.begin() + n);
  return r;
}

struct ReplayResult {
  std::vector<std::uint64_t> input_tokens, hit_tokens, miss_tokens, written_tokens;
  std::uint64_t total_input = 0, total_hit = 0, total_miss = 0;
  double phr = 0.0;
};

// simulate(prompts, {capacity, EvictionPolicy::none, min_cacheable}, tok).
inline ReplayResult simulate_unbounded(const std::vector<std::string>& prompts,
                                       std::uint64_t min_cacheable_prefix_tokens,
                                       const Tokenizer& tok) {
  std::string arena;
  std::vector<std::uint64_t> off;
  pack_strings(prompts, arena, off);
  const std::uint64_t n = prompts.size();
  ReplayResult r;
  for (auto* v : {&r.input_tokens, &r.hit_tokens, &r.miss_tokens, &r.written_tokens})
    v->assign(n ? n : 1, 0);
  std::uint64_t tot[3] = {0, 0, 0};
  detail::check(po_replay_unbounded(n, reinterpret_cast<const std::uint8_t*>(arena.data()),
                                    off.data(), PO_LOC_HOST, detail::tokenizer_kind(tok),
                                    min_cacheable_prefix_tokens, r.input_tokens.data(),
                                    r.hit_tokens.data(), r.miss_tokens.data(),
                                    r.written_tokens.data(), tot, nullptr));
  for (auto* v : {&r.input_tokens, &r.hit_tokens, &r.miss_tokens, &r.written_tokens}) v->resize(n);
  r.total_input = tot[0];
  r.total_hit = tot[1];
  r.total_miss = tot[2];
  r.phr = tot[0] ? static_cast<double>(tot[1]) / static_cast<double>(tot[0]) : 0.0;
  return r;
}

// load_csv (table.hpp:188-215) of CSV text.
inline Table load_csv(std::string_view text) {
  po_csv* h = nullptr;
  detail::check(po_load_csv(reinterpret_cast<const std::uint8_t*>(text.data()), text.size(),
                            PO_LOC_HOST, &h, nullptr));
  std::uint64_t rows = 0, ab = 0, nb = 0;
  std::uint32_t fields = 0;
  po_csv_info(h, &rows, &fields, &ab, &nb);
  std::string arena(ab ? ab : 1, '\0'), names(nb ? nb : 1, '\0');
  std::vector<std::uint64_t> off(rows * fields + 1), noff(fields + 1);
  const int rc = po_csv_copy(h, PO_LOC_HOST, reinterpret_cast<std::uint8_t*>(arena.data()),
                             off.data(), reinterpret_cast<std::uint8_t*>(names.data()),
                             noff.data(), nullptr);
  po_csv_free(h);
  detail::check(rc);
  std::vector<std::string> field_names;
  for (std::uint32_t f = 0; f < fields; ++f)
    field_names.push_back(names.substr(noff[f], noff[f + 1] - noff[f]));
  std::vector<std::vector<std::string>> table_rows(rows);
  for (std::uint64_t r = 0; r < rows; ++r)
    for (std::uint32_t f = 0; f < fields; ++f) {
      const std::uint64_t i = r * fields + f;
      table_rows[r].push_back(arena.substr(off[i], off[i + 1] - off[i]));
    }
  return Table(std::move(field_names), std::move(table_rows));
}

}  // namespace prefixopt::b200
