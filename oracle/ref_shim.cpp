// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference implementation (the header-only library
// under /root/reference/proj/include, compiled in place by oracle/Makefile)
// through the oracle C interface with the `ref_` prefix. Nothing here
// re-implements the algorithm: each entry point builds a prefixopt::Table
// from the ABI view and calls the reference function named in its comment.
// The output goes to oracle/_ref/ (git-ignored, shipped to the GPU box).

#include <chrono>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "prefixopt/cache_sim.hpp"
#include "prefixopt/cost.hpp"
#include "prefixopt/fd.hpp"
#include "prefixopt/ggr.hpp"
#include "prefixopt/objective.hpp"
#include "prefixopt/stats.hpp"

#include "oracle.h"

namespace {

thread_local std::string g_err;

prefixopt::Table to_table(const po_table* t) {
  if (!t || t->location != PO_LOC_HOST) throw std::invalid_argument("ref shim needs host table");
  std::vector<std::string> names;
  for (uint32_t f = 0; f < t->n_fields; ++f)
    names.emplace_back(t->field_names[f], t->field_name_lens[f]);
  std::vector<std::vector<std::string>> rows(t->n_rows);
  for (uint64_t r = 0; r < t->n_rows; ++r) {
    rows[r].reserve(t->n_fields);
    for (uint32_t f = 0; f < t->n_fields; ++f) {
      uint64_t i = r * t->n_fields + f;
      rows[r].emplace_back(reinterpret_cast<const char*>(t->arena) + t->offsets[i],
                           t->offsets[i + 1] - t->offsets[i]);
    }
  }
  return prefixopt::Table(std::move(names), std::move(rows));
}

// A deterministic tokenizer defined by the caller's per-cell lengths: maps
// the exact text the reference passes to count() (the value, or the rendered
// fragment in full_fragment mode) to its length.
class TableTokenizer final : public prefixopt::Tokenizer {
 public:
  TableTokenizer(const po_table* t, const prefixopt::Table& tab, prefixopt::SegmentScoring s) {
    for (uint64_t r = 0; r < tab.row_count(); ++r)
      for (uint32_t f = 0; f < tab.field_count(); ++f) {
        const std::string& v = tab.cell(r, f);
        std::string key = s == prefixopt::SegmentScoring::value_only
                              ? v
                              : prefixopt::fragment_text(tab.field_name(f), v);
        lens_[key] = t->cell_lens[r * t->n_fields + f];
      }
  }
  std::string_view name() const override { return "custom"; }
  std::vector<std::string_view> tokens(std::string_view) const override {
    throw std::logic_error("not used on this path");
  }
  std::size_t count(std::string_view text) const override {
    auto it = lens_.find(std::string(text));
    if (it == lens_.end()) throw std::logic_error("custom tokenizer: unknown text");
    return it->second;
  }

 private:
  std::unordered_map<std::string, std::size_t> lens_;
};

struct Tok {
  std::unique_ptr<TableTokenizer> custom;
  const prefixopt::Tokenizer* tok = nullptr;
};

Tok make_tok(int kind, const po_table* t, const prefixopt::Table& tab,
             prefixopt::SegmentScoring s) {
  Tok out;
  if (kind == PO_TOK_CHAR) out.tok = &prefixopt::char_tokenizer();
  else if (kind == PO_TOK_WORD) out.tok = &prefixopt::word_tokenizer();
  else {
    out.custom = std::make_unique<TableTokenizer>(t, tab, s);
    out.tok = out.custom.get();
  }
  return out;
}

prefixopt::SegmentScoring scoring_of(int s) {
  return s == PO_SCORE_VALUE ? prefixopt::SegmentScoring::value_only
                             : prefixopt::SegmentScoring::full_fragment;
}

prefixopt::StatsScoreVariant variant_of(int v) {
  if (v == PO_STATS_SQUARED) return prefixopt::StatsScoreVariant::squared_length;
  if (v == PO_STATS_LENFREQ) return prefixopt::StatsScoreVariant::length_frequency;
  return prefixopt::StatsScoreVariant::cardinality_weighted_squared;
}

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return PO_OK;
  } catch (const prefixopt::schema_error& e) {
    g_err = e.what();
    return PO_ERR_SCHEMA;
  } catch (const prefixopt::domain_error& e) {
    g_err = e.what();
    return PO_ERR_DOMAIN;
  } catch (const prefixopt::structural_error& e) {
    g_err = e.what();
    return PO_ERR_STRUCTURAL;
  } catch (const prefixopt::size_error& e) {
    g_err = e.what();
    return PO_ERR_SIZE;
  } catch (const prefixopt::error& e) {
    g_err = e.what();
    return PO_ERR_ERROR;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return PO_ERR_OUT_OF_RANGE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PO_ERR_ERROR;
  }
}

}  // namespace

extern "C" {

// prefixopt::ggr (ggr.hpp:367-394)
int ref_ggr(const po_table* tv, const po_fd_groups* fds, const po_ggr_config* cfg, int32_t tok,
            int32_t scoring, uint64_t* out_rows, uint64_t* out_offsets, int32_t* out_fields,
            uint64_t cap, uint64_t* out_phc, po_solve_stats* out_stats) {
  return guarded([&] {
    prefixopt::Table t = to_table(tv);
    auto sc = scoring_of(scoring);
    Tok tk = make_tok(tok, tv, t, sc);
    prefixopt::FunctionalDependencySet set;
    if (fds)
      for (uint32_t g = 0; g < fds->n_groups; ++g) {
        std::vector<std::string> names;
        for (uint32_t k = fds->group_offsets[g]; k < fds->group_offsets[g + 1]; ++k)
          names.push_back(t.field_name(fds->members[k]));
        set.groups.push_back(std::move(names));
      }
    prefixopt::GgrConfig c;
    c.row_recursion_depth = cfg->row_recursion_depth;
    c.column_recursion_depth = cfg->column_recursion_depth;
    c.hitcount_stop_threshold = cfg->hitcount_stop_threshold;
    c.use_fds = cfg->use_fds != 0;
    c.stats_variant = variant_of(cfg->stats_variant);
    prefixopt::SolveResult res = prefixopt::ggr(t, set, c, *tk.tok, sc);
    uint64_t at = 0;
    for (const auto& e : res.schedule.entries) at += e.field_order.size();
    if (at > cap) throw prefixopt::size_error("ref shim: field capacity too small");
    at = 0;
    out_offsets[0] = 0;
    for (size_t i = 0; i < res.schedule.entries.size(); ++i) {
      const auto& e = res.schedule.entries[i];
      out_rows[i] = e.row_id;
      for (int f : e.field_order) out_fields[at++] = f;
      out_offsets[i + 1] = at;
    }
    *out_phc = res.phc_score;
    if (out_stats) {
      out_stats->recursive_calls = res.stats.recursive_calls;
      out_stats->candidates_examined = res.stats.candidates_examined;
      out_stats->max_depth = res.stats.max_depth;
      out_stats->wall_ms = res.stats.wall_ms;
    }
  });
}

// prefixopt::phc (objective.hpp:94-99)
int ref_phc(const po_table* tv, int32_t tok, int32_t scoring, uint64_t n, const uint64_t* rows,
            const uint64_t* offs, const int32_t* fields, uint64_t* out_phc) {
  return guarded([&] {
    prefixopt::Table t = to_table(tv);
    auto sc = scoring_of(scoring);
    Tok tk = make_tok(tok, tv, t, sc);
    prefixopt::RequestSchedule s;
    for (uint64_t i = 0; i < n; ++i)
      s.entries.push_back({rows[i], std::vector<int>(fields + offs[i], fields + offs[i + 1])});
    *out_phc = prefixopt::phc(s, t, *tk.tok, sc);
  });
}

// prefixopt::sort_rows_fixed_order (objective.hpp:154-171)
int ref_sort_rows_fixed_order(const po_table* tv, const int32_t* order, uint64_t* out_rows) {
  return guarded([&] {
    prefixopt::Table t = to_table(tv);
    std::vector<int> o(order, order + tv->n_fields);
    prefixopt::RequestSchedule s = prefixopt::sort_rows_fixed_order(t, o);
    for (size_t i = 0; i < s.entries.size(); ++i) out_rows[i] = s.entries[i].row_id;
  });
}

// prefixopt::compute_stats (stats.hpp:25-45); total_len is recovered from
// avg_len * n, which is exact for the integer sums the tests use (< 2^53).
int ref_compute_stats(const po_table* tv, int32_t tok, int32_t scoring, uint64_t* out_card,
                      uint64_t* out_total) {
  return guarded([&] {
    prefixopt::Table t = to_table(tv);
    auto sc = scoring_of(scoring);
    Tok tk = make_tok(tok, tv, t, sc);
    prefixopt::ColumnStats st = prefixopt::compute_stats(t, *tk.tok, sc);
    for (size_t f = 0; f < st.fields.size(); ++f) {
      out_card[f] = st.fields[f].cardinality;
      out_total[f] = static_cast<uint64_t>(st.fields[f].avg_len * double(t.row_count()) + 0.5);
    }
  });
}

// prefixopt::fixed_order_by_hitcount_stats (ggr.hpp:59-84)
int ref_fixed_order_by_hitcount_stats(uint32_t m, uint64_t total_rows, const uint64_t* card,
                                      const double* avg, int32_t variant, int32_t* out) {
  return guarded([&] {
    prefixopt::ColumnStats st;
    st.total_rows = total_rows;
    for (uint32_t f = 0; f < m; ++f) st.fields.push_back({"f" + std::to_string(f), card[f], avg[f]});
    std::vector<int> o = prefixopt::fixed_order_by_hitcount_stats(st, variant_of(variant));
    std::copy(o.begin(), o.end(), out);
  });
}

// prefixopt::validate_fds (fd.hpp:66-109). Groups arrive as field indices;
// agree/differ fields are returned as indices.
int ref_validate_fds(const po_table* tv, const po_fd_groups* fds, uint8_t* out_satisfied,
                     uint8_t* out_has_witness, uint64_t* out_row_a, uint64_t* out_row_b,
                     int32_t* out_agree, int32_t* out_differ) {
  return guarded([&] {
    prefixopt::Table t = to_table(tv);
    prefixopt::FunctionalDependencySet set;
    for (uint32_t g = 0; g < fds->n_groups; ++g) {
      std::vector<std::string> names;
      for (uint32_t k = fds->group_offsets[g]; k < fds->group_offsets[g + 1]; ++k)
        names.push_back(t.field_name(fds->members[k]));
      set.groups.push_back(names);
    }
    const prefixopt::FdValidationReport rep = prefixopt::validate_fds(t, set);
    for (size_t g = 0; g < rep.groups.size(); ++g) {
      const auto& gr = rep.groups[g];
      out_satisfied[g] = gr.satisfied ? 1 : 0;
      out_has_witness[g] = gr.witness ? 1 : 0;
      if (gr.witness) {
        out_row_a[g] = gr.witness->row_a;
        out_row_b[g] = gr.witness->row_b;
        out_agree[g] = t.require_field(gr.witness->agree_field);
        out_differ[g] = t.require_field(gr.witness->differ_field);
      }
    }
  });
}

// prefixopt::discover_fds (fd.hpp:114-141): out_group_of_field[f] = index of
// the reported group holding field f, -1 when f is in no group.
int ref_discover_fds(const po_table* tv, uint64_t max_rows, int32_t* out_group_of_field) {
  return guarded([&] {
    prefixopt::Table t = to_table(tv);
    const prefixopt::FunctionalDependencySet set = prefixopt::discover_fds(t, max_rows);
    for (size_t f = 0; f < t.field_count(); ++f) out_group_of_field[f] = -1;
    for (size_t g = 0; g < set.groups.size(); ++g)
      for (const auto& nm : set.groups[g]) out_group_of_field[t.require_field(nm)] = int32_t(g);
  });
}

// prefixopt::render_prompt (objective.hpp:118-131) of every entry; sizes
// first (out_bytes == NULL), then the bytes.
int ref_render_prompts(const po_table* tv, uint64_t n_entries, const uint64_t* rows,
                       const uint64_t* offs, const int32_t* fields, const uint8_t* sp,
                       uint64_t sp_len, const uint8_t* q, uint64_t q_len, uint64_t* out_offsets,
                       uint8_t* out_bytes, uint64_t capacity, uint64_t* out_total) {
  return guarded([&] {
    prefixopt::Table t = to_table(tv);
    const std::string_view spv(reinterpret_cast<const char*>(sp), sp ? sp_len : 0);
    const std::string_view qv(reinterpret_cast<const char*>(q), q ? q_len : 0);
    uint64_t pos = 0;
    out_offsets[0] = 0;
    for (uint64_t i = 0; i < n_entries; ++i) {
      prefixopt::ScheduleEntry e;
      e.row_id = rows[i];
      e.field_order.assign(fields + offs[i], fields + offs[i + 1]);
      const std::string p = prefixopt::render_prompt(e, t, spv, qv);
      if (out_bytes && pos + p.size() <= capacity) std::memcpy(out_bytes + pos, p.data(), p.size());
      pos += p.size();
      out_offsets[i + 1] = pos;
    }
    *out_total = pos;
  });
}

// prefixopt::dedup (cost.hpp:171-186)
int ref_dedup(uint64_t n, const uint8_t* arena, const uint64_t* offsets, uint64_t* out_expansion,
              uint64_t* out_unique_first, uint64_t* out_n_unique) {
  return guarded([&] {
    std::vector<std::string> prompts;
    for (uint64_t i = 0; i < n; ++i)
      prompts.emplace_back(reinterpret_cast<const char*>(arena) + offsets[i],
                           offsets[i + 1] - offsets[i]);
    const prefixopt::DedupResult d = prefixopt::dedup(prompts);
    std::vector<char> seen(d.uniques.size(), 0);
    for (uint64_t i = 0; i < n; ++i) {
      out_expansion[i] = d.expansion_map[i];
      if (!seen[d.expansion_map[i]]) {
        seen[d.expansion_map[i]] = 1;
        out_unique_first[d.expansion_map[i]] = i;
      }
    }
    *out_n_unique = d.uniques.size();
  });
}

// prefixopt::simulate (cache_sim.hpp:223-285): eviction 0 = none, 1 = lru.
int ref_simulate(uint64_t n, const uint8_t* arena, const uint64_t* offsets, int32_t tok,
                 uint64_t capacity, int32_t eviction, uint64_t min_cacheable, uint64_t* out_input,
                 uint64_t* out_hit, uint64_t* out_miss, uint64_t* out_written,
                 uint8_t* out_uncacheable, uint64_t* out_totals) {
  return guarded([&] {
    std::vector<std::string> prompts;
    for (uint64_t i = 0; i < n; ++i)
      prompts.emplace_back(reinterpret_cast<const char*>(arena) + offsets[i],
                           offsets[i + 1] - offsets[i]);
    prefixopt::CacheConfig cfg;
    cfg.capacity_tokens = capacity;
    cfg.eviction = eviction ? prefixopt::EvictionPolicy::lru : prefixopt::EvictionPolicy::none;
    cfg.min_cacheable_prefix_tokens = min_cacheable;
    const prefixopt::Tokenizer& tk =
        tok == PO_TOK_WORD ? prefixopt::word_tokenizer() : prefixopt::char_tokenizer();
    const prefixopt::SimReport r = prefixopt::simulate(prompts, cfg, tk);
    for (uint64_t i = 0; i < n; ++i) {
      out_input[i] = r.requests[i].input_tokens;
      out_hit[i] = r.requests[i].hit_tokens;
      out_miss[i] = r.requests[i].miss_tokens;
      out_written[i] = r.requests[i].written_tokens;
      out_uncacheable[i] = r.requests[i].uncacheable ? 1 : 0;
    }
    out_totals[0] = r.total_input;
    out_totals[1] = r.total_hit;
    out_totals[2] = r.total_miss;
    out_totals[3] = r.evicted_tokens;
  });
}

}  // extern "C"

namespace {
// A loaded table as sizes (out_arena == NULL) or as row-major arena +
// offsets and names (the layout po_csv_copy / po_jsonl_copy produce).
void emit_table(const prefixopt::Table& t, uint64_t* out_rows, uint32_t* out_fields,
                uint64_t* out_arena_bytes, uint64_t* out_names_bytes, uint8_t* out_arena,
                uint64_t* out_offsets, uint8_t* out_names, uint64_t* out_name_offsets) {
  uint64_t ab = 0, nb = 0;
  for (size_t r = 0; r < t.row_count(); ++r)
    for (size_t f = 0; f < t.field_count(); ++f) ab += t.cell(r, f).size();
  for (const auto& nm : t.field_names()) nb += nm.size();
  *out_rows = t.row_count();
  *out_fields = uint32_t(t.field_count());
  *out_arena_bytes = ab;
  *out_names_bytes = nb;
  if (!out_arena) return;
  uint64_t pos = 0, k = 0;
  out_offsets[0] = 0;
  for (size_t r = 0; r < t.row_count(); ++r)
    for (size_t f = 0; f < t.field_count(); ++f) {
      const std::string& c = t.cell(r, f);
      std::memcpy(out_arena + pos, c.data(), c.size());
      pos += c.size();
      out_offsets[++k] = pos;
    }
  pos = 0;
  out_name_offsets[0] = 0;
  for (size_t f = 0; f < t.field_count(); ++f) {
    const std::string& nm = t.field_name(f);
    std::memcpy(out_names + pos, nm.data(), nm.size());
    pos += nm.size();
    out_name_offsets[f + 1] = pos;
  }
}
}  // namespace

extern "C" {

// prefixopt::load_csv (table.hpp:188-215) on `len` bytes; sizes first
// (out_arena == NULL), then the table.
int ref_load_csv(const uint8_t* data, uint64_t len, uint64_t* out_rows, uint32_t* out_fields,
                 uint64_t* out_arena_bytes, uint64_t* out_names_bytes, uint8_t* out_arena,
                 uint64_t* out_offsets, uint8_t* out_names, uint64_t* out_name_offsets) {
  return guarded([&] {
    std::istringstream in(std::string(reinterpret_cast<const char*>(data), len));
    emit_table(prefixopt::load_csv(in), out_rows, out_fields, out_arena_bytes, out_names_bytes,
               out_arena, out_offsets, out_names, out_name_offsets);
  });
}

// prefixopt::load_jsonl (table.hpp:225-269), same calling convention.
int ref_load_jsonl(const uint8_t* data, uint64_t len, uint64_t* out_rows, uint32_t* out_fields,
                   uint64_t* out_arena_bytes, uint64_t* out_names_bytes, uint8_t* out_arena,
                   uint64_t* out_offsets, uint8_t* out_names, uint64_t* out_name_offsets) {
  return guarded([&] {
    std::istringstream in(std::string(reinterpret_cast<const char*>(data), len));
    emit_table(prefixopt::load_jsonl(in), out_rows, out_fields, out_arena_bytes, out_names_bytes,
               out_arena, out_offsets, out_names, out_name_offsets);
  });
}

const char* ref_last_error(void) { return g_err.c_str(); }

}  // extern "C"
