// ORACLE — TEST INFRASTRUCTURE ONLY. Never linked into or called by the
// product path (paper_2403_05821_b200/ and proj/include/). Loaded only by
// tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg.
//
// CPU restatement of the reference GGR reorder + PHC path
// (/root/reference/proj/include/prefixopt/*.hpp), written independently from
// the algorithm's specification: grouping is done by sorting instead of
// hashing, the recursion threads a field-order prefix downwards instead of
// stitching results upwards, and every function cites the reference lines
// whose behaviour it restates. Pinned against the reference itself
// (oracle/_ref, tests/test_oracle_pinning.py) and the golden fixtures in
// tests/golden/.
//
// Exported with the `oracle_` prefix; see oracle.h.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "oracle.h"

namespace {

thread_local std::string g_err;

struct OracleError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, std::string msg) { throw OracleError{code, std::move(msg)}; }

// A table view over the ABI's row-major arena (table.hpp:24-104 semantics:
// cells are opaque bytes, row ids are ingestion order).
struct Tab {
  uint64_t n = 0;
  uint32_t m = 0;
  std::vector<std::string_view> names;
  const uint8_t* arena = nullptr;
  const uint64_t* off = nullptr;
  const uint64_t* lens = nullptr;

  explicit Tab(const po_table* t) {
    if (!t) fail(PO_ERR_INVALID_ARG, "null table");
    if (t->location != PO_LOC_HOST) fail(PO_ERR_INVALID_ARG, "oracle needs host buffers");
    n = t->n_rows;
    m = t->n_fields;
    for (uint32_t f = 0; f < m; ++f)
      names.emplace_back(t->field_names[f], t->field_name_lens[f]);
    arena = t->arena;
    off = t->offsets;
    lens = t->cell_lens;
  }
  // Table::cell (table.hpp:62-64) throws std::out_of_range via .at().
  std::string_view cell(uint64_t r, int64_t f) const {
    if (r >= n || f < 0 || f >= int64_t(m)) fail(PO_ERR_OUT_OF_RANGE, "cell index out of range");
    uint64_t i = r * m + uint64_t(f);
    return std::string_view(reinterpret_cast<const char*>(arena) + off[i], off[i + 1] - off[i]);
  }
};

// tokenizer.hpp:76-78 — the six ASCII whitespace bytes.
bool ws(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v';
}

// WordTokenizer::count (tokenizer.hpp:64-73): maximal non-whitespace runs.
uint64_t words(std::string_view s) {
  uint64_t runs = 0;
  for (size_t i = 0; i < s.size(); ++i)
    if (!ws(s[i]) && (i == 0 || ws(s[i - 1]))) ++runs;
  return runs;
}

// json_escape (scoring.hpp:33-57).
std::string escape(std::string_view s) {
  static const char hexd[] = "0123456789abcdef";
  std::string o;
  for (char ch : s) {
    unsigned char u = static_cast<unsigned char>(ch);
    if (ch == '"') o += "\\\"";
    else if (ch == '\\') o += "\\\\";
    else if (ch == '\b') o += "\\b";
    else if (ch == '\f') o += "\\f";
    else if (ch == '\n') o += "\\n";
    else if (ch == '\r') o += "\\r";
    else if (ch == '\t') o += "\\t";
    else if (u < 0x20) {
      o += "\\u00";
      o += hexd[u >> 4];
      o += hexd[u & 15];
    } else {
      o += ch;
    }
  }
  return o;
}

// fragment_text (scoring.hpp:62-69): "<field>": "<value>", with both escaped.
std::string fragment(std::string_view field, std::string_view value) {
  return "\"" + escape(field) + "\": \"" + escape(value) + "\", ";
}

// segment_len (scoring.hpp:72-76) through Tokenizer::count.
uint64_t seglen(const Tab& t, uint64_t r, int f, int tok, int scoring) {
  if (tok == PO_TOK_CUSTOM) {
    if (!t.lens) fail(PO_ERR_INVALID_ARG, "custom tokenizer without cell_lens");
    return t.lens[r * t.m + uint64_t(f)];
  }
  std::string_view v = t.cell(r, f);
  if (scoring == PO_SCORE_VALUE) return tok == PO_TOK_CHAR ? v.size() : words(v);
  std::string frag = fragment(t.names[f], v);
  return tok == PO_TOK_CHAR ? frag.size() : words(frag);
}

void check_modes(int tok, int scoring) {
  if (tok < 0 || tok > 2) fail(PO_ERR_INVALID_ARG, "bad tokenizer");
  if (scoring < 0 || scoring > 1) fail(PO_ERR_INVALID_ARG, "bad scoring");
}

// fixed_order_by_hitcount_stats (ggr.hpp:59-84): double score per field,
// descending, ties kept in schema order (stable).
std::vector<int> hitcount_order(uint64_t total_rows, const std::vector<uint64_t>& card,
                                const std::vector<double>& avg, int variant) {
  size_t k = card.size();
  std::vector<double> score(k, 0.0);
  for (size_t f = 0; f < k; ++f) {
    if (card[f] == 0) continue;
    double ratio = static_cast<double>(total_rows) / static_cast<double>(card[f]);
    if (variant == PO_STATS_WEIGHTED) score[f] = avg[f] * avg[f] * (ratio - 1.0);
    else if (variant == PO_STATS_SQUARED) score[f] = avg[f] * avg[f];
    else score[f] = avg[f] * ratio;
  }
  std::vector<int> idx(k);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return score[a] > score[b]; });
  return idx;
}

struct Entry {
  uint64_t row;
  std::vector<int> fields;
};

// hit (objective.hpp:70-91): squared segment lengths over the leading run of
// positions whose field and cell both match the previous request.
uint64_t hit_of(const Tab& t, const std::vector<Entry>& s, size_t r, int tok, int scoring) {
  if (r == 0) return 0;
  const Entry& a = s[r];
  const Entry& b = s[r - 1];
  size_t lim = std::min(a.fields.size(), b.fields.size());
  uint64_t sum = 0;
  for (size_t p = 0; p < lim; ++p) {
    int f = a.fields[p];
    if (f != b.fields[p]) break;
    if (t.cell(a.row, f) != t.cell(b.row, f)) break;
    uint64_t l = seglen(t, a.row, f, tok, scoring);
    sum += l * l;
  }
  return sum;
}

// phc (objective.hpp:94-99).
uint64_t phc_of(const Tab& t, const std::vector<Entry>& s, int tok, int scoring) {
  uint64_t total = 0;
  for (size_t r = 1; r < s.size(); ++r) total += hit_of(t, s, r, tok, scoring);
  return total;
}

// Lexicographic row order by concatenated fragments under one field order,
// ties by row id (objective.hpp:154-171; ggr.hpp:340-350).
std::vector<uint64_t> fragment_sort(const Tab& t, std::vector<uint64_t> rows,
                                    const std::vector<int>& order) {
  std::vector<std::pair<std::string, uint64_t>> keyed;
  keyed.reserve(rows.size());
  for (uint64_t r : rows) {
    std::string key;
    for (int f : order) key += fragment(t.names[f], t.cell(r, f));
    keyed.emplace_back(std::move(key), r);
  }
  std::sort(keyed.begin(), keyed.end());  // (key, row): row breaks ties like stable_sort
  for (size_t i = 0; i < keyed.size(); ++i) rows[i] = keyed[i].second;
  return rows;
}

// Greedy Group Recursion (ggr.hpp:135-357) restated top-down: the block
// field prefix is carried into the recursion and rows are appended to `out`
// in emission order (block subtree before rest subtree, ggr.hpp:303-313).
class Ggr {
 public:
  Ggr(const Tab& t, const po_fd_groups* fds, const po_ggr_config& cfg, int tok, int scoring)
      : t_(t), cfg_(cfg), tok_(tok), scoring_(scoring) {
    // len_[r][f] (ggr.hpp:149-152)
    len_.resize(t.n * t.m);
    for (uint64_t r = 0; r < t.n; ++r)
      for (uint32_t f = 0; f < t.m; ++f) len_[r * t.m + f] = seglen(t, r, int(f), tok, scoring);
    // partners_[f]: other members of every FD group holding f, each group's
    // members in ascending index order (ggr.hpp:154-164).
    partners_.assign(t.m, {});
    if (cfg.use_fds && fds) {
      for (uint32_t g = 0; g < fds->n_groups; ++g) {
        std::vector<int> mem(fds->members + fds->group_offsets[g],
                             fds->members + fds->group_offsets[g + 1]);
        for (int f : mem)
          if (f < 0 || f >= int(t.m)) fail(PO_ERR_SCHEMA, "unknown field in FD group");
        std::sort(mem.begin(), mem.end());
        for (int f : mem)
          for (int o : mem)
            if (o != f) partners_[f].push_back(o);
      }
    }
  }

  uint64_t calls = 0, cands = 0, maxdepth = 0;

  void solve(std::vector<Entry>& out) {
    std::vector<uint64_t> rows(t_.n);
    std::iota(rows.begin(), rows.end(), 0);
    std::vector<int> cols(t_.m);
    std::iota(cols.begin(), cols.end(), 0);
    node(rows, cols, 0, 0, 0, {}, out);
  }

 private:
  const Tab& t_;
  po_ggr_config cfg_;
  int tok_, scoring_;
  std::vector<uint64_t> len_;
  std::vector<std::vector<int>> partners_;

  uint64_t L(uint64_t r, int f) const { return len_[r * t_.m + uint64_t(f)]; }

  struct Cand {
    unsigned __int128 numer = 0;
    uint64_t count = 0;
    int col = -1;
    std::string_view value;
  };
  // Candidate::better_than (ggr.hpp:189-197): exact rational compare with
  // u128 cross products, then larger count, lower field index, smaller bytes.
  static bool beats(const Cand& a, const Cand& b) {
    unsigned __int128 l = a.numer * b.count, r = b.numer * a.count;
    if (l != r) return l > r;
    if (a.count != b.count) return a.count > b.count;
    if (a.col != b.col) return a.col < b.col;
    return a.value < b.value;
  }

  static void emit(std::vector<Entry>& out, uint64_t row, const std::vector<int>& prefix,
                   const std::vector<int>& tail) {
    Entry e{row, prefix};
    e.fields.insert(e.fields.end(), tail.begin(), tail.end());
    out.push_back(std::move(e));
  }

  // recurse (ggr.hpp:207-314)
  void node(std::vector<uint64_t> rows, const std::vector<int>& cols, uint64_t rd, uint64_t cd,
            uint64_t depth, const std::vector<int>& prefix, std::vector<Entry>& out) {
    ++calls;  // every entry counts, base cases included (ggr.hpp:210-211)
    maxdepth = std::max(maxdepth, depth);
    if (rows.empty()) return;
    if (cols.empty()) {  // ascending row ids, no fields
      std::sort(rows.begin(), rows.end());
      for (uint64_t r : rows) emit(out, r, prefix, {});
      return;
    }
    if (rows.size() == 1) {
      emit(out, rows[0], prefix, cols);
      return;
    }
    if (cols.size() == 1) {  // raw-byte order, then row id (ggr.hpp:221-231)
      int c = cols[0];
      std::stable_sort(rows.begin(), rows.end(), [&](uint64_t a, uint64_t b) {
        std::string_view va = t_.cell(a, c), vb = t_.cell(b, c);
        if (va != vb) return va < vb;
        return a < b;
      });
      for (uint64_t r : rows) emit(out, r, prefix, cols);
      return;
    }
    if (rd > cfg_.row_recursion_depth || cd > cfg_.column_recursion_depth) {
      leaf_fallback(rows, cols, prefix, out);
      return;
    }

    std::vector<char> active(t_.m, 0);
    for (int c : cols) active[c] = 1;

    // Candidate scan (ggr.hpp:239-273), grouping by sorting row ids on the
    // cell bytes so that each run of equal values is one group.
    Cand best;
    bool have = false;
    for (int c : cols) {
      std::vector<int> ap;
      for (int o : partners_[c])
        if (active[o]) ap.push_back(o);
      std::vector<uint64_t> order = rows;
      std::stable_sort(order.begin(), order.end(),
                       [&](uint64_t a, uint64_t b) { return t_.cell(a, c) < t_.cell(b, c); });
      size_t i = 0;
      while (i < order.size()) {
        std::string_view v = t_.cell(order[i], c);
        size_t j = i;
        uint64_t ptot = 0;
        while (j < order.size() && t_.cell(order[j], c) == v) {
          for (int o : ap) ptot += L(order[j], o);
          ++j;
        }
        uint64_t cnt = j - i;
        // value length from the group's first row in `rows` order, i.e. the
        // smallest row id of the run (ggr.hpp:255)
        uint64_t vl = L(*std::min_element(order.begin() + i, order.begin() + j), c);
        ++cands;
        unsigned __int128 numer =
            (static_cast<unsigned __int128>(vl) * vl * cnt + ptot) * (cnt - 1);
        Cand cand{numer, cnt, c, v};
        if (!have || beats(cand, best)) {
          best = cand;
          have = true;
        }
        i = j;
      }
    }
    // Early stop (ggr.hpp:276-278).
    if (!have || best.numer == 0 ||
        best.numer < static_cast<unsigned __int128>(cfg_.hitcount_stop_threshold) * best.count) {
      leaf_fallback(rows, cols, prefix, out);
      return;
    }
    // Split + FD merge (ggr.hpp:280-296).
    std::vector<int> bcols{best.col};
    for (int o : partners_[best.col])
      if (active[o]) bcols.push_back(o);
    std::vector<uint64_t> in, rest;
    for (uint64_t r : rows) (t_.cell(r, best.col) == best.value ? in : rest).push_back(r);
    std::vector<int> sub;
    for (int c : cols)
      if (std::find(bcols.begin(), bcols.end(), c) == bcols.end()) sub.push_back(c);
    std::vector<int> p2 = prefix;
    p2.insert(p2.end(), bcols.begin(), bcols.end());
    node(std::move(in), sub, rd, cd + 1, depth + 1, p2, out);
    node(std::move(rest), cols, rd + 1, cd, depth + 1, prefix, out);
  }

  // fallback (ggr.hpp:318-356): local stats -> stats-ranked field order ->
  // fragment-key row sort.
  void leaf_fallback(const std::vector<uint64_t>& rows, const std::vector<int>& cols,
                     const std::vector<int>& prefix, std::vector<Entry>& out) {
    std::vector<uint64_t> card(cols.size());
    std::vector<double> avg(cols.size());
    for (size_t k = 0; k < cols.size(); ++k) {
      int c = cols[k];
      std::vector<std::string_view> vals;
      uint64_t tot = 0;
      for (uint64_t r : rows) {
        vals.push_back(t_.cell(r, c));
        tot += L(r, c);
      }
      std::sort(vals.begin(), vals.end());
      card[k] = uint64_t(std::unique(vals.begin(), vals.end()) - vals.begin());
      avg[k] = rows.empty() ? 0.0 : static_cast<double>(tot) / rows.size();
    }
    std::vector<int> local = hitcount_order(rows.size(), card, avg, cfg_.stats_variant);
    std::vector<int> order;
    for (int i : local) order.push_back(cols[i]);
    for (uint64_t r : fragment_sort(t_, rows, order)) emit(out, r, prefix, order);
  }
};

void stats_of(const Tab& t, int tok, int scoring, std::vector<uint64_t>& card,
              std::vector<uint64_t>& total) {
  // compute_stats (stats.hpp:25-45)
  card.assign(t.m, 0);
  total.assign(t.m, 0);
  for (uint32_t f = 0; f < t.m; ++f) {
    std::vector<std::string_view> vals;
    vals.reserve(t.n);
    for (uint64_t r = 0; r < t.n; ++r) {
      vals.push_back(t.cell(r, f));
      total[f] += seglen(t, r, int(f), tok, scoring);
    }
    std::sort(vals.begin(), vals.end());
    card[f] = uint64_t(std::unique(vals.begin(), vals.end()) - vals.begin());
  }
}

// validate_field_permutation (objective.hpp:140-149).
void check_perm(uint32_t m, const int32_t* order) {
  std::vector<char> seen(m, 0);
  for (uint32_t i = 0; i < m; ++i) {
    int f = order[i];
    if (f < 0 || f >= int(m) || seen[f])
      fail(PO_ERR_SCHEMA, "field order is not a permutation of the schema");
    seen[f] = 1;
  }
}

// partition_signature (fd.hpp:56-64) restated by sorting: rows ordered by
// (value bytes, row id); every row's signature is the first row of its run.
std::vector<uint64_t> signature(const Tab& t, int f) {
  std::vector<uint64_t> idx(t.n), sig(t.n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(),
                   [&](uint64_t a, uint64_t b) { return t.cell(a, f) < t.cell(b, f); });
  for (uint64_t i = 0; i < t.n; ++i)
    sig[idx[i]] = (i > 0 && t.cell(idx[i], f) == t.cell(idx[i - 1], f)) ? sig[idx[i - 1]] : idx[i];
  return sig;
}

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return PO_OK;
  } catch (const OracleError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PO_ERR_ERROR;
  }
}

}  // namespace

extern "C" {

int oracle_ggr(const po_table* tv, const po_fd_groups* fds, const po_ggr_config* cfg,
               int32_t tok, int32_t scoring, uint64_t* out_rows, uint64_t* out_offsets,
               int32_t* out_fields, uint64_t cap, uint64_t* out_phc, po_solve_stats* out_stats) {
  return guarded([&] {
    auto t0 = std::chrono::steady_clock::now();
    check_modes(tok, scoring);
    if (!cfg) fail(PO_ERR_INVALID_ARG, "null config");
    Tab t(tv);
    Ggr solver(t, fds, *cfg, tok, scoring);
    std::vector<Entry> sched;
    sched.reserve(t.n);
    solver.solve(sched);
    uint64_t score = phc_of(t, sched, tok, scoring);
    // Whole-table fallback competition (ggr.hpp:379-387): replace only when
    // strictly better.
    if (t.n > 0 && t.m > 0) {
      std::vector<uint64_t> card, tot;
      stats_of(t, tok, scoring, card, tot);
      std::vector<double> avg(t.m);
      for (uint32_t f = 0; f < t.m; ++f) avg[f] = static_cast<double>(tot[f]) / t.n;
      std::vector<int> order = hitcount_order(t.n, card, avg, cfg->stats_variant);
      std::vector<uint64_t> all(t.n);
      std::iota(all.begin(), all.end(), 0);
      std::vector<Entry> fb;
      for (uint64_t r : fragment_sort(t, all, order)) fb.push_back({r, order});
      uint64_t fscore = phc_of(t, fb, tok, scoring);
      if (fscore > score) {
        sched = std::move(fb);
        score = fscore;
      }
    }
    uint64_t at = 0;
    for (const auto& e : sched) at += e.fields.size();
    if (at > cap) fail(PO_ERR_SIZE, "oracle: field capacity too small");
    at = 0;
    out_offsets[0] = 0;
    for (uint64_t i = 0; i < sched.size(); ++i) {
      out_rows[i] = sched[i].row;
      for (int f : sched[i].fields) out_fields[at++] = f;
      out_offsets[i + 1] = at;
    }
    *out_phc = score;
    if (out_stats) {
      out_stats->recursive_calls = solver.calls;
      out_stats->candidates_examined = solver.cands;
      out_stats->max_depth = solver.maxdepth;
      out_stats->wall_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

int oracle_phc(const po_table* tv, int32_t tok, int32_t scoring, uint64_t n_entries,
               const uint64_t* row_ids, const uint64_t* order_offsets,
               const int32_t* order_fields, uint64_t* out_phc) {
  return guarded([&] {
    check_modes(tok, scoring);
    Tab t(tv);
    std::vector<Entry> s(n_entries);
    for (uint64_t i = 0; i < n_entries; ++i) {
      s[i].row = row_ids[i];
      s[i].fields.assign(order_fields + order_offsets[i], order_fields + order_offsets[i + 1]);
    }
    *out_phc = phc_of(t, s, tok, scoring);
  });
}

int oracle_sort_rows_fixed_order(const po_table* tv, const int32_t* field_order,
                                 uint64_t* out_rows) {
  return guarded([&] {
    Tab t(tv);
    check_perm(t.m, field_order);
    std::vector<uint64_t> all(t.n);
    std::iota(all.begin(), all.end(), 0);
    std::vector<int> order(field_order, field_order + t.m);
    std::vector<uint64_t> s = fragment_sort(t, all, order);
    std::copy(s.begin(), s.end(), out_rows);
  });
}

int oracle_compute_stats(const po_table* tv, int32_t tok, int32_t scoring, uint64_t* out_card,
                         uint64_t* out_total) {
  return guarded([&] {
    check_modes(tok, scoring);
    Tab t(tv);
    std::vector<uint64_t> card, tot;
    stats_of(t, tok, scoring, card, tot);
    std::copy(card.begin(), card.end(), out_card);
    std::copy(tot.begin(), tot.end(), out_total);
  });
}

int oracle_fixed_order_by_hitcount_stats(uint32_t m, uint64_t total_rows, const uint64_t* card,
                                         const double* avg, int32_t variant, int32_t* out) {
  return guarded([&] {
    std::vector<uint64_t> c(card, card + m);
    std::vector<double> a(avg, avg + m);
    std::vector<int> o = hitcount_order(total_rows, c, a, variant);
    std::copy(o.begin(), o.end(), out);
  });
}

// validate_fds (fd.hpp:66-109): overlap check, then per group the first
// member whose signature differs from the first member's; the witness row
// pair is the earlier row of the matching side and the first differing row.
int oracle_validate_fds(const po_table* tv, const po_fd_groups* fds, uint8_t* out_satisfied,
                        uint8_t* out_has_witness, uint64_t* out_row_a, uint64_t* out_row_b,
                        int32_t* out_agree, int32_t* out_differ) {
  return guarded([&] {
    Tab t(tv);
    std::vector<char> claimed(t.m, 0);
    for (uint32_t k = 0; k < fds->group_offsets[fds->n_groups]; ++k) {
      const int32_t f = fds->members[k];
      if (f < 0 || f >= int32_t(t.m)) fail(PO_ERR_SCHEMA, "unknown field");
      if (claimed[f]) fail(PO_ERR_SCHEMA, "field appears in more than one FD group");
      claimed[f] = 1;
    }
    for (uint32_t g = 0; g < fds->n_groups; ++g) {
      const uint32_t b0 = fds->group_offsets[g], b1 = fds->group_offsets[g + 1];
      out_satisfied[g] = 1;
      out_has_witness[g] = 0;
      if (b1 - b0 < 2 || t.n < 2) continue;
      const int32_t base = fds->members[b0];
      const std::vector<uint64_t> bs = signature(t, base);
      for (uint32_t k = b0 + 1; k < b1 && out_satisfied[g]; ++k) {
        const std::vector<uint64_t> os = signature(t, fds->members[k]);
        for (uint64_t r = 0; r < t.n; ++r) {
          if (bs[r] == os[r]) continue;
          out_satisfied[g] = 0;
          out_has_witness[g] = 1;
          const bool base_earlier = bs[r] != r;
          out_row_a[g] = base_earlier ? bs[r] : os[r];
          out_row_b[g] = r;
          out_agree[g] = base_earlier ? base : fds->members[k];
          out_differ[g] = base_earlier ? fds->members[k] : base;
          break;
        }
      }
    }
  });
}

// discover_fds (fd.hpp:114-141): size cap, then fields joined to the first
// earlier class with an identical signature; singleton classes dropped.
int oracle_discover_fds(const po_table* tv, uint64_t max_rows, int32_t* out_group_of_field) {
  return guarded([&] {
    Tab t(tv);
    if (t.n > max_rows) fail(PO_ERR_SIZE, "discover_fds: table exceeds the row cap");
    std::vector<std::vector<uint64_t>> class_sig;
    std::vector<std::vector<int>> members;
    for (uint32_t f = 0; f < t.m; ++f) {
      std::vector<uint64_t> sg = signature(t, int(f));
      size_t c = 0;
      while (c < class_sig.size() && class_sig[c] != sg) ++c;
      if (c == class_sig.size()) {
        class_sig.push_back(std::move(sg));
        members.push_back({});
      }
      members[c].push_back(int(f));
    }
    int32_t g = 0;
    for (uint32_t f = 0; f < t.m; ++f) out_group_of_field[f] = -1;
    for (const auto& mem : members) {
      if (mem.size() < 2) continue;
      for (int f : mem) out_group_of_field[f] = g;
      ++g;
    }
  });
}

// render_prompt (objective.hpp:118-131) = [sp '\n'][q '\n'] + render_body
// (objective.hpp:102-115) = '{' + join(", ", '"' esc(name) '": "' esc(v) '"') + '}'.
int oracle_render_prompts(const po_table* tv, uint64_t n_entries, const uint64_t* rows,
                          const uint64_t* offs, const int32_t* fields, const uint8_t* sp,
                          uint64_t sp_len, const uint8_t* q, uint64_t q_len,
                          uint64_t* out_offsets, uint8_t* out_bytes, uint64_t capacity,
                          uint64_t* out_total) {
  return guarded([&] {
    Tab t(tv);
    std::string prefix;
    if (sp && sp_len) prefix += std::string(reinterpret_cast<const char*>(sp), sp_len) + "\n";
    if (q && q_len) prefix += std::string(reinterpret_cast<const char*>(q), q_len) + "\n";
    uint64_t pos = 0;
    out_offsets[0] = 0;
    for (uint64_t i = 0; i < n_entries; ++i) {
      std::string p = prefix + "{";
      for (uint64_t k = offs[i]; k < offs[i + 1]; ++k) {
        if (k > offs[i]) p += ", ";
        const std::string_view v = t.cell(rows[i], fields[k]);  // range-checked
        p += "\"" + escape(t.names[fields[k]]) + "\": \"" + escape(v) + "\"";
      }
      p += "}";
      if (out_bytes && pos + p.size() <= capacity) std::memcpy(out_bytes + pos, p.data(), p.size());
      pos += p.size();
      out_offsets[i + 1] = pos;
    }
    *out_total = pos;
  });
}

// dedup (cost.hpp:171-186) restated by sorting: stable order by bytes, the
// first index of each run of equal strings names the unique; uniques are
// numbered by first occurrence.
int oracle_dedup(uint64_t n, const uint8_t* arena, const uint64_t* offsets,
                 uint64_t* out_expansion, uint64_t* out_unique_first, uint64_t* out_n_unique) {
  return guarded([&] {
    auto str = [&](uint64_t i) {
      return std::string_view(reinterpret_cast<const char*>(arena) + offsets[i],
                              offsets[i + 1] - offsets[i]);
    };
    std::vector<uint64_t> idx(n), first(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) { return str(a) < str(b); });
    for (uint64_t k = 0; k < n; ++k)
      first[idx[k]] = (k > 0 && str(idx[k]) == str(idx[k - 1])) ? first[idx[k - 1]] : idx[k];
    std::vector<uint64_t> uid(n, 0);
    uint64_t nu = 0;
    for (uint64_t i = 0; i < n; ++i)
      if (first[i] == i) {
        uid[i] = nu;
        out_unique_first[nu++] = i;
      }
    for (uint64_t i = 0; i < n; ++i) out_expansion[i] = uid[first[i]];
    *out_n_unique = nu;
  });
}

const char* oracle_last_error(void) { return g_err.c_str(); }

}  // extern "C"
