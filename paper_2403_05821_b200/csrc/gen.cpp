// Deterministic synthetic tables for the BASELINE configs C1..C5
// (SURVEY.md §8d). Counter-based: every cell is a pure function of
// (config, seed, column, row), so any row range can be generated
// independently (row-sharded multi-GPU runs, CPU-baseline subsamples) and
// both the GPU path and the CPU reference read byte-identical tables.
//
// Built into libpogen.so (host only, not part of the product path).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

inline uint64_t mix(uint64_t x) {  // SplitMix64 finaliser
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
inline uint64_t h3(uint64_t a, uint64_t b, uint64_t c) { return mix(mix(mix(a) ^ b) ^ c); }
inline double unit(uint64_t h) { return double(h >> 11) * (1.0 / 9007199254740992.0); }

struct Vocab {
  std::vector<std::string> words;
  explicit Vocab(uint64_t seed) {
    for (int i = 0; i < 2048; ++i) {
      uint64_t h = h3(seed, 0xABCDEF, uint64_t(i));
      int len = 2 + int(h % 8);
      std::string w;
      for (int k = 0; k < len; ++k) w += char('a' + (mix(h + k) % 26));
      if ((h >> 40) % 7 == 0) w[0] = char(w[0] - 32);
      words.push_back(w);
    }
  }
};

// Zipf(s) over K values by inverse CDF.
struct Zipf {
  std::vector<double> cdf;
  Zipf() = default;
  Zipf(uint64_t K, double s) {
    cdf.resize(K);
    double acc = 0;
    for (uint64_t k = 0; k < K; ++k) {
      acc += 1.0 / std::pow(double(k + 1), s);
      cdf[k] = acc;
    }
    for (auto& c : cdf) c /= acc;
  }
  uint64_t sample(double u) const {
    return uint64_t(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
  }
};

enum Kind { UNIFORM, ZIPF, SAME_AS, UNIQUE, CATEGORICAL, ID, GROUP3 };

struct Col {
  const char* name;
  Kind kind;
  uint64_t card;     // UNIFORM/ZIPF/CATEGORICAL
  double s;          // ZIPF exponent
  int len;           // mean text length
  int src;           // SAME_AS: column whose value id this column reuses
  int pool;          // text namespace (equal pool + id => equal bytes)
  std::vector<std::string> cats;  // CATEGORICAL fixed texts
  std::vector<double> weights;    // CATEGORICAL probabilities
  Zipf zipf;
};

struct Config {
  std::vector<Col> cols;
  bool inject = false;      // escapable / non-ASCII bytes in ~1% of distinct values
  double dup_rows = 0.0;    // fraction of exact-duplicate rows
};

Config make_config(int id) {
  Config c;
  auto col = [](const char* name, Kind k, uint64_t card, double s, int len, int src, int pool) {
    Col x;
    x.name = name;
    x.kind = k;
    x.card = card;
    x.s = s;
    x.len = len;
    x.src = src;
    x.pool = pool;
    return x;
  };
  auto cat = [](const char* name, std::vector<std::string> v, std::vector<double> w) {
    Col x;
    x.name = name;
    x.kind = CATEGORICAL;
    x.card = v.size();
    x.cats = std::move(v);
    x.weights = std::move(w);
    return x;
  };
  switch (id) {
    case 1:  // demo 10K x 4, controlled cardinality, uniform
      c.cols = {col("category", UNIFORM, 8, 0, 32, -1, 1), col("brand", UNIFORM, 100, 0, 16, -1, 2),
                col("product", UNIFORM, 2000, 0, 48, -1, 3), col("note", UNIQUE, 0, 0, 24, -1, 4)};
      c.inject = true;
      break;
    case 2:  // Amazon-products shape 1M x 6
      c.cols = {col("title", ZIPF, 50000, 1.1, 60, -1, 1),
                col("description", SAME_AS, 0, 0, 400, 0, 2),
                col("reviewerName", ZIPF, 200000, 1.05, 14, -1, 3),
                cat("rating", {"5.0", "4.0", "3.0", "2.0", "1.0"}, {0.55, 0.2, 0.1, 0.06, 0.09}),
                cat("verified_purchase", {"True", "False"}, {0.8, 0.2}),
                col("reviewText", UNIQUE, 0, 0, 250, -1, 6)};
      c.inject = true;
      break;
    case 3:  // Movies shape 10M x 5, movie_title <-> movie_info
      c.cols = {col("movie_title", ZIPF, 200000, 1.0, 20, -1, 1),
                col("movie_info", SAME_AS, 0, 0, 300, 0, 2),
                cat("review_type", {"Fresh", "Rotten"}, {0.6, 0.4}),
                cat("top_critic", {"True", "False"}, {0.2, 0.8}),
                col("review_content", UNIQUE, 0, 0, 120, -1, 5)};
      c.inject = true;
      break;
    case 4:  // mixed 100M x 8
      c.cols = {cat("flag", {"True", "False"}, {0.5, 0.5}),
                cat("digit", {"0", "1", "2", "3", "4", "5", "6", "7", "8", "9"},
                    std::vector<double>(10, 0.1)),
                col("category", UNIFORM, 300, 0, 24, -1, 3), col("item", ZIPF, 1000000, 1.0, 200, -1, 4),
                col("item_detail", SAME_AS, 0, 0, 600, 3, 5), col("vendor", UNIFORM, 100000, 0, 40, -1, 6),
                col("uid", ID, 0, 0, 12, -1, 7), col("group3", GROUP3, 0, 0, 90, -1, 8)};
      break;
    case 5:  // FEVER/SQuAD shape 20M x 5, ~2 KB evidence, 20% duplicate rows
      c.cols = {col("claim", ZIPF, 10000000, 0.8, 80, -1, 1),
                col("evidence1", ZIPF, 2000000, 1.0, 2048, -1, 9),
                col("evidence2", ZIPF, 2000000, 1.0, 2048, -1, 9),
                col("evidence3", ZIPF, 2000000, 1.0, 2048, -1, 9),
                col("evidence4", ZIPF, 2000000, 1.0, 2048, -1, 9)};
      c.dup_rows = 0.2;
      break;
    default:
      break;
  }
  for (auto& x : c.cols)
    if (x.kind == ZIPF) x.zipf = Zipf(x.card, x.s);
  return c;
}

struct Gen {
  Config cfg;
  uint64_t seed;
  Vocab vocab;
  Gen(int id, uint64_t sd) : cfg(make_config(id)), seed(sd), vocab(sd) {}

  uint64_t source_row(uint64_t r) const {
    if (cfg.dup_rows <= 0) return r;
    for (int guard = 0; guard < 64 && r > 0; ++guard) {
      uint64_t h = h3(seed, 0xD0D0, r);
      if (unit(h) >= cfg.dup_rows) return r;
      r = r - 1 - (mix(h) % std::min<uint64_t>(r, 1000));
    }
    return r;
  }

  // value id of column c in row r
  uint64_t value_id(int c, uint64_t r) const {
    const Col& x = cfg.cols[c];
    uint64_t h = h3(seed, uint64_t(c) + 1, r);
    switch (x.kind) {
      case UNIFORM: return h % x.card;
      case ZIPF: return x.zipf.sample(unit(h));
      case SAME_AS: return value_id(x.src, r);
      case UNIQUE:
      case ID: return r;
      case GROUP3: return r / 3;
      case CATEGORICAL: {
        double u = unit(h), acc = 0;
        for (size_t k = 0; k < x.weights.size(); ++k) {
          acc += x.weights[k];
          if (u < acc) return k;
        }
        return x.weights.size() - 1;
      }
    }
    return 0;
  }

  void text(int c, uint64_t v, std::string& out) const {
    const Col& x = cfg.cols[c];
    out.clear();
    if (x.kind == CATEGORICAL) {
      out = x.cats[v];
      return;
    }
    if (x.kind == ID) {
      char buf[32];
      snprintf(buf, sizeof buf, "id-%09llu", (unsigned long long)v);
      out = buf;
      return;
    }
    uint64_t h = h3(seed ^ 0x5151, uint64_t(x.pool), v);
    int target = std::max(1, x.len / 2 + int(h % uint64_t(x.len + 1)));
    if (x.kind == UNIQUE || x.kind == GROUP3) {
      char buf[32];
      snprintf(buf, sizeof buf, "#%llu ", (unsigned long long)v);
      out = buf;
    }
    for (uint64_t k = 0; int(out.size()) < target; ++k) {
      if (!out.empty() && out.back() != ' ') out += ' ';
      out += vocab.words[mix(h + 0x77 * (k + 1)) % vocab.words.size()];
    }
    if (int(out.size()) > target) out.resize(target);
    if (cfg.inject && (mix(h ^ 0xE5C) % 100) == 0) {
      static const char* specials[] = {"\"", "\\", "\n", "\x01", "\xC3\xA9", "\t"};
      uint64_t g = mix(h ^ 0xF00D);
      out.insert(g % (out.size() + 1), specials[(g >> 20) % 6]);
    }
  }
};

}  // namespace

extern "C" {

int pogen_n_fields(int config) { return int(make_config(config).cols.size()); }

const char* pogen_field_name(int config, int f) {
  static thread_local Config c;
  c = make_config(config);
  return (f >= 0 && f < int(c.cols.size())) ? c.cols[f].name : nullptr;
}

// Generates rows [row_begin, row_begin + n_rows) of config `config`.
// Pass 1 (arena == NULL): fills offsets (n_rows*m + 1, starting at 0) and
// returns the arena size. Pass 2: writes the bytes. Returns -1 on bad config.
long long pogen_generate_cols(int config, uint64_t seed, uint64_t row_begin, uint64_t n_rows,
                              uint64_t colmask, uint64_t* offsets, uint8_t* arena, int n_threads);

long long pogen_generate(int config, uint64_t seed, uint64_t row_begin, uint64_t n_rows,
                         uint64_t* offsets, uint8_t* arena, int n_threads) {
  return pogen_generate_cols(config, seed, row_begin, n_rows, ~0ull, offsets, arena, n_threads);
}

// Same as pogen_generate restricted to the columns whose bit is set in
// colmask (value ids still come from the full row, so FDs are preserved).
long long pogen_generate_cols(int config, uint64_t seed, uint64_t row_begin, uint64_t n_rows,
                              uint64_t colmask, uint64_t* offsets, uint8_t* arena, int n_threads) {
  Gen g(config, seed);
  std::vector<int> sel;
  for (int c = 0; c < int(g.cfg.cols.size()); ++c)
    if ((colmask >> c) & 1) sel.push_back(c);
  const int m = int(sel.size());
  if (m == 0) return -1;
  if (n_threads <= 0) n_threads = int(std::max(1u, std::thread::hardware_concurrency()));
  n_threads = int(std::min<uint64_t>(uint64_t(n_threads), std::max<uint64_t>(1, n_rows / 1024 + 1)));
  std::vector<std::thread> th;
  if (!arena) {
    // lengths, then an exclusive prefix sum
    auto work = [&](int t) {
      std::string s;
      uint64_t lo = n_rows * t / n_threads, hi = n_rows * (t + 1) / n_threads;
      for (uint64_t i = lo; i < hi; ++i) {
        uint64_t r = g.source_row(row_begin + i);
        for (int k = 0; k < m; ++k) {
          g.text(sel[k], g.value_id(sel[k], r), s);
          offsets[i * m + k + 1] = s.size();
        }
      }
    };
    for (int t = 0; t < n_threads; ++t) th.emplace_back(work, t);
    for (auto& x : th) x.join();
    offsets[0] = 0;
    for (uint64_t i = 1; i <= n_rows * m; ++i) offsets[i] += offsets[i - 1];
    return (long long)offsets[n_rows * m];
  }
  auto work = [&](int t) {
    std::string s;
    uint64_t lo = n_rows * t / n_threads, hi = n_rows * (t + 1) / n_threads;
    for (uint64_t i = lo; i < hi; ++i) {
      uint64_t r = g.source_row(row_begin + i);
      for (int k = 0; k < m; ++k) {
        g.text(sel[k], g.value_id(sel[k], r), s);
        std::memcpy(arena + offsets[i * m + k], s.data(), s.size());
      }
    }
  };
  for (int t = 0; t < n_threads; ++t) th.emplace_back(work, t);
  for (auto& x : th) x.join();
  return (long long)offsets[n_rows * m];
}

}  // extern "C"
