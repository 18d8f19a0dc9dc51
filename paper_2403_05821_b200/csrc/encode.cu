// K3 rank_sort + id remap + counts around the K1/K2 dictionary (dict.cu):
// exact per-column dictionary encoding of the table on the GPU.
//
// Reference behaviour replaced:
//   * every std::unordered_map/set<string_view> over cells (ggr.hpp:251,
//     ggr.hpp:324, stats.hpp:33) and every string == (ggr.hpp:286,
//     objective.hpp:86) becomes an integer compare on `vid`;
//   * std::string < in the single-column base case (ggr.hpp:223-228) and the
//     candidate tie-break (ggr.hpp:196) becomes vid order (vid IS the raw-byte
//     rank);
//   * the fragment-key compare of the statistics fallback (ggr.hpp:340-350,
//     objective.hpp:156-166) becomes esc_rank order;
//   * segment_len/Tokenizer::count (scoring.hpp:72-76, tokenizer.hpp:44,
//     64-73) is evaluated once per distinct value.
//
// The cell bytes are read once, by the fused dictionary pass (dict.cu);
// everything here works on its per-distinct output.

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "internal.cuh"

namespace po {

namespace {

__global__ void k_iota_pos(uint32_t* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    a[i] = uint32_t(i);
}

// Items of the ranked columns only: item k -> distinct index d (the ranked
// columns' d-ranges, rbase[j] .. + (rpre[j+1] - rpre[j]), concatenated).
__global__ void k_ranked_items(const uint64_t* rbase, const uint64_t* rpre, uint32_t nr,
                               uint64_t total, const uint32_t* d_col, uint32_t* sub_d,
                               uint32_t* sub_col) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t j = 0;
    while (j + 1 < nr && rpre[j + 1] <= k) ++j;
    const uint64_t d = rbase[j] + (k - rpre[j]);
    sub_d[k] = uint32_t(d);
    sub_col[k] = d_col[d];
  }
}

__global__ void k_scatter_sub(const uint32_t* sub_d, const uint32_t* sub_pos, uint64_t total,
                              uint32_t* pos) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x)
    pos[sub_d[k]] = sub_pos[k];
}


// pos[d] (escaped order) of every distinct value d (compaction order): its
// id map, and its bytes / representative row / column scattered into vid
// order.
__global__ void k_scatter_pos(const uint32_t* pos_of, const uint32_t* d_col, const uint64_t* colbase,
                              uint64_t D, const uint64_t* val_off, const uint32_t* val_len,
                              const uint32_t* rep_row, uint32_t* cid2vid, uint64_t* off_by_pos,
                              uint32_t* len_by_pos, uint32_t* row_by_pos, uint32_t* col_by_pos) {
  for (uint64_t d = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; d < D;
       d += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t p = pos_of[d];
    const uint32_t c = d_col[d];
    cid2vid[d] = uint32_t(p - colbase[c]);
    off_by_pos[p] = val_off[d];
    len_by_pos[p] = val_len[d];
    row_by_pos[p] = rep_row[d];
    col_by_pos[p] = c;
  }
}

__device__ __forceinline__ bool is_ws(uint8_t c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v';
}

// Escaped length of one byte under json_escape (scoring.hpp:33-57).
__device__ __forceinline__ uint32_t esc_len(uint8_t c) {
  if (c == '"' || c == '\\' || c == '\b' || c == '\f' || c == '\n' || c == '\r' || c == '\t')
    return 2;
  return c < 0x20 ? 6 : 1;
}

struct TextLen {
  uint64_t bytes, esc_bytes, word_runs, space_runs;
  bool empty, lead_space, trail_space;
};

// One pass over a byte string: raw length, escaped length, word runs under
// the six-byte whitespace set (WordTokenizer), and runs of non-' ' bytes
// (the only whitespace left after json_escape).
__device__ TextLen text_len(const uint8_t* p, uint64_t len) {
  TextLen t{len, 0, 0, 0, len == 0, false, false};
  bool prev_ws = true, prev_sp = true;
  for (uint64_t j = 0; j < len; ++j) {
    uint8_t c = p[j];
    t.esc_bytes += esc_len(c);
    bool w = is_ws(c), sp = c == ' ';
    if (!w && prev_ws) ++t.word_runs;
    if (!sp && prev_sp) ++t.space_runs;
    prev_ws = w;
    prev_sp = sp;
  }
  if (len) {
    t.lead_space = p[0] == ' ';
    t.trail_space = p[len - 1] == ' ';
  }
  return t;
}

// Word count of `"X":` / `"X",` where X is an escaped string whose only
// whitespace is ' ': runs(X) + [X empty or starts with ' '] + [X ends with ' '].
__device__ __forceinline__ uint64_t frag_words(const TextLen& t) {
  return t.space_runs + ((t.empty || t.lead_space) ? 1 : 0) + ((!t.empty && t.trail_space) ? 1 : 0);
}

// Segment length of every distinct value (segment_len, scoring.hpp:72-76).
// fragment = '"' esc(f) '": "' esc(v) '", ' => char: |esc f| + |esc v| + 8;
// word: frag_words(f) + frag_words(v).
__global__ void k_vlen(const uint8_t* vals, const uint64_t* val_off, const uint32_t* val_len,
                       const uint64_t* cell_lens, const uint32_t* row_by_pos,
                       const uint32_t* col_by_pos, uint64_t D, uint32_t m, int tok, int scoring,
                       const uint64_t* name_char_len, const uint64_t* name_word_len,
                       uint64_t* vlen) {
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < D;
       p += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t c = col_by_pos[p];
    if (tok == PO_TOK_CUSTOM) {
      vlen[p] = cell_lens[uint64_t(row_by_pos[p]) * m + c];
      continue;
    }
    const uint64_t len = val_len[p];
    if (tok == PO_TOK_CHAR && scoring == PO_SCORE_VALUE) {
      vlen[p] = len;  // CharTokenizer::count == byte length (tokenizer.hpp:44)
      continue;
    }
    TextLen t = text_len(vals + val_off[p], len);
    uint64_t L;
    if (scoring == PO_SCORE_VALUE)
      L = tok == PO_TOK_CHAR ? t.bytes : t.word_runs;
    else
      L = tok == PO_TOK_CHAR ? name_char_len[c] + t.esc_bytes + 8 : name_word_len[c] + frag_words(t);
    vlen[p] = L;
  }
}

// Dictionary ids (first-claim order) -> vids (escaped order), in place.
__global__ void k_vid(uint32_t* ids, uint64_t n, uint32_t m, const uint64_t* colbase,
                      const uint32_t* cid2vid) {
  const uint64_t total = n * m;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t c = uint32_t(i % m);
    ids[i] = cid2vid[colbase[c] + ids[i]];
  }
}

// Occurrence count per (column, vid), all columns in one pass over the vid
// matrix: low-cardinality columns are counted in a shared-memory histogram
// (soff[c] = their bin offset, kSmemBins total), the others with spread
// global atomics.
constexpr uint32_t kSmemBins = 12288;
constexpr uint32_t kLargeCol = 0xFFFFFFFFu;
constexpr uint32_t kUniqueCol = 0xFFFFFFFEu;  // card == n: every count is 1

__global__ void __launch_bounds__(512) k_count(const uint32_t* vid, uint64_t n, uint32_t m,
                                               const uint32_t* soff, uint32_t nbins,
                                               const uint64_t* colbase, uint32_t* count) {
  extern __shared__ uint32_t h[];
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  // Warps walk 32 rows column by column; lanes holding the same value (the
  // frequent values of skewed columns) add once per warp (one atomic per
  // distinct value in the warp instead of one per cell).
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t ntiles = (n + 31) / 32;
  for (uint64_t tile = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; tile < ntiles;
       tile += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    const uint64_t r = tile * 32 + lane;
    const bool live = r < n;
    const uint32_t act = __ballot_sync(0xffffffffu, live);
    for (uint32_t c = 0; c < m; ++c) {
      const uint32_t o = soff[c];
      if (o == kUniqueCol) {
        if (live) count[colbase[c] + vid[r * m + c]] = 1u;
        continue;
      }
      if (!live) continue;
      const uint32_t v = vid[r * m + c];
      const uint32_t peers = __match_any_sync(act, v);
      if (lane != uint32_t(__ffs(peers) - 1)) continue;
      const uint32_t k = uint32_t(__popc(peers));
      if (o != kLargeCol) atomicAdd(&h[o + v], k);
      else atomicAdd(&count[colbase[c] + v], k);
    }
  }
  __syncthreads();
  // flush: the small column owning bin b is the one with the largest
  // offset <= b (columns are few; linear scan)
  for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x)
    if (h[b]) {
      uint32_t owner = 0, best = 0;
      for (uint32_t cc = 0; cc < m; ++cc)
        if (soff[cc] < kUniqueCol && soff[cc] <= b && soff[cc] >= best) {
          best = soff[cc];
          owner = cc;
        }
      atomicAdd(&count[colbase[owner] + (b - soff[owner])], h[b]);
    }
}

// Per-column sum of count*vlen (stats.hpp:38). Dictionary positions are
// grouped by column, so each thread sums a contiguous run of kTotRun entries
// in a register and flushes only at column changes; the m per-block
// accumulators in shared memory then take one global atomic each.
constexpr uint32_t kTotRun = 16;

__global__ void k_total_len(const uint32_t* count, const uint64_t* vlen, const uint32_t* col_by_pos,
                            uint64_t D, uint32_t m, unsigned long long* total) {
  extern __shared__ unsigned long long acc[];
  const bool priv = m <= 4096;
  if (priv)
    for (uint32_t c = threadIdx.x; c < m; c += blockDim.x) acc[c] = 0;
  __syncthreads();
  auto flush = [&](uint32_t c, unsigned long long v) {
    if (!v) return;
    if (priv) atomicAdd(&acc[c], v);
    else atomicAdd(&total[c], v);
  };
  const uint64_t runs = (D + kTotRun - 1) / kTotRun;
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < runs;
       q += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t lo = q * kTotRun, hi = lo + kTotRun < D ? lo + kTotRun : D;
    uint32_t cur = col_by_pos[lo];
    unsigned long long sum = 0;
    for (uint64_t p = lo; p < hi; ++p) {
      const uint32_t c = col_by_pos[p];
      if (c != cur) {
        flush(cur, sum);
        cur = c;
        sum = 0;
      }
      sum += uint64_t(count[p]) * vlen[p];
    }
    flush(cur, sum);
  }
  if (priv) {
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < m; c += blockDim.x)
      if (acc[c]) atomicAdd(&total[c], acc[c]);
  }
}

uint64_t word_count_host(const std::string& s) {
  uint64_t n = 0;
  bool prev = true;
  for (unsigned char c : s) {
    bool w = c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v';
    if (!w && prev) ++n;
    prev = w;
  }
  return n;
}

std::string json_escape_host(const std::string& s) {
  static const char hexd[] = "0123456789abcdef";
  std::string o;
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          o += "\\u00";
          o += hexd[c >> 4];
          o += hexd[c & 15];
        } else {
          o += char(c);
        }
    }
  }
  return o;
}

}  // namespace

void make_device_table(const po_table* t, int tok, cudaStream_t s, DeviceTable& out,
                       bool stream_host) {
  if (!t) fail(PO_ERR_INVALID_ARG, "null table");
  if (t->location != PO_LOC_HOST && t->location != PO_LOC_DEVICE)
    fail(PO_ERR_INVALID_ARG, "bad table location");
  out.n = t->n_rows;
  out.m = t->n_fields;
  if (out.m && !t->field_names) fail(PO_ERR_INVALID_ARG, "null field names");
  out.names.clear();
  for (uint32_t f = 0; f < out.m; ++f)
    out.names.emplace_back(t->field_names[f], t->field_name_lens ? t->field_name_lens[f]
                                                                  : strlen(t->field_names[f]));
  const uint64_t cells = out.n * out.m;
  if (cells >= (uint64_t(1) << 32) || out.n >= 0xFFFFFFFFull)
    fail(PO_ERR_SIZE, "table too large for one device (rows*fields must be < 2^32)");
  if (cells == 0) return;
  if (!t->offsets) fail(PO_ERR_INVALID_ARG, "null offsets");
  if (tok == PO_TOK_CUSTOM && !t->cell_lens)
    fail(PO_ERR_INVALID_ARG, "custom tokenizer requires cell_lens");
  if (t->location == PO_LOC_HOST) {
    out.arena_bytes = t->offsets[cells];
  } else {
    PO_CUDA(cudaMemcpyAsync(&out.arena_bytes, t->offsets + cells, sizeof(uint64_t),
                            cudaMemcpyDeviceToHost, s));
    sync(s);
  }
  // an all-empty table may come with a null arena (an empty std::vector's
  // data(), a size-0 device tensor): the kernels get a valid dummy byte
  if (!t->arena && out.arena_bytes) fail(PO_ERR_INVALID_ARG, "null arena");
  static const uint8_t kEmptyByte = 0;
  if (t->location == PO_LOC_HOST) {
    if (tok == PO_TOK_CUSTOM) {
      out.own_lens.alloc(cells, s);
      out.own_lens.upload(t->cell_lens, cells);
      out.cell_lens = out.own_lens.get();
    }
    if (stream_host) {  // the dictionary pass copies row chunks itself
      out.h_arena = t->arena ? t->arena : &kEmptyByte;
      out.h_offsets = t->offsets;
      return;
    }
    out.own_offsets.alloc(cells + 1, s);
    out.own_offsets.upload(t->offsets, cells + 1);
    out.own_arena.alloc(std::max<uint64_t>(out.arena_bytes, 1), s);
    out.own_arena.upload(t->arena, out.arena_bytes);
    out.arena = out.own_arena.get();
    out.offsets = out.own_offsets.get();
  } else {
    if (t->arena) {
      out.arena = t->arena;
    } else {
      out.own_arena.alloc(1, s);
      out.arena = out.own_arena.get();
    }
    out.offsets = t->offsets;
    out.cell_lens = tok == PO_TOK_CUSTOM ? t->cell_lens : nullptr;
  }
}

void encode(const DeviceTable& t, int tok, int scoring, cudaStream_t s, Encoded& e,
            uint32_t hash_bits_debug, bool ordered, bool rank_unique) {
  e.n = t.n;
  e.m = t.m;
  e.card.assign(t.m, 0);
  e.colbase.assign(t.m + 1, 0);
  e.total_len.assign(t.m, 0);
  e.D = 0;
  const uint64_t n = t.n, m = t.m, cells = n * m;
  if (cells == 0) {
    e.d_colbase = to_device(e.colbase, s);
    return;
  }
  // K1 + K2: dictionary ids per cell (first-claim order) in e.vid
  e.vid.alloc_auto(cells, s);
  DictResult dr;
  build_dictionary(t, hash_bits_debug, s, e.vid.get(), dr);
  timing_mark("dict", s);
  e.card = dr.card;
  e.colbase = dr.colbase;
  e.D = dr.D;
  const uint64_t D = e.D;
  e.d_colbase = std::move(dr.d_colbase);
  e.val_arena = dr.val_arena;
  e.val_bytes = dr.val_bytes;
  e.own_vals = std::move(dr.own_vals);

  // Escaped fragment-key order (json_escape(v) + '"') of the distinct values
  // of each column -> vid. Raw-byte order is only needed for candidate ties
  // and single-column leaves; the solver ranks those few values on demand.
  DevBuf<uint32_t> esc_pos(D, s);
  RefineKey ek;
  ek.kind = 1;
  ek.arena = e.val_arena;
  ek.arena_bytes = e.val_bytes;
  ek.str_off = dr.val_off.get();
  ek.str_len = dr.val_len.get();
  // rank_unique = false: a column with a distinct value per row (n > 1)
  // keeps ids in first-claim order (Encoded::unranked); its order is only
  // needed to break ties inside a sort, which sorts by its bytes instead.
  e.unranked.assign(m, 0);
  if (ordered && !rank_unique && n > 1)
    for (uint32_t c = 0; c < m; ++c) e.unranked[c] = e.card[c] == n;
  std::vector<uint64_t> rbase, rpre{0};
  for (uint32_t c = 0; c < m; ++c)
    if (!e.unranked[c] && e.card[c]) {
      rbase.push_back(e.colbase[c]);
      rpre.push_back(rpre.back() + e.card[c]);
    }
  const uint64_t n_ranked = rpre.back();
  if (!ordered || n_ranked < D)  // identity (dedup, FD checks, unranked columns)
    PO_LAUNCH(k_iota_pos, grid_for(D, 256), 256, 0, s, esc_pos.get(), D);
  if (ordered && n_ranked) {
    // round 0 groups the distinct values by column index
    std::vector<uint32_t> cb32(m);
    for (uint32_t c = 0; c < m; ++c) cb32[c] = uint32_t(e.colbase[c]);
    DevBuf<uint32_t> d_cb32 = to_device(cb32, s);
    RefineJob je;
    je.n_groups = uint32_t(m);
    je.grp_max = uint32_t(D);
    je.key = ek;
    je.d_grp_start = d_cb32.get();
    if (n_ranked == D) {
      je.n_items = uint32_t(D);
      je.d_grp_init = dr.d_col.get();
      je.d_out_pos = esc_pos.get();
      refine_sort_multi({je}, s);
    } else {
      DevBuf<uint64_t> d_rbase = to_device(rbase, s), d_rpre = to_device(rpre, s);
      DevBuf<uint32_t> sub_d(n_ranked, s), sub_col(n_ranked, s), sub_pos(n_ranked, s);
      PO_LAUNCH(k_ranked_items, grid_for(n_ranked, 256), 256, 0, s, d_rbase.get(), d_rpre.get(),
                uint32_t(rbase.size()), n_ranked, dr.d_col.get(), sub_d.get(), sub_col.get());
      je.n_items = uint32_t(n_ranked);
      je.d_grp_init = sub_col.get();
      je.key.item_ref = sub_d.get();
      je.d_out_pos = sub_pos.get();
      refine_sort_multi({je}, s);
      PO_LAUNCH(k_scatter_sub, grid_for(n_ranked, 256), 256, 0, s, sub_d.get(), sub_pos.get(),
                n_ranked, esc_pos.get());
    }
  }
  timing_mark("rank_sort", s);

  DevBuf<uint32_t> cid2vid(D, s), col_by_pos(D, s);
  e.rep_row.alloc_auto(D, s);
  e.val_off.alloc_auto(D, s);
  e.val_len.alloc_auto(D, s);
  PO_LAUNCH(k_scatter_pos, grid_for(D, 256), 256, 0, s, esc_pos.get(), dr.d_col.get(),
            e.d_colbase.get(), D, dr.val_off.get(), dr.val_len.get(), dr.rep_row.get(),
            cid2vid.get(), e.val_off.get(), e.val_len.get(), e.rep_row.get(), col_by_pos.get());
  timing_mark("scatter_pos", s);

  // Segment length per distinct value.
  std::vector<uint64_t> nchar(m), nword(m);
  for (uint32_t c = 0; c < m; ++c) {
    std::string esc = json_escape_host(t.names[c]);
    nchar[c] = esc.size();
    // frag_words for the name, computed on the host with the same rule
    uint64_t runs = 0;
    bool prev = true;
    for (unsigned char ch : esc) {
      bool sp = ch == ' ';
      if (!sp && prev) ++runs;
      prev = sp;
    }
    bool empty = esc.empty();
    nword[c] = runs + ((empty || esc.front() == ' ') ? 1 : 0) + ((!empty && esc.back() == ' ') ? 1 : 0);
  }
  (void)word_count_host;
  DevBuf<uint64_t> d_nchar = to_device(nchar, s), d_nword = to_device(nword, s);
  e.vlen.alloc_auto(D, s);
  PO_LAUNCH(k_vlen, grid_for(D, 256), 256, 0, s, e.val_arena, e.val_off.get(), e.val_len.get(),
            t.cell_lens, e.rep_row.get(), col_by_pos.get(), D, uint32_t(m), tok, scoring,
            d_nchar.get(), d_nword.get(), e.vlen.get());
  timing_mark("vlen", s);

  // vid matrix (row-major, in place) and occurrence counts.
  PO_LAUNCH(k_vid, grid_for(cells, 256), 256, 0, s, e.vid.get(), n, uint32_t(m), e.d_colbase.get(),
            cid2vid.get());
  timing_mark("vid", s);
  e.count.alloc_auto(D, s);
  e.count.zero();
  {
    std::vector<uint32_t> soff(m, kLargeCol);
    uint32_t nbins = 0;
    for (uint32_t c = 0; c < m; ++c)
      if (e.card[c] == n) soff[c] = kUniqueCol;
      else if (nbins + e.card[c] <= kSmemBins) {
        soff[c] = nbins;
        nbins += uint32_t(e.card[c]);
      }
    auto d_soff = to_device(soff, s);
    PO_LAUNCH(k_count, grid_for(((n + 31) / 32) * 32, 512, 2), 512, nbins * sizeof(uint32_t), s, e.vid.get(), n,
              uint32_t(m), d_soff.get(), nbins, e.d_colbase.get(), e.count.get());
  }
  timing_mark("count", s);
  DevBuf<unsigned long long> tot(m, s);
  tot.zero();
  PO_LAUNCH(k_total_len, grid_for((D + kTotRun - 1) / kTotRun, 256, 2), 256, m <= 4096 ? m * 8 : 0, s, e.count.get(),
            e.vlen.get(), col_by_pos.get(), D, uint32_t(m), tot.get());
  std::vector<unsigned long long> htot(m);
  d2h_sync(htot.data(), tot.get(), (m) * sizeof(*tot.get()), s);
  for (uint32_t c = 0; c < m; ++c) e.total_len[c] = htot[c];
  timing_mark("encode_tail", s);
}

}  // namespace po
