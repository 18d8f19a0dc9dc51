// K1 cell_scan + K2 dict_encode + K3 rank_sort: exact per-column dictionary
// encoding of the table on the GPU.
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
// One pass over the arena: each thread hashes its cell, probes its column's
// open-addressing table keyed by the 64-bit hash and, when the slot is owned
// by another cell, verifies equality on the bytes (the representative stays
// L2-resident for popular values). Different strings with equal hashes keep
// probing, so the dictionary is exact regardless of hash collisions.

#include <cub/cub.cuh>

#include <algorithm>

#include "internal.cuh"

namespace po {

namespace {

constexpr uint32_t kEmptyRep = 0xFFFFFFFFu;

constexpr uint64_t kShortCell = 32;  // longer cells are hashed/compared by the whole warp

// K1+K2 fused. A warp takes 32 consecutive cells (contiguous in the row-major
// arena). Short cells are hashed by their own lane; long cells one at a time
// by the whole warp with coalesced 8-byte word loads. Each lane then probes
// its column's table; a slot owned by another cell with the same hash is
// verified on the bytes (cooperatively for long cells) and probing continues
// on a mismatch, so value identity is exact.
__global__ void __launch_bounds__(256) k_dict_insert(
    const uint8_t* __restrict__ arena, const uint8_t* arena_end,
    const uint64_t* __restrict__ offsets, uint64_t n, uint32_t m, uint64_t cap,
    unsigned long long* keys, uint32_t* reps, uint32_t* slot_of_cell, uint64_t hash_mask) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t total = n * m;
  const uint64_t warp0 = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t base = warp0 * 32; base < total; base += nwarps * 32) {
    const uint64_t i = base + lane;
    const bool valid = i < total;
    uint64_t o0 = 0, len = 0, r = 0;
    uint32_t c = 0;
    if (valid) {
      o0 = offsets[i];
      len = offsets[i + 1] - o0;
      r = i / m;
      c = uint32_t(i - r * m);
    }
    const bool is_long = valid && len > kShortCell;
    uint64_t h = 0;
    if (valid && !is_long) h = hash_bytes(arena + o0, len, arena_end);
    for (unsigned lm = __ballot_sync(0xffffffffu, is_long); lm; lm &= lm - 1) {
      const int src = __ffs(lm) - 1;
      const uint64_t so = __shfl_sync(0xffffffffu, o0, src);
      const uint64_t sl = __shfl_sync(0xffffffffu, len, src);
      const uint64_t hh = warp_hash_bytes(arena + so, sl, arena_end, lane);
      if (int(lane) == src) h = hh;
    }
    h &= hash_mask;
    if (h == 0) h = 1;
    unsigned long long* K = keys + uint64_t(c) * cap;
    uint32_t* R = reps + uint64_t(c) * cap;
    uint64_t slot = h & (cap - 1);
    bool done = !valid;
    for (;;) {
      // per-lane probing until inserted, matched (short) or a long match awaits verification
      bool verify = false;
      uint64_t rep_off = 0;
      while (!done && !verify) {
        unsigned long long k = K[slot];
        if (k == 0) {
          const unsigned long long prev = atomicCAS(&K[slot], 0ull, (unsigned long long)h);
          if (prev == 0) {
            atomicExch(&R[slot], uint32_t(r));
            done = true;
            break;
          }
          k = prev;
        }
        if (k == h) {
          uint32_t rep;
          while ((rep = ld_relaxed_u32(&R[slot])) == kEmptyRep) {
          }
          const uint64_t j = uint64_t(rep) * m + c;
          const uint64_t q0 = offsets[j];
          if (offsets[j + 1] - q0 == len) {
            if (!is_long) {
              if (bytes_equal(arena + o0, arena + q0, len, arena_end)) {
                done = true;
                break;
              }
            } else {
              verify = true;
              rep_off = q0;
              break;
            }
          }
        }
        slot = (slot + 1) & (cap - 1);
      }
      // cooperative verification of long matches
      for (unsigned vm = __ballot_sync(0xffffffffu, verify); vm; vm &= vm - 1) {
        const int src = __ffs(vm) - 1;
        const uint64_t a = __shfl_sync(0xffffffffu, o0, src);
        const uint64_t b = __shfl_sync(0xffffffffu, rep_off, src);
        const uint64_t sl = __shfl_sync(0xffffffffu, len, src);
        const bool eq = warp_bytes_equal(arena + a, arena + b, sl, arena_end, lane);
        if (int(lane) == src) {
          if (eq) done = true;
          else slot = (slot + 1) & (cap - 1);  // same hash, different bytes: keep probing
        }
      }
      if (__all_sync(0xffffffffu, done)) break;
    }
    if (valid) slot_of_cell[i] = uint32_t(slot);
  }
}

__global__ void k_occupied(const unsigned long long* keys, uint64_t cap, uint8_t* flags) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < cap;
       i += uint64_t(gridDim.x) * blockDim.x)
    flags[i] = keys[i] != 0;
}

__global__ void k_distinct_info(const uint32_t* sel_slot, uint64_t cnt, uint64_t base, uint32_t c,
                                uint64_t cap, const uint32_t* reps, uint32_t* d_col,
                                uint32_t* d_row) {
  for (uint64_t d = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; d < cnt;
       d += uint64_t(gridDim.x) * blockDim.x) {
    d_col[base + d] = c;
    d_row[base + d] = reps[uint64_t(c) * cap + sel_slot[base + d]];
  }
}

__global__ void k_grp_from_col(const uint32_t* col, const uint64_t* colbase, uint64_t D,
                               uint32_t* grp) {
  for (uint64_t d = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; d < D;
       d += uint64_t(gridDim.x) * blockDim.x)
    grp[d] = uint32_t(colbase[col[d]]);
}

// raw_pos[d] -> vid; scatter representative row / column into position order.
__global__ void k_scatter_raw(const uint32_t* raw_pos, const uint32_t* d_col, const uint32_t* d_row,
                              const uint32_t* sel_slot, const uint64_t* colbase, uint64_t D,
                              uint64_t cap, uint32_t* slot2vid, uint32_t* row_by_pos,
                              uint32_t* col_by_pos) {
  for (uint64_t d = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; d < D;
       d += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t p = raw_pos[d];
    uint32_t c = d_col[d];
    slot2vid[uint64_t(c) * cap + sel_slot[d]] = uint32_t(p - colbase[c]);
    row_by_pos[p] = d_row[d];
    col_by_pos[p] = c;
  }
}

__global__ void k_esc_rank(const uint32_t* esc_pos, const uint32_t* col_by_pos,
                           const uint64_t* colbase, uint64_t D, uint32_t* esc_rank) {
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < D;
       p += uint64_t(gridDim.x) * blockDim.x)
    esc_rank[p] = uint32_t(esc_pos[p] - colbase[col_by_pos[p]]);
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
__global__ void k_vlen(const uint8_t* arena, const uint64_t* offsets, const uint64_t* cell_lens,
                       const uint32_t* row_by_pos, const uint32_t* col_by_pos, uint64_t D,
                       uint32_t m, int tok, int scoring, const uint64_t* name_char_len,
                       const uint64_t* name_word_len, uint64_t* vlen) {
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < D;
       p += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t c = col_by_pos[p];
    uint64_t i = uint64_t(row_by_pos[p]) * m + c;
    if (tok == PO_TOK_CUSTOM) {
      vlen[p] = cell_lens[i];
      continue;
    }
    uint64_t o0 = offsets[i], len = offsets[i + 1] - o0;
    if (tok == PO_TOK_CHAR && scoring == PO_SCORE_VALUE) {
      vlen[p] = len;  // CharTokenizer::count == byte length (tokenizer.hpp:44)
      continue;
    }
    TextLen t = text_len(arena + o0, len);
    uint64_t L;
    if (scoring == PO_SCORE_VALUE)
      L = tok == PO_TOK_CHAR ? t.bytes : t.word_runs;
    else
      L = tok == PO_TOK_CHAR ? name_char_len[c] + t.esc_bytes + 8 : name_word_len[c] + frag_words(t);
    vlen[p] = L;
  }
}

__global__ void k_vid(const uint32_t* slot_of_cell, const uint32_t* slot2vid, uint64_t n, uint32_t m,
                      uint64_t cap, uint32_t* vid) {
  const uint64_t total = n * m;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t c = uint32_t(i % m);
    vid[i] = slot2vid[uint64_t(c) * cap + slot_of_cell[i]];
  }
}

// Occurrence count per (column, vid): shared-memory privatised histogram for
// low-cardinality columns, spread global atomics otherwise.
constexpr uint32_t kSmemBins = 12288;

__global__ void k_count(const uint32_t* vid, uint64_t n, uint32_t m, uint32_t c, uint64_t card,
                        uint64_t base, uint32_t* count) {
  extern __shared__ uint32_t h[];
  const bool priv = card <= kSmemBins;
  if (priv)
    for (uint32_t b = threadIdx.x; b < card; b += blockDim.x) h[b] = 0;
  __syncthreads();
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t v = vid[r * m + c];
    if (priv) atomicAdd(&h[v], 1u);
    else atomicAdd(&count[base + v], 1u);
  }
  if (priv) {
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < card; b += blockDim.x)
      if (h[b]) atomicAdd(&count[base + b], h[b]);
  }
}

// Per-column sum of count*vlen (stats.hpp:38), privatised per block in
// shared memory (m accumulators) so the global atomics are m per block.
__global__ void k_total_len(const uint32_t* count, const uint64_t* vlen, const uint32_t* col_by_pos,
                            uint64_t D, uint32_t m, unsigned long long* total) {
  extern __shared__ unsigned long long acc[];
  const bool priv = m <= 4096;
  if (priv)
    for (uint32_t c = threadIdx.x; c < m; c += blockDim.x) acc[c] = 0;
  __syncthreads();
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < D;
       p += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned long long v = uint64_t(count[p]) * vlen[p];
    if (priv) atomicAdd(&acc[col_by_pos[p]], v);
    else atomicAdd(&total[col_by_pos[p]], v);
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

void make_device_table(const po_table* t, int tok, cudaStream_t s, DeviceTable& out) {
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
  if (!t->arena || !t->offsets) fail(PO_ERR_INVALID_ARG, "null arena/offsets");
  if (tok == PO_TOK_CUSTOM && !t->cell_lens)
    fail(PO_ERR_INVALID_ARG, "custom tokenizer requires cell_lens");
  if (t->location == PO_LOC_HOST) {
    out.arena_bytes = t->offsets[cells];
    out.own_offsets.alloc(cells + 1, s);
    out.own_offsets.upload(t->offsets, cells + 1);
    out.own_arena.alloc(out.arena_bytes, s);
    out.own_arena.upload(t->arena, out.arena_bytes);
    out.arena = out.own_arena.get();
    out.offsets = out.own_offsets.get();
    if (tok == PO_TOK_CUSTOM) {
      out.own_lens.alloc(cells, s);
      out.own_lens.upload(t->cell_lens, cells);
      out.cell_lens = out.own_lens.get();
    }
  } else {
    PO_CUDA(cudaMemcpyAsync(&out.arena_bytes, t->offsets + cells, sizeof(uint64_t),
                            cudaMemcpyDeviceToHost, s));
    sync(s);
    out.arena = t->arena;
    out.offsets = t->offsets;
    out.cell_lens = tok == PO_TOK_CUSTOM ? t->cell_lens : nullptr;
  }
}

void encode(const DeviceTable& t, int tok, int scoring, cudaStream_t s, Encoded& e,
            uint32_t hash_bits_debug) {
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
  uint64_t cap = 64;
  while (cap < 2 * n) cap <<= 1;
  const uint8_t* arena_end = t.arena + t.arena_bytes;

  DevBuf<unsigned long long> keys(m * cap, s);
  keys.zero();
  DevBuf<uint32_t> reps(m * cap, s);
  reps.fill_bytes(0xFF);
  DevBuf<uint32_t> slot_of_cell(cells, s);
  uint64_t hmask = hash_bits_debug >= 64 ? ~uint64_t(0) : ((uint64_t(1) << hash_bits_debug) - 1);
  PO_LAUNCH(k_dict_insert, grid_for(cells, 256), 256, 0, s, t.arena, arena_end, t.offsets, n,
            uint32_t(m), cap, keys.get(), reps.get(), slot_of_cell.get(), hmask);

  // Distinct values per column (occupied slots), in column order.
  DevBuf<uint8_t> flags(cap, s);
  DevBuf<uint32_t> sel(cells, s);  // per distinct: slot within its column
  DevBuf<int> nsel(1, s);
  size_t tmp_bytes = 0;
  cub::CountingInputIterator<uint32_t> it(0);
  PO_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, it, flags.get(), sel.get(), nsel.get(),
                                     int(cap), s));
  DevBuf<uint8_t> tmp(tmp_bytes, s);
  for (uint32_t c = 0; c < m; ++c) {
    PO_LAUNCH(k_occupied, grid_for(cap, 256), 256, 0, s, keys.get() + uint64_t(c) * cap, cap,
              flags.get());
    PO_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tmp_bytes, it, flags.get(),
                                       sel.get() + e.colbase[c], nsel.get(), int(cap), s));
    int k = 0;
    PO_CUDA(cudaMemcpyAsync(&k, nsel.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    sync(s);
    e.card[c] = uint64_t(k);
    e.colbase[c + 1] = e.colbase[c] + uint64_t(k);
  }
  e.D = e.colbase[m];
  const uint64_t D = e.D;
  e.d_colbase = to_device(e.colbase, s);

  DevBuf<uint32_t> d_col(D, s), d_row(D, s);
  for (uint32_t c = 0; c < m; ++c)
    PO_LAUNCH(k_distinct_info, grid_for(e.card[c], 256), 256, 0, s, sel.get(), e.card[c],
              e.colbase[c], c, cap, reps.get(), d_col.get(), d_row.get());

  // Raw-byte order of the distinct values of each column -> vid.
  DevBuf<uint32_t> grp(D, s), raw_pos(D, s);
  PO_LAUNCH(k_grp_from_col, grid_for(D, 256), 256, 0, s, d_col.get(), e.d_colbase.get(), D,
            grp.get());
  RefineKey rk;
  rk.kind = 0;
  rk.arena = t.arena;
  rk.arena_bytes = t.arena_bytes;
  rk.offsets = t.offsets;
  rk.item_cell_row = d_row.get();
  rk.item_col = d_col.get();
  rk.m = uint32_t(m);
  refine_sort(uint32_t(D), grp.get(), uint32_t(D), rk, raw_pos.get(), s);

  DevBuf<uint32_t> slot2vid(m * cap, s), col_by_pos(D, s);
  e.rep_row.alloc(D, s);
  PO_LAUNCH(k_scatter_raw, grid_for(D, 256), 256, 0, s, raw_pos.get(), d_col.get(), d_row.get(),
            sel.get(), e.d_colbase.get(), D, cap, slot2vid.get(), e.rep_row.get(),
            col_by_pos.get());
  keys.release();
  flags.release();

  // Escaped fragment-key order (json_escape(v) + '"') -> esc_rank.
  PO_LAUNCH(k_grp_from_col, grid_for(D, 256), 256, 0, s, col_by_pos.get(), e.d_colbase.get(), D,
            grp.get());
  RefineKey ek = rk;
  ek.kind = 1;
  ek.item_cell_row = e.rep_row.get();
  ek.item_col = col_by_pos.get();
  DevBuf<uint32_t> esc_pos(D, s);
  refine_sort(uint32_t(D), grp.get(), uint32_t(D), ek, esc_pos.get(), s);
  e.esc_rank.alloc(D, s);
  PO_LAUNCH(k_esc_rank, grid_for(D, 256), 256, 0, s, esc_pos.get(), col_by_pos.get(),
            e.d_colbase.get(), D, e.esc_rank.get());

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
  e.vlen.alloc(D, s);
  PO_LAUNCH(k_vlen, grid_for(D, 256), 256, 0, s, t.arena, t.offsets, t.cell_lens,
            e.rep_row.get(), col_by_pos.get(), D, uint32_t(m), tok, scoring, d_nchar.get(),
            d_nword.get(), e.vlen.get());

  // vid matrix (row-major) and occurrence counts.
  e.vid.alloc(cells, s);
  PO_LAUNCH(k_vid, grid_for(cells, 256), 256, 0, s, slot_of_cell.get(), slot2vid.get(), n,
            uint32_t(m), cap, e.vid.get());
  slot_of_cell.release();
  slot2vid.release();
  e.count.alloc(D, s);
  e.count.zero();
  for (uint32_t c = 0; c < m; ++c) {
    size_t smem = e.card[c] <= kSmemBins ? e.card[c] * sizeof(uint32_t) : 0;
    PO_LAUNCH(k_count, grid_for(n, 512, 4), 512, smem, s, e.vid.get(), n, uint32_t(m), c,
              e.card[c], e.colbase[c], e.count.get());
  }
  DevBuf<unsigned long long> tot(m, s);
  tot.zero();
  PO_LAUNCH(k_total_len, grid_for(D, 256, 2), 256, m <= 4096 ? m * 8 : 0, s, e.count.get(),
            e.vlen.get(), col_by_pos.get(), D, uint32_t(m), tot.get());
  std::vector<unsigned long long> htot(m);
  tot.download(htot.data(), m);
  sync(s);
  for (uint32_t c = 0; c < m; ++c) e.total_len[c] = htot[c];
}

}  // namespace po
