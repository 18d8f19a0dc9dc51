// Segmented refinement sort: the engine behind K3 rank_sort (distinct values
// in raw-byte and escaped-fragment order) and K8 multikey_sort (leaf row
// sorts of the statistics fallback, objective.hpp:154-171 / ggr.hpp:340-350,
// and the raw single-column base case, ggr.hpp:221-231).
//
// MSD by key chunks: each round stable-radix-sorts the still-unresolved items
// on one 64-bit word (group << shift | chunk) and splits groups where the
// chunk changes. Round 0 names groups by a small index (column, leaf) whose
// start positions come from a table, so its chunk is as wide as possible;
// later rounds name groups by their final start position. Most items resolve
// in round 0, later rounds touch only the long shared prefixes.

#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>
#include <memory>
#include <mutex>

#include "internal.cuh"
#include "msort.cuh"

namespace po {

namespace {

__constant__ uint16_t c_esc_code[257];  // byte -> code in escaped order; [256] = end

constexpr uint16_t kRawEnd = 1;  // raw codes: end = 1, byte b = b + 2

__device__ __forceinline__ uint32_t end_code(const RefineKey& K) {
  return K.kind == 1 ? c_esc_code[256] : kRawEnd;  // raw bytes / symbol streams: 1
}

// Symbols [base, base + nsym) of a string as 9-bit codes (the end marker at
// position len, zero padding after). Raw order: end < every byte (a prefix
// sorts first). Escaped order: the code of each byte is the rank of its
// json_escape expansion and the end marker is the closing '"' (0x22) of the
// fragment, so comparing code strings == comparing escaped fragment keys (the
// expansions are prefix-free).
// Location of item i's string: offset and length in symbols.
__device__ __forceinline__ void str_at(const RefineKey& K, uint32_t item, uint64_t& o0,
                                       uint64_t& len) {
  const uint32_t r = K.item_ref ? K.item_ref[item] : item;
  o0 = K.str_off[r];
  len = K.str_len ? uint64_t(K.str_len[r]) : K.str_off[r + 1] - o0;
}

__device__ __forceinline__ uint64_t string_chunk(const RefineKey& K, uint32_t item, uint64_t base,
                                                 uint32_t nsym) {
  uint64_t o0, len;
  str_at(K, item, o0, len);
  const uint8_t* p = K.arena + o0;
  const uint16_t* p16 = reinterpret_cast<const uint16_t*>(K.arena) + o0;
  uint64_t chunk = 0;
  for (uint32_t j = 0; j < nsym; ++j) {
    const uint64_t pos = base + j + K.skip;
    uint32_t code;
    if (pos < len) {
      if (K.kind == 3) {
        code = p16[pos];  // symbol streams hold their codes (>= 2)
      } else {
        const uint8_t b = p[pos];
        code = K.kind == 0 ? uint32_t(b) + 2 : c_esc_code[b];
      }
    } else {
      code = pos == len ? end_code(K) : 0;
    }
    chunk = (chunk << 9) | code;
  }
  return chunk;
}

__device__ __forceinline__ bool string_terminal(const RefineKey& K, uint64_t chunk, uint32_t nsym) {
  const uint32_t e = end_code(K);
  for (uint32_t j = 0; j < nsym; ++j)
    if (((chunk >> (9 * j)) & 511u) == e) return true;
  return false;
}

// Chunk k of a row: the packed ranks of its leaf's k-th key group.
__device__ __forceinline__ uint64_t row_chunk(const RefineKey& K, uint32_t row, uint32_t k) {
  const uint32_t leaf = K.row_leaf[row];
  if (k >= K.leaf_nchunks[leaf]) return 0;
  const uint32_t ch = K.leaf_chunk_off[leaf] + k;
  const uint32_t k0 = K.chunk_key_off[ch], nk = K.chunk_nkeys[ch];
  uint64_t chunk = 0;
  for (uint32_t j = 0; j < nk; ++j) {
    const int32_t f = K.key_field[k0 + j];
    // vids are ranks in the escaped fragment-key order (the fallback order)
    chunk = (chunk << K.key_bits[k0 + j]) | K.vid[uint64_t(row) * K.m + f];
  }
  return chunk;
}

__device__ __forceinline__ bool row_terminal(const RefineKey& K, uint32_t row, uint32_t k) {
  return k + 1 >= K.leaf_nchunks[K.row_leaf[row]];
}

// Per-round layout of a string key: two 64-bit words per round. Round 0:
// word A = nsym0 symbols next to the group id, word B = the next nsym (7);
// later rounds: A and B each nsym symbols (segments carry the group).
struct StrRound {
  uint64_t base;
  uint32_t nsym;
};
__device__ __forceinline__ StrRound str_round(const RefineKey& K, uint32_t k) {
  if (k == 0) return {0, K.nsym0};
  return {uint64_t(K.nsym0) + uint64_t(K.nsym) + uint64_t(k - 1) * 2 * K.nsym, K.nsym};
}
__device__ __forceinline__ StrRound str_round_b(const RefineKey& K, uint32_t k) {
  const StrRound a = str_round(K, k);
  return {a.base + a.nsym, K.nsym};
}

__global__ void k_build_keys(const uint32_t* items, const uint32_t* grp, uint32_t A, uint32_t k,
                             uint32_t shift, uint32_t nsym_a, RefineKey K, uint64_t* keys,
                             uint64_t* keys_b) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x) {
    uint64_t chunk;
    if (K.kind == 2) {
      chunk = row_chunk(K, items[i], k);
    } else {
      // per-item offset: rounds consume 2 words, segments skip shared prefixes
      const uint32_t na = nsym_a;
      const uint64_t base = K.item_off[items[i]];
      chunk = string_chunk(K, items[i], base, na);
      if (keys_b) keys_b[i] = string_chunk(K, items[i], base + na, K.nsym);
    }
    keys[i] = shift < 64 ? ((uint64_t(grp[i]) << shift) | chunk) : chunk;
  }
}

// String rounds: symbols consumed by the round for every item still active.
__global__ void k_advance(const uint32_t* items, const int* count, uint32_t consumed,
                          uint32_t* item_off) {
  const uint32_t A = uint32_t(*count);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x)
    item_off[items[i]] += consumed;
}

// Shared-prefix skip of the next round's segments: the symbols every member
// shares with its segment's head (members share their offset), minimum per
// segment. Long common prefixes then cost one round instead of one round per
// 14 symbols.
__device__ __forceinline__ uint64_t sym_lcp(const RefineKey& K, uint32_t a, uint32_t b,
                                            uint64_t off) {
  uint64_t oa, la, ob, lb;
  str_at(K, a, oa, la);
  str_at(K, b, ob, lb);
  const uint64_t st = off + K.skip;
  if (st >= la || st >= lb) return 0;
  const uint64_t n = (la < lb ? la : lb) - st;  // symbols to compare
  const uint32_t us = K.kind == 3 ? 2u : 1u;    // bytes per symbol
  const uint8_t* pa = K.arena + (oa + st) * us;
  const uint8_t* pb = K.arena + (ob + st) * us;
  const uint8_t* lim = K.arena + K.arena_bytes;
  return first_diff(pa, pb, n * us, lim) / us;
}

__global__ void k_skip_init(const uint8_t* flags, const int* count, uint32_t* seg_skip) {
  const uint32_t A = uint32_t(*count);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x)
    if (flags[i]) seg_skip[i] = 0xFFFFFFFFu;
}

__global__ void k_skip_lcp(const uint32_t* items, const uint32_t* head, const int* count,
                           RefineKey K, uint32_t* seg_skip) {
  // items of a segment are contiguous: the lanes of a warp that share a head
  // take their minimum first (one atomic per segment per warp; a segment
  // holding most items would otherwise serialise on one address)
  const uint32_t A = uint32_t(*count);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < A; base += stride) {
    const uint32_t i = base + lane;
    uint32_t h = 0xFFFFFFFFu, v = 0xFFFFFFFFu;
    if (i < A) {
      h = head[i];
      if (h == i) h = 0xFFFFFFFFu;
      else {
        const uint64_t l = sym_lcp(K, items[i], items[h], K.item_off[items[i]]);
        v = uint32_t(l < 0xFFFFFFFEull ? l : 0xFFFFFFFEull);
      }
    }
    const unsigned peers = __match_any_sync(0xffffffffu, h);
    v = __reduce_min_sync(peers, v);
    if (h != 0xFFFFFFFFu && int(lane) == __ffs(peers) - 1) atomicMin(&seg_skip[h], v);
  }
}

__global__ void k_skip_apply(const uint32_t* items, const uint32_t* head, const int* count,
                             const uint32_t* seg_skip, uint32_t* item_off) {
  const uint32_t A = uint32_t(*count);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x) {
    const uint32_t sk = seg_skip[head[i]];
    if (sk != 0xFFFFFFFFu) item_off[items[i]] += sk;
  }
}

bool two_words_round0() {  // experiment knob: two key words in round 0 too
  static const bool on = [] {
    const char* v = std::getenv("PO_TWO_WORDS_ROUND0");
    return !(v && *v == '0');
  }();
  return on;
}

// Round-0 string keys of at most this many items are sorted by one merge
// sort on the 128-bit (word A, word B) key instead of two 64-bit radix sorts
// (16 onesweep passes, latency-bound at these sizes). PO_MERGE_ROUND0_MAX.
uint32_t merge_round0_max() {
  static const uint32_t v = [] {
    const char* e = std::getenv("PO_MERGE_ROUND0_MAX");
    return e && *e ? uint32_t(std::strtoul(e, nullptr, 10)) : (1u << 19);
  }();
  return v;
}

// round-0 record of the two-word merge path: (word A, word B) key + item
struct Rec128 {
  uint64_t a, b;
  uint32_t v, pad;
};
struct Less128 {
  __device__ __forceinline__ bool operator()(const Rec128& x, const Rec128& y) const {
    return x.a < y.a || (x.a == y.a && x.b < y.b);
  }
};

__global__ void k_pack128(const uint64_t* a, const uint64_t* b, const uint32_t* items, uint32_t n,
                          Rec128* r) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    r[i] = Rec128{a[i], b[i], items[i], 0u};
}

__global__ void k_unpack128(const Rec128* r, uint32_t n, uint64_t* a, uint64_t* b, uint32_t* v) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    a[i] = r[i].a;
    b[i] = r[i].b;
    v[i] = r[i].v;
  }
}

// PO_MSORT=cub: the library merge sort on the small-job paths (comparison runs)
bool msort_cub() {
  static const bool v = [] {
    const char* e = std::getenv("PO_MSORT");
    return e && std::string(e) == "cub";
  }();
  return v;
}

bool seg_radix_rows() {  // experiment knob: row-key rounds by radix with segment prefix
  static const bool on = [] {
    const char* v = std::getenv("PO_SEGRADIX_ROWS");
    return v && *v == '1';
  }();
  return on;
}

struct FlagU32 {
  const uint8_t* flags;
  __device__ __forceinline__ uint32_t operator()(uint32_t i) const { return flags[i]; }
};
__global__ void k_minus_one(uint32_t* a, uint32_t A) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x) a[i] -= 1;
}

struct HeadOf {  // segment head position of active index i (max-scan input)
  const uint8_t* flags;
  __device__ __forceinline__ uint32_t operator()(uint32_t i) const { return flags[i] ? i : 0u; }
};
struct MaxU32 {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

__global__ void k_gather_kv(const uint32_t* perm, uint32_t A, const uint64_t* k_in,
                            const uint32_t* v_in, uint64_t* k_out, uint32_t* v_out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x) {
    const uint32_t p = perm[i];
    k_out[i] = k_in[p];
    v_out[i] = v_in[p];
  }
}

__global__ void k_seg_end(uint32_t* seg_begin, const int* nseg, const int* count) {
  seg_begin[*nseg] = uint32_t(*count);
}

// Boundary markers for one pair max-scan: (start index of each item's
// group, start index of its (group, chunk) run). Computed on the fly by the
// scan's input iterator; rounds >= 1 take group boundaries from the segment
// flags, round 0 from the group bits of the key.
struct Marks {
  const uint64_t* keys;
  const uint8_t* flags;  // null: round 0
  uint32_t shift;
  const uint64_t* keys_b;  // string rounds: the second key word (null: row keys)
  __device__ __forceinline__ uint2 operator()(uint32_t i) const {
    if (i == 0) return make_uint2(0, 0);
    const uint64_t a = keys[i], b = keys[i - 1];
    const bool gb = flags ? flags[i] != 0 : (shift < 64 && (a >> shift) != (b >> shift));
    const bool rb = gb || a != b || (keys_b && keys_b[i] != keys_b[i - 1]);
    return make_uint2(gb ? i : 0, rb ? i : 0);
  }
};

struct Max2 {
  __device__ __forceinline__ uint2 operator()(const uint2& a, const uint2& b) const {
    return make_uint2(a.x > b.x ? a.x : b.x, a.y > b.y ? a.y : b.y);
  }
};

// Resolved items get their final position; the others keep (new group start,
// item) packed in one word for a single compaction. `start` maps round-0
// group indices to start positions (null: the group id is the start).
__global__ void k_resolve(const uint64_t* keys, const uint64_t* keys_b, const uint32_t* items,
                          const uint2* starts,
                          uint32_t A, uint32_t k, uint32_t shift, uint32_t nsym_a,
                          const uint32_t* start, const uint32_t* seg_grp, RefineKey K,
                          uint32_t* out_pos, uint8_t* keep, uint64_t* packed) {
  const uint64_t cmask = shift >= 64 ? ~0ull : ((1ull << shift) - 1);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x) {
    const uint32_t item = items[i];
    uint32_t g;
    if (seg_grp) {
      g = seg_grp[i];  // segmented rounds: group start aligned with the active array
    } else {
      const uint32_t gid = shift < 64 ? uint32_t(keys[i] >> shift) : 0u;
      g = start ? start[gid] : gid;
    }
    const uint2 st = starts[i];
    const uint32_t pos = g + (i - st.x);
    const bool run_head = st.y == i;
    const bool next_head = i + 1 >= A || starts[i + 1].y == i + 1;
    bool term;
    if (K.kind == 2) term = row_terminal(K, item, k);
    else
      term = string_terminal(K, keys[i] & cmask, nsym_a) ||
             (keys_b && string_terminal(K, keys_b[i], K.nsym));
    if ((run_head && next_head) || term) {
      out_pos[item] = pos;
      keep[i] = 0;
    } else {
      keep[i] = 1;
    }
    packed[i] = (uint64_t(g + (st.y - st.x)) << 32) | item;
  }
}

// Unpack the compacted (group start, item) words and flag the segment starts
// of the next round (runs of equal group start). Flags are written over the
// previous round's item count: positions at or past the new count are
// cleared so the selection over the old range only yields real starts.
__global__ void k_unpack(const uint64_t* packed, const int* count, uint32_t old_count,
                         uint32_t* items, uint32_t* grp, uint8_t* flags) {
  const uint32_t A = uint32_t(*count);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < old_count;
       i += gridDim.x * blockDim.x) {
    uint8_t f = 0;
    if (i < A) {
      const uint64_t v = packed[i];
      items[i] = uint32_t(v);
      grp[i] = uint32_t(v >> 32);
      f = (i == 0 || (v >> 32) != (packed[i - 1] >> 32)) ? 1 : 0;
    }
    flags[i] = f;
  }
}

__global__ void k_iota(uint32_t* a, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[i] = i;
}

bool g_esc_table_ready = false;
std::mutex g_esc_mu;

void ensure_esc_table() {
  std::lock_guard<std::mutex> lk(g_esc_mu);
  if (g_esc_table_ready) return;
  uint16_t code[257];
  esc_code_table(code);
  PO_CUDA(cudaMemcpyToSymbol(c_esc_code, code, sizeof(code)));
  g_esc_table_ready = true;
}

// One sort's device state across rounds.
struct Job {
  RefineJob spec;
  RefineKey key;
  uint32_t A = 0, k = 0;
  uint32_t shift0 = 0, shift = 0;  // chunk bits of round 0 / of later rounds
  int end_bit0 = 0, end_bit = 0;
  size_t tb = 0;
  DevBuf<uint32_t> items, items2, grp;
  DevBuf<uint2> starts;
  DevBuf<uint64_t> keys, keys2, pk, pk2;
  // string kinds: second key word (by position, then sorted), gather scratch
  DevBuf<uint64_t> kb, kb2, k1g;
  DevBuf<uint32_t> perm1, perm2, pos_iota, itg, item_off, head, seg_skip, segidx;
  DevBuf<uint8_t> keep, tmp, segflags;
  DevBuf<uint32_t> seg_begin;
  uint32_t nseg = 0;
  size_t seg_tb = 0;
  DevBuf<uint8_t> seg_tmp;
};

}  // namespace

// Symbol value of each byte in escaped text (scoring.hpp:33-57): plain
// bytes keep their value; escapes start with '\' (0x5C) then the escape
// letter; \u00XX escapes append the byte itself (hex digits sort like the
// byte). The fragment terminator '"' closes every value. code[b] is the rank
// of byte b's expansion, code[256] the rank of the terminator.
void esc_code_table(uint16_t code[257]) {
  std::vector<std::pair<uint32_t, int>> sym;
  for (int b = 0; b < 256; ++b) {
    uint32_t v;
    switch (b) {
      case '"': v = (0x5Cu << 16) | (0x22u << 8); break;
      case '\\': v = (0x5Cu << 16) | (0x5Cu << 8); break;
      case '\b': v = (0x5Cu << 16) | (uint32_t('b') << 8); break;
      case '\f': v = (0x5Cu << 16) | (uint32_t('f') << 8); break;
      case '\n': v = (0x5Cu << 16) | (uint32_t('n') << 8); break;
      case '\r': v = (0x5Cu << 16) | (uint32_t('r') << 8); break;
      case '\t': v = (0x5Cu << 16) | (uint32_t('t') << 8); break;
      default:
        v = b < 0x20 ? ((0x5Cu << 16) | (uint32_t('u') << 8) | uint32_t(b)) : (uint32_t(b) << 16);
    }
    sym.push_back({v, b});
  }
  sym.push_back({0x22u << 16, 256});
  std::sort(sym.begin(), sym.end());
  for (size_t r = 0; r < sym.size(); ++r) code[sym[r].second] = uint16_t(r + 1);
}

uint32_t refine_chunk_bits(uint32_t grp_max) { return 64u - uint32_t(bits_for(grp_max)); }

namespace {

// One-pass exact string sort (kinds 0 and 1, small jobs): a stable merge sort
// of (group, first 14 symbols as two words, item) records whose comparator
// falls back to the remaining symbols when the words tie, so no refinement
// rounds are needed. Equal strings keep their item order (stable), exactly as
// the refinement sort leaves them.
struct StrRec {
  uint32_t g, item;
  uint64_t k0, k1;
};

__device__ __forceinline__ uint32_t sym_code(const RefineKey& K, const uint8_t* p, uint64_t len,
                                             uint64_t pos) {
  if (pos < len) return K.kind == 0 ? uint32_t(p[pos]) + 2 : c_esc_code[p[pos]];
  return pos == len ? end_code(K) : 0u;
}

struct StrLess {
  RefineKey K;
  __device__ __forceinline__ bool operator()(const StrRec& a, const StrRec& b) const {
    if (a.g != b.g) return a.g < b.g;
    if (a.k0 != b.k0) return a.k0 < b.k0;
    if (a.k1 != b.k1) return a.k1 < b.k1;
    // symbols [14, ...) of both strings
    uint64_t oa, la, ob, lb;
    str_at(K, a.item, oa, la);
    str_at(K, b.item, ob, lb);
    const uint8_t* pa = K.arena + oa;
    const uint8_t* pb = K.arena + ob;
    const uint8_t* lim = K.arena + K.arena_bytes;
    // eight bytes at a time while both strings last: symbol codes are a
    // one-to-one function of the byte, so the first differing byte decides
    uint64_t pos = 14 + K.skip;
    while (pos < la && pos < lb) {
      const uint64_t ra = la - pos, rb = lb - pos;
      const uint32_t w = uint32_t(ra < rb ? (ra < 8 ? ra : 8) : (rb < 8 ? rb : 8));
      const uint64_t x = load8_unaligned(pa + pos, lim), y = load8_unaligned(pb + pos, lim);
      const uint64_t d = mask_low_bytes(x ^ y, w);
      if (d) {
        const uint32_t sh = uint32_t(__ffsll(static_cast<long long>(d)) - 1) & ~7u;
        const uint32_t bx = uint32_t(x >> sh) & 0xFF, by = uint32_t(y >> sh) & 0xFF;
        return K.kind == 0 ? bx < by : c_esc_code[bx] < c_esc_code[by];
      }
      pos += w;
    }
    // one string ends here: end code against a byte code (or both ended)
    const uint32_t ca = sym_code(K, pa, la, pos), cb = sym_code(K, pb, lb, pos);
    return ca < cb;
  }
};

__global__ void k_str_recs(RefineKey K, const uint32_t* grp_init, uint32_t n, StrRec* recs) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    recs[i] = StrRec{grp_init[i], i, string_chunk(K, i, 0, 7), string_chunk(K, i, 7, 7)};
}

__global__ void k_str_first(const StrRec* recs, uint32_t n, uint32_t* first) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (i == 0 || recs[i - 1].g != recs[i].g) first[recs[i].g] = i;
}

__global__ void k_str_place(const StrRec* recs, uint32_t n, const uint32_t* first,
                            const uint32_t* grp_start, uint32_t* out_pos) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t g = recs[i].g;
    out_pos[recs[i].item] = (grp_start ? grp_start[g] : g) + (i - first[g]);
  }
}

// PO_MERGE_RANK=0 disables the one-pass path
bool merge_rank_enabled() {
  const char* e = std::getenv("PO_MERGE_RANK");
  return !(e && *e == '0');
}

}  // namespace

// True when the job was sorted here (kinds 0/1 up to merge_round0_max items).
bool merge_rank_job(const RefineJob& sp, cudaStream_t s) {
  if (!merge_rank_enabled() || (sp.key.kind != 0 && sp.key.kind != 1) ||
      sp.n_items > merge_round0_max() || sp.key.item_off)
    return false;
  if (sp.key.kind == 1) ensure_esc_table();
  const uint32_t n = sp.n_items;
  ProfScope ps(msort_cub() ? "cub_merge_sort" : "merge_sort", s);
  DevBuf<StrRec> recs(n, s);
  PO_LAUNCH(k_str_recs, grid_for(n, 256), 256, 0, s, sp.key, sp.d_grp_init, n, recs.get());
  StrLess less{sp.key};
  if (msort_cub()) {
    size_t need = 0;
    PO_CUDA(cub::DeviceMergeSort::StableSortKeys(nullptr, need, recs.get(), int(n), less, s));
    DevBuf<uint8_t> tmp(need, s);
    PO_CUDA(cub::DeviceMergeSort::StableSortKeys(tmp.get(), need, recs.get(), int(n), less, s));
  } else {
    DevBuf<StrRec> tmp(n, s);
    stable_merge_sort(recs.get(), tmp.get(), n, less, s);
  }
  const uint32_t ng = sp.d_grp_start ? sp.n_groups : sp.grp_max + 1;
  DevBuf<uint32_t> first(std::max<uint32_t>(ng, 1), s);
  PO_LAUNCH(k_str_first, grid_for(n, 256), 256, 0, s, recs.get(), n, first.get());
  PO_LAUNCH(k_str_place, grid_for(n, 256), 256, 0, s, recs.get(), n, first.get(), sp.d_grp_start,
            sp.d_out_pos);
  return true;
}

void refine_sort_multi(const std::vector<RefineJob>& specs, cudaStream_t s) {
  std::vector<std::unique_ptr<Job>> jobs;
  for (const RefineJob& sp : specs) {
    if (sp.n_items == 0) continue;
    if (merge_rank_job(sp, s)) continue;
    auto j = std::make_unique<Job>();
    j->spec = sp;
    j->key = sp.key;
    // group ids of round 0: indices < n_groups (with a start table) or start
    // positions; later rounds: start positions <= grp_max
    const uint32_t g0max = sp.d_grp_start ? (sp.n_groups ? sp.n_groups - 1 : 0) : sp.grp_max;
    const uint32_t cb0 = refine_chunk_bits(g0max), cb = refine_chunk_bits(sp.grp_max);
    // rounds >= 1 sort inside segments: the key is the chunk alone (64 bits)
    (void)cb;
    if (j->key.kind != 2) {
      if (cb0 < 9) fail(PO_ERR_SIZE, "too many columns to rank");
      j->key.nsym0 = cb0 / 9;
      j->key.nsym = 7;
      j->shift0 = 9 * j->key.nsym0;
      j->shift = 64;
    } else {
      j->shift0 = std::min(sp.row_chunk_bits0 ? sp.row_chunk_bits0 : cb0, cb0);
      j->shift = 64;
    }
    j->key.chunk_bits = cb;
    j->end_bit0 = int(j->shift0) + bits_for(g0max);
    j->end_bit = 64;
    if (j->key.kind == 1) ensure_esc_table();
    const uint32_t n = sp.n_items;
    j->items.alloc_auto(n, s);
    j->items2.alloc_auto(n, s);
    j->grp.alloc_auto(n, s);
    j->keys.alloc_auto(n, s);
    j->keys2.alloc_auto(n, s);
    j->pk.alloc_auto(n, s);
    j->pk2.alloc_auto(n, s);
    j->starts.alloc_auto(n, s);
    j->keep.alloc_auto(n, s);
    j->segflags.alloc_auto(n, s);
    j->seg_begin.alloc_auto(n + 1, s);
    j->segidx.alloc_auto(n, s);
    PO_LAUNCH(k_iota, grid_for(n, 256), 256, 0, s, j->items.get(), n);
    if (j->key.kind != 2) {
      j->kb.alloc_auto(n, s);
      j->kb2.alloc_auto(n, s);
      j->k1g.alloc_auto(n, s);
      j->perm1.alloc_auto(n, s);
      j->perm2.alloc_auto(n, s);
      j->pos_iota.alloc_auto(n, s);
      j->itg.alloc_auto(n, s);
      j->item_off.alloc_auto(n, s);
      j->item_off.zero();
      j->head.alloc_auto(n, s);
      j->seg_skip.alloc_auto(n, s);
      j->key.item_off = j->item_off.get();
      PO_LAUNCH(k_iota, grid_for(n, 256), 256, 0, s, j->pos_iota.get(), n);
    }
    PO_CUDA(cudaMemcpyAsync(j->grp.get(), sp.d_grp_init, n * sizeof(uint32_t),
                            cudaMemcpyDeviceToDevice, s));
    size_t sort_bytes = 0, scan_bytes = 0, sel_bytes = 0;
    int* nullcount = nullptr;
    PO_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, j->keys.get(), j->keys2.get(),
                                            j->items.get(), j->items2.get(), n, 0, 64, s));
    {
      cub::TransformInputIterator<uint2, Marks, cub::CountingInputIterator<uint32_t>> mk(
          cub::CountingInputIterator<uint32_t>(0), Marks{j->keys2.get(), nullptr, 0, nullptr});
      PO_CUDA(cub::DeviceScan::InclusiveScan(nullptr, scan_bytes, mk, j->starts.get(), Max2(), n, s));
    }
    PO_CUDA(cub::DeviceSelect::Flagged(nullptr, sel_bytes, j->pk2.get(), j->keep.get(),
                                       j->pk.get(), nullcount, n, s));
    j->tb = std::max(sort_bytes, std::max(scan_bytes, sel_bytes));
    j->tmp.alloc(j->tb, s);
    j->A = n;
    jobs.push_back(std::move(j));
  }
  DevBuf<int> nsel(std::max<size_t>(1, 2 * jobs.size()), s);  // per job: active, segments
  std::vector<int> hn(2 * jobs.size());
  for (;;) {
    bool any = false;
    for (size_t q = 0; q < jobs.size(); ++q) {
      Job& j = *jobs[q];
      if (!j.A) continue;
      any = true;
      const uint32_t A = j.A;
      const bool seg = j.k > 0;  // rounds >= 1: sorts inside the unresolved groups
      const uint32_t* start = seg ? nullptr : j.spec.d_grp_start;
      const bool strk = j.key.kind != 2;  // string keys
      // two key words per round (LSD) — in round 0 only when asked: there the
      // extra pass covers every item, later rounds only the unresolved ones
      const bool two = strk && (seg || two_words_round0());
      // Rounds >= 1: one global radix sort with the segment index in the high
      // key bits (segments keep their positions) when the chunk still fits,
      // else CUB's segmented sort.
      uint32_t shift = seg ? 64u : j.shift0;
      uint32_t nsym_a = seg ? j.key.nsym : j.key.nsym0;
      bool segradix = false;
      if (seg) {
        const uint32_t sbits = uint32_t(bits_for(j.nseg ? j.nseg - 1 : 0));
        if (two && (64 - sbits) / 9 >= 1) {
          segradix = true;
          shift = 64 - sbits;
          nsym_a = std::min<uint32_t>(j.key.nsym, shift / 9);
        } else if (!two && seg_radix_rows() &&
                   sbits + (j.spec.row_chunk_bits ? j.spec.row_chunk_bits : 64) <= 64) {
          segradix = true;
          shift = 64 - sbits;
        }
        if (segradix) {  // segment index of every active position
          ProfScope ps("cub_scan", s);
          cub::TransformInputIterator<uint32_t, FlagU32, cub::CountingInputIterator<uint32_t>> fi(
              cub::CountingInputIterator<uint32_t>(0), FlagU32{j.segflags.get()});
          size_t hb = 0;
          PO_CUDA(cub::DeviceScan::InclusiveSum(nullptr, hb, fi, j.segidx.get(), A, s));
          if (hb > j.tb) {
            j.tmp.alloc(hb, s);
            j.tb = hb;
          }
          PO_CUDA(cub::DeviceScan::InclusiveSum(j.tmp.get(), hb, fi, j.segidx.get(), A, s));
          PO_LAUNCH(k_minus_one, grid_for(A, 256), 256, 0, s, j.segidx.get(), A);
        }
      }
      PO_LAUNCH(k_build_keys, grid_for(A, 256), 256, 0, s, j.items.get(),
                segradix ? j.segidx.get() : j.grp.get(), A, j.k, shift, nsym_a, j.key,
                j.keys.get(), two ? j.kb.get() : nullptr);
      size_t b = j.tb;
      // one stable sort pass over the active items: a radix sort in round 0,
      // a segmented sort inside the unresolved groups later
      auto sort_pass = [&](const uint64_t* kin, uint64_t* kout, const uint32_t* vin, uint32_t* vout,
                           int end_bit) {
        if (!seg || segradix) {
          radix_sort_pairs(kin, kout, vin, vout, A, 0, end_bit, s);
          return;
        }
        ProfScope ps("cub_segmented_sort", s);
        size_t need = 0;
        PO_CUDA(cub::DeviceSegmentedSort::StableSortPairs(nullptr, need, kin, kout, vin, vout,
                                                          int(A), int(j.nseg), j.seg_begin.get(),
                                                          j.seg_begin.get() + 1, s));
        if (need > j.seg_tb) {
          j.seg_tmp.alloc(need, s);
          j.seg_tb = need;
        }
        PO_CUDA(cub::DeviceSegmentedSort::StableSortPairs(j.seg_tmp.get(), need, kin, kout, vin,
                                                          vout, int(A), int(j.nseg),
                                                          j.seg_begin.get(), j.seg_begin.get() + 1,
                                                          s));
      };
      if (two && !seg && A <= merge_round0_max()) {
        // one stable merge sort by (word A, word B): the same order as the
        // two LSD passes below
        ProfScope ps(msort_cub() ? "cub_merge_sort" : "merge_sort", s);
        DevBuf<Rec128> r128(A, s), t128(A, s);
        PO_LAUNCH(k_pack128, grid_for(A, 256), 256, 0, s, j.keys.get(), j.kb.get(), j.items.get(),
                  A, r128.get());
        if (msort_cub()) {
          size_t need = 0;
          PO_CUDA(cub::DeviceMergeSort::StableSortKeys(nullptr, need, r128.get(), int(A), Less128(), s));
          if (need > j.tb) {
            j.tmp.alloc(need, s);
            j.tb = need;
          }
          PO_CUDA(cub::DeviceMergeSort::StableSortKeys(j.tmp.get(), need, r128.get(), int(A),
                                                       Less128(), s));
        } else {
          stable_merge_sort(r128.get(), t128.get(), A, Less128(), s);
        }
        PO_LAUNCH(k_unpack128, grid_for(A, 256), 256, 0, s, r128.get(), A, j.keys2.get(), j.kb.get(),
                  j.items2.get());
      } else if (two) {
        // LSD over the two words: by word B, then stably by word A
        sort_pass(j.kb.get(), j.kb2.get(), j.pos_iota.get(), j.perm1.get(), 64);
        PO_LAUNCH(k_gather_kv, grid_for(A, 256), 256, 0, s, j.perm1.get(), A, j.keys.get(),
                  j.items.get(), j.k1g.get(), j.itg.get());
        sort_pass(j.k1g.get(), j.keys2.get(), j.pos_iota.get(), j.perm2.get(),
                  seg ? 64 : j.end_bit0);  // segradix: the segment index is in the top bits
        PO_LAUNCH(k_gather_kv, grid_for(A, 256), 256, 0, s, j.perm2.get(), A, j.kb2.get(),
                  j.itg.get(), j.kb.get(), j.items2.get());
      } else {
        sort_pass(j.keys.get(), j.keys2.get(), j.items.get(), j.items2.get(),
                  seg ? 64 : j.end_bit0);
      }
      {
        ProfScope ps("cub_scan", s);
        b = j.tb;
        cub::TransformInputIterator<uint2, Marks, cub::CountingInputIterator<uint32_t>> mk(
            cub::CountingInputIterator<uint32_t>(0),
            Marks{j.keys2.get(), seg ? j.segflags.get() : nullptr, shift,
                  two ? j.kb.get() : nullptr});
        PO_CUDA(cub::DeviceScan::InclusiveScan(j.tmp.get(), b, mk, j.starts.get(), Max2(), A, s));
      }
      PO_LAUNCH(k_resolve, grid_for(A, 256), 256, 0, s, j.keys2.get(), two ? j.kb.get() : nullptr,
                j.items2.get(),
                j.starts.get(), A, j.k, shift, nsym_a, start, seg ? j.grp.get() : nullptr,
                j.key, j.spec.d_out_pos, j.keep.get(), j.pk2.get());
      {
        ProfScope ps("cub_select", s);
        b = j.tb;
        PO_CUDA(cub::DeviceSelect::Flagged(j.tmp.get(), b, j.pk2.get(), j.keep.get(), j.pk.get(),
                                           nsel.get() + 2 * q, A, s));
      }
      // segments of the next round: runs of equal group start
      PO_LAUNCH(k_unpack, grid_for(A, 256), 256, 0, s, j.pk.get(), nsel.get() + 2 * q, A,
                j.items.get(), j.grp.get(), j.segflags.get());
      {
        ProfScope ps("cub_select", s);
        b = j.tb;
        cub::CountingInputIterator<uint32_t> it(0);
        PO_CUDA(cub::DeviceSelect::Flagged(j.tmp.get(), b, it, j.segflags.get(), j.seg_begin.get(),
                                           nsel.get() + 2 * q + 1, A, s));
      }
      PO_LAUNCH(k_seg_end, 1, 1, 0, s, j.seg_begin.get(), nsel.get() + 2 * q + 1,
                nsel.get() + 2 * q);
      if (strk) {
        // next round: advance past this round's symbols, then skip the
        // prefix every member of a segment shares
        const int* cnt = nsel.get() + 2 * q;
        PO_LAUNCH(k_advance, grid_for(A, 256), 256, 0, s, j.items.get(), cnt,
                  nsym_a + (two ? j.key.nsym : 0), j.item_off.get());
        {
          ProfScope ps("cub_scan", s);
          size_t hb = 0;
          cub::TransformInputIterator<uint32_t, HeadOf, cub::CountingInputIterator<uint32_t>> hi(
              cub::CountingInputIterator<uint32_t>(0), HeadOf{j.segflags.get()});
          PO_CUDA(cub::DeviceScan::InclusiveScan(nullptr, hb, hi, j.head.get(), MaxU32(), A, s));
          if (hb > j.tb) {
            j.tmp.alloc(hb, s);
            j.tb = hb;
          }
          PO_CUDA(cub::DeviceScan::InclusiveScan(j.tmp.get(), hb, hi, j.head.get(), MaxU32(), A, s));
        }
        PO_LAUNCH(k_skip_init, grid_for(A, 256), 256, 0, s, j.segflags.get(), cnt, j.seg_skip.get());
        PO_LAUNCH(k_skip_lcp, grid_for(A, 256), 256, 0, s, j.items.get(), j.head.get(), cnt, j.key,
                  j.seg_skip.get());
        PO_LAUNCH(k_skip_apply, grid_for(A, 256), 256, 0, s, j.items.get(), j.head.get(), cnt,
                  j.seg_skip.get(), j.item_off.get());
      }
      ++j.k;
    }
    if (!any) break;
    PO_CUDA(cudaMemcpyAsync(hn.data(), nsel.get(), 2 * jobs.size() * sizeof(int),
                            cudaMemcpyDeviceToHost, s));
    sync(s);
    if (debug_timing()) {
      fprintf(stderr, "[po refine] round:");
      for (size_t q = 0; q < jobs.size(); ++q)
        fprintf(stderr, " job%zu %u->%d (%d groups)", q, jobs[q]->A, jobs[q]->A ? hn[2 * q] : 0,
                jobs[q]->A ? hn[2 * q + 1] : 0);
      fprintf(stderr, "\n");
    }
    for (size_t q = 0; q < jobs.size(); ++q)
      if (jobs[q]->A) {
        jobs[q]->A = uint32_t(hn[2 * q]);
        jobs[q]->nseg = uint32_t(hn[2 * q + 1]);
      }
  }
}

namespace {

// -1 / 1: a before / after b in escaped fragment order (distinct strings).
// The expansions are prefix-free, so the first differing raw byte (or the
// end of the shorter string, the closing '"') decides.
__device__ __forceinline__ bool esc_less(const uint8_t* a, uint64_t la, const uint8_t* b,
                                         uint64_t lb) {
  const uint64_t mn = la < lb ? la : lb;
  uint64_t i = 0;
  while (i < mn && a[i] == b[i]) ++i;
  const uint32_t ca = i < la ? c_esc_code[a[i]] : c_esc_code[256];
  const uint32_t cb = i < lb ? c_esc_code[b[i]] : c_esc_code[256];
  return ca < cb;
}

// Thread per position of a short run (2..max_len rows of one leaf, distinct
// values of column col_of_leaf[leaf]): its rank among the run's values.
__global__ void k_rank_short_runs(CellStr cs, const uint32_t* perm, const uint32_t* run,
                                  const uint32_t* run_len, const uint32_t* row_leaf,
                                  const int32_t* col_of_leaf, uint64_t n, uint32_t max_len,
                                  uint32_t* pos) {
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < n;
       q += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t st = run[q], L = run_len[st];
    if (L < 2 || L > max_len) continue;
    const uint32_t r = perm[q];
    const uint32_t c = uint32_t(col_of_leaf[row_leaf[r]]);
    const uint8_t* a;
    uint64_t la;
    cs.get(r, c, a, la);
    uint32_t rank = 0;
    for (uint32_t j = st; j < st + L; ++j) {
      if (j == q) continue;
      const uint8_t* b;
      uint64_t lb;
      cs.get(perm[j], c, b, lb);
      rank += esc_less(b, lb, a, la);
    }
    pos[r] = st + rank;
  }
}

// Escaped codes of symbols [7w, 7w + 7) of a string, 9 bits each (end marker
// at len, zero padding after): comparing (word 0, word 1) orders the first 14
// symbols of the fragment keys.
__device__ __forceinline__ uint64_t esc_word(const uint8_t* p, uint64_t len, uint32_t w) {
  uint64_t chunk = 0;
  for (uint32_t j = 0; j < 7; ++j) {
    const uint64_t i = 7ull * w + j;
    const uint32_t code = i < len ? c_esc_code[p[i]] : (i == len ? c_esc_code[256] : 0u);
    chunk = (chunk << 9) | code;
  }
  return chunk;
}

__global__ void k_long_keys(CellStr cs, const uint32_t* perm, const uint32_t* row_leaf,
                            const int32_t* col_of_leaf, const uint32_t* items, uint32_t nt,
                            uint64_t* k0, uint64_t* k1) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nt; k += gridDim.x * blockDim.x) {
    const uint32_t q = items[k], r = perm[q];
    const uint8_t* p;
    uint64_t len;
    cs.get(r, uint32_t(col_of_leaf[row_leaf[r]]), p, len);
    k0[q] = esc_word(p, len, 0);
    k1[q] = esc_word(p, len, 1);
  }
}

// Positions of long runs: part p of the run (kLongPart positions
// from st + y * kLongPart) is counted against the position's 14-symbol keys;
// keys equal on all 14 symbols fall back to a full escaped comparison. Runs
// are split so the longest one does not serialise on a few warps; positions
// of one run are consecutive in items[], so a warp's loads of k0[j] / k1[j]
// coincide.
constexpr uint32_t kLongPart = 512;

__global__ void k_rank_long_runs(CellStr cs, const uint32_t* perm, const uint32_t* run, const uint32_t* run_len,
                                 const uint32_t* row_leaf, const int32_t* col_of_leaf,
                                 const uint32_t* items, uint32_t nt, const uint64_t* __restrict__ k0,
                                 const uint64_t* __restrict__ k1, uint32_t gx, uint32_t* rank_out) {
  const uint32_t part = blockIdx.x / gx;  // blocks [part * gx, (part + 1) * gx): one part
  const uint32_t k = (blockIdx.x - part * gx) * blockDim.x + threadIdx.x;
  if (k >= nt) return;
  const uint32_t q = items[k], st = run[q], L = run_len[st];
  const uint32_t lo = st + part * kLongPart;
  if (lo >= st + L) return;
  const uint32_t hi = min(st + L, lo + kLongPart);
  const uint64_t a0 = k0[q], a1 = k1[q];
  uint32_t rank = 0, eq = 0;
#pragma unroll 8
  for (uint32_t j = lo; j < hi; ++j) {
    const uint64_t b0 = k0[j], b1 = k1[j];
    rank += (b0 < a0) | ((b0 == a0) & (b1 < a1));
    eq += (b0 == a0) & (b1 == a1);
  }
  if (eq > uint32_t(q >= lo && q < hi)) {  // shared 14-symbol prefixes: compare bytes
    const uint32_t r = perm[q];
    const uint32_t c = uint32_t(col_of_leaf[row_leaf[r]]);
    const uint8_t* a;
    uint64_t la;
    cs.get(r, c, a, la);
    for (uint32_t j = lo; j < hi; ++j) {
      if (j == q || k0[j] != a0 || k1[j] != a1) continue;
      const uint8_t* b;
      uint64_t lb;
      cs.get(perm[j], c, b, lb);
      rank += esc_less(b, lb, a, la);
    }
  }
  if (rank) atomicAdd(rank_out + k, rank);
}

__global__ void k_long_place(const uint32_t* items, uint32_t nt, const uint32_t* perm,
                             const uint32_t* run, const uint32_t* rank, uint32_t* pos) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nt; k += gridDim.x * blockDim.x) {
    const uint32_t q = items[k];
    pos[perm[q]] = run[q] + rank[k];
  }
}

}  // namespace

CellStr cell_str(const Encoded& e) {
  return CellStr{e.val_arena, e.val_arena + e.val_bytes, e.val_off.get(), e.val_len.get(),
                 e.vid.get(), e.d_colbase.get(), e.m};
}

void rank_short_runs(const CellStr& cs, const uint32_t* perm, const uint32_t* run,
                     const uint32_t* run_len, const uint32_t* row_leaf, const int32_t* col_of_leaf,
                     uint64_t n, uint32_t max_len, uint32_t* pos, cudaStream_t s) {
  if (n == 0) return;
  ensure_esc_table();
  PO_LAUNCH(k_rank_short_runs, grid_for(n, 256), 256, 0, s, cs, perm, run, run_len, row_leaf,
            col_of_leaf, n, max_len, pos);
}

void rank_long_runs(const CellStr& cs, const uint32_t* perm, const uint32_t* run,
                    const uint32_t* run_len, const uint32_t* row_leaf, const int32_t* col_of_leaf,
                    const uint32_t* items, uint32_t nt, uint64_t n, uint32_t max_len, uint32_t* pos,
                    cudaStream_t s) {
  if (nt == 0) return;
  ensure_esc_table();
  DevBuf<uint64_t> k0(n, s), k1(n, s);
  PO_LAUNCH(k_long_keys, grid_for(nt, 256), 256, 0, s, cs, perm, row_leaf, col_of_leaf, items, nt,
            k0.get(), k1.get());
  DevBuf<uint32_t> rank(nt, s);
  rank.zero();
  const uint32_t gx = (nt + 255) / 256, parts = (max_len + kLongPart - 1) / kLongPart;
  PO_LAUNCH(k_rank_long_runs, gx * parts, 256, 0, s, cs, perm, run, run_len, row_leaf, col_of_leaf,
            items, nt, k0.get(), k1.get(), gx, rank.get());
  PO_LAUNCH(k_long_place, grid_for(nt, 256), 256, 0, s, items, nt, perm, run, rank.get(), pos);
}

void refine_sort(uint32_t n_items, const uint32_t* d_grp_init, uint32_t grp_max,
                 const RefineKey& key, uint32_t* d_out_pos, cudaStream_t s, uint32_t row_chunk_bits) {
  RefineJob j;
  j.n_items = n_items;
  j.d_grp_init = d_grp_init;
  j.grp_max = grp_max;
  j.key = key;
  j.d_out_pos = d_out_pos;
  j.row_chunk_bits = row_chunk_bits;
  refine_sort_multi({j}, s);
}

// po_debug_merge_sort: stable_merge_sort on (a, b, value) records (test hook)
void debug_merge_sort(const uint64_t* a, const uint64_t* b, const uint32_t* v, uint32_t n,
                      uint64_t* oa, uint64_t* ob, uint32_t* ov, cudaStream_t s) {
  DevBuf<uint64_t> da(n, s), db(n, s);
  DevBuf<uint32_t> dv(n, s);
  DevBuf<Rec128> r(n, s), t(n, s);
  if (!n) return;
  PO_CUDA(cudaMemcpyAsync(da.get(), a, n * 8ull, cudaMemcpyHostToDevice, s));
  PO_CUDA(cudaMemcpyAsync(db.get(), b, n * 8ull, cudaMemcpyHostToDevice, s));
  PO_CUDA(cudaMemcpyAsync(dv.get(), v, n * 4ull, cudaMemcpyHostToDevice, s));
  PO_LAUNCH(k_pack128, grid_for(n, 256), 256, 0, s, da.get(), db.get(), dv.get(), n, r.get());
  stable_merge_sort(r.get(), t.get(), n, Less128(), s);
  PO_LAUNCH(k_unpack128, grid_for(n, 256), 256, 0, s, r.get(), n, da.get(), db.get(), dv.get());
  PO_CUDA(cudaMemcpyAsync(oa, da.get(), n * 8ull, cudaMemcpyDeviceToHost, s));
  PO_CUDA(cudaMemcpyAsync(ob, db.get(), n * 8ull, cudaMemcpyDeviceToHost, s));
  PO_CUDA(cudaMemcpyAsync(ov, dv.get(), n * 4ull, cudaMemcpyDeviceToHost, s));
  sync(s);
}

}  // namespace po
