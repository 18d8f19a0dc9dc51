// K1 cell_scan + K2 dict_encode in ONE read of the arena: exact per-column
// dictionaries (a dense value id per cell) sized from the observed
// cardinality, over resident tables or streamed host row chunks.
//
// Reference behaviour replaced: the hashing and string equality inside every
// std::unordered_map/set<string_view> over cells (ggr.hpp:251, 286, 324;
// stats.hpp:33; objective.hpp:86). After this pass every later equality is an
// integer compare.
//
// Kernel k_dict_build (one launch per row chunk). A tile is 32 rows; each
// column c is handled by groups of G_c lanes (G_c from the column's average
// length: 1 lane for short cells up to the whole warp for ~2 KB cells), so a
// warp takes 32/G_c cells of one column at a time. A group
//   1. loads its cell as 16-byte aligned chunks (lane gl: chunks gl, gl+G, ..;
//      coalesced) and keeps up to kRmax chunks per lane in registers,
//   2. computes the 64-bit cell hash (a sum of per-word terms, so lanes add
//      their own words and the group reduces with shuffles),
//   3. the group leader probes the column's open-addressing table: an empty
//      slot is claimed (the cell becomes the representative of a new value:
//      id = the column's next dense id), a slot with the same hash yields the
//      candidate value,
//   4. the group compares its registers with the representative's bytes
//      (L2-resident for popular values); a mismatch (a 64-bit collision)
//      continues probing, so the dictionary is exact.
// Cells longer than the register window are hashed and compared window by
// window (the second read is an L1/L2 hit).
//
// Capacity: tables are sized per column from the distinct count observed on a
// first row chunk (linear extrapolation, at most n). A table whose id space
// or slots run out mid-chunk flags the column; the host grows it (rehash from
// the stored hashes) and reruns the chunk, which is idempotent for values
// already present. Streamed (host) tables copy each new value's bytes into a
// compact value arena after its chunk, so later phases never need the table
// bytes again.

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <future>
#include <thread>
#include <cstdlib>
#include <string>

#include "internal.cuh"

namespace po {

namespace {

constexpr uint32_t kNoCid = 0xFFFFFFFFu;    // slot claimed, id not yet published
constexpr uint32_t kOverCid = 0xFFFFFFFEu;  // slot claimed past the id capacity
constexpr uint64_t kInVals = 1ull << 63;    // voff: representative in the value arena
constexpr uint64_t kUnsetOff = ~0ull;       // voff / vlen of an id not yet written
constexpr uint32_t kUnsetLen = 0xFFFFFFFFu;
constexpr uint32_t kRmax = 4;               // 16-byte chunks per lane held in registers
constexpr uint32_t kTileRows = 32;
constexpr uint32_t kBuildBlock = 256;

struct ColDict {
  unsigned long long* keys;   // [cap] 64-bit hash, 0 = empty
  uint32_t* cids;             // [cap] value id of the slot
  unsigned long long* vhash;  // [cidcap] hash of value id
  unsigned long long* voff;   // [cidcap] representative byte offset (| kInVals)
  uint32_t* vlen;             // [cidcap] byte length
  uint32_t* vrow;             // [cidcap] (global) row of the representative
  uint64_t cap;               // power of two
  uint32_t cidcap;
  uint32_t G;                 // lanes per cell
  uint32_t item0;             // first work item of the column inside a tile
};

struct BuildArgs {
  const uint8_t* chunk;      // byte at absolute offset o: chunk[o - base]
  uint64_t base;
  const uint8_t* chunk_lim;  // loads start before this address
  const uint8_t* vals;       // value arena (representatives flagged kInVals)
  const uint8_t* vals_lim;
  const uint64_t* offs;      // offsets of the chunk's cells: index (r - r0) * m + c
  uint64_t r0, r1;
  uint32_t m;
  uint32_t items;            // work items per tile (sum of G)
  uint64_t hmask;
  const ColDict* cols;
  uint32_t* ncid;            // [m] ids handed out per column
  uint32_t* overflow;        // [m]
  uint32_t* cid_mat;         // [n*m] value id of cell (r, c) at r*m + c
  uint32_t prefetch;         // L2 bulk prefetch of each block's next tile
};

__device__ __forceinline__ uint4 ld16(const uint8_t* p, const uint8_t* lim) {
  return p < lim ? __ldg(reinterpret_cast<const uint4*>(p)) : make_uint4(0u, 0u, 0u, 0u);
}
__device__ __forceinline__ uint64_t lo64(uint4 v) { return (uint64_t(v.y) << 32) | v.x; }
__device__ __forceinline__ uint64_t hi64(uint4 v) { return (uint64_t(v.w) << 32) | v.z; }
__device__ __forceinline__ uint64_t funnel(uint64_t a, uint64_t b, uint32_t sh) {
  return sh ? ((a >> sh) | (b << (64 - sh))) : a;
}

// One group's cell: 16-byte chunks [a0, a0 + 16*nchunks) cover its bytes.
struct CellGeom {
  const uint8_t* a0;
  uint32_t len, nwords, nchunks;
  uint32_t s8, sh;  // cell start = word s8 of chunk 0, bit shift sh
};

__device__ __forceinline__ CellGeom cell_geom(const uint8_t* p, uint32_t len) {
  CellGeom g;
  const uintptr_t ad = reinterpret_cast<uintptr_t>(p);
  g.a0 = reinterpret_cast<const uint8_t*>(ad & ~uintptr_t(15));
  g.len = len;
  g.nwords = (len + 7) / 8;
  g.nchunks = len ? uint32_t(((ad + len + 15) >> 4) - (ad >> 4)) : 0u;
  g.s8 = uint32_t((ad >> 3) & 1);
  g.sh = uint32_t(ad & 7) * 8;
  return g;
}

// Register window of kRmax chunk rounds from round w0: chunk j = gl + round*G
// of the cell (16 bytes) plus the first 8 bytes of chunk j + 1 (the
// neighbour lane's chunk, an L1 hit), so every lane forms its two cell words
// without shuffles. Only the cell's last word carries bytes past its end
// (masked where used).
struct Window {
  uint4 b[kRmax];
  uint64_t nx[kRmax];
};

__device__ __forceinline__ void load_window(Window& W, const CellGeom& g, uint32_t w0, uint32_t gl,
                                            uint32_t G) {
#pragma unroll
  for (uint32_t t = 0; t < kRmax; ++t) {
    const uint32_t j = gl + (w0 + t) * G;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    uint64_t x = 0;
    if (j < g.nchunks) {  // chunk starts before the cell end: inside the arena
      v = __ldg(reinterpret_cast<const uint4*>(g.a0 + 16 * j));
      if (j + 1 < g.nchunks) x = __ldg(reinterpret_cast<const unsigned long long*>(g.a0 + 16 * (j + 1)));
    }
    W.b[t] = v;
    W.nx[t] = x;
  }
}

// The lane's two cell words of round w0 + t: word k0 = x0, word k0 + 1 = x1
// (k0 = 2*(gl + round*G) - s8 may be -1: that word precedes the cell).
__device__ __forceinline__ void window_words(const Window& W, uint32_t t, uint32_t sh, uint64_t& x0,
                                             uint64_t& x1) {
  const uint64_t lo = lo64(W.b[t]), hi = hi64(W.b[t]);
  x0 = funnel(lo, hi, sh);
  x1 = funnel(hi, W.nx[t], sh);
}

// word_term(x, k) with kc = k * 0x9E3779B97F4A7C15 (common.cuh)
__device__ __forceinline__ uint64_t word_term_kc(uint64_t w, uint64_t kc) {
  const uint64_t x = (w ^ kc) * 0xff51afd7ed558ccdULL;
  return x ^ (x >> 32);
}
constexpr uint64_t kWordC = 0x9E3779B97F4A7C15ULL;

// Representative words k0 and k0 + 1 (k0 >= 0): three aligned loads.
__device__ __forceinline__ void rep_words(const uint8_t* rep, int64_t k0, const uint8_t* lim,
                                          uint64_t& y0, uint64_t& y1) {
  const uintptr_t ad = reinterpret_cast<uintptr_t>(rep) + 8 * uint64_t(k0);
  const uint64_t* p = reinterpret_cast<const uint64_t*>(ad & ~uintptr_t(7));
  const uint64_t* l =
      reinterpret_cast<const uint64_t*>((reinterpret_cast<uintptr_t>(lim) + 7) & ~uintptr_t(7));
  const uint32_t sh = uint32_t(ad & 7) * 8;
  const uint64_t w0 = p < l ? __ldg(p) : 0, w1 = p + 1 < l ? __ldg(p + 1) : 0;
  const uint64_t w2 = (sh && p + 2 < l) ? __ldg(p + 2) : 0;
  y0 = funnel(w0, w1, sh);
  y1 = funnel(w1, w2, sh);
}

// Write-once fields read by other threads while the kernel runs (slot id,
// representative offset and length) carry no fences: each starts at a
// sentinel that is never a valid value, so a reader that sees the sentinel
// (not yet visible, or a stale L1 line) re-reads it from L2 until it is set.
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}
__device__ __forceinline__ uint64_t ld_volatile_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

enum : uint32_t { kFound = 0, kClaimed = 1, kOverflow = 2 };

// Leader: from `slot`, find the first slot holding hash h (returns its id)
// or claim an empty one for a new value.
__device__ __forceinline__ uint32_t probe(const ColDict& D, uint32_t c, uint64_t h, uint64_t& slot,
                                          uint32_t& cid, uint64_t off, uint64_t len, uint32_t row,
                                          uint32_t* ncid, uint32_t* overflow) {
  for (uint64_t tries = 0;; ++tries) {
    if (tries > D.cap) {  // no empty slot left
      atomicOr(&overflow[c], 1u);
      return kOverflow;
    }
    // plain (L1-cached) loads on the hot path: a slot's key and id change
    // once (0 -> h, kNoCid -> id), so a stale line can only show the
    // unclaimed / unpublished state, which the slow paths re-check in L2
    unsigned long long k = D.keys[slot];
    if (k == 0) {
      const unsigned long long prev = atomicCAS(&D.keys[slot], 0ull, (unsigned long long)h);
      if (prev == 0) {
        const uint32_t id = atomicAdd(&ncid[c], 1u);
        if (id >= D.cidcap) {
          D.cids[slot] = kOverCid;
          atomicOr(&overflow[c], 1u);
          return kOverflow;
        }
        D.vhash[id] = h;
        D.voff[id] = off;
        D.vlen[id] = uint32_t(len);
        D.vrow[id] = row;
        D.cids[slot] = id;
        cid = id;
        return kClaimed;
      }
      k = prev;
    }
    if (k == h) {
      uint32_t id = D.cids[slot];
      while (id == kNoCid) {
        __nanosleep(20);
        id = ld_volatile_u32(&D.cids[slot]);
      }
      if (id == kOverCid) {
        atomicOr(&overflow[c], 1u);
        return kOverflow;
      }
      cid = id;
      return kFound;
    }
    slot = (slot + 1) & (D.cap - 1);
  }
}

enum : uint32_t { kSearching = 3 };

// One lockstep probe round of a warp whose lanes probe the same column (all
// 32 lanes call it; lanes with search = false only join the ballot). A lane
// examines one slot: its hash there -> kFound (id), an empty slot it wins ->
// kClaimed, a foreign key -> next slot (kSearching), its hash with the id not
// yet visible -> the same slot again next round (kSearching). The round's
// claims reserve their ids with one atomic per warp.
__device__ __forceinline__ uint32_t probe_round(const ColDict& D, uint32_t c, uint64_t h,
                                                uint64_t& slot, uint64_t& tries, bool search,
                                                uint32_t& id, uint64_t off, uint32_t len,
                                                uint32_t row, uint32_t* ncid, uint32_t* overflow) {
  uint32_t res = kSearching;
  bool claim = false;
  if (search) {
    unsigned long long k = D.keys[slot];  // plain load: stale only as 0
    if (k == 0) {
      const unsigned long long prev = atomicCAS(&D.keys[slot], 0ull, (unsigned long long)h);
      if (prev == 0) claim = true;
      else k = prev;
    }
    if (!claim) {
      if (k == h) {
        uint32_t v = D.cids[slot];
        if (v == kNoCid) v = ld_volatile_u32(&D.cids[slot]);
        if (v == kOverCid) {
          atomicOr(&overflow[c], 1u);
          res = kOverflow;
        } else if (v != kNoCid) {
          id = v;
          res = kFound;
        }
      } else if (++tries > D.cap) {
        atomicOr(&overflow[c], 1u);
        res = kOverflow;
      } else {
        slot = (slot + 1) & (D.cap - 1);
      }
    }
  }
  const uint32_t lane = threadIdx.x & 31;
  const unsigned cm = __ballot_sync(0xffffffffu, claim);
  if (cm) {
    const int leader = __ffs(cm) - 1;
    uint32_t base = 0;
    if (int(lane) == leader) base = atomicAdd(&ncid[c], uint32_t(__popc(cm)));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (claim) {
      const uint32_t v = base + uint32_t(__popc(cm & ((1u << lane) - 1u)));
      if (v >= D.cidcap) {
        D.cids[slot] = kOverCid;
        atomicOr(&overflow[c], 1u);
        res = kOverflow;
      } else {
        D.vhash[v] = h;
        D.voff[v] = off;
        D.vlen[v] = len;
        D.vrow[v] = row;
        D.cids[slot] = v;
        id = v;
        res = kClaimed;
      }
    }
  }
  return res;
}

constexpr uint32_t kMaxSmemItems = 8192;  // item -> column table in shared memory
constexpr uint32_t kMaxSmemCols = 128;     // column descriptors in shared memory

// A block takes tiles of 32 rows; its warps take the tile's work items
// (column c: G_c items of 32/G_c cells). Control flow is warp-uniform (loops
// run to the warp's longest cell, lanes past their own cell are predicated
// off), so the group shuffles and ballots use the full mask; only the
// leaders' probe loops diverge, with no collective inside.
__global__ void __launch_bounds__(kBuildBlock, 3) k_dict_build(BuildArgs A) {
  extern __shared__ uint16_t s_col[];  // [items] when smem_cols
  __shared__ ColDict s_dict[kMaxSmemCols];
  const bool smem_cols = A.items <= kMaxSmemItems && A.m <= 65535;
  const bool smem_dict = A.m <= kMaxSmemCols;
  if (smem_cols)
    for (uint32_t c = 0; c < A.m; ++c) {
      const uint32_t i0 = A.cols[c].item0, G = A.cols[c].G;
      for (uint32_t j = threadIdx.x; j < G; j += blockDim.x) s_col[i0 + j] = uint16_t(c);
    }
  if (smem_dict)
    for (uint32_t c = threadIdx.x; c < A.m; c += blockDim.x) s_dict[c] = A.cols[c];
  __syncthreads();
  constexpr unsigned kFull = 0xffffffffu;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t rows = A.r1 - A.r0;
  const uint64_t ntiles = (rows + kTileRows - 1) / kTileRows;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
  for (uint32_t w = warp; w < A.items; w += kBuildBlock / 32) {
    if (w == 0 && lane == 0 && A.prefetch && tile + gridDim.x < ntiles) {
      // stream the block's next tile (a contiguous byte range: whole rows)
      // into L2 while this one is processed
      const uint64_t t1 = tile + gridDim.x;
      const uint64_t e1 = (t1 + 1) * kTileRows < rows ? (t1 + 1) * kTileRows : rows;
      const uintptr_t b0 =
          reinterpret_cast<uintptr_t>(A.chunk + (A.offs[t1 * kTileRows * A.m] - A.base)) & ~uintptr_t(15);
      const uintptr_t b1 = reinterpret_cast<uintptr_t>(A.chunk + (A.offs[e1 * A.m] - A.base));
      const uintptr_t lim = reinterpret_cast<uintptr_t>(A.chunk_lim) & ~uintptr_t(15);
      const uintptr_t b1a = (b1 + 15) & ~uintptr_t(15);
      const uintptr_t end = b1a <= lim ? b1a : lim;
      if (end > b0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b0), "r"(uint32_t(end - b0))
                     : "memory");
    }
    uint32_t c;
    if (smem_cols) {
      c = s_col[w];
    } else {  // last c with item0 <= w
      uint32_t lo = 0, hi = A.m;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (A.cols[mid].item0 <= w) lo = mid;
        else hi = mid;
      }
      c = lo;
    }
    const ColDict& D = smem_dict ? s_dict[c] : A.cols[c];
    const uint32_t G = D.G;
    const uint32_t gl = lane & (G - 1);
    const uint32_t gshift = lane & ~(G - 1);  // first lane of the group
    const uint64_t rl = tile * kTileRows + (w - D.item0) * (32 / G) + lane / G;
    const bool valid = rl < rows;
    uint64_t o0 = 0;
    uint32_t len = 0;
    if (valid) {
      const uint64_t li = rl * A.m + c;
      o0 = A.offs[li];
      len = uint32_t(A.offs[li + 1] - o0);
    }
    const CellGeom g = cell_geom(A.chunk + (o0 - A.base), len);
    const uint32_t steps = (g.nchunks + G - 1) / G;
    const uint32_t wsteps = __reduce_max_sync(kFull, steps);  // warp-uniform
    const bool fits = wsteps <= kRmax;
    // word index and k * C of this lane's first word; per round +2G
    const int32_t kfirst = int32_t(2 * gl) - int32_t(g.s8);
    const uint64_t kstep = 2ull * G;
    const uint64_t lastmask = (len & 7) ? ((uint64_t(1) << (8 * (len & 7))) - 1) : ~0ull;
    // 1-2: hash
    Window W;
    unsigned long long sum = 0;
    for (uint32_t w0 = 0; w0 < wsteps; w0 += kRmax) {
      load_window(W, g, w0, gl, G);
#pragma unroll
      for (uint32_t t = 0; t < kRmax; ++t) {
        if (w0 + t >= wsteps) break;  // warp-uniform
        uint64_t x0, x1;
        window_words(W, t, g.sh, x0, x1);
        const int64_t k0 = int64_t(kfirst) + int64_t((w0 + t) * kstep);
        const uint64_t kc = uint64_t(k0) * kWordC;
        if (k0 + 1 == int64_t(g.nwords)) x0 &= lastmask;  // the cell's last word
        if (k0 + 2 == int64_t(g.nwords)) x1 &= lastmask;
        if (k0 >= 0 && uint64_t(k0) < g.nwords) sum += word_term_kc(x0, kc);
        if (uint64_t(k0 + 1) < g.nwords) sum += word_term_kc(x1, kc + kWordC);
      }
    }
    for (uint32_t d = G >> 1; d > 0; d >>= 1) sum += __shfl_xor_sync(kFull, sum, d, G);
    uint64_t h = hash_finish(sum, len) & A.hmask;
    h = h ? h : 1;
    // 3-4: probe, verify, continue past collisions (warp-uniform rounds)
    uint64_t slot = h & (D.cap - 1);
    uint32_t cid = kNoCid;
    bool done = !valid;
    uint64_t tries = 0;
    while (__any_sync(kFull, !done)) {
      uint32_t res = kSearching, id = 0;
      uint64_t sl = slot;
      {  // the group leaders probe in lockstep rounds until each has an answer
        bool search = !done && gl == 0;
        while (__any_sync(kFull, search)) {
          const uint32_t r = probe_round(D, c, h, sl, tries, search, id, o0, len,
                                         uint32_t(A.r0 + rl), A.ncid, A.overflow);
          if (search && r != kSearching) {
            res = r;
            search = false;
          }
        }
      }
      res = __shfl_sync(kFull, res, 0, G);
      id = __shfl_sync(kFull, id, 0, G);
      sl = __shfl_sync(kFull, sl, 0, G);
      bool check = false;
      const uint8_t* rep = nullptr;
      const uint8_t* rlim = nullptr;
      uint64_t rlen = 0;
      if (!done) {
        if (res == kOverflow) {
          done = true;
        } else if (res == kClaimed) {
          cid = id;
          done = true;
        } else {
          // representative locator: written once before the id's slot; a
          // stale L1 line shows the initial sentinels -> re-read from L2
          uint64_t ro = D.voff[id];
          rlen = D.vlen[id];
          while (ro == kUnsetOff || rlen == kUnsetLen) {
            ro = ld_volatile_u64(&D.voff[id]);
            rlen = ld_volatile_u32(&D.vlen[id]);
          }
          const bool in_vals = (ro & kInVals) != 0;
          rep = in_vals ? A.vals + (ro & ~kInVals) : A.chunk + (ro - A.base);
          rlim = in_vals ? A.vals_lim : A.chunk_lim;
          check = rlen == len && len > 0;
          if (rlen == len && len == 0) {  // equal empty strings
            cid = id;
            done = true;
          }
        }
      }
      uint64_t diff = 0;
      if (__any_sync(kFull, check)) {
        for (uint32_t w0 = 0; w0 < wsteps; w0 += kRmax) {
          if (!fits) load_window(W, g, w0, gl, G);
#pragma unroll
          for (uint32_t t = 0; t < kRmax; ++t) {
            if (w0 + t >= wsteps) break;
            if (!check) continue;
            uint64_t x0, x1;
            window_words(W, t, g.sh, x0, x1);
            const int64_t k0 = int64_t(kfirst) + int64_t((w0 + t) * kstep);
            if (k0 >= 0 && uint64_t(k0) < g.nwords) {
              uint64_t y0, y1;
              rep_words(rep, k0, rlim, y0, y1);
              diff |= (x0 ^ y0) & (uint64_t(k0) + 1 == g.nwords ? lastmask : ~0ull);
              if (uint64_t(k0 + 1) < g.nwords)
                diff |= (x1 ^ y1) & (uint64_t(k0) + 2 == g.nwords ? lastmask : ~0ull);
            } else if (k0 < 0 && g.nwords) {  // only word 0 is this lane's
              diff |= (x1 ^ load8_unaligned(rep, rlim)) & (g.nwords == 1 ? lastmask : ~0ull);
            }
          }
        }
      }
      const unsigned bad = __ballot_sync(kFull, diff != 0);
      const unsigned gbits = G == 32 ? kFull : (((1u << G) - 1u) << gshift);
      if (!done && res == kFound) {
        if (rlen == len && !(bad & gbits)) {
          cid = id;
          done = true;
        } else {
          slot = (sl + 1) & (D.cap - 1);  // a different value with the same hash
        }
      }
    }
    if (valid && gl == 0) A.cid_mat[(A.r0 + rl) * A.m + c] = cid;
  }
}

// ---------------------------------------------------------------------------
// Default path: three kernels per chunk (the fused group kernel above is
// slower on C2 and C5: profiles/r2_dict_experiments.md).
//   K1+K2a k_hash_probe thread per cell, warps walk 32 rows column by column
//                     (lanes of a warp hash cells of one column: similar
//                     lengths), 4 aligned 8-byte loads per 4 words; then the
//                     warp probes the column's table in lockstep rounds:
//                     claim (new value id) or find the slot of the cell's
//                     hash (id marked pending)
//   K2b k_verify_cells every pending cell byte-compared with its value's
//                     representative; a mismatch (64-bit collision) goes to
//   K2c k_fixup_cells exact re-probe with byte verification at every equal key
// ---------------------------------------------------------------------------
constexpr uint32_t kPending = 0x80000000u;  // cid_mat: found, not yet verified

// Cell hash of (row r, column c) of the chunk (thread per cell): the last
// aligned word of a step is the first of the next, carried (four loads per
// four words).
template <int STEP = 4>
__device__ __forceinline__ uint64_t cell_hash(const uint8_t* __restrict__ chunk, uint64_t base,
                                              const uint64_t* lim, uint64_t o0, uint64_t len,
                                              uint64_t hash_mask) {
  const uintptr_t ad = reinterpret_cast<uintptr_t>(chunk + (o0 - base));
  const uint64_t* p = reinterpret_cast<const uint64_t*>(ad & ~uintptr_t(7));
  const uint32_t sh = uint32_t(ad & 7) * 8;
  const uint64_t words = (len + 7) / 8;
  uint64_t sum = 0;
  uint64_t carry = (words && p < lim) ? __ldg(p) : 0;
  for (uint64_t k = 0; k < words; k += STEP) {
    uint64_t w[STEP + 1];
    w[0] = carry;
#pragma unroll
    for (int u = 1; u < STEP + 1; ++u) w[u] = (p + k + u < lim) ? __ldg(p + k + u) : 0;
    carry = w[STEP];
#pragma unroll
    for (int u = 0; u < STEP; ++u) {
      const uint64_t kk = k + u;
      if (kk < words) {
        uint64_t x = funnel(w[u], w[u + 1], sh);
        const uint64_t rem = len - 8 * kk;
        if (rem < 8) x = mask_low_bytes(x, uint32_t(rem));
        sum += word_term(x, kk);
      }
    }
  }
  const uint64_t h = hash_finish(sum, len) & hash_mask;
  return h ? h : 1;
}

// Whole-warp hash of one long cell (same value as cell_hash): lane l takes
// words 2l, 2l+1, 2l+64, ... with three aligned 8-byte loads per word pair
// (consecutive lanes read consecutive 16 bytes: coalesced), then the warp
// reduces the word terms. (A variant loading aligned 16-byte chunks and
// shifting them through shuffles was slower on C5: 12.2 vs 8.8 ms per 3M rows.)
__device__ __forceinline__ uint64_t warp_cell_hash(const uint8_t* p, uint64_t len, const uint8_t* lim,
                                                   uint64_t hash_mask, uint32_t lane) {
  const uint64_t nwords = (len + 7) / 8;
  const uint64_t lastmask = (len & 7) ? ((uint64_t(1) << (8 * (len & 7))) - 1) : ~0ull;
  unsigned long long sum = 0;
  for (uint64_t k0 = 2 * lane; k0 < nwords; k0 += 64) {
    uint64_t x0, x1;
    rep_words(p, int64_t(k0), lim, x0, x1);
    if (k0 + 1 == nwords) x0 &= lastmask;
    sum += word_term(x0, k0);
    if (k0 + 1 < nwords) {
      if (k0 + 2 == nwords) x1 &= lastmask;
      sum += word_term(x1, k0 + 1);
    }
  }
  const uint64_t h = hash_finish(warp_sum_u64(sum), len) & hash_mask;
  return h ? h : 1;
}

// Whole-warp byte equality of two strings of length len (same lane layout).
__device__ __forceinline__ bool warp_equal(const uint8_t* a, const uint8_t* a_lim, const uint8_t* b,
                                           const uint8_t* b_lim, uint64_t len, uint32_t lane) {
  const uint64_t nwords = (len + 7) / 8;
  const uint64_t lastmask = (len & 7) ? ((uint64_t(1) << (8 * (len & 7))) - 1) : ~0ull;
  uint64_t diff = 0;
  for (uint64_t k0 = 2 * lane; k0 < nwords; k0 += 64) {
    uint64_t x0, x1, y0, y1;
    rep_words(a, int64_t(k0), a_lim, x0, x1);
    rep_words(b, int64_t(k0), b_lim, y0, y1);
    diff |= (x0 ^ y0) & (k0 + 1 == nwords ? lastmask : ~0ull);
    if (k0 + 1 < nwords) diff |= (x1 ^ y1) & (k0 + 2 == nwords ? lastmask : ~0ull);
  }
  return !__any_sync(0xffffffffu, diff != 0);
}

// K1 + K2a: warps take 32 rows and walk them column by column (lanes of a
// warp hash cells of one column: similar lengths; one row's bytes are read
// by the same lane in consecutive iterations, so boundary sectors hit L1),
// then probe the column's table with the hashes in lockstep rounds
// (probe_round: each round's claims reserve their ids with one atomic per
// warp; a lane meeting its hash in a slot whose id is not yet visible
// retries it next round). Claimed cells get their new id, found cells the
// slot's id marked pending (byte verification follows).
template <int MINB, int STEP>
__global__ void __launch_bounds__(256, MINB) k_hash_probe(const uint8_t* __restrict__ chunk, uint64_t base,
                                                    const uint8_t* chunk_lim,
                                                    const uint64_t* __restrict__ offs, uint64_t rows,
                                                    uint64_t r0, uint32_t m, uint64_t hash_mask,
                                                    const ColDict* __restrict__ cols, uint32_t* ncid,
                                                    uint32_t* overflow, uint32_t* cid_mat,
                                                    uint64_t long_min) {
  constexpr unsigned kFull = 0xffffffffu;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t ntiles = (rows + 31) / 32;
  const uint64_t* lim =
      reinterpret_cast<const uint64_t*>((reinterpret_cast<uintptr_t>(chunk_lim) + 7) & ~uintptr_t(7));
  for (uint64_t tile = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; tile < ntiles;
       tile += (uint64_t(gridDim.x) * blockDim.x) >> 5)
    for (uint32_t c = 0; c < m; ++c) {
      const uint64_t r = tile * 32 + lane;
      bool search = r < rows;
      const uint64_t i = r * m + c;
      uint64_t o0 = 0, len = 0, h = 0;
      if (search) {
        o0 = offs[i];
        len = offs[i + 1] - o0;
      }
      // cells of at least long_min bytes are hashed by the whole warp
      // (coalesced), the others by their own lane
      const bool coop = search && len >= long_min;
      if (search && !coop) h = cell_hash<STEP>(chunk, base, lim, o0, len, hash_mask);
      for (unsigned lm = __ballot_sync(kFull, coop); lm; lm &= lm - 1) {
        const int src = __ffs(lm) - 1;
        const uint64_t so = __shfl_sync(kFull, o0, src), sl = __shfl_sync(kFull, len, src);
        const uint64_t sh = warp_cell_hash(chunk + (so - base), sl, chunk_lim, hash_mask, lane);
        if (int(lane) == src) h = sh;
      }
      const ColDict& D = cols[c];
      uint64_t slot = h & (D.cap - 1), tries = 0;
      uint32_t out = kNoCid;
      while (__any_sync(kFull, search)) {
        uint32_t id = 0;
        const uint32_t res = probe_round(D, c, h, slot, tries, search, id, o0, uint32_t(len),
                                         uint32_t(r0 + r), ncid, overflow);
        if (search && res != kSearching) {
          out = res == kClaimed ? id : (res == kFound ? (id | kPending) : kNoCid);
          // a cell of at most 8 bytes is one masked word: for a fixed length
          // the full 64-bit hash is a bijection of it (odd multiply,
          // xor-shift, fmix64), so an equal hash and an equal length mean
          // equal bytes — no byte compare (not for h == 1, the image of the
          // remapped 0, nor under debug hash masks)
          if (res == kFound && len <= 8 && h != 1 && hash_mask == ~0ull &&
              ld_volatile_u32(&D.vlen[id]) == uint32_t(len))
            out = id;
          search = false;
        }
      }
      if (r < rows) cid_mat[(r0 + r) * m + c] = out;
    }
}

// Four words of a byte string from five aligned words, the first passed in
// (the previous step's last) and the new last handed back.
struct Step4 {
  uint64_t w[4];
};
__device__ __forceinline__ Step4 load_step4_carry(const uint64_t* p, uint32_t sh, const uint64_t* lim,
                                                  uint64_t& carry) {
  uint64_t a[5];
  a[0] = carry;
#pragma unroll
  for (int u = 1; u < 5; ++u) a[u] = (p + u < lim) ? __ldg(p + u) : 0;
  carry = a[4];
  Step4 r;
#pragma unroll
  for (int u = 0; u < 4; ++u) r.w[u] = funnel(a[u], a[u + 1], sh);
  return r;
}

// Byte equality of two strings of length len (4 words per step, 8 loads in
// flight).
__device__ __forceinline__ bool equal_bytes4(const uint8_t* a, const uint8_t* a_lim, const uint8_t* b,
                                             const uint8_t* b_lim, uint64_t len) {
  if (!len) return true;
  const uintptr_t aa = reinterpret_cast<uintptr_t>(a), bb = reinterpret_cast<uintptr_t>(b);
  const uint64_t* pa = reinterpret_cast<const uint64_t*>(aa & ~uintptr_t(7));
  const uint64_t* pb = reinterpret_cast<const uint64_t*>(bb & ~uintptr_t(7));
  const uint64_t* la =
      reinterpret_cast<const uint64_t*>((reinterpret_cast<uintptr_t>(a_lim) + 7) & ~uintptr_t(7));
  const uint64_t* lb =
      reinterpret_cast<const uint64_t*>((reinterpret_cast<uintptr_t>(b_lim) + 7) & ~uintptr_t(7));
  const uint32_t sa = uint32_t(aa & 7) * 8, sb = uint32_t(bb & 7) * 8;
  const uint64_t words = (len + 7) / 8;
  uint64_t ca = pa < la ? __ldg(pa) : 0, cb = pb < lb ? __ldg(pb) : 0;
  for (uint64_t k = 0; k < words; k += 4) {
    const Step4 x = load_step4_carry(pa + k, sa, la, ca);
    const Step4 y = load_step4_carry(pb + k, sb, lb, cb);
    uint64_t d = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t kk = k + u;
      if (kk < words) {
        const uint64_t rem = len - 8 * kk;
        d |= mask_low_bytes(x.w[u] ^ y.w[u], rem >= 8 ? 8u : uint32_t(rem));
      }
    }
    if (d) return false;
  }
  return true;
}

__device__ __forceinline__ void rep_loc(const ColDict& D, uint32_t id, const BuildArgs& A,
                                        const uint8_t*& rep, const uint8_t*& rlim, uint64_t& rlen) {
  uint64_t ro = D.voff[id];
  rlen = D.vlen[id];
  while (ro == kUnsetOff || rlen == kUnsetLen) {  // published in this kernel (fix-up races)
    ro = ld_volatile_u64(&D.voff[id]);
    rlen = ld_volatile_u32(&D.vlen[id]);
  }
  const bool in_vals = (ro & kInVals) != 0;
  rep = in_vals ? A.vals + (ro & ~kInVals) : A.chunk + (ro - A.base);
  rlim = in_vals ? A.vals_lim : A.chunk_lim;
}

template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_verify_cells(BuildArgs A, uint32_t* collided,
                                                      uint32_t* n_collided, uint64_t long_min) {
  // warps take 32 rows of one column (similar lengths); a lane compares its
  // own cell with its value's representative, cells of at least long_min
  // bytes are compared by the whole warp (coalesced)
  constexpr unsigned kFull = 0xffffffffu;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t rows = A.r1 - A.r0;
  const uint64_t ntiles = (rows + 31) / 32;
  for (uint64_t tile = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; tile < ntiles;
       tile += (uint64_t(gridDim.x) * blockDim.x) >> 5)
    for (uint32_t c = 0; c < A.m; ++c) {
      const uint64_t r = tile * 32 + lane;
      const uint64_t gi = (A.r0 + r) * A.m + c;
      const uint32_t v = r < rows ? A.cid_mat[gi] : kNoCid;
      const bool pending = (v & kPending) && v != kNoCid;
      const uint32_t id = v & ~kPending;
      const uint64_t i = r * A.m + c;
      uint64_t o0 = 0, len = 0, rlen = 0;
      const uint8_t* rep = nullptr;
      const uint8_t* rlim = nullptr;
      if (pending) {
        o0 = A.offs[i];
        len = A.offs[i + 1] - o0;
        rep_loc(A.cols[c], id, A, rep, rlim, rlen);
      }
      const uint8_t* cell = A.chunk + (o0 - A.base);
      const bool coop = pending && rlen == len && len >= long_min;
      bool eq = false;
      if (pending && !coop) eq = rlen == len && equal_bytes4(cell, A.chunk_lim, rep, rlim, len);
      for (unsigned lm = __ballot_sync(kFull, coop); lm; lm &= lm - 1) {
        const int src = __ffs(lm) - 1;
        const uint8_t* sc = reinterpret_cast<const uint8_t*>(
            __shfl_sync(kFull, reinterpret_cast<uintptr_t>(cell), src));
        const uint8_t* sr = reinterpret_cast<const uint8_t*>(
            __shfl_sync(kFull, reinterpret_cast<uintptr_t>(rep), src));
        const uint8_t* srl = reinterpret_cast<const uint8_t*>(
            __shfl_sync(kFull, reinterpret_cast<uintptr_t>(rlim), src));
        const uint64_t sl = __shfl_sync(kFull, len, src);
        const bool e = warp_equal(sc, A.chunk_lim, sr, srl, sl, lane);
        if (int(lane) == src) eq = e;
      }
      if (pending) {
        if (eq) A.cid_mat[gi] = id;
        else collided[atomicAdd(n_collided, 1u)] = uint32_t(i);
      }
    }
}

// Rare path: a cell whose hash slot holds a different string re-probes its
// column with byte verification at every slot of its hash.
__global__ void k_fixup_cells(BuildArgs A, const uint32_t* collided, const uint32_t* n_collided_dev) {
  const uint32_t nc = *n_collided_dev;  // read on the device: no host round trip
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nc; q += gridDim.x * blockDim.x) {
    const uint64_t i = collided[q];
    const uint64_t r = i / A.m;
    const uint32_t c = uint32_t(i - r * A.m);
    const ColDict& D = A.cols[c];
    const uint64_t o0 = A.offs[i], len = A.offs[i + 1] - o0;
    const uint64_t* lim = reinterpret_cast<const uint64_t*>(
        (reinterpret_cast<uintptr_t>(A.chunk_lim) + 7) & ~uintptr_t(7));
    const uint64_t h = cell_hash(A.chunk, A.base, lim, o0, len, A.hmask);
    const uint8_t* cell = A.chunk + (o0 - A.base);
    uint64_t slot = h & (D.cap - 1);
    uint32_t out = kNoCid;
    for (;;) {
      uint32_t id = 0;
      const uint32_t res = probe(D, c, h, slot, id, o0, len, uint32_t(A.r0 + r), A.ncid, A.overflow);
      if (res == kOverflow) break;
      if (res == kClaimed) {
        out = id;
        break;
      }
      const uint8_t* rep;
      const uint8_t* rlim;
      uint64_t rlen;
      rep_loc(D, id, A, rep, rlim, rlen);
      if (rlen == len && equal_bytes4(cell, A.chunk_lim, rep, rlim, len)) {
        out = id;
        break;
      }
      slot = (slot + 1) & (D.cap - 1);
    }
    A.cid_mat[(A.r0 + r) * A.m + c] = out;
  }
}

// Per-column byte totals of up to `ns` evenly spaced rows (lane-count choice).
__global__ void k_sample_col_bytes(const uint64_t* offsets, uint64_t n, uint32_t m, uint32_t ns,
                                   unsigned long long* sums) {
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < uint64_t(ns) * m;
       q += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = q / m;
    const uint32_t c = uint32_t(q - k * m);
    const uint64_t r = ns >= n ? k : (k * n) / ns;
    const uint64_t i = r * m + c;
    atomicAdd(&sums[c], (unsigned long long)(offsets[i + 1] - offsets[i]));
  }
}

// Re-inserts ids [0, count) of a column into a fresh (zeroed keys, kNoCid
// ids) table of capacity cap from their stored hashes. Every id keeps its
// own slot (equal hashes of different values stay separate entries).
__global__ void k_rehash(const unsigned long long* vhash, uint32_t count, unsigned long long* keys,
                         uint32_t* cids, uint64_t cap) {
  for (uint32_t id = blockIdx.x * blockDim.x + threadIdx.x; id < count; id += gridDim.x * blockDim.x) {
    const unsigned long long h = vhash[id];
    uint64_t slot = h & (cap - 1);
    for (;;) {
      if (atomicCAS(&keys[slot], 0ull, h) == 0ull) {
        cids[slot] = id;
        break;
      }
      slot = (slot + 1) & (cap - 1);
    }
  }
}

// New values of a chunk (streamed tables): flat index q over the columns'
// new id ranges (segment s: column seg_col[s], ids from seg_id0[s], flat
// start seg_q0[s]).
struct NewVals {
  const uint32_t* seg_col;
  const uint32_t* seg_id0;
  const uint64_t* seg_q0;
  uint32_t nseg;
  const ColDict* cols;
};

__device__ __forceinline__ void new_val(const NewVals& V, uint64_t q, uint32_t& c, uint32_t& id) {
  uint32_t lo = 0, hi = V.nseg;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (V.seg_q0[mid] <= q) lo = mid;
    else hi = mid;
  }
  c = V.seg_col[lo];
  id = V.seg_id0[lo] + uint32_t(q - V.seg_q0[lo]);
}

__global__ void k_new_val_sizes(NewVals V, uint64_t total, uint64_t* sizes) {
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < total;
       q += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t c, id;
    new_val(V, q, c, id);
    sizes[q] = (uint64_t(V.cols[c].vlen[id]) + 7) & ~uint64_t(7);  // 8-byte slots
  }
}

// Warp per new value: copy its bytes from the chunk into the value arena
// (8-byte aligned slot at vals_used + pos[q]) and repoint its offset.
__global__ void k_copy_new_vals(NewVals V, uint64_t total, const uint64_t* pos, uint64_t vals_used,
                                const uint8_t* chunk, uint64_t base, const uint8_t* chunk_end,
                                uint8_t* vals) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t q = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; q < total;
       q += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
    uint32_t c, id;
    new_val(V, q, c, id);
    const ColDict& D = V.cols[c];
    const uint64_t off = D.voff[id];
    const uint64_t len = D.vlen[id];
    const uint8_t* src = chunk + (off - base);
    uint64_t* dst = reinterpret_cast<uint64_t*>(vals + vals_used + pos[q]);
    for (uint64_t k = lane; 8 * k < len; k += 32) dst[k] = load8_unaligned(src + 8 * k, chunk_end);
    __syncwarp();
    if (lane == 0) D.voff[id] = kInVals | (vals_used + pos[q]);
  }
}

// Dense arrays over all distinct values in compaction order: d = colbase[c] + id.
__global__ void k_gather_dict(const ColDict* cols, const uint64_t* colbase, uint32_t m, uint64_t D,
                              uint64_t* val_off, uint32_t* val_len, uint32_t* rep_row,
                              uint32_t* d_col) {
  for (uint64_t d = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; d < D;
       d += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t lo = 0, hi = m;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (colbase[mid] <= d) lo = mid;
      else hi = mid;
    }
    const uint32_t c = lo;
    const uint32_t id = uint32_t(d - colbase[c]);
    val_off[d] = cols[c].voff[id] & ~kInVals;
    val_len[d] = cols[c].vlen[id];
    rep_row[d] = cols[c].vrow[id];
    d_col[d] = c;
  }
}

uint64_t pow2_at_least(uint64_t x) {
  uint64_t p = 64;
  while (p < x) p <<= 1;
  return p;
}

struct ColBufs {
  DevBuf<unsigned long long> keys, vhash, voff;
  DevBuf<uint32_t> cids, vlen, vrow;
};

class Builder {
 public:
  Builder(uint64_t n, uint32_t m, uint64_t hmask, cudaStream_t s)
      : n_(n), m_(m), hmask_(hmask), s_(s), bufs_(m), h_(m), cnt2_(2 * size_t(m), s),
        d_cols_(m, s) {
    cnt2_.zero();
  }

  // lanes per cell from the columns' average lengths
  void set_lanes(const std::vector<double>& avg) {
    row_bytes_ = 0;
    for (double a : avg) row_bytes_ += a;
    uint32_t item = 0;
    for (uint32_t c = 0; c < m_; ++c) {
      // fewest lanes whose register window holds a cell of about the
      // column's average length (unaligned: up to two extra chunks)
      const double chunks = avg[c] / 16.0 + 1.5;
      static const uint32_t max_lanes = [] {  // PO_DICT_LANES: experiment knob
        const char* v = std::getenv("PO_DICT_LANES");
        const int x = v && *v ? std::atoi(v) : 32;
        return uint32_t(x >= 1 && x <= 32 ? x : 32);
      }();
      uint32_t G = 1;
      while (G < max_lanes && double(G) * kRmax < chunks) G <<= 1;
      h_[c].G = G;
      h_[c].item0 = item;
      item += G;  // a tile of 32 rows = G items of 32/G cells
    }
    items_ = item;
  }

  // capacity for at least `want` ids (<= n) per column; rehashes existing ones
  void reserve(uint32_t c, uint64_t want) {
    want = std::max<uint64_t>(1, std::min<uint64_t>(want, n_));
    ColDict& D = h_[c];
    if (D.keys && want <= D.cidcap) return;
    const uint32_t keep = D.keys ? std::min<uint32_t>(count_[c], D.cidcap) : 0;
    const uint32_t cidcap = uint32_t(want);
    const uint64_t cap = pow2_at_least(2 * want);
    HostScope hs("dict_reserve");
    ProfScope ps("dict_reserve", s_);
    ColBufs nb;
    nb.keys.alloc_auto(cap, s_);
    nb.cids.alloc_auto(cap, s_);
    nb.keys.zero();
    nb.cids.fill_bytes(0xFF);
    nb.vhash.alloc_auto(cidcap, s_);
    nb.voff.alloc_auto(cidcap, s_);
    nb.vlen.alloc_auto(cidcap, s_);
    nb.vrow.alloc_auto(cidcap, s_);
    nb.voff.fill_bytes(0xFF);  // kUnsetOff / kUnsetLen
    nb.vlen.fill_bytes(0xFF);
    if (keep) {
      PO_CUDA(cudaMemcpyAsync(nb.vhash.get(), D.vhash, keep * 8ull, cudaMemcpyDeviceToDevice, s_));
      PO_CUDA(cudaMemcpyAsync(nb.voff.get(), D.voff, keep * 8ull, cudaMemcpyDeviceToDevice, s_));
      PO_CUDA(cudaMemcpyAsync(nb.vlen.get(), D.vlen, keep * 4ull, cudaMemcpyDeviceToDevice, s_));
      PO_CUDA(cudaMemcpyAsync(nb.vrow.get(), D.vrow, keep * 4ull, cudaMemcpyDeviceToDevice, s_));
      PO_LAUNCH(k_rehash, grid_for(keep, 256), 256, 0, s_, nb.vhash.get(), keep, nb.keys.get(),
                nb.cids.get(), cap);
    }
    bufs_[c] = std::move(nb);
    D.keys = bufs_[c].keys.get();
    D.cids = bufs_[c].cids.get();
    D.vhash = bufs_[c].vhash.get();
    D.voff = bufs_[c].voff.get();
    D.vlen = bufs_[c].vlen.get();
    D.vrow = bufs_[c].vrow.get();
    D.cap = cap;
    D.cidcap = cidcap;
    dirty_ = true;
  }

  // First reservation of every column at once: one allocation holding all
  // columns' arrays, grouped so that two memsets initialise them (slot keys
  // zero; cids and the value offsets / lengths all-ones).
  void reserve_all(uint64_t want_each) {
    HostScope hs("dict_reserve_all");
    ProfScope ps("dict_reserve_all", s_);
    const uint64_t want = std::max<uint64_t>(1, std::min<uint64_t>(want_each, n_));
    const uint64_t cap = pow2_at_least(2 * want);
    auto al = [](uint64_t b) { return (b + 255) & ~uint64_t(255); };
    const uint64_t zb = al(cap * 8), fb = al(cap * 4) + al(want * 8) + al(want * 4),
                   ub = al(want * 8) + al(want * 4);
    shared_.alloc_auto(m_ * (zb + fb + ub), s_);
    uint8_t* z = shared_.get();
    uint8_t* f = z + m_ * zb;
    uint8_t* u = f + m_ * fb;
    PO_CUDA(cudaMemsetAsync(z, 0, m_ * zb, s_));
    PO_CUDA(cudaMemsetAsync(f, 0xFF, m_ * fb, s_));
    for (uint32_t c = 0; c < m_; ++c) {
      ColDict& D = h_[c];
      bufs_[c] = ColBufs{};
      D.keys = reinterpret_cast<unsigned long long*>(z + c * zb);
      uint8_t* fc = f + c * fb;
      D.cids = reinterpret_cast<uint32_t*>(fc);
      D.voff = reinterpret_cast<unsigned long long*>(fc + al(cap * 4));
      D.vlen = reinterpret_cast<uint32_t*>(fc + al(cap * 4) + al(want * 8));
      uint8_t* uc = u + c * ub;
      D.vhash = reinterpret_cast<unsigned long long*>(uc);
      D.vrow = reinterpret_cast<uint32_t*>(uc + al(want * 8));
      D.cap = cap;
      D.cidcap = uint32_t(want);
    }
    dirty_ = true;
  }

  void init_counts() { count_.assign(m_, 0); }
  void set_avg_cell_bytes(double v) { avg_cell_bytes_ = v; }

  // one chunk of rows [r0, r1), retried with grown tables until no column
  // overflows; leaves count_ = the per-column distinct counts
  void run_chunk(const uint8_t* chunk, uint64_t base, const uint8_t* chunk_lim, const uint8_t* vals,
                 const uint8_t* vals_lim, const uint64_t* offs, uint64_t r0, uint64_t r1,
                 uint32_t* cid_mat) {
    if (r1 <= r0) return;
    for (int attempt = 0;; ++attempt) {
      push_state();
      BuildArgs A;
      A.chunk = chunk;
      A.base = base;
      A.chunk_lim = chunk_lim;
      A.vals = vals ? vals : chunk;
      A.vals_lim = vals ? vals_lim : chunk_lim;
      A.offs = offs;
      A.r0 = r0;
      A.r1 = r1;
      A.m = m_;
      A.items = items_;
      A.hmask = hmask_;
      A.cols = d_cols_.get();
      A.ncid = ncid();
      A.overflow = over();
      A.cid_mat = cid_mat;
      const uint64_t work = ((r1 - r0 + kTileRows - 1) / kTileRows) * items_;
      const uint64_t tiles = (r1 - r0 + kTileRows - 1) / kTileRows;
      // persistent: the resident blocks stride over the tiles
      const unsigned grid = unsigned(std::min<uint64_t>(tiles, uint64_t(kSMs) * 3));
      // next-tile prefetch while two waves of tiles fit well inside L2
      {
        static const int pf_env = [] {
          const char* v = std::getenv("PO_DICT_PREFETCH");
          return v && *v ? std::atoi(v) : -1;
        }();
        const double tile_bytes = row_bytes_ * kTileRows;
        A.prefetch = pf_env >= 0 ? uint32_t(pf_env) : uint32_t(2.0 * grid * tile_bytes < 48e6);
      }
      (void)work;
      const unsigned smem = items_ <= kMaxSmemItems ? ((items_ * 2 + 15) & ~15u) : 0u;
      if (fused_) {
        PO_LAUNCH(k_dict_build, grid, kBuildBlock, smem, s_, A);
      } else {
        const uint64_t cells = (r1 - r0) * m_;
        collided_.alloc_auto(cells, s_);
        DevBuf<uint32_t> ncol(1, s_);
        ncol.zero();
        const unsigned gw = grid_for(((r1 - r0 + 31) / 32) * 32, 256, 8);
        // PO_LONG_CELL: cells of at least this many bytes are hashed and
        // verified by a whole warp (C5's ~2 KB cells: verify 15.7 -> 10.9 ms
        // per 3M rows; C2's cells stay below it)
        static const uint64_t long_min = [] {
          const char* v = std::getenv("PO_LONG_CELL");
          return v && *v ? uint64_t(std::strtoull(v, nullptr, 10)) : uint64_t(1024);
        }();
        // occupancy (measured, tools/probe_shape_sweep.sh): the probe at 6
        // blocks per SM (40 registers); the verify at 4, or at 8 when the cells
        // average at least long_min bytes (they take the whole-warp compare,
        // which needs few registers: C5 verify 10.8 -> 8.1 ms per 3M rows)
        PO_LAUNCH((k_hash_probe<6, 4>), gw, 256, 0, s_, chunk, base, chunk_lim, offs, r1 - r0, r0, m_,
                  hmask_, d_cols_.get(), ncid(), over(), cid_mat, long_min);
        if (avg_cell_bytes_ >= double(long_min))
          PO_LAUNCH((k_verify_cells<8>), gw, 256, 0, s_, A, collided_.get(), ncol.get(), long_min);
        else
          PO_LAUNCH((k_verify_cells<4>), gw, 256, 0, s_, A, collided_.get(), ncol.get(), long_min);
        PO_LAUNCH(k_fixup_cells, kSMs, 128, 0, s_, A, collided_.get(), ncol.get());
      }
      std::vector<uint32_t> hc(2 * m_);
      d2h_sync(hc.data(), cnt2_.get(), 2 * size_t(m_) * sizeof(uint32_t), s_);
      bool any = false;
      for (uint32_t c = 0; c < m_; ++c) {
        count_[c] = hc[c];
        if (hc[m_ + c]) any = true;
      }
      if (!any) return;
      if (attempt > 40) fail(PO_ERR_ERROR, "internal: dictionary growth did not converge");
      // ids at or past a column's old capacity were never published: the
      // grown table keeps ids [0, keep) and the counter restarts there
      for (uint32_t c = 0; c < m_; ++c)
        if (hc[m_ + c]) {
          const uint32_t keep = std::min<uint32_t>(hc[c], h_[c].cidcap);
          const uint64_t want =
              std::max<uint64_t>(2ull * h_[c].cidcap, uint64_t(hc[c]) + (r1 - r0) / 4);
          count_[c] = keep;
          reserve(c, want);
          hc[c] = keep;
        }
      std::fill(hc.begin() + m_, hc.end(), 0u);
      cnt2_.upload(hc.data(), 2 * size_t(m_));
    }
  }

  const std::vector<uint32_t>& counts() const { return count_; }
  const ColDict* d_cols() {
    push_state();
    return d_cols_.get();
  }
  const ColDict& col(uint32_t c) const { return h_[c]; }
  bool fused() const { return fused_; }
  uint32_t lanes(uint32_t c) const { return h_[c].G; }

 private:
  void push_state() {
    if (!dirty_) return;
    h2d_async(d_cols_.get(), h_.data(), sizeof(ColDict) * m_, s_);
    dirty_ = false;
  }

  uint64_t n_;
  uint32_t m_;
  uint64_t hmask_;
  cudaStream_t s_;
  std::vector<ColBufs> bufs_;
  std::vector<ColDict> h_;
  DevBuf<uint32_t> cnt2_;  // [new ids per column][overflow flags per column]
  DevBuf<uint8_t> shared_;  // reserve_all's arrays of every column
  double avg_cell_bytes_ = 0;
  uint32_t* ncid() { return cnt2_.get(); }
  uint32_t* over() { return cnt2_.get() + m_; }
  DevBuf<ColDict> d_cols_;
  uint32_t items_ = 0;
  double row_bytes_ = 0;
  // PO_DICT_KERNEL=fused: the one-kernel group path (experiment)
  bool fused_ = [] {
    const char* v = std::getenv("PO_DICT_KERNEL");
    return v && std::string(v) == "fused";
  }();
  DevBuf<uint32_t> collided_;
  bool dirty_ = true;
  std::vector<uint32_t> count_;
};

}  // namespace

void exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, cudaStream_t s) {
  if (!n) return;
  size_t tb = 0;
  PO_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, int64_t(n), s));
  DevBuf<uint8_t> tmp(tb, s);
  ProfScope ps("cub_scan", s);
  PO_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, in, out, int64_t(n), s));
}

namespace {

// Pageable host input (a std::vector or numpy arena): the driver copies it
// through its own small bounce buffers at ~8 GB/s. Instead, host threads
// copy each row chunk into one of two pinned slots in parallel (the slots
// are kept per host thread across calls: pinning memory is slow), and the
// slot is copied to the device asynchronously; the staging of chunk k+1
// runs while chunk k is copied and encoded.
struct PinnedSlot {
  uint8_t* p = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;  // the last H2D out of the slot
  int dev = -1;
  bool pending = false;
};
// A thread's slots go back to a process-wide list when it exits (buffers
// are never freed: pinning is slow and cudaFreeHost synchronises the
// device), so a caller that runs each call on a fresh thread reuses them.
std::mutex g_slot_mu;
std::vector<std::pair<uint8_t*, size_t>> g_slot_free;

struct PinnedSlots {
  PinnedSlot slot[2];
  ~PinnedSlots() {
    std::lock_guard<std::mutex> lk(g_slot_mu);
    for (auto& x : slot) {
      if (x.pending) cudaEventSynchronize(x.done);
      if (x.done) cudaEventDestroy(x.done);
      if (x.p) g_slot_free.push_back({x.p, x.cap});
    }
  }
};
thread_local PinnedSlots g_slots;

PinnedSlot& pinned_slot(int i, size_t bytes) {
  PinnedSlot& x = g_slots.slot[i];
  int dev = 0;
  PO_CUDA(cudaGetDevice(&dev));
  if (x.pending) {
    PO_CUDA(cudaEventSynchronize(x.done));
    x.pending = false;
  }
  if (x.cap < bytes) {
    std::lock_guard<std::mutex> lk(g_slot_mu);
    if (x.p) g_slot_free.push_back({x.p, x.cap});
    x.p = nullptr;
    x.cap = 0;
    size_t best = g_slot_free.size();
    for (size_t k = 0; k < g_slot_free.size(); ++k)  // smallest free buffer that fits
      if (g_slot_free[k].second >= bytes &&
          (best == g_slot_free.size() || g_slot_free[k].second < g_slot_free[best].second))
        best = k;
    if (best < g_slot_free.size()) {
      x.p = g_slot_free[best].first;
      x.cap = g_slot_free[best].second;
      g_slot_free.erase(g_slot_free.begin() + best);
    } else {
      PO_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&x.p), bytes, cudaHostAllocPortable));
      x.cap = bytes;
    }
  }
  if (x.dev != dev) {
    if (x.done) cudaEventDestroy(x.done);
    PO_CUDA(cudaEventCreateWithFlags(&x.done, cudaEventDisableTiming));
    x.dev = dev;
  }
  return x;
}

// memcpy with several host threads (bandwidth of one thread: ~10 GB/s)
void parallel_copy(uint8_t* dst, const uint8_t* src, size_t bytes) {
  const size_t kPiece = 16u << 20;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned nt = unsigned(std::min<size_t>(std::min(8u, hw), (bytes + kPiece - 1) / kPiece));
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (bytes + nt - 1) / nt;
  for (unsigned i = 0; i < nt; ++i) {
    const size_t lo = i * per, hi = std::min(bytes, lo + per);
    if (lo < hi) th.emplace_back([=] { std::memcpy(dst + lo, src + lo, hi - lo); });
  }
  for (auto& x : th) x.join();
}

bool host_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

}  // namespace

void build_dictionary(const DeviceTable& t, uint32_t hash_bits, cudaStream_t s, uint32_t* cid_mat,
                      DictResult& out) {
  const uint64_t n = t.n, m = t.m, cells = n * m;
  out = DictResult{};
  out.card.assign(m, 0);
  out.colbase.assign(m + 1, 0);
  if (cells == 0) return;
  if (n >= (uint64_t(1) << 31)) fail(PO_ERR_SIZE, "table too large for one device (rows must be < 2^31)");
  const uint64_t hmask = hash_bits >= 64 ? ~uint64_t(0) : ((uint64_t(1) << hash_bits) - 1);
  Builder B(n, uint32_t(m), hmask, s);
  B.init_counts();
  B.set_avg_cell_bytes(double(t.arena_bytes) / double(cells));
  const bool streamed = t.h_arena != nullptr;
  const uint64_t* h_offs = streamed ? t.h_offsets : nullptr;

  // per-column average lengths from a sample of rows (lanes per cell of the
  // fused kernel)
  std::vector<double> avg(m, 0.0);
  if (B.fused()) {
    const uint32_t ns = uint32_t(std::min<uint64_t>(n, 4096));
    std::vector<unsigned long long> sums(m, 0);
    if (streamed) {
      for (uint32_t k = 0; k < ns; ++k) {
        const uint64_t r = ns >= n ? k : (uint64_t(k) * n) / ns;
        for (uint64_t c = 0; c < m; ++c) sums[c] += h_offs[r * m + c + 1] - h_offs[r * m + c];
      }
    } else {
      DevBuf<unsigned long long> d_sums(m, s);
      d_sums.zero();
      PO_LAUNCH(k_sample_col_bytes, grid_for(uint64_t(ns) * m, 256, 4), 256, 0, s, t.offsets, n,
                uint32_t(m), ns, d_sums.get());
      d2h_sync(sums.data(), d_sums.get(), (m) * sizeof(*d_sums.get()), s);
    }
    for (uint64_t c = 0; c < m; ++c) avg[c] = double(sums[c]) / double(std::max<uint32_t>(ns, 1));
  }
  B.set_lanes(avg);

  // Capacity. When every column sized for n distinct values fits a small
  // budget (about 48 B per cell), one chunk with exact worst-case tables;
  // otherwise a first chunk with room for all its rows to be new, then
  // tables sized from its distinct counts.
  const double worst = 48.0 * double(n) * double(m);
  bool exact_caps = worst <= 1e9;  // no driver query on the common path
  if (!exact_caps && worst <= 4e9) {
    size_t free_b = 0, total_b = 0;
    PO_CUDA(cudaMemGetInfo(&free_b, &total_b));
    exact_caps = worst <= 0.1 * double(free_b);
  }
  const uint64_t R0 = (exact_caps || n <= 131072) ? n : std::max<uint64_t>(65536, n / 16);
  B.reserve_all(exact_caps ? n : R0);

  if (!streamed) {
    const uint8_t* lim = t.arena + t.arena_bytes;
    B.run_chunk(t.arena, 0, lim, nullptr, nullptr, t.offsets, 0, R0, cid_mat);
    if (R0 < n) {
      // extrapolate each column's distinct count to the whole table
      for (uint32_t c = 0; c < m; ++c) {
        const double d0 = double(B.counts()[c]);
        const double est = d0 >= double(R0) ? double(n) : d0 + d0 / double(R0) * double(n - R0) * 1.1 + 1024.0;
        B.reserve(c, uint64_t(std::min(double(n), est)));
      }
      B.run_chunk(t.arena, 0, lim, nullptr, nullptr, t.offsets + R0 * m, R0, n, cid_mat);
    }
    out.val_arena = t.arena;
    out.val_bytes = t.arena_bytes;
  } else {
    // streamed: row chunks of at most kChunkBytes through two device buffers
    // (the copy of chunk k+1 overlaps the dictionary pass over chunk k); new
    // values are copied into a compact value arena after their chunk
    const uint64_t total_bytes = t.arena_bytes;
    const uint64_t kChunkBytes = std::max<uint64_t>(64ull << 20, std::min<uint64_t>(512ull << 20, total_bytes / 4));
    std::vector<std::pair<uint64_t, uint64_t>> chunks;  // row ranges
    {
      uint64_t r = 0;
      const uint64_t first_rows = R0;
      while (r < n) {
        uint64_t lo = r + 1, hi = std::min(n, chunks.empty() ? first_rows : n);
        // largest row end with bytes <= kChunkBytes (at least one row)
        const uint64_t b0 = h_offs[r * m];
        while (lo < hi) {
          const uint64_t mid = lo + (hi - lo + 1) / 2;
          if (h_offs[mid * m] - b0 <= kChunkBytes) lo = mid;
          else hi = mid - 1;
        }
        chunks.push_back({r, lo});
        r = lo;
      }
    }
    cudaStream_t cs = copy_stream();
    uint64_t max_rows = 0, max_bytes = 0;
    for (auto [a, b] : chunks) {
      max_rows = std::max(max_rows, b - a);
      max_bytes = std::max(max_bytes, h_offs[b * m] - h_offs[a * m]);
    }
    DevBuf<uint8_t> cbuf[2];
    DevBuf<uint64_t> obuf[2];
    cudaEvent_t copied[2], used[2];
    for (int b = 0; b < 2; ++b) {
      cbuf[b].alloc_auto(max_bytes + 64, s);
      obuf[b].alloc_auto(max_rows * m + 1, s);
      PO_CUDA(cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming));
      PO_CUDA(cudaEventCreateWithFlags(&used[b], cudaEventDisableTiming));
      PO_CUDA(cudaEventRecord(used[b], s));  // buffers allocated on s
    }
    struct EvGuard {
      cudaEvent_t* e;
      ~EvGuard() {
        for (int b = 0; b < 4; ++b) cudaEventDestroy(e[b]);
      }
    };
    cudaEvent_t evs[4] = {copied[0], copied[1], used[0], used[1]};
    EvGuard guard{evs};
    const bool pageable = host_pageable(t.h_arena) || host_pageable(h_offs);
    // pageable input: chunk k's bytes and offsets staged into pinned slot k%2
    // the slot is taken on the calling thread (it owns the slots and its
    // device is current); the returned task only copies host bytes
    auto stage = [&](size_t k) -> std::function<void()> {
      const int b = int(k & 1);
      const auto [a, e] = chunks[k];
      const uint64_t b0 = h_offs[a * m], b1 = h_offs[e * m];
      const size_t ob = ((e - a) * m + 1) * 8, ab = (b1 - b0 + 15) & ~size_t(15);
      uint8_t* dst = pinned_slot(b, ab + ob).p;
      const uint8_t* src = t.h_arena + b0;
      const uint64_t* so = h_offs + a * m;
      return [=] {
        parallel_copy(dst, src, b1 - b0);
        std::memcpy(dst + ab, so, ob);
      };
    };
    auto issue = [&](size_t k) {
      const int b = int(k & 1);
      const auto [a, e] = chunks[k];
      const uint64_t b0 = h_offs[a * m], b1 = h_offs[e * m];
      const size_t ob = ((e - a) * m + 1) * 8;
      PO_CUDA(cudaStreamWaitEvent(cs, used[b], 0));
      const uint8_t* src_a = t.h_arena + b0;
      const void* src_o = h_offs + a * m;
      if (pageable) {
        PinnedSlot& ps = g_slots.slot[b];
        src_a = ps.p;
        src_o = ps.p + ((b1 - b0 + 15) & ~size_t(15));
      }
      if (b1 > b0) PO_CUDA(cudaMemcpyAsync(cbuf[b].get(), src_a, b1 - b0, cudaMemcpyHostToDevice, cs));
      PO_CUDA(cudaMemcpyAsync(obuf[b].get(), src_o, ob, cudaMemcpyHostToDevice, cs));
      PO_CUDA(cudaEventRecord(copied[b], cs));
      if (pageable) {
        PinnedSlot& ps = g_slots.slot[b];
        PO_CUDA(cudaEventRecord(ps.done, cs));
        ps.pending = true;
      }
    };
    DevBuf<uint8_t> vals;
    uint64_t vals_cap = 0, vals_used = 0;
    std::vector<uint32_t> prev(m, 0);
    if (pageable) stage(0)();
    issue(0);
    for (size_t k = 0; k < chunks.size(); ++k) {
      const int b = int(k & 1);
      const auto [a, e] = chunks[k];
      const uint64_t b0 = h_offs[a * m], b1 = h_offs[e * m];
      // value arena room for every byte of this chunk being new
      if (vals_used + (b1 - b0) + 8 * (e - a) * m + 64 > vals_cap) {
        const uint64_t ncap = std::max<uint64_t>(vals_used + (b1 - b0) + 8 * (e - a) * m + 64,
                                                 vals_cap + vals_cap / 2);
        DevBuf<uint8_t> nv;
        nv.alloc_auto(ncap + 64, s);
        if (vals_used)
          PO_CUDA(cudaMemcpyAsync(nv.get(), vals.get(), vals_used, cudaMemcpyDeviceToDevice, s));
        vals = std::move(nv);
        vals_cap = ncap;
      }
      if (k > 0) {  // re-estimate the columns for the rest of the table
        const uint64_t done = a, left = n - a;
        for (uint32_t c = 0; c < m; ++c) {
          const double d = double(B.counts()[c]);
          const double rate = double(B.counts()[c] - prev[c]) / double(std::max<uint64_t>(1, chunks[k - 1].second - chunks[k - 1].first));
          (void)done;
          const double est = d + std::min(rate, 1.0) * double(std::min<uint64_t>(left, e - a)) * 1.1 + 1024.0;
          B.reserve(c, uint64_t(std::min(double(n), est)));
          prev[c] = B.counts()[c];
        }
      }
      PO_CUDA(cudaStreamWaitEvent(s, copied[b], 0));
      // next chunk: pinned input is copied now (overlapping this pass);
      // pageable input is staged by host threads meanwhile, copied after
      std::future<void> staging;
      if (k + 1 < chunks.size()) {
        if (pageable) staging = std::async(std::launch::async, stage(k + 1));
        else issue(k + 1);
      }
      const uint8_t* cb = cbuf[b].get();
      const uint8_t* clim = cb + (b1 - b0);
      const std::vector<uint32_t> before = B.counts();
      B.run_chunk(cb, b0, clim, vals.get(), vals.get() + vals_used, obuf[b].get(), a, e, cid_mat);
      // copy this chunk's new values into the value arena
      std::vector<uint32_t> seg_col, seg_id0;
      std::vector<uint64_t> seg_q0;
      uint64_t tot = 0;
      for (uint32_t c = 0; c < m; ++c)
        if (B.counts()[c] > before[c]) {
          seg_col.push_back(c);
          seg_id0.push_back(before[c]);
          seg_q0.push_back(tot);
          tot += B.counts()[c] - before[c];
        }
      if (tot) {
        auto d_sc = to_device(seg_col, s);
        auto d_si = to_device(seg_id0, s);
        auto d_sq = to_device(seg_q0, s);
        NewVals V{d_sc.get(), d_si.get(), d_sq.get(), uint32_t(seg_col.size()), B.d_cols()};
        DevBuf<uint64_t> sizes(tot + 1, s), pos(tot + 1, s);
        PO_LAUNCH(k_new_val_sizes, grid_for(tot, 256), 256, 0, s, V, tot, sizes.get());
        exclusive_scan_u64(sizes.get(), pos.get(), tot + 1, s);
        PO_LAUNCH(k_copy_new_vals, grid_for(tot * 32, 256), 256, 0, s, V, tot, pos.get(), vals_used,
                  cb, b0, clim, vals.get());
        uint64_t added = 0;
        PO_CUDA(cudaMemcpyAsync(&added, pos.get() + tot, 8, cudaMemcpyDeviceToHost, s));
        sync(s);
        vals_used += added;
      }
      PO_CUDA(cudaEventRecord(used[b], s));
      if (staging.valid()) {
        staging.get();
        issue(k + 1);
      }
    }
    out.own_vals = std::move(vals);
    out.val_arena = out.own_vals.get();
    out.val_bytes = vals_used;
    if (!out.val_arena) {  // every value empty
      out.own_vals.alloc(1, s);
      out.val_arena = out.own_vals.get();
    }
  }

  // dense per-distinct arrays (compaction order)
  for (uint32_t c = 0; c < m; ++c) {
    out.card[c] = B.counts()[c];
    out.colbase[c + 1] = out.colbase[c] + out.card[c];
  }
  const uint64_t D = out.colbase[m];
  out.D = D;
  out.d_colbase = to_device(out.colbase, s);
  out.val_off.alloc_auto(D, s);
  out.val_len.alloc_auto(D, s);
  out.rep_row.alloc_auto(D, s);
  out.d_col.alloc_auto(D, s);
  PO_LAUNCH(k_gather_dict, grid_for(D, 256), 256, 0, s, B.d_cols(), out.d_colbase.get(), uint32_t(m),
            D, out.val_off.get(), out.val_len.get(), out.rep_row.get(), out.d_col.get());
}

}  // namespace po
