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
#include <cstdlib>
#include <string>

#include "internal.cuh"

namespace po {

namespace {

constexpr uint32_t kEmptyRep = 0xFFFFFFFFu;

// Reader of an arbitrarily aligned byte string as little-endian 8-byte words
// from either shared memory (staged tile) or global memory, loading only
// 8-byte-aligned words that start before `lim`.
template <bool kShared>
struct Words {
  const uint64_t* p;
  const uint64_t* lim;
  uint32_t sh;
  uint64_t cur;
  __device__ __forceinline__ static uint64_t ld(const uint64_t* q) {
    if constexpr (kShared) return *q;
    else return __ldg(q);
  }
  __device__ __forceinline__ Words(const uint8_t* a, const uint8_t* limit) {
    const uintptr_t ad = reinterpret_cast<uintptr_t>(a);
    p = reinterpret_cast<const uint64_t*>(ad & ~uintptr_t(7));
    lim = reinterpret_cast<const uint64_t*>((reinterpret_cast<uintptr_t>(limit) + 7) & ~uintptr_t(7));
    sh = uint32_t(ad & 7) * 8;
    cur = p < lim ? ld(p) : 0;
  }
  __device__ __forceinline__ uint64_t next() {
    const uint64_t* q = p + 1;
    const uint64_t nxt = q < lim ? ld(q) : 0;
    const uint64_t w = sh ? ((cur >> sh) | (nxt << (64 - sh))) : cur;
    cur = nxt;
    p = q;
    return w;
  }
};

template <bool kShared>
__device__ __forceinline__ uint64_t hash_cell(const uint8_t* a, uint64_t len, const uint8_t* limit) {
  uint64_t sum = 0;
  if (len) {
    Words<kShared> rd(a, limit);
    uint64_t k = 0;
    for (; 8 * (k + 1) <= len; ++k) sum += word_term(rd.next(), k);
    if (8 * k < len) sum += word_term(mask_low_bytes(rd.next(), uint32_t(len - 8 * k)), k);
  }
  return hash_finish(sum, len);
}

// Cell (shared or global) vs representative (global), 4 words per step so
// several independent loads of the representative are in flight.
template <bool kShared>
__device__ __forceinline__ bool equal_cell_rep(const uint8_t* a, const uint8_t* a_lim,
                                               const uint8_t* b, const uint8_t* b_lim,
                                               uint64_t len) {
  Words<kShared> ra(a, a_lim);
  Words<false> rb(b, b_lim);
  uint64_t left = len;
  while (left >= 32) {
    const uint64_t b0 = rb.next(), b1 = rb.next(), b2 = rb.next(), b3 = rb.next();
    const uint64_t a0 = ra.next(), a1 = ra.next(), a2 = ra.next(), a3 = ra.next();
    if ((a0 ^ b0) | (a1 ^ b1) | (a2 ^ b2) | (a3 ^ b3)) return false;
    left -= 32;
  }
  while (left) {
    const uint32_t take = left >= 8 ? 8u : uint32_t(left);
    if (mask_low_bytes(ra.next(), take) != mask_low_bytes(rb.next(), take)) return false;
    left -= take;
  }
  return true;
}

// Probe column c's table for the cell's value: claim an empty slot (the cell
// becomes the representative) or find the slot whose representative has the
// same bytes. Equal hashes with different bytes keep probing (exact).
// Representative locator stored next to each claimed slot: arena offset
// (high 40 bits) and byte length (low 24 bits; kLongRep = look it up).
constexpr uint64_t kLongRep = 0xFFFFFF;
__device__ __forceinline__ uint64_t pack_rep(uint64_t off, uint64_t len) {
  return (off << 24) | (len < kLongRep ? len : kLongRep);
}

// Claims slot `slot` for the cell (representative) — publishes the locator
// before the row (readers spin on the row with acquire semantics).
__device__ __forceinline__ void publish_rep(uint32_t* R, unsigned long long* RO, uint64_t slot,
                                            uint32_t row, uint64_t off, uint64_t len) {
  RO[slot] = pack_rep(off, len);
  __threadfence();
  atomicExch(&R[slot], row);
}

__device__ __forceinline__ void read_rep(const uint32_t* R, const unsigned long long* RO,
                                         uint64_t slot, uint32_t m, uint32_t c,
                                         const uint64_t* __restrict__ offsets, uint64_t& off,
                                         uint64_t& len) {
  uint32_t rep;
  while ((rep = ld_acquire_u32(&R[slot])) == kEmptyRep) {
  }
  const uint64_t pk = RO[slot];
  off = pk >> 24;
  len = pk & kLongRep;
  if (len == kLongRep) {
    const uint64_t j = uint64_t(rep) * m + c;
    len = offsets[j + 1] - offsets[j];
  }
}

// Probe column c's table for the cell's value: claim an empty slot (the cell
// becomes the representative) or find the slot whose representative has the
// same bytes. Equal hashes with different bytes keep probing (exact).
template <bool kShared>
__device__ __forceinline__ uint64_t probe_insert(unsigned long long* K, uint32_t* R,
                                                 unsigned long long* RO, uint64_t cap, uint64_t h,
                                                 uint64_t slot, uint32_t row, uint32_t c,
                                                 uint32_t m, uint64_t o0, const uint8_t* cell,
                                                 const uint8_t* cell_lim, uint64_t len,
                                                 const uint8_t* arena, const uint8_t* arena_end,
                                                 const uint64_t* __restrict__ offsets) {
  for (;;) {
    unsigned long long k = K[slot];
    if (k == 0) {
      const unsigned long long prev = atomicCAS(&K[slot], 0ull, (unsigned long long)h);
      if (prev == 0) {
        publish_rep(R, RO, slot, row, o0, len);
        return slot;
      }
      k = prev;
    }
    if (k == h) {
      uint64_t q0, ql;
      read_rep(R, RO, slot, m, c, offsets, q0, ql);
      if (ql == len && equal_cell_rep<kShared>(cell, cell_lim, arena + q0, arena_end, len))
        return slot;
    }
    slot = (slot + 1) & (cap - 1);
  }
}

// 8 bytes of a staged tile at byte offset `off` (two aligned shared loads).
__device__ __forceinline__ uint64_t smem_word(const uint64_t* s64, uint32_t off) {
  const uint32_t q = off >> 3, sh = (off & 7) * 8;
  const uint64_t w0 = s64[q];
  return sh ? ((w0 >> sh) | (s64[q + 1] << (64 - sh))) : w0;
}

constexpr uint32_t kDictBlock = 256;

// ---------------------------------------------------------------------------
// K1 cell_scan: tile-staged hashing of every cell.
// A block takes a tile of whole rows (rows_per_tile * m <= 256 cells, one per
// thread); one elected thread streams the tile's 16-byte-aligned byte range
// into shared memory with a TMA bulk copy, double-buffered so the next tile
// is in flight while this one is hashed. Threads take the tile's cells in
// column-major order, so the 32 lanes of a warp hash cells of the same
// column (similar lengths: little divergence) out of shared memory. Output:
// the 64-bit hash of every cell. A tile larger than a staging buffer is
// hashed from global memory (same hash).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kDictBlock) k_cell_hash(
    const uint8_t* __restrict__ arena, const uint8_t* arena_end,
    const uint64_t* __restrict__ offsets, uint64_t total, uint32_t m, uint32_t rows_per_tile,
    uint32_t stage_bytes, uint64_t hash_mask, unsigned long long* __restrict__ hashes) {
  extern __shared__ __align__(128) uint8_t sbuf_all[];
  __shared__ __align__(8) uint64_t s_bar[2];
  const uint32_t tile = rows_per_tile * m;  // cells per tile
  const uint32_t buf_bytes = (stage_bytes + 64 + 127) & ~127u;
  const uint64_t ntiles = (total + tile - 1) / tile;
  const uint32_t tid = threadIdx.x;
  auto tile_range = [&](uint64_t t, uintptr_t& a0, uintptr_t& b1) {
    const uint64_t j0 = t * tile;
    const uint64_t j1 = j0 + tile < total ? j0 + tile : total;
    a0 = reinterpret_cast<uintptr_t>(arena + offsets[j0]) & ~uintptr_t(15);
    b1 = (reinterpret_cast<uintptr_t>(arena + offsets[j1]) + 15) & ~uintptr_t(15);
  };
  auto issue = [&](uint64_t t, int b) {
    uintptr_t a0, b1;
    tile_range(t, a0, b1);
    if (b1 - a0 > stage_bytes) return;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&s_bar[b], uint32_t(b1 - a0));
    bulk_g2s(sbuf_all + b * buf_bytes, reinterpret_cast<const void*>(a0), uint32_t(b1 - a0),
             &s_bar[b]);
  };
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0 && blockIdx.x < ntiles) issue(blockIdx.x, 0);
  // column-major position of this thread inside a tile
  const uint32_t col = tid / rows_per_tile, row = tid - col * rows_per_tile;
  const bool active = tid < tile;
  uint32_t uses[2] = {0u, 0u};
  uint32_t kiter = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++kiter) {
    const int bsel = int(kiter & 1);
    const uint8_t* sb = sbuf_all + bsel * buf_bytes;
    uintptr_t gA0, gB1;
    tile_range(t, gA0, gB1);
    const bool staged = gB1 - gA0 <= stage_bytes;
    if (tid == 0 && t + gridDim.x < ntiles) issue(t + gridDim.x, bsel ^ 1);
    const uint64_t i = t * tile + uint64_t(row) * m + col;
    const bool mine = active && i < total;
    const uint64_t o0 = mine ? offsets[i] : 0;
    const uint64_t len = mine ? offsets[i + 1] - o0 : 0;
    if (staged) {
      mbar_wait(&s_bar[bsel], uses[bsel] & 1u);
      ++uses[bsel];
      if (mine) {
        const uint8_t* cell = sb + (reinterpret_cast<uintptr_t>(arena + o0) - gA0);
        const uint64_t h = hash_cell<true>(cell, len, sb + (gB1 - gA0) + 16) & hash_mask;
        hashes[i] = h ? h : 1;
      }
    } else if (mine) {
      const uint64_t h = hash_cell<false>(arena + o0, len, arena_end) & hash_mask;
      hashes[i] = h ? h : 1;
    }
    __syncthreads();  // buffer bsel is refilled by the next-but-one issue
  }
}

// K1 cell_scan (segment-parallel, TMA-staged): the default hashing kernel.
// A block streams tiles of T consecutive cells (row-major: a contiguous byte
// range of the arena) into shared memory with one bulk copy per tile,
// double-buffered so the next tile's copy overlaps this tile's hashing. The
// work inside a tile is split into 64-byte segments of cells (a cell of len
// bytes has max(1, ceil(len/64)) segments), so long and short cells balance
// across threads: each thread hashes whole segments out of shared memory and
// adds its partial word sum to the cell's accumulator (shared atomics; the
// hash is a sum of per-word terms, so the order does not matter), then one
// thread per cell finishes the hash. The arena is read exactly once, as
// large aligned bulk copies. A tile whose byte range exceeds the staging
// buffer (or ends past the arena) is hashed from global memory with the
// same segment split.
constexpr uint32_t kSegBlock = 256;
constexpr uint32_t kSegMaxCells = 1023;
constexpr uint32_t kSegQ = 4;  // offsets held per thread: (kSegMaxCells + 1) / kSegBlock
constexpr uint32_t kSegStages = 4;

__device__ __forceinline__ uint64_t smem_word8(const uint8_t* base, uint32_t off) {
  const uint64_t* s64 = reinterpret_cast<const uint64_t*>(base);
  const uint32_t q = off >> 3, sh = (off & 7) * 8;
  const uint64_t w0 = s64[q];
  return sh ? ((w0 >> sh) | (s64[q + 1] << (64 - sh))) : w0;
}

template <uint32_t G>  // lanes per cell: 8, 16 or 32
__global__ void __launch_bounds__(kSegBlock, 3) k_cell_hash_seg(
    const uint8_t* __restrict__ arena, const uint8_t* arena_end,
    const uint64_t* __restrict__ offsets, uint64_t n, uint32_t m, uint32_t R,
    uint32_t stage_bytes, uint64_t hash_mask, unsigned long long* __restrict__ hashes) {
  extern __shared__ __align__(128) uint8_t sbuf_all[];
  __shared__ __align__(8) uint64_t s_bar[kSegStages];
  __shared__ uint64_t s_off[kSegMaxCells + 1];
  const uint32_t buf_bytes = stage_bytes + 128;  // slack: 8-byte reads past the data
  const uint64_t total = n * m;
  const uint32_t T = R * m;  // cells per tile: R whole rows
  const uint64_t ntiles = (n + R - 1) / R;
  const uint32_t tid = threadIdx.x;
  const uint32_t gl = tid % G;  // lane within its group of G lanes (one cell)
  const uintptr_t end_addr = reinterpret_cast<uintptr_t>(arena_end);
  auto cells_of = [&](uint64_t t) -> uint32_t {
    const uint64_t j0 = t * T;
    return uint32_t((j0 + T < total ? j0 + T : total) - j0);
  };
  auto stageable = [&](uintptr_t a0, uintptr_t b1) {
    return b1 > a0 && b1 - a0 <= stage_bytes && b1 <= end_addr;  // never read past the arena
  };
  auto issue = [&](uint64_t t, int b) {
    const uint64_t j0 = t * T;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(arena + offsets[j0]) & ~uintptr_t(15);
    const uintptr_t b1 =
        (reinterpret_cast<uintptr_t>(arena + offsets[j0 + cells_of(t)]) + 15) & ~uintptr_t(15);
    if (!stageable(a0, b1)) return;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&s_bar[b], uint32_t(b1 - a0));
    bulk_g2s(sbuf_all + b * buf_bytes, reinterpret_cast<const void*>(a0), uint32_t(b1 - a0),
             &s_bar[b]);
  };
  auto load_offs = [&](uint64_t t, uint64_t* r) {
    const uint64_t j0 = t * T;
    const uint32_t nc = cells_of(t);
#pragma unroll
    for (uint32_t q = 0; q < kSegQ; ++q) {
      const uint32_t c = tid + q * kSegBlock;
      r[q] = c <= nc ? __ldg(offsets + j0 + c) : 0;
    }
  };
  if (tid == 0) {
    for (uint32_t b = 0; b < kSegStages; ++b) mbar_init(&s_bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t roff[kSegQ];
  if (blockIdx.x < ntiles) {  // ring of kSegStages buffers: stages-1 tiles ahead
    if (tid == 0)
      for (uint32_t b = 0; b + 1 < kSegStages; ++b)
        if (blockIdx.x + uint64_t(b) * gridDim.x < ntiles) issue(blockIdx.x + uint64_t(b) * gridDim.x, int(b));
    load_offs(blockIdx.x, roff);
  }
  uint32_t parity = 0;  // bit b: phase of buffer b
  uint32_t kiter = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++kiter) {
    const int bsel = int(kiter % kSegStages);
    const uint8_t* sb = sbuf_all + bsel * buf_bytes;
    const uint64_t j0 = t * T;
    const uint32_t nc = cells_of(t);
    const uint32_t rows = nc / m;
#pragma unroll
    for (uint32_t q = 0; q < kSegQ; ++q) {
      const uint32_t c = tid + q * kSegBlock;
      if (c <= nc) s_off[c] = roff[q];
    }
    __syncthreads();
    const uintptr_t gA0 = reinterpret_cast<uintptr_t>(arena + s_off[0]) & ~uintptr_t(15);
    const uintptr_t gB1 = (reinterpret_cast<uintptr_t>(arena + s_off[nc]) + 15) & ~uintptr_t(15);
    const bool staged = stageable(gA0, gB1);
    if (tid == 0) {  // refill the buffer freed by the previous tile
      const uint64_t ahead = t + uint64_t(kSegStages - 1) * gridDim.x;
      if (ahead < ntiles) issue(ahead, int((kiter + kSegStages - 1) % kSegStages));
    }
    if (t + gridDim.x < ntiles) load_offs(t + gridDim.x, roff);  // next tile's offsets
    if (staged) {
      mbar_wait(&s_bar[bsel], (parity >> bsel) & 1u);
      parity ^= 1u << bsel;
    }
    // cells in column-major order (the groups of a warp take consecutive rows
    // of one column: similar lengths); a group walks its cell 8*G bytes at a
    // time, lane gl taking words gl, gl+G, ...
    // warp-uniform loop: the shuffles below need every lane of the warp
    for (uint32_t kb = (tid >> 5) * (32 / G); kb < nc; kb += kSegBlock / G) {
      const uint32_t k = kb + (tid & 31) / G;
      const bool valid = k < nc;
      uint32_t ci = 0;
      uint64_t len = 0;
      unsigned long long sum = 0;
      if (valid) {
        const uint32_t col = k / rows, row = k - col * rows;
        ci = row * m + col;
        const uint64_t o0 = s_off[ci];
        len = s_off[ci + 1] - o0;
        const uint8_t* cell = arena + o0;
        const uint32_t sbase = uint32_t(reinterpret_cast<uintptr_t>(cell) - gA0);
        for (uint64_t b = 8 * gl; b < len; b += 8 * G) {
          const uint32_t take = len - b >= 8 ? 8u : uint32_t(len - b);
          const uint64_t x = staged ? smem_word8(sb, sbase + uint32_t(b))
                                    : load8_unaligned(cell + b, arena_end);
          sum += word_term(mask_low_bytes(x, take), b >> 3);
        }
      }
#pragma unroll
      for (uint32_t d = G / 2; d > 0; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
      if (valid && gl == 0) {
        const uint64_t h = hash_finish(sum, len) & hash_mask;
        hashes[j0 + ci] = h ? h : 1;
      }
    }
    __syncthreads();  // s_off and buffer bsel are reused
  }
}

// K1 cell_scan (direct): one thread per cell, warps assigned column-major
// over tiles of 32 rows so the 32 lanes of a warp hash cells of the same
// column (similar lengths: converged loops). Each step covers 4 words of the
// cell with 4 independent aligned 8-byte loads (the fifth aligned word a
// step needs is the previous step's last, kept in a register), so every
// thread keeps several loads in flight without shared-memory staging or
// block barriers.
__global__ void __launch_bounds__(256) k_cell_hash_cols(
    const uint8_t* __restrict__ arena, const uint8_t* arena_end,
    const uint64_t* __restrict__ offsets, uint64_t n, uint32_t m, uint64_t hash_mask,
    unsigned long long* __restrict__ hashes) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t ntiles = (n + 31) / 32;
  const uint64_t* lim =
      reinterpret_cast<const uint64_t*>((reinterpret_cast<uintptr_t>(arena_end) + 7) & ~uintptr_t(7));
  for (uint64_t tile = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; tile < ntiles;
       tile += (uint64_t(gridDim.x) * blockDim.x) >> 5)
  for (uint32_t c = 0; c < m; ++c) {
    // the warp walks its 32 rows column by column: the bytes of one row are
    // read by the same lane in consecutive iterations (boundary sectors hit L1)
    const uint64_t r = tile * 32 + lane;
    if (r >= n) continue;
    const uint64_t i = r * m + c;
    const uint64_t o0 = offsets[i], len = offsets[i + 1] - o0;
    const uintptr_t ad = reinterpret_cast<uintptr_t>(arena + o0);
    const uint64_t* p = reinterpret_cast<const uint64_t*>(ad & ~uintptr_t(7));
    const uint32_t sh = uint32_t(ad & 7) * 8;
    const uint64_t words = (len + 7) / 8;
    uint64_t sum = 0;
    // the last aligned word of a step is the first of the next: carried in a
    // register (four loads per four words)
    uint64_t carry = (words && p < lim) ? __ldg(p) : 0;
    for (uint64_t k = 0; k < words; k += 4) {
      uint64_t w[5];
      w[0] = carry;
#pragma unroll
      for (int u = 1; u < 5; ++u) w[u] = (p + k + u < lim) ? __ldg(p + k + u) : 0;
      carry = w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t kk = k + u;
        if (kk < words) {
          uint64_t x = sh ? ((w[u] >> sh) | (w[u + 1] << (64 - sh))) : w[u];
          const uint64_t rem = len - 8 * kk;
          if (rem < 8) x = mask_low_bytes(x, uint32_t(rem));
          sum += word_term(x, kk);
        }
      }
    }
    const uint64_t h = hash_finish(sum, len) & hash_mask;
    hashes[i] = h ? h : 1;
  }
}


// ---------------------------------------------------------------------------
// K2a probe: one thread per cell, full occupancy, no barriers. The first
// cell to reach an empty slot claims it and records itself as the value's
// representative (row + arena locator); a cell meeting a slot with its hash
// is tentatively that slot's value (verified on the bytes by K2b). Claims
// and records become visible to K2b at the kernel boundary, so no fences or
// spin-waits are needed here.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_dict_probe(
    const unsigned long long* __restrict__ hashes, const uint64_t* __restrict__ offsets,
    uint64_t total, uint32_t m, uint64_t cap, unsigned long long* keys, uint32_t* reps,
    unsigned long long* repoffs, uint32_t* slot_of_cell) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / m;
    const uint32_t c = uint32_t(i - r * m);
    const unsigned long long h = hashes[i];
    unsigned long long* K = keys + uint64_t(c) * cap;
    uint64_t slot = h & (cap - 1);
    for (;;) {
      unsigned long long k = K[slot];
      if (k == 0) {
        const unsigned long long prev = atomicCAS(&K[slot], 0ull, h);
        if (prev == 0) {
          const uint64_t o0 = offsets[i];
          reps[uint64_t(c) * cap + slot] = uint32_t(r);
          repoffs[uint64_t(c) * cap + slot] = pack_rep(o0, offsets[i + 1] - o0);
          break;
        }
        k = prev;
      }
      if (k == h) break;
      slot = (slot + 1) & (cap - 1);
    }
    slot_of_cell[i] = uint32_t(slot);
  }
}

// ---------------------------------------------------------------------------
// K2b verify: every cell whose slot is owned by another row is compared
// byte for byte with the representative (4 words of each string per step,
// 4 aligned loads each). A mismatch — two different strings with the same
// 64-bit hash — flags the cell for K2c.
// ---------------------------------------------------------------------------
// Unaligned 4-word step of a byte string.
struct Step4 {
  uint64_t w[4];
};
// Four words of a byte string from five aligned words, the first passed in
// (the previous step's last one) and the new last one handed back: four
// loads per step.
__device__ __forceinline__ Step4 load_step4_carry(const uint64_t* p, uint32_t sh,
                                                  const uint64_t* lim, uint64_t& carry) {
  uint64_t a[5];
  a[0] = carry;
#pragma unroll
  for (int u = 1; u < 5; ++u) a[u] = (p + u < lim) ? __ldg(p + u) : 0;
  carry = a[4];
  Step4 r;
#pragma unroll
  for (int u = 0; u < 4; ++u) r.w[u] = sh ? ((a[u] >> sh) | (a[u + 1] << (64 - sh))) : a[u];
  return r;
}

__global__ void __launch_bounds__(256) k_dict_verify(
    const uint8_t* __restrict__ arena, const uint8_t* arena_end,
    const uint64_t* __restrict__ offsets, uint64_t n, uint32_t m, uint64_t cap,
    const uint32_t* __restrict__ reps, const unsigned long long* __restrict__ repoffs,
    const uint32_t* __restrict__ slot_of_cell, uint32_t* collided, uint32_t* n_collided) {
  // Warps take 32 rows of one column (similar lengths); every lane compares
  // its own cell with the representative, 4 words per step with all 8 loads
  // in flight.
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t ntiles = (n + 31) / 32;
  const uint64_t* lim =
      reinterpret_cast<const uint64_t*>((reinterpret_cast<uintptr_t>(arena_end) + 7) & ~uintptr_t(7));
  for (uint64_t tile = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; tile < ntiles;
       tile += (uint64_t(gridDim.x) * blockDim.x) >> 5)
  for (uint32_t c = 0; c < m; ++c) {
    const uint64_t r = tile * 32 + lane;
    if (r >= n) continue;
    const uint64_t i = r * m + c;
    const uint64_t sidx = uint64_t(c) * cap + slot_of_cell[i];
    const uint32_t rep = reps[sidx];
    if (rep == uint32_t(r)) continue;  // the representative itself
    const uint64_t o0 = offsets[i], len = offsets[i + 1] - o0;
    const uint64_t pk = repoffs[sidx];
    const uint64_t q0 = pk >> 24;
    uint64_t ql = pk & kLongRep;
    if (ql == kLongRep) {
      const uint64_t j = uint64_t(rep) * m + c;
      ql = offsets[j + 1] - offsets[j];
    }
    bool eq = ql == len;
    if (eq && len) {
      const uintptr_t aa = reinterpret_cast<uintptr_t>(arena + o0);
      const uintptr_t bb = reinterpret_cast<uintptr_t>(arena + q0);
      const uint64_t* pa = reinterpret_cast<const uint64_t*>(aa & ~uintptr_t(7));
      const uint64_t* pb = reinterpret_cast<const uint64_t*>(bb & ~uintptr_t(7));
      const uint32_t sa = uint32_t(aa & 7) * 8, sb = uint32_t(bb & 7) * 8;
      const uint64_t words = (len + 7) / 8;
      uint64_t ca = pa < lim ? __ldg(pa) : 0, cb = pb < lim ? __ldg(pb) : 0;
      for (uint64_t k = 0; k < words && eq; k += 4) {
        const Step4 x = load_step4_carry(pa + k, sa, lim, ca);
        const Step4 y = load_step4_carry(pb + k, sb, lim, cb);
        uint64_t d = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t kk = k + u;
          if (kk < words) {
            const uint64_t rem = len - 8 * kk;
            d |= mask_low_bytes(x.w[u] ^ y.w[u], rem >= 8 ? 8u : uint32_t(rem));
          }
        }
        eq = d == 0;
      }
    }
    if (!eq) collided[atomicAdd(n_collided, 1u)] = uint32_t(i);
  }
}

// ---------------------------------------------------------------------------
// K2c collision fix-up (rare path): a cell whose hash slot belongs to a
// different string keeps probing past that slot with byte verification,
// claiming or joining slots with the publish/acquire protocol (several
// colliding cells of the same string may race here).
// ---------------------------------------------------------------------------
__global__ void k_dict_fixup(const uint8_t* __restrict__ arena, const uint8_t* arena_end,
                             const uint64_t* __restrict__ offsets, uint32_t m, uint64_t cap,
                             const unsigned long long* __restrict__ hashes,
                             unsigned long long* keys, uint32_t* reps, unsigned long long* repoffs,
                             const uint32_t* collided, const uint32_t* n_collided_dev,
                             uint32_t* slot_of_cell) {
  const uint32_t n_collided = *n_collided_dev;  // read on the device: no host round trip
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n_collided;
       q += gridDim.x * blockDim.x) {
    const uint64_t i = collided[q];
    const uint64_t r = i / m;
    const uint32_t c = uint32_t(i - r * m);
    const uint64_t o0 = offsets[i], len = offsets[i + 1] - o0;
    const uint64_t base = uint64_t(c) * cap;
    const uint64_t slot = probe_insert<false>(
        keys + base, reps + base, repoffs + base, cap, hashes[i], (slot_of_cell[i] + 1) & (cap - 1),
        uint32_t(r), c, m, o0, arena + o0, arena_end, len, arena, arena_end, offsets);
    slot_of_cell[i] = uint32_t(slot);
  }
}

// Occupied dictionary slots of every column, compacted per column into
// sel[c*cap ..] (any order: the rank sort orders them; unranked and
// equality-only ids use it only as identity). A block takes a chunk of
// kCompactChunk slots of one column (cap is a power of two >= 64; chunks never
// straddle columns), counts its occupied slots and reserves them with ONE
// atomic.
constexpr uint32_t kCompactChunk = 4096;
__global__ void __launch_bounds__(256) k_compact_slots(const unsigned long long* __restrict__ keys,
                                                       uint64_t cap, uint64_t total, uint32_t* sel,
                                                       int* count) {
  __shared__ int s_warp[8];
  __shared__ int s_base;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t chunk = cap < kCompactChunk ? cap : kCompactChunk;
  if (chunk == kCompactChunk) {
    // one coalesced pass: thread t owns slots c0 + u*256 + t (u < 16) as a
    // bit mask, a block scan of the per-thread counts places them
    typedef cub::BlockScan<int, 256> BS;
    __shared__ typename BS::TempStorage ts;
    for (uint64_t c0 = blockIdx.x * chunk; c0 < total; c0 += uint64_t(gridDim.x) * chunk) {
      const uint64_t col = c0 / cap;
      uint32_t occ = 0;
#pragma unroll
      for (int u = 0; u < int(kCompactChunk / 256); ++u)
        occ |= uint32_t(keys[c0 + u * 256 + threadIdx.x] != 0) << u;
      int before = 0, tot = 0;
      BS(ts).ExclusiveSum(__popc(occ), before, tot);
      if (threadIdx.x == 0) s_base = tot ? atomicAdd(&count[col], tot) : 0;
      __syncthreads();
      uint32_t* out = sel + col * cap + s_base + before;
      const uint32_t rel0 = uint32_t(c0 - col * cap) + threadIdx.x;
      for (int u = 0; occ; ++u, occ >>= 1)
        if (occ & 1u) *out++ = rel0 + uint32_t(u) * 256u;
      __syncthreads();  // s_base and the scan storage are reused
    }
    return;
  }
  for (uint64_t c0 = blockIdx.x * chunk; c0 < total; c0 += uint64_t(gridDim.x) * chunk) {
    const uint64_t col = c0 / cap;
    int mine = 0;
    for (uint64_t i = c0 + threadIdx.x; i < c0 + chunk; i += 256) mine += keys[i] != 0;
    for (int d = 16; d > 0; d >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, d);
    if (lane == 0) s_warp[wid] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < 8; ++w) t += s_warp[w];
      s_base = t ? atomicAdd(&count[col], t) : 0;
    }
    __syncthreads();
    int base = s_base;
    // ordered write: 256 slots per step, block-wide exclusive prefix of the step
    for (uint64_t b = c0; b < c0 + chunk; b += 256) {
      const bool occ = b + threadIdx.x < c0 + chunk && keys[b + threadIdx.x] != 0;
      const unsigned bal = __ballot_sync(0xffffffffu, occ);
      if (lane == 0) s_warp[wid] = __popc(bal);
      __syncthreads();
      int before = 0, step = 0;
      for (int w = 0; w < 8; ++w) {
        before += w < int(wid) ? s_warp[w] : 0;
        step += s_warp[w];
      }
      if (occ)
        sel[col * cap + base + before + __popc(bal & ((1u << lane) - 1))] = uint32_t(b + threadIdx.x - col * cap);
      base += step;
      __syncthreads();
    }
  }
}

__global__ void k_iota_pos(uint32_t* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    a[i] = uint32_t(i);
}

// Items of the ranked columns only: item k -> distinct index d (the ranked
// columns' d-ranges, rbase[j] .. + (rpre[j+1] - rpre[j]), concatenated).
__global__ void k_ranked_items(const uint64_t* rbase, const uint64_t* rpre, uint32_t nr,
                               uint64_t total, const uint32_t* d_row, const uint32_t* d_col,
                               uint32_t* sub_d, uint32_t* sub_row, uint32_t* sub_col) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t j = 0;
    while (j + 1 < nr && rpre[j + 1] <= k) ++j;
    const uint64_t d = rbase[j] + (k - rpre[j]);
    sub_d[k] = uint32_t(d);
    sub_row[k] = d_row[d];
    sub_col[k] = d_col[d];
  }
}

__global__ void k_scatter_sub(const uint32_t* sub_d, const uint32_t* sub_pos, uint64_t total,
                              uint32_t* pos) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x)
    pos[sub_d[k]] = sub_pos[k];
}


// Per distinct value d (column-major dictionary order): its column (binary
// search over colbase), its slot and its representative row; one launch for
// every column.
__global__ void k_distinct_info(const uint32_t* stage_sel, uint64_t D, const uint64_t* colbase,
                                uint32_t m, uint64_t cap, const uint32_t* reps, uint32_t* sel_slot,
                                uint32_t* d_col, uint32_t* d_row) {
  for (uint64_t d = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; d < D;
       d += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t lo = 0, hi = m;  // last c with colbase[c] <= d
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (colbase[mid] <= d) lo = mid;
      else hi = mid;
    }
    const uint32_t c = lo;
    const uint32_t slot = stage_sel[uint64_t(c) * cap + (d - colbase[c])];
    sel_slot[d] = slot;
    d_col[d] = c;
    d_row[d] = reps[uint64_t(c) * cap + slot];
  }
}


// pos[d] (escaped order) -> vid; scatter representative row / column into
// vid order.
__global__ void k_scatter_pos(const uint32_t* pos_of, const uint32_t* d_col, const uint32_t* d_row,
                              const uint32_t* sel_slot, const uint64_t* colbase, uint64_t D,
                              uint64_t cap, uint32_t* slot2vid, uint32_t* row_by_pos,
                              uint32_t* col_by_pos) {
  for (uint64_t d = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; d < D;
       d += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t p = pos_of[d];
    const uint32_t c = d_col[d];
    slot2vid[uint64_t(c) * cap + sel_slot[d]] = uint32_t(p - colbase[c]);
    row_by_pos[p] = d_row[d];
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
            uint32_t hash_bits_debug, bool ordered, bool rank_unique) {
  e.n = t.n;
  e.m = t.m;
  e.arena = t.arena;
  e.offsets = t.offsets;
  e.arena_bytes = t.arena_bytes;
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

  // the large transient tables come from the block cache (common.cuh)
  DevBuf<unsigned long long> keys;
  keys.alloc_cached(m * cap, s);
  keys.zero();
  DevBuf<uint32_t> reps;
  reps.alloc_cached(m * cap, s);
  reps.fill_bytes(0xFF);
  DevBuf<unsigned long long> repoffs;
  repoffs.alloc_cached(m * cap, s);
  DevBuf<uint32_t> slot_of_cell;
  slot_of_cell.alloc_cached(cells, s);
  uint64_t hmask = hash_bits_debug >= 64 ? ~uint64_t(0) : ((uint64_t(1) << hash_bits_debug) - 1);
  {
    // K1: hash every cell. Tiles of whole rows sized so a typical tile uses
    // about 60% of a staging buffer.
    // 32 rows per tile when a row has <= 8 cells: each warp then hashes 32
    // cells of ONE column (similar lengths, converged loops).
    const double row_bytes = double(t.arena_bytes) / double(n);
    uint32_t rows_per_tile = m <= kDictBlock / 32 ? 32u : std::max<uint32_t>(1, kDictBlock / uint32_t(m));
    uint32_t stage = 32 * 1024;
    while (stage < 96 * 1024 && row_bytes * rows_per_tile > stage * 0.6) stage += 16 * 1024;
    while (rows_per_tile > 1 && row_bytes * rows_per_tile > stage * 0.6) rows_per_tile >>= 1;
    const uint32_t smem = 2 * ((stage + 64 + 127) & ~127u);
    static int attr_set = 0;
    if (attr_set < int(smem)) {
      PO_CUDA(cudaFuncSetAttribute(k_cell_hash, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
      attr_set = int(smem);
    }
    DevBuf<unsigned long long> hashes;
    hashes.alloc_cached(cells, s);
    // cols (default) | seg (TMA ring, group per cell) | tile (TMA, thread per cell)
    const char* hk = std::getenv("PO_HASH_KERNEL");
    const std::string hsel = hk && *hk ? hk : "cols";
    if (hsel == "seg" && m <= kSegMaxCells) {
      const double row_bytes = double(t.arena_bytes) / double(n);
      const uint32_t sstage = 16 * 1024;
      uint32_t R = uint32_t(std::max(1.0, 0.6 * sstage / std::max(row_bytes, 1.0)));
      R = std::min<uint32_t>(R, kSegMaxCells / uint32_t(m));
      R = std::max<uint32_t>(R, 1);
      const uint32_t ssmem = kSegStages * (sstage + 128);
      static bool seg_attr = false;
      if (!seg_attr) {
        PO_CUDA(cudaFuncSetAttribute(k_cell_hash_seg<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(ssmem)));
        PO_CUDA(cudaFuncSetAttribute(k_cell_hash_seg<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(ssmem)));
        PO_CUDA(cudaFuncSetAttribute(k_cell_hash_seg<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(ssmem)));
        seg_attr = true;
      }
      const uint64_t ntiles = (n + R - 1) / R;
      const unsigned grid = unsigned(std::min<uint64_t>(ntiles, uint64_t(kSMs) * 3));
      const double cell_bytes = double(t.arena_bytes) / double(cells);
      if (cell_bytes >= 384)
        PO_LAUNCH(k_cell_hash_seg<32>, grid, kSegBlock, ssmem, s, t.arena, arena_end, t.offsets, n,
                  uint32_t(m), R, sstage, hmask, hashes.get());
      else if (cell_bytes >= 160)
        PO_LAUNCH(k_cell_hash_seg<16>, grid, kSegBlock, ssmem, s, t.arena, arena_end, t.offsets, n,
                  uint32_t(m), R, sstage, hmask, hashes.get());
      else
        PO_LAUNCH(k_cell_hash_seg<8>, grid, kSegBlock, ssmem, s, t.arena, arena_end, t.offsets, n,
                  uint32_t(m), R, sstage, hmask, hashes.get());
    } else if (hsel == "tile" && m <= kDictBlock) {
      const uint64_t ntiles = (cells + rows_per_tile * m - 1) / (rows_per_tile * m);
      PO_LAUNCH(k_cell_hash, unsigned(std::min<uint64_t>(ntiles, uint64_t(kSMs) * 3)), kDictBlock,
                smem, s, t.arena, arena_end, t.offsets, cells, uint32_t(m), rows_per_tile, stage,
                hmask, hashes.get());
    } else {
      static const unsigned hb = [] {  // resident blocks per SM (experiment knob)
        const char* v = std::getenv("PO_HASH_BLOCKS_PER_SM");
        return v && *v ? unsigned(std::atoi(v)) : 0u;
      }();
      const unsigned g = hb ? std::min<unsigned>(grid_for(((n + 31) / 32) * 32, 256, 8), kSMs * hb)
                            : grid_for(((n + 31) / 32) * 32, 256, 8);
      PO_LAUNCH(k_cell_hash_cols, g, 256, 0, s, t.arena,
                arena_end, t.offsets, n, uint32_t(m), hmask, hashes.get());
    }
    // K2a/K2b: probe + claim, then byte verification of every duplicate
    PO_LAUNCH(k_dict_probe, grid_for(cells, 256, 32), 256, 0, s, hashes.get(), t.offsets, cells,
              uint32_t(m), cap, keys.get(), reps.get(), repoffs.get(), slot_of_cell.get());
    DevBuf<uint32_t> collided, ncol(1, s);
    collided.alloc_cached(cells, s);
    ncol.zero();
    PO_LAUNCH(k_dict_verify, grid_for(((n + 31) / 32) * 32, 256, 8), 256, 0, s, t.arena,
              arena_end, t.offsets, n, uint32_t(m), cap, reps.get(), repoffs.get(), slot_of_cell.get(),
              collided.get(), ncol.get());
    // K2c: exact resolution of 64-bit hash collisions (almost always no work)
    PO_LAUNCH(k_dict_fixup, kSMs, 128, 0, s, t.arena, arena_end, t.offsets, uint32_t(m), cap,
              hashes.get(), keys.get(), reps.get(), repoffs.get(), collided.get(), ncol.get(),
              slot_of_cell.get());
  }

  timing_mark("dict", s);
  // Distinct values per column (occupied slots): every column is compacted
  // into its own region of `stage` without host round trips, then one D2H of
  // the m counts gives the cardinalities and the packed layout.
  DevBuf<uint32_t> stage_sel;
  stage_sel.alloc_cached(m * cap, s);
  DevBuf<int> nsel(m, s);
  nsel.zero();
  {
    const uint64_t chunks = (m * cap + kCompactChunk - 1) / kCompactChunk;
    PO_LAUNCH(k_compact_slots, unsigned(std::min<uint64_t>(chunks, uint64_t(kSMs) * 8)), 256, 0, s,
              keys.get(), cap, m * cap, stage_sel.get(), nsel.get());
  }
  {
    std::vector<int> hk(m);
    nsel.download(hk.data(), m);  // pageable D2H: completes before returning
    sync(s);
    for (uint32_t c = 0; c < m; ++c) {
      e.card[c] = uint64_t(hk[c]);
      e.colbase[c + 1] = e.colbase[c] + uint64_t(hk[c]);
    }
  }
  e.D = e.colbase[m];
  const uint64_t D = e.D;
  e.d_colbase = to_device(e.colbase, s);

  DevBuf<uint32_t> sel(D, s);  // per distinct (column order): slot within its column
  DevBuf<uint32_t> d_col(D, s), d_row(D, s);
  PO_LAUNCH(k_distinct_info, grid_for(D, 256), 256, 0, s, stage_sel.get(), D,
            e.d_colbase.get(), uint32_t(m), cap, reps.get(), sel.get(), d_col.get(),
            d_row.get());
  stage_sel.release();

  // Escaped fragment-key order (json_escape(v) + '"') of the distinct values
  // of each column -> vid. Raw-byte order is only needed for candidate ties
  // and single-column leaves; the solver ranks those few values on demand.
  DevBuf<uint32_t> esc_pos(D, s);
  RefineKey ek;
  ek.kind = 1;
  ek.arena = t.arena;
  ek.arena_bytes = t.arena_bytes;
  ek.offsets = t.offsets;
  ek.item_cell_row = d_row.get();
  ek.item_col = d_col.get();
  ek.m = uint32_t(m);
  timing_mark("distinct", s);
  // rank_unique = false: a column with a distinct value per row (n > 1)
  // keeps ids in compaction order (Encoded::unranked); its order is only
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
      je.d_grp_init = d_col.get();
      je.d_out_pos = esc_pos.get();
      refine_sort_multi({je}, s);
    } else {
      DevBuf<uint64_t> d_rbase = to_device(rbase, s), d_rpre = to_device(rpre, s);
      DevBuf<uint32_t> sub_d(n_ranked, s), sub_row(n_ranked, s), sub_col(n_ranked, s),
          sub_pos(n_ranked, s);
      PO_LAUNCH(k_ranked_items, grid_for(n_ranked, 256), 256, 0, s, d_rbase.get(), d_rpre.get(),
                uint32_t(rbase.size()), n_ranked, d_row.get(), d_col.get(), sub_d.get(),
                sub_row.get(), sub_col.get());
      je.n_items = uint32_t(n_ranked);
      je.d_grp_init = sub_col.get();
      je.key.item_cell_row = sub_row.get();
      je.key.item_col = sub_col.get();
      je.d_out_pos = sub_pos.get();
      refine_sort_multi({je}, s);
      PO_LAUNCH(k_scatter_sub, grid_for(n_ranked, 256), 256, 0, s, sub_d.get(), sub_pos.get(),
                n_ranked, esc_pos.get());
    }
  }
  timing_mark("rank_sort", s);

  DevBuf<uint32_t> slot2vid, col_by_pos(D, s);
  slot2vid.alloc_cached(m * cap, s);
  e.rep_row.alloc_auto(D, s);
  timing_mark("scatter_alloc", s);
  PO_LAUNCH(k_scatter_pos, grid_for(D, 256), 256, 0, s, esc_pos.get(), d_col.get(), d_row.get(),
            sel.get(), e.d_colbase.get(), D, cap, slot2vid.get(), e.rep_row.get(),
            col_by_pos.get());
  keys.release();
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
  PO_LAUNCH(k_vlen, grid_for(D, 256), 256, 0, s, t.arena, t.offsets, t.cell_lens,
            e.rep_row.get(), col_by_pos.get(), D, uint32_t(m), tok, scoring, d_nchar.get(),
            d_nword.get(), e.vlen.get());

  timing_mark("vlen", s);
  // vid matrix (row-major) and occurrence counts.
  e.vid.alloc_auto(cells, s);
  PO_LAUNCH(k_vid, grid_for(cells, 256), 256, 0, s, slot_of_cell.get(), slot2vid.get(), n,
            uint32_t(m), cap, e.vid.get());
  slot_of_cell.release();
  slot2vid.release();
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
  tot.download(htot.data(), m);
  sync(s);
  for (uint32_t c = 0; c < m; ++c) e.total_len[c] = htot[c];
  timing_mark("encode_tail", s);
}

}  // namespace po
