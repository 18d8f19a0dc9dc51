// Prompt rendering and byte-exact dedup: the step
// after the path in cmd_solve (run.hpp:457-466).
//
// render_prompt (objective.hpp:118-131): [system_prompt '\n'] [question '\n']
// then render_body (objective.hpp:102-115): '{' then, per field of the
// entry's order, [", "] '"' esc(name) '": "' esc(value) '"', then '}'.
// Escaping is json_escape (scoring.hpp:33-57). One warp per request: pass 1
// sums the escaped lengths (lanes stride over each cell's bytes, warp sum),
// an exclusive scan gives every prompt's offset, pass 2 writes the bytes —
// 32 input bytes per step, each lane's expansion (1, 2 or 6 bytes) placed
// by a warp prefix sum, so the output is written in order without gaps.
//
// dedup (cost.hpp:171-186): uniques in first-occurrence order + expansion
// map, from the exact dictionary of the prompts (encode() on a one-column
// table: equal ids <=> equal bytes) and the first index of every id.

#include <cub/cub.cuh>

#include <cstdlib>
#include <functional>

#include "internal.cuh"

namespace po {

namespace {

__device__ __forceinline__ uint32_t esc_len_b(uint8_t c) {
  if (c == '"' || c == '\\' || c == '\b' || c == '\f' || c == '\n' || c == '\r' || c == '\t')
    return 2;
  return c < 0x20 ? 6 : 1;
}

__device__ __forceinline__ void esc_write(uint8_t c, uint8_t* o) {
  switch (c) {
    case '"': o[0] = '\\'; o[1] = '"'; return;
    case '\\': o[0] = '\\'; o[1] = '\\'; return;
    case '\b': o[0] = '\\'; o[1] = 'b'; return;
    case '\f': o[0] = '\\'; o[1] = 'f'; return;
    case '\n': o[0] = '\\'; o[1] = 'n'; return;
    case '\r': o[0] = '\\'; o[1] = 'r'; return;
    case '\t': o[0] = '\\'; o[1] = 't'; return;
    default:
      if (c < 0x20) {
        o[0] = '\\'; o[1] = 'u'; o[2] = '0'; o[3] = '0';
        const uint8_t lo = c & 15;
        o[4] = uint8_t('0' + (c >> 4));  // c < 0x20: the high digit is 0 or 1
        o[5] = uint8_t(lo < 10 ? '0' + lo : 'a' + lo - 10);
      } else {
        o[0] = c;
      }
  }
}

struct Sched {
  const uint64_t* rows;
  const uint64_t* offs;
  const int32_t* fields;
};

__global__ void k_prompt_len(const uint8_t* __restrict__ arena, const uint8_t* arena_end,
                             const uint64_t* __restrict__ offsets,
                             uint64_t n_rows, uint32_t m, Sched sc, uint64_t n_entries,
                             const uint64_t* __restrict__ name_esc_len, uint64_t prefix_len,
                             uint64_t* out_len, int* err) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; i < n_entries;
       i += warps) {
    const uint64_t r = sc.rows[i];
    const uint64_t a = sc.offs[i], b = sc.offs[i + 1];
    uint64_t tot = 0;
    for (uint64_t p = a; p < b; ++p) {
      const int32_t f = sc.fields[p];
      if (r >= n_rows || f < 0 || uint32_t(f) >= m) {
        if (lane == 0) atomicExch(err, 1);
        break;
      }
      const uint64_t c = r * m + f;
      const uint8_t* v = arena + offsets[c];
      const uint64_t len = offsets[c + 1] - offsets[c];
      for (uint64_t j = 8 * lane; j < len; j += 256) {  // 8 bytes per lane per step
        const uint64_t w = load8_unaligned(v + j, arena_end);
        const uint32_t nb = len - j >= 8 ? 8u : uint32_t(len - j);
        for (uint32_t k = 0; k < nb; ++k) tot += esc_len_b(uint8_t(w >> (8 * k)));
      }
      if (lane == 0) tot += (p > a ? 2 : 0) + 1 + name_esc_len[f] + 4 + 1;
    }
    for (int d = 16; d > 0; d >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, d);
    if (lane == 0) out_len[i] = prefix_len + 2 + tot;
  }
}

// ---------------------------------------------------------------------------
// Dense schedules (the ggr() output covers every cell): escaped lengths come
// from one pass over the table in storage order (k_cell_esc_extra: thread
// per cell, a warp's 32 cells are one contiguous byte range), then a
// thread per request sums its fields (k_prompt_len_cells).
// ---------------------------------------------------------------------------
constexpr unsigned kFullMask = 0xffffffffu;
constexpr uint32_t kHigh32 = 0x80808080u, kLow32 = 0x7F7F7F7Fu;
constexpr uint64_t kHigh64 = 0x8080808080808080ull, kLow64 = 0x7F7F7F7F7F7F7F7Full;

// high bit of every byte json_escape expands: < 0x20, '"' or '\\' (exact
// per byte: no carry crosses a byte)
__device__ __forceinline__ uint64_t esc_flags64(uint64_t x) {
  const uint64_t ctrl = ~(x | ((x & kLow64) + 0x6060606060606060ull)) & kHigh64;
  const uint64_t y1 = x ^ 0x2222222222222222ull, y2 = x ^ 0x5C5C5C5C5C5C5C5Cull;
  const uint64_t z1 = ~(((y1 & kLow64) + kLow64) | y1) & kHigh64;
  const uint64_t z2 = ~(((y2 & kLow64) + kLow64) | y2) & kHigh64;
  return ctrl | z1 | z2;
}
__device__ __forceinline__ uint32_t esc_flags32(uint32_t x) {
  const uint32_t ctrl = ~(x | ((x & kLow32) + 0x60606060u)) & kHigh32;
  const uint32_t y1 = x ^ 0x22222222u, y2 = x ^ 0x5C5C5C5Cu;
  const uint32_t z1 = ~(((y1 & kLow32) + kLow32) | y1) & kHigh32;
  const uint32_t z2 = ~(((y2 & kLow32) + kLow32) | y2) & kHigh32;
  return ctrl | z1 | z2;
}

constexpr uint32_t kExtraBig = 0xFFFFFFFFu;

// extra bytes json_escape adds to arena[o, e), one thread (cells too long for
// k_cell_esc_extra's 32-bit counts)
__device__ uint64_t esc_extra_serial(const uint8_t* arena, uint64_t o, uint64_t e) {
  uint64_t x = 0;
  for (uint64_t i = o; i < e; ++i) x += esc_len_b(arena[i]) - 1;
  return x;
}

// Escaped-length extras of every cell (escaped length = len + extra). A
// warp takes 32 consecutive cells — one contiguous byte range of the arena —
// and scans the range once with coalesced 16-byte loads; a byte to escape
// (rare) is charged to its cell by a binary search over the warp's 33 cell
// offsets in shared memory.
constexpr uint32_t kEscWarps = 8;
__global__ void __launch_bounds__(kEscWarps * 32)
    k_cell_esc_extra(const uint8_t* __restrict__ arena, const uint64_t* __restrict__ offsets,
                     uint64_t cells, uint32_t* __restrict__ extra) {
  __shared__ uint64_t s_off[kEscWarps][33];
  __shared__ uint32_t s_cnt[kEscWarps][32];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t nw = (cells + 31) / 32;
  const uintptr_t base = reinterpret_cast<uintptr_t>(arena);
  for (uint64_t wi = blockIdx.x * uint64_t(kEscWarps) + wid; wi < nw;
       wi += uint64_t(gridDim.x) * kEscWarps) {
    const uint64_t c0 = wi * 32;
    const uint32_t nc = cells - c0 < 32 ? uint32_t(cells - c0) : 32u;
    s_off[wid][lane] = offsets[c0 + (lane < nc ? lane : nc)];
    if (lane == 0) s_off[wid][32] = offsets[c0 + nc];
    s_cnt[wid][lane] = 0;
    __syncwarp();
    const uint64_t lo = s_off[wid][0], hi = s_off[wid][32];
    // arena offset of the first aligned chunk (negative when the arena
    // itself is not 16-byte aligned)
    const int64_t a0 = int64_t((base + lo) & ~uintptr_t(15)) - int64_t(base);
#pragma unroll 4
    for (int64_t a = a0 + 16 * int64_t(lane); a < int64_t(hi); a += 512) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(arena + a));
      const uint64_t w0 = uint64_t(v.x) | (uint64_t(v.y) << 32), w1 = uint64_t(v.z) | (uint64_t(v.w) << 32);
      // bytes of the chunk inside [lo, hi)
      const uint32_t b0 = a < int64_t(lo) ? uint32_t(int64_t(lo) - a) : 0u;
      const uint32_t b1 = int64_t(hi) - a >= 16 ? 16u : uint32_t(int64_t(hi) - a);
      const uint64_t k0 = (b1 >= 8 ? ~0ull : ((1ull << (8 * b1)) - 1)) & (b0 >= 8 ? 0ull : ~((1ull << (8 * b0)) - 1));
      const uint64_t k1 = (b1 <= 8 ? 0ull : (b1 == 16 ? ~0ull : ((1ull << (8 * (b1 - 8))) - 1))) &
                          (b0 <= 8 ? ~0ull : ~((1ull << (8 * (b0 - 8))) - 1));
      uint64_t f[2] = {esc_flags64(w0) & k0, esc_flags64(w1) & k1};
      const uint64_t w[2] = {w0, w1};
#pragma unroll
      for (int h = 0; h < 2; ++h)
        while (f[h]) {
          const uint32_t k = uint32_t(__ffsll((long long)f[h]) - 1) >> 3;
          f[h] &= f[h] - 1;
          const uint64_t pos = uint64_t(a + 8 * h + k);
          uint32_t j0 = 0, j1 = nc - 1;  // last cell with offset <= pos (empty cells skipped)
          while (j0 < j1) {
            const uint32_t mid = (j0 + j1 + 1) / 2;
            if (s_off[wid][mid] <= pos) j0 = mid;
            else j1 = mid - 1;
          }
          atomicAdd(&s_cnt[wid][j0], esc_len_b(uint8_t(w[h] >> (8 * k))) - 1);
        }
    }
    __syncwarp();
    if (lane < nc) {
      // a cell whose extra may not fit 32 bits is summed by its reader instead
      const bool big = s_off[wid][lane + 1] - s_off[wid][lane] > 0xFFFFFFFFull / 6;
      extra[c0 + lane] = big ? kExtraBig : s_cnt[wid][lane];
    }
    __syncwarp();
  }
}

__global__ void k_prompt_len_cells(const uint8_t* __restrict__ arena,
                                   const uint64_t* __restrict__ offsets,
                                   const uint32_t* __restrict__ extra, uint64_t n_rows, uint32_t m,
                                   Sched sc, uint64_t n_entries,
                                   const uint64_t* __restrict__ name_esc_len, uint64_t prefix_len,
                                   uint64_t* out_len, int* err) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n_entries;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = sc.rows[i];
    const uint64_t a = sc.offs[i], b = sc.offs[i + 1];
    uint64_t tot = 0;
    for (uint64_t p = a; p < b; ++p) {
      const int32_t f = sc.fields[p];
      if (r >= n_rows || f < 0 || uint32_t(f) >= m) {
        atomicExch(err, 1);
        break;
      }
      const uint64_t c = r * m + f;
      const uint64_t o = offsets[c], len = offsets[c + 1] - o;
      uint64_t x = extra[c];
      if (x == kExtraBig) x = esc_extra_serial(arena, o, o + len);  // a cell of > 700 MB
      tot += (p > a ? 2 : 0) + 1 + name_esc_len[f] + 4 + len + x + 1;
    }
    out_len[i] = prefix_len + 2 + tot;
  }
}

// ---------------------------------------------------------------------------
// k_prompt_write: a warp renders a contiguous range of requests (their
// prompts are one contiguous output range) into a shared-memory staging
// buffer laid out at the output's 16-byte alignment, and writes it out in
// aligned 16-byte stores (bytes only at the range's two ends). Copies move
// 128 bytes per warp step: lane l builds output word l of the step from two
// aligned source words (the second is lane l+1's first: one shuffle) with a
// byte permute; a step whose bytes need escaping is redone 32 input bytes
// at a time with a warp prefix sum of the escaped sizes.
// ---------------------------------------------------------------------------
constexpr uint32_t kRenderWarps = 8;
constexpr uint32_t kRenderBuf = 4096;  // staging bytes per warp (multiple of 16)
struct Stage {
  uint8_t* buf;    // shared, 16-byte aligned
  uint8_t* gbase;  // output address of buf[0] (16-byte aligned)
  uint32_t bp;     // next buf byte
  uint32_t from;   // first buf byte of this warp's output not yet written
};

__device__ __forceinline__ void stage_write(const Stage& st, uint32_t from, uint32_t upto,
                                            uint32_t lane) {
  if (upto <= from) return;
  const uint32_t a = (from + 15) & ~15u, b = upto & ~15u;
  if (a >= b) {
    for (uint32_t x = from + lane; x < upto; x += 32) st.gbase[x] = st.buf[x];
    return;
  }
  for (uint32_t x = from + lane; x < a; x += 32) st.gbase[x] = st.buf[x];
  for (uint32_t x = b + lane; x < upto; x += 32) st.gbase[x] = st.buf[x];
  for (uint32_t x = a + 16 * lane; x < b; x += 512)
    *reinterpret_cast<uint4*>(st.gbase + x) = *reinterpret_cast<const uint4*>(st.buf + x);
}

// write the buffer's aligned part, keep the tail (< 16 bytes) at its start
__device__ __forceinline__ void stage_flush(Stage& st, uint32_t lane) {
  __syncwarp();
  const uint32_t cut = st.bp & ~15u;
  if (!cut) return;
  stage_write(st, st.from, cut, lane);
  const uint32_t tail = st.bp - cut;
  const uint8_t v = lane < tail ? st.buf[cut + lane] : 0;
  __syncwarp();
  if (lane < tail) st.buf[lane] = v;
  __syncwarp();
  st.gbase += cut;
  st.bp = tail;
  st.from = st.from > cut ? st.from - cut : 0;
}

__device__ __forceinline__ void stage_ensure(Stage& st, uint32_t need, uint32_t lane) {
  if (st.bp + need > kRenderBuf) stage_flush(st, lane);
}

// up to 4 literal bytes (little-endian in `bytes`)
__device__ __forceinline__ void stage_put(Stage& st, uint32_t bytes, uint32_t n, uint32_t lane) {
  stage_ensure(st, 4, lane);
  __syncwarp();
  if (lane < n) st.buf[st.bp + lane] = uint8_t(bytes >> (8 * lane));
  st.bp += n;
  __syncwarp();
}

// append src[0, len) (device memory), json-escaped when kEscape. A step
// fills up to 32 output words (128 bytes): lane l builds word l from the two
// aligned source words under it with a byte permute, only the step's first
// and last words are merged with their neighbours' bytes. (Steps of 2 and 4
// words per lane measured slower on C2: most cells are short.)
template <bool kEscape>
__device__ __forceinline__ void stage_append(Stage& st, const uint8_t* src, uint64_t len, uint32_t lane) {
  uint32_t* buf32 = reinterpret_cast<uint32_t*>(st.buf);
  while (len) {
    stage_ensure(st, 132, lane);
    __syncwarp();
    const uint32_t bp = st.bp;
    const uint32_t head = bp & 3u;  // bytes of the first word before bp
    const uint32_t take = len < 128u - head ? uint32_t(len) : 128u - head;
    // this lane's word starts at source offset r0 (lane 0: up to 3 before src)
    const int32_t r0 = int32_t(4 * lane) - int32_t(head);
    const uintptr_t sa = reinterpret_cast<uintptr_t>(src) + intptr_t(r0);
    const uint32_t sh = uint32_t(sa & 3);
    const int32_t ra = r0 - int32_t(sh);  // aligned word under it, relative to src
    const uint32_t* A = reinterpret_cast<const uint32_t*>(sa - sh);
    // only aligned words holding a byte of [0, take) are read
    const uint32_t lo = (ra > -4 && ra < int32_t(take)) ? __ldg(A) : 0u;
    const uint32_t hi = (ra > -8 && ra + 4 < int32_t(take)) ? __ldg(A + 1) : 0u;
    const uint32_t val = __byte_perm(lo, hi, 0x3210u + 0x1111u * sh);
    const int32_t b0 = r0 < 0 ? -r0 : 0;
    const int32_t b1 = min(int32_t(take) - r0, 4);
    const uint32_t keep = b1 > b0 ? (0xFFFFFFFFu >> (8 * (4 - (b1 - b0)))) << (8 * b0) : 0u;
    bool special = false;
    if (kEscape) special = __any_sync(kFullMask, (esc_flags32(val) & keep) != 0);
    if (!special) {
      const uint32_t w = (bp >> 2) + lane;
      if (keep == ~0u) buf32[w] = val;
      else if (keep) buf32[w] = (buf32[w] & ~keep) | (val & keep);
      st.bp = bp + take;
    } else {
      // the same input bytes, escaped, 32 at a time
      for (uint32_t j0 = 0; j0 < take; j0 += 32) {
        stage_ensure(st, 6 * 32, lane);
        __syncwarp();
        const uint32_t j = j0 + lane;
        uint8_t c = 0;
        uint32_t e = 0;
        if (j < take) {
          c = src[j];
          e = esc_len_b(c);
        }
        uint32_t incl = e;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(kFullMask, incl, d);
          if (int(lane) >= d) incl += y;
        }
        if (e) esc_write(c, st.buf + st.bp + incl - e);
        st.bp += __shfl_sync(kFullMask, incl, 31);
      }
    }
    src += take;
    len -= take;
  }
  __syncwarp();
}

// Bytes [r, r + 4) of src[0, len) (r may be negative or past the end: those
// bytes are garbage, masked by the caller); only aligned words holding a
// byte of [0, len) are read.
__device__ __forceinline__ uint32_t word_at(const uint8_t* src, int32_t r, int32_t len) {
  const uintptr_t sa = reinterpret_cast<uintptr_t>(src) + intptr_t(r);
  const uint32_t sh = uint32_t(sa & 3);
  const int32_t ra = r - int32_t(sh);
  const uint32_t* A = reinterpret_cast<const uint32_t*>(sa - sh);
  const uint32_t lo = (ra > -4 && ra < len) ? __ldg(A) : 0u;
  const uint32_t hi = (ra > -8 && ra + 4 < len) ? __ldg(A + 1) : 0u;
  return __byte_perm(lo, hi, 0x3210u + 0x1111u * sh);
}
// byte mask of the word bytes whose offset (relative to the word start r)
// falls in [lo, hi)
__device__ __forceinline__ uint32_t range_keep(int32_t r, int32_t lo, int32_t hi) {
  const int32_t b0 = max(lo - r, 0), b1 = min(hi - r, 4);
  return b1 > b0 ? (0xFFFFFFFFu >> (8 * (4 - (b1 - b0)))) << (8 * b0) : 0u;
}

// A field's name template a[0, la) followed by its value b[0, lb), escaped:
// one copy step when both fit one 32-word window and the value has nothing
// to escape (most short cells), else the two appends.
__device__ __forceinline__ void stage_append_pair(Stage& st, const uint8_t* a, uint64_t la,
                                                  const uint8_t* b, uint64_t lb, uint32_t lane) {
  if (la + lb + 4 <= 128) {
    stage_ensure(st, 132, lane);
    __syncwarp();
    const uint32_t bp = st.bp;
    const uint32_t head = bp & 3u;
    const int32_t LA = int32_t(la), T = int32_t(la + lb);
    if (uint32_t(T) <= 128u - head) {
      const int32_t r0 = int32_t(4 * lane) - int32_t(head);  // word start, relative to a[0]
      const uint32_t va = word_at(a, r0, LA), vb = word_at(b, r0 - LA, T - LA);
      const uint32_t ka = range_keep(r0, 0, LA), kb = range_keep(r0, LA, T);
      if (!__any_sync(kFullMask, (esc_flags32(vb) & kb) != 0)) {
        uint32_t* buf32 = reinterpret_cast<uint32_t*>(st.buf);
        const uint32_t val = (va & ka) | (vb & kb), keep = ka | kb;
        const uint32_t w = (bp >> 2) + lane;
        if (keep == ~0u) buf32[w] = val;
        else if (keep) buf32[w] = (buf32[w] & ~keep) | (val & keep);
        st.bp = bp + uint32_t(T);
        __syncwarp();
        return;
      }
    }
  }
  stage_append<false>(st, a, la, lane);
  stage_append<true>(st, b, lb, lane);
}

__global__ void __launch_bounds__(kRenderWarps * 32)
    k_prompt_write(const uint8_t* __restrict__ arena, const uint64_t* __restrict__ offsets,
                   uint32_t m, Sched sc, uint64_t n_entries, uint64_t per_warp,
                   const uint8_t* __restrict__ tmpl, const uint64_t* __restrict__ tmpl_off,
                   const uint8_t* prefix, uint64_t prefix_len,
                   const uint64_t* __restrict__ out_off, uint8_t* out) {
  __shared__ __align__(16) uint8_t sbuf[kRenderWarps][kRenderBuf];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t gw = blockIdx.x * uint64_t(kRenderWarps) + wid;
  const uint64_t i0 = gw * per_warp;
  if (i0 >= n_entries) return;
  const uint64_t i1 = i0 + per_warp < n_entries ? i0 + per_warp : n_entries;
  Stage st;
  st.buf = sbuf[wid];
  {
    uint8_t* g = out + out_off[i0];
    st.gbase = reinterpret_cast<uint8_t*>(reinterpret_cast<uintptr_t>(g) & ~uintptr_t(15));
    st.bp = st.from = uint32_t(g - st.gbase);
  }
  for (uint64_t i = i0; i < i1; ++i) {
    const uint64_t r = sc.rows[i];
    const uint64_t a = sc.offs[i], b = sc.offs[i + 1];
    if (prefix_len) stage_append<false>(st, prefix, prefix_len, lane);
    if (a == b) stage_put(st, 0x7D7Bu, 2, lane);  // {}
    for (uint64_t p0 = a; p0 < b; p0 += 32) {
      // the next 32 fields' cells and name templates, one per lane
      uint64_t co = 0, cl = 0, to = 0, tl = 0;
      if (p0 + lane < b) {
        const int32_t f = sc.fields[p0 + lane];
        const uint64_t c = r * m + uint32_t(f);
        co = offsets[c];
        cl = offsets[c + 1] - co;
        const uint32_t q = 2 * uint32_t(f) + (p0 + lane > a ? 1 : 0);
        to = tmpl_off[q];
        tl = tmpl_off[q + 1] - to;
      }
      const uint32_t cnt = b - p0 < 32 ? uint32_t(b - p0) : 32u;
      for (uint32_t k = 0; k < cnt; ++k) {
        const uint64_t o = __shfl_sync(kFullMask, co, k), l = __shfl_sync(kFullMask, cl, k);
        const uint64_t tO = __shfl_sync(kFullMask, to, k), tL = __shfl_sync(kFullMask, tl, k);
        stage_append_pair(st, tmpl + tO, tL, arena + o, l, lane);  // [{ or ", ]"name": "value
      }
    }
    if (a != b) stage_put(st, 0x7D22u, 2, lane);  // "}
  }
  __syncwarp();
  stage_write(st, st.from, st.bp, lane);
}

__global__ void k_first_index(const uint32_t* vid, uint64_t n, uint32_t* first) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    if (first[vid[i]] > uint32_t(i)) atomicMin(&first[vid[i]], uint32_t(i));  // see k_first_row (fd.cu)
}

__global__ void k_is_first(const uint32_t* vid, uint64_t n, const uint32_t* first, uint32_t* flag) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    flag[i] = first[vid[i]] == uint32_t(i) ? 1u : 0u;
}

__global__ void k_expand(const uint32_t* vid, uint64_t n, const uint32_t* first,
                         const uint32_t* uidx_excl, uint64_t* expansion, uint64_t* unique_first) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t f = first[vid[i]];
    expansion[i] = uidx_excl[f];
    if (f == uint32_t(i)) unique_first[uidx_excl[i]] = i;
  }
}

}  // namespace

std::string json_escape_bytes(const std::string& s) {
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

void render_prompts_device(const DeviceTable& t, uint64_t n_entries, const uint64_t* rows,
                           const uint64_t* order_offsets, const int32_t* fields, uint64_t n_fields,
                           const std::string& system_prompt, const std::string& question,
                           DevBuf<uint64_t>& out_off, uint64_t& total,
                           const std::function<uint8_t*(uint64_t)>& dst_for, cudaStream_t s) {
  const uint32_t m = t.m;
  std::string prefix;
  if (!system_prompt.empty()) prefix += system_prompt + "\n";
  if (!question.empty()) prefix += question + "\n";
  std::vector<uint64_t> name_len(std::max<uint32_t>(m, 1), 0);
  for (uint32_t f = 0; f < m; ++f) name_len[f] = json_escape_bytes(t.names[f]).size();
  auto d_name_len = to_device(name_len, s);
  // per field the text before its value: first field '{"name": "', later
  // fields '", "name": "' (the previous value's closing quote)
  std::string tmpl;
  std::vector<uint64_t> tmpl_off(2 * size_t(m) + 1, 0);
  for (uint32_t f = 0; f < m; ++f) {
    const std::string e = json_escape_bytes(t.names[f]);
    tmpl += "{\"" + e + "\": \"";
    tmpl_off[2 * f + 1] = tmpl.size();
    tmpl += "\", \"" + e + "\": \"";
    tmpl_off[2 * f + 2] = tmpl.size();
  }
  std::vector<uint8_t> tb8(tmpl.begin(), tmpl.end());
  tb8.resize((tb8.size() + 16) & ~size_t(15), 0);
  auto d_tmpl = to_device(tb8, s);
  auto d_tmpl_off = to_device(tmpl_off, s);
  // padded to 16 bytes: the copy reads whole aligned words
  std::vector<uint8_t> pb(prefix.begin(), prefix.end());
  pb.resize((pb.size() + 16) & ~size_t(15), 0);
  auto d_prefix = to_device(pb, s);
  out_off.alloc(n_entries + 1, s);
  total = 0;
  if (n_entries == 0) {
    out_off.zero();
    dst_for(0);
    return;
  }
  Sched sc{rows, order_offsets, fields};
  DevBuf<uint64_t> lens(n_entries + 1, s);
  lens.zero();
  DevBuf<int> err(1, s);
  err.zero();
  const uint64_t cells = t.n * uint64_t(m);
  int herr = 0;
  if (cells && n_fields * 2 >= cells) {
    // dense schedule: escaped lengths of all cells in storage order
    DevBuf<uint32_t> extra(cells, s);
    PO_LAUNCH(k_cell_esc_extra, grid_for(cells, kEscWarps * 32), kEscWarps * 32, 0, s, t.arena,
              t.offsets, cells, extra.get());
    PO_LAUNCH(k_prompt_len_cells, grid_for(n_entries, 256), 256, 0, s, t.arena, t.offsets, extra.get(),
              t.n, m, sc, n_entries, d_name_len.get(), uint64_t(prefix.size()), lens.get(),
              err.get());
  } else {
    PO_LAUNCH(k_prompt_len, grid_for(n_entries * 32, 256), 256, 0, s, t.arena,
              t.arena + t.arena_bytes, t.offsets, t.n, m, sc,
              n_entries, d_name_len.get(), uint64_t(prefix.size()), lens.get(), err.get());
  }
  size_t tb = 0;
  PO_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, lens.get(), out_off.get(), int64_t(n_entries + 1), s));
  DevBuf<uint8_t> tmp(tb, s);
  PO_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, lens.get(), out_off.get(), int64_t(n_entries + 1), s));
  err.download(&herr, 1);
  PO_CUDA(cudaMemcpyAsync(&total, out_off.get() + n_entries, 8, cudaMemcpyDeviceToHost, s));
  sync(s);
  if (herr) fail(PO_ERR_OUT_OF_RANGE, "schedule references a row or field outside the table");
  uint8_t* dst = dst_for(total);
  if (!dst || !total) return;
  // a warp per contiguous request range: about one range per resident warp
  int bps = 0;
  PO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_prompt_write, kRenderWarps * 32, 0));
  {
    const uint64_t max_warps = uint64_t(kSMs) * std::max(bps, 1) * kRenderWarps;
    const uint64_t warps = std::min<uint64_t>(n_entries, max_warps);
    const uint64_t per_warp = (n_entries + warps - 1) / warps;
    const uint64_t used = (n_entries + per_warp - 1) / per_warp;
    PO_LAUNCH(k_prompt_write, unsigned((used + kRenderWarps - 1) / kRenderWarps), kRenderWarps * 32, 0, s,
              t.arena, t.offsets, m, sc, n_entries, per_warp, d_tmpl.get(), d_tmpl_off.get(),
            d_prefix.get(), uint64_t(prefix.size()), out_off.get(), dst);
  }
}

void dedup_device(const DeviceTable& t, uint64_t* d_expansion, uint64_t* d_unique_first,
                  uint64_t& n_unique, cudaStream_t s) {
  const uint64_t n = t.n;
  n_unique = 0;
  if (n == 0) return;
  Encoded e;
  encode(t, PO_TOK_CHAR, PO_SCORE_VALUE, s, e, debug_hash_bits(), /*ordered=*/false);
  DevBuf<uint32_t> first(e.D, s), flag(n + 1, s), uex(n + 1, s);
  first.fill_bytes(0xFF);
  PO_LAUNCH(k_first_index, grid_for(n, 256), 256, 0, s, e.vid.get(), n, first.get());
  flag.zero();
  PO_LAUNCH(k_is_first, grid_for(n, 256), 256, 0, s, e.vid.get(), n, first.get(), flag.get());
  size_t tb = 0;
  PO_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.get(), uex.get(), int64_t(n + 1), s));
  DevBuf<uint8_t> tmp(tb, s);
  PO_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, flag.get(), uex.get(), int64_t(n + 1), s));
  PO_LAUNCH(k_expand, grid_for(n, 256), 256, 0, s, e.vid.get(), n, first.get(), uex.get(),
            d_expansion, d_unique_first);
  n_unique = e.D;
}

}  // namespace po
