// Prefix-cache replay under an UNBOUNDED cache:
// prefixopt::simulate with EvictionPolicy::none (cache_sim.hpp:223-285).
//
// With nothing ever evicted, the store holds every token prefix of every
// earlier prompt, so request i's raw hit (TokenTrie::match) is
//   raw_hit(i) = max_{j < i} LCP_tokens(prompt_i, prompt_j).
// In lexicographic order of the token sequences the LCP of two prompts is
// the minimum of the adjacent LCPs between them, and the best earlier prompt
// is one of the two nearest positions (left / right) holding an earlier
// request. So:
//   1. token sequences as sort keys — char tokenizer: the bytes; word
//      tokenizer: a u16 symbol stream, token bytes (b+3) each token closed by
//      a separator (2) below every byte, so stream order == token-sequence
//      order (tokenizer.hpp:47-73);
//   2. one refine sort of the prompts (common prefix of all prompts skipped);
//   3. adjacent LCPs in tokens (8 bytes per compare step; word: separators
//      inside the common prefix);
//   4. sparse tables of request index and of adjacent LCP over the sorted
//      order; per position a descent finds the nearest earlier request on
//      each side and a range-min gives its LCP.
// hit = raw_hit if >= min_cacheable_prefix_tokens else 0; miss = input - hit;
// written = input - raw_hit (cache_sim.hpp:266-272). LRU eviction is
// sequential by definition (the order is the experiment) and not provided.

#include <cub/cub.cuh>

#include "internal.cuh"

namespace po {

namespace {

__device__ __forceinline__ bool is_ws(uint8_t c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v';
}

constexpr uint16_t kSymSep = 2;  // token separator; bytes are b + 3

// input tokens per prompt; word mode also the symbol-stream length
__global__ void k_tok_counts(const uint8_t* __restrict__ arena, const uint64_t* __restrict__ off,
                             uint64_t n, int word, uint64_t* ntok, uint64_t* nsym) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; i < n; i += warps) {
    const uint8_t* p = arena + off[i];
    const uint64_t len = off[i + 1] - off[i];
    uint64_t tok = 0, nonws = 0;
    if (word)
      for (uint64_t j = lane; j < len; j += 32) {
        const bool nw = !is_ws(p[j]);
        nonws += nw;
        tok += nw && (j == 0 || is_ws(p[j - 1]));
      }
    for (int d = 16; d > 0; d >>= 1) {
      tok += __shfl_xor_sync(0xffffffffu, tok, d);
      nonws += __shfl_xor_sync(0xffffffffu, nonws, d);
    }
    if (lane == 0) {
      ntok[i] = word ? tok : len;
      if (nsym) nsym[i] = nonws + tok;
    }
  }
}

// word tokens as symbol streams (one warp per prompt, warp prefix sums)
__global__ void k_word_syms(const uint8_t* __restrict__ arena, const uint64_t* __restrict__ off,
                            uint64_t n, const uint64_t* __restrict__ soff, uint16_t* sym) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; i < n; i += warps) {
    const uint8_t* p = arena + off[i];
    const uint64_t len = off[i + 1] - off[i];
    uint64_t pos = soff[i];
    for (uint64_t base = 0; base < len; base += 32) {
      const uint64_t j = base + lane;
      uint8_t c = 0;
      uint32_t cnt = 0;
      bool end = false;
      if (j < len) {
        c = p[j];
        if (!is_ws(c)) {
          end = j + 1 == len || is_ws(p[j + 1]);
          cnt = 1 + (end ? 1 : 0);
        }
      }
      uint32_t incl = cnt;
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (int(lane) >= d) incl += y;
      }
      if (cnt) {
        const uint64_t at = pos + incl - cnt;
        sym[at] = uint16_t(c) + 3;
        if (end) sym[at + 1] = kSymSep;
      }
      pos += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

// Common prefix (in key units: bytes or symbols) of two keys (first_diff);
// word mode also counts the separators (= whole tokens) inside it.
struct Lcp {
  uint64_t units, tokens;
};
__device__ __forceinline__ Lcp key_lcp(const uint8_t* a, uint64_t la, const uint8_t* b, uint64_t lb,
                                       const uint8_t* lim, int word) {
  const uint32_t us = word ? 2 : 1;  // bytes per key unit
  const uint64_t n = (la < lb ? la : lb) * us;
  const uint64_t units = first_diff(a, b, n, lim) / us;
  uint64_t tokens = 0;
  if (word)  // separators among the common prefix's symbols (bytes just read: cache hits)
    for (uint64_t i = 0; i < 2 * units; i += 8) {
      const uint64_t x = load8_unaligned(a + i, lim);
      const uint64_t take = 2 * units - i < 8 ? 2 * units - i : 8;
      for (uint32_t k = 0; k + 2 <= take; k += 2) tokens += ((x >> (8 * k)) & 0xFFFF) == kSymSep;
    }
  return {units, tokens};
}

__global__ void k_lcp_first(const uint8_t* __restrict__ keys, const uint64_t* __restrict__ off,
                            uint64_t n, const uint8_t* lim, int word, unsigned long long* out) {
  // one atomic per block: a million atomics on one address serialise
  const uint32_t us = word ? 2 : 1;
  unsigned long long mn = ~0ull;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const Lcp l = key_lcp(keys + off[0] * us, off[1] - off[0], keys + off[i] * us,
                          off[i + 1] - off[i], lim, word);
    mn = l.units < mn ? l.units : mn;
  }
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, mn, d);
    mn = o < mn ? o : mn;
  }
  __shared__ unsigned long long s_min;
  if (threadIdx.x == 0) s_min = ~0ull;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && mn != ~0ull) atomicMin(&s_min, mn);
  __syncthreads();
  if (threadIdx.x == 0 && s_min != ~0ull) atomicMin(out, s_min);
}

// lcp[p] = LCP in tokens of sorted positions p-1 and p (lcp[0] = 0)
__global__ void k_adj_lcp(const uint32_t* __restrict__ perm, uint64_t n, const uint8_t* keys,
                          const uint64_t* __restrict__ off, const uint8_t* lim, int word,
                          uint32_t* lcp) {
  const uint32_t us = word ? 2 : 1;
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n;
       p += uint64_t(gridDim.x) * blockDim.x) {
    if (p == 0) {
      lcp[0] = 0;
      continue;
    }
    const uint32_t a = perm[p - 1], b = perm[p];
    const Lcp l = key_lcp(keys + off[a] * us, off[a + 1] - off[a], keys + off[b] * us,
                          off[b + 1] - off[b], lim, word);
    lcp[p] = uint32_t(word ? l.tokens : l.units);
  }
}

__global__ void k_seq(uint32_t* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    a[i] = uint32_t(i);
}

__global__ void k_st_level(const uint32_t* prev, uint64_t n, uint64_t half, uint32_t* cur) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    cur[i] = i + half < n ? min(prev[i], prev[i + half]) : prev[i];
}

// raw hit of the request at sorted position p (written at its request index)
__global__ void k_replay_query(uint64_t n, uint32_t K, const uint32_t* __restrict__ st_t,
                               const uint32_t* __restrict__ st_l, unsigned long long* raw) {
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n;
       p += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t t = st_t[p];  // level 0 = request index at p
    auto lmin = [&](uint64_t l, uint64_t r) -> uint32_t {  // min lcp[l..r], l <= r
      uint32_t k = 31 - __clz(uint32_t(r - l + 1));
      return min(st_l[uint64_t(k) * n + l], st_l[uint64_t(k) * n + r - (uint64_t(1) << k) + 1]);
    };
    uint32_t best = 0;
    // nearest earlier request on the left: shrink [pos, p) while its min > t
    uint64_t pos = p;
    for (int k = int(K) - 1; k >= 0; --k) {
      const uint64_t w = uint64_t(1) << k;
      if (pos >= w && st_t[uint64_t(k) * n + pos - w] > t) pos -= w;
    }
    if (pos > 0) best = max(best, lmin(pos, p));  // LCP(pos-1, p) = min lcp[pos..p]
    // nearest earlier request on the right
    pos = p + 1;
    for (int k = int(K) - 1; k >= 0; --k) {
      const uint64_t w = uint64_t(1) << k;
      if (pos + w <= n && st_t[uint64_t(k) * n + pos] > t) pos += w;
    }
    if (pos < n) best = max(best, lmin(p + 1, pos));
    raw[t] = best;
  }
}

}  // namespace

void replay_unbounded_device(const DeviceTable& pt, int tok, uint64_t* d_input, uint64_t* d_raw,
                             cudaStream_t s) {
  const uint64_t n = pt.n;
  if (n == 0) return;
  const int word = tok == PO_TOK_WORD ? 1 : 0;
  DevBuf<uint64_t> nsym;
  if (word) nsym.alloc(n + 1, s);
  PO_LAUNCH(k_tok_counts, grid_for(n * 32, 256), 256, 0, s, pt.arena, pt.offsets, n, word, d_input,
            word ? nsym.get() : nullptr);
  // sort keys: the bytes, or the word symbol streams
  const uint8_t* keys = pt.arena;
  const uint64_t* koff = pt.offsets;
  uint64_t key_bytes = pt.arena_bytes;
  DevBuf<uint64_t> soff;
  DevBuf<uint16_t> sym;
  if (word) {
    soff.alloc(n + 1, s);
    PO_CUDA(cudaMemsetAsync(nsym.get() + n, 0, 8, s));
    size_t tb = 0;
    PO_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, nsym.get(), soff.get(), int64_t(n + 1), s));
    DevBuf<uint8_t> tmp(tb, s);
    PO_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, nsym.get(), soff.get(), int64_t(n + 1), s));
    uint64_t total = 0;
    PO_CUDA(cudaMemcpyAsync(&total, soff.get() + n, 8, cudaMemcpyDeviceToHost, s));
    sync(s);
    sym.alloc(std::max<uint64_t>(total, 1), s);
    PO_LAUNCH(k_word_syms, grid_for(n * 32, 256), 256, 0, s, pt.arena, pt.offsets, n, soff.get(),
              sym.get());
    keys = reinterpret_cast<const uint8_t*>(sym.get());
    koff = soff.get();
    key_bytes = 2 * total;
  }
  const uint8_t* lim = keys + key_bytes;
  // prefix shared by every prompt (system prompt, question, JSON opening)
  DevBuf<unsigned long long> common(1, s);
  common.fill_bytes(0xFF);
  PO_LAUNCH(k_lcp_first, grid_for(n, 256), 256, 0, s, keys, koff, n, lim, word, common.get());
  unsigned long long skip = 0;
  common.download(&skip, 1);
  sync(s);
  // lexicographic order of the token sequences (ties: request order)
  DevBuf<uint32_t> iota(n, s), zeros(n, s), pos(n, s), perm(n, s), start(1, s);
  zeros.zero();
  start.zero();
  PO_LAUNCH(k_seq, grid_for(n, 256), 256, 0, s, iota.get(), n);
  RefineJob j;
  j.n_items = uint32_t(n);
  j.d_grp_init = zeros.get();
  j.d_grp_start = start.get();
  j.n_groups = 1;
  j.grp_max = uint32_t(n);
  j.key.kind = word ? 3 : 0;
  j.key.arena = keys;
  j.key.arena_bytes = key_bytes;
  j.key.str_off = koff;  // string i = prompt i (consecutive offsets)
  j.key.skip = skip;
  j.d_out_pos = pos.get();
  refine_sort_multi({j}, s);
  PO_LAUNCH(k_invert, grid_for(n, 256), 256, 0, s, pos.get(), n, perm.get());
  // sparse tables over the sorted order: request index and adjacent LCP
  uint32_t K = 1;
  while ((uint64_t(1) << K) <= n) ++K;
  DevBuf<uint32_t> st_t(uint64_t(K) * n, s), st_l(uint64_t(K) * n, s);
  PO_CUDA(cudaMemcpyAsync(st_t.get(), perm.get(), n * 4, cudaMemcpyDeviceToDevice, s));
  PO_LAUNCH(k_adj_lcp, grid_for(n, 256), 256, 0, s, perm.get(), n, keys, koff, lim, word,
            st_l.get());
  for (uint32_t k = 1; k < K; ++k) {
    PO_LAUNCH(k_st_level, grid_for(n, 256), 256, 0, s, st_t.get() + uint64_t(k - 1) * n, n,
              uint64_t(1) << (k - 1), st_t.get() + uint64_t(k) * n);
    PO_LAUNCH(k_st_level, grid_for(n, 256), 256, 0, s, st_l.get() + uint64_t(k - 1) * n, n,
              uint64_t(1) << (k - 1), st_l.get() + uint64_t(k) * n);
  }
  PO_LAUNCH(k_replay_query, grid_for(n, 256), 256, 0, s, n, K, st_t.get(), st_l.get(),
            reinterpret_cast<unsigned long long*>(d_raw));
}

// simulate()'s per-request report from the replay (cache_sim.hpp:266-279):
// hit = raw LCP when it reaches min_cacheable, else 0; miss = input - hit;
// written = input - raw; totals of input, hit and miss (atomics per warp).
__global__ void k_replay_report(const uint64_t* __restrict__ in, uint64_t* raw_to_written, uint64_t n,
                                uint64_t min_cacheable, uint64_t* hit, uint64_t* miss,
                                unsigned long long* totals) {
  unsigned long long ti = 0, th = 0, tm = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t a = in[i], r = raw_to_written[i];
    const uint64_t h = r >= min_cacheable ? r : 0;
    hit[i] = h;
    miss[i] = a - h;
    raw_to_written[i] = a - r;
    ti += a;
    th += h;
    tm += a - h;
  }
  ti = warp_sum_u64(ti);
  th = warp_sum_u64(th);
  tm = warp_sum_u64(tm);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&totals[0], ti);
    atomicAdd(&totals[1], th);
    atomicAdd(&totals[2], tm);
  }
}

void replay_report_device(const uint64_t* d_input, uint64_t* d_raw, uint64_t n, uint64_t min_cacheable,
                          uint64_t* d_hit, uint64_t* d_miss, unsigned long long* d_totals,
                          cudaStream_t s) {
  PO_CUDA(cudaMemsetAsync(d_totals, 0, 3 * sizeof(unsigned long long), s));
  PO_LAUNCH(k_replay_report, grid_for(n, 256), 256, 0, s, d_input, d_raw, n, min_cacheable, d_hit,
            d_miss, d_totals);
}

}  // namespace po
