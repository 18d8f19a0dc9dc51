// Shared device/host helpers for the sm_100a GGR + PHC path.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <chrono>
#include <cstring>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/prefixopt_cuda.h"

namespace po {

// ---------------------------------------------------------------------------
// errors: mapped to PO_ERR_* at the ABI boundary (abi.cu)
// ---------------------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    fail(PO_ERR_ERROR, std::string("CUDA error in ") + what + " (" + file + ":" +
                           std::to_string(line) + "): " + cudaGetErrorString(e));
}
#define PO_CUDA(x) ::po::cuda_check((x), #x, __FILE__, __LINE__)

extern std::atomic<uint64_t> g_launches;
extern std::atomic<int> g_profile;

// Per-kernel CUDA-event timing (po_profile_enable / po_profile_report):
// events recorded on the launching stream around each launch.
void profile_begin(const char* name, cudaStream_t s, void** token);
void profile_end(void* token, cudaStream_t s);

// Times a library call (CUB building blocks) like a kernel when profiling.
struct ProfScope {
  void* tok = nullptr;
  cudaStream_t s;
  ProfScope(const char* name, cudaStream_t st) : s(st) {
    if (g_profile.load(std::memory_order_relaxed)) profile_begin(name, st, &tok);
  }
  ~ProfScope() {
    if (tok) profile_end(tok, s);
  }
};

// Host wall time of a section (profile mode only, no synchronisation):
// reported as "host:<name>" next to the kernels.
void profile_host(const char* name, double ms);
struct HostScope {
  const char* name;
  std::chrono::steady_clock::time_point t0;
  bool on;
  explicit HostScope(const char* n) : name(n), on(g_profile.load(std::memory_order_relaxed)) {
    if (on) t0 = std::chrono::steady_clock::now();
  }
  ~HostScope() {
    if (on)
      profile_host(name, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};

// Every kernel of this library is launched through PO_LAUNCH so bench.py can
// report how many of OUR kernels ran (po_kernel_launch_count) and time them.
#define PO_LAUNCH(kernel, grid, block, smem, stream, ...)                    \
  do {                                                                       \
    if ((grid) > 0) {                                                        \
      void* po_tok_ = nullptr;                                               \
      if (::po::g_profile.load(std::memory_order_relaxed))                   \
        ::po::profile_begin(#kernel, (stream), &po_tok_);                    \
      kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);            \
      ::po::g_launches.fetch_add(1, std::memory_order_relaxed);              \
      PO_CUDA(cudaGetLastError());                                           \
      if (po_tok_) ::po::profile_end(po_tok_, (stream));                     \
    }                                                                        \
  } while (0)

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

inline unsigned grid_for(uint64_t work, unsigned block, unsigned max_waves = 16) {
  uint64_t g = (work + block - 1) / block;
  uint64_t cap = uint64_t(kSMs) * max_waves * (1024 / block);
  if (g > cap) g = cap;
  return unsigned(g);
}

// Small host->device copies (per-level descriptors, key schedules, column
// tables) are staged through a per-thread pinned arena so cudaMemcpyAsync
// stays asynchronous (a copy from pageable memory may synchronise the
// stream and stall the launch queue). Larger copies (caller data) go direct.
constexpr size_t kPinnedSmallCopy = 1 << 20;
void h2d_async(void* dst, const void* src, size_t bytes, cudaStream_t s);
// device -> host copy, then the stream synchronised (pinned bounce buffer)
void d2h_sync(void* dst, const void* src, size_t bytes, cudaStream_t s,
              const char* file = __builtin_FILE(), int line = __builtin_LINE());

// Large transient buffers (the dictionary tables, per-cell arrays) come from
// a per-device cache of cudaMalloc'd blocks that are never returned to the
// driver: a block is reused by the next call that needs one of about its size
// (the new stream waits on an event recorded where the block was released),
// so repeated calls map no memory. Returns the block's pointer.
void* cached_block_acquire(size_t bytes, cudaStream_t s);
void cached_block_release(void* p, cudaStream_t s);

// ---------------------------------------------------------------------------
// stream-ordered device buffer (cudaMallocAsync on the call's stream)
// ---------------------------------------------------------------------------
template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t s) { alloc(n, s); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      s_ = o.s_;
      cached_ = o.cached_;
      o.p_ = nullptr;
      o.n_ = 0;
      o.cached_ = false;
    }
    return *this;
  }
  // Buffers of 16 MB and more come from the block cache (identical sizes
  // recur call after call, so steady-state calls map no memory and the two
  // allocators never compete for the same GBs), smaller ones from the
  // stream-ordered pool.
  void alloc(size_t n, cudaStream_t s) {
    if (n * sizeof(T) >= (16u << 20)) {
      alloc_cached(n, s);
      return;
    }
    release();
    s_ = s;
    n_ = n;
    if (n) PO_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T) + 64, s));
  }
  void alloc_auto(size_t n, cudaStream_t s) { alloc(n, s); }
  // the same from the block cache (cached_block_acquire)
  void alloc_cached(size_t n, cudaStream_t s) {
    release();
    s_ = s;
    n_ = n;
    if (n) {
      p_ = static_cast<T*>(cached_block_acquire(n * sizeof(T) + 64, s));
      cached_ = true;
    }
  }
  void zero() {
    if (n_) PO_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s_));
  }
  void fill_bytes(int v) {
    if (n_) PO_CUDA(cudaMemsetAsync(p_, v, n_ * sizeof(T), s_));
  }
  void release() {
    if (p_) {
      if (cached_) cached_block_release(p_, s_);
      else cudaFreeAsync(p_, s_);
    }
    p_ = nullptr;
    n_ = 0;
    cached_ = false;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  void upload(const T* h, size_t n) {
    if (n) h2d_async(p_, h, n * sizeof(T), s_);
  }
  void download(T* h, size_t n) const {
    if (n) PO_CUDA(cudaMemcpyAsync(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost, s_));
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t s_ = nullptr;
  bool cached_ = false;
};

// a buffer from alloc_auto (block cache when large)
template <class T>
DevBuf<T> dev_auto(size_t n, cudaStream_t s) {
  DevBuf<T> b;
  b.alloc_auto(n, s);
  return b;
}

template <class T>
DevBuf<T> to_device(const std::vector<T>& v, cudaStream_t s) {
  DevBuf<T> d(v.size(), s);
  d.upload(v.data(), v.size());
  return d;
}

extern thread_local uint64_t g_syncs;  // host synchronisations of this thread (debug timing)
bool debug_syncs();  // PO_DEBUG_SYNCS=1: print the call site of every stream sync
inline void sync(cudaStream_t s, const char* file = __builtin_FILE(), int line = __builtin_LINE()) {
  HostScope hs("sync");
  ++g_syncs;
  if (debug_syncs()) fprintf(stderr, "[po sync] %s:%d\n", file, line);
  PO_CUDA(cudaStreamSynchronize(s));
}

// Host wall-time breakdown of one call (PO_DEBUG_TIMING=1): synchronises the
// stream at every mark, so it perturbs the timing it reports; debug only.
bool debug_timing();
void timing_mark(const char* phase, cudaStream_t s);
void timing_report(const char* call);

inline int bits_for(uint64_t max_value) {  // bits to hold values 0..max_value
  int b = 0;
  while (b < 64 && (max_value >> b)) ++b;
  return b == 0 ? 1 : b;
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

__device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

// Sequential reader of an arbitrarily aligned byte string as little-endian
// 8-byte words, using only 8-byte-aligned loads that never start at or past
// `limit` (the end of the arena), so no load leaves the allocation.
struct WordReader {
  const uint64_t* p;
  const uint64_t* lim;  // first aligned word that starts at/after the arena end
  uint32_t sh;
  uint64_t cur;
  __device__ __forceinline__ WordReader(const uint8_t* a, const uint8_t* limit) {
    uintptr_t ad = reinterpret_cast<uintptr_t>(a);
    p = reinterpret_cast<const uint64_t*>(ad & ~uintptr_t(7));
    lim = reinterpret_cast<const uint64_t*>((reinterpret_cast<uintptr_t>(limit) + 7) & ~uintptr_t(7));
    sh = uint32_t(ad & 7) * 8;
    cur = p < lim ? __ldg(p) : 0;
  }
  __device__ __forceinline__ uint64_t next() {
    const uint64_t* q = p + 1;
    uint64_t nxt = q < lim ? __ldg(q) : 0;
    uint64_t w = sh ? ((cur >> sh) | (nxt << (64 - sh))) : cur;
    cur = nxt;
    p = q;
    return w;
  }
};

__device__ __forceinline__ uint64_t mask_low_bytes(uint64_t w, uint32_t nbytes) {
  return nbytes >= 8 ? w : (w & ((uint64_t(1) << (8 * nbytes)) - 1));
}

// 64-bit hash of a cell's bytes (value identity for the dictionary; exact
// equality is always verified on the bytes, so quality only affects speed).
// h = fmix64(len*C + sum_k term(word_k, k)) over the cell's 8-byte words
// (little-endian, zero-padded), so a warp can hash a long cell cooperatively
// (lane l takes words l, l+32, ...) and get the same value as one lane.
__device__ __forceinline__ uint64_t word_term(uint64_t w, uint64_t k) {
  const uint64_t x = (w ^ (k * 0x9E3779B97F4A7C15ULL)) * 0xff51afd7ed558ccdULL;
  return x ^ (x >> 32);
}

__device__ __forceinline__ uint64_t hash_finish(uint64_t sum, uint64_t len) {
  uint64_t h = fmix64(sum + len * 0xC2B2AE3D27D4EB4FULL);
  return h ? h : 1;  // 0 marks an empty slot
}

__device__ __forceinline__ uint64_t hash_bytes(const uint8_t* a, uint64_t len, const uint8_t* limit) {
  uint64_t sum = 0;
  if (len) {
    WordReader rd(a, limit);
    uint64_t left = len;
    for (uint64_t k = 0; left; ++k) {
      uint32_t take = left >= 8 ? 8u : uint32_t(left);
      sum += word_term(mask_low_bytes(rd.next(), take), k);
      left -= take;
    }
  }
  return hash_finish(sum, len);
}

// 8 bytes at an arbitrary address (two aligned loads, none past `limit`).
__device__ __forceinline__ uint64_t load8_unaligned(const uint8_t* a, const uint8_t* limit) {
  const uintptr_t ad = reinterpret_cast<uintptr_t>(a);
  const uint64_t* p = reinterpret_cast<const uint64_t*>(ad & ~uintptr_t(7));
  const uint64_t* lim =
      reinterpret_cast<const uint64_t*>((reinterpret_cast<uintptr_t>(limit) + 7) & ~uintptr_t(7));
  const uint32_t sh = uint32_t(ad & 7) * 8;
  const uint64_t w0 = p < lim ? __ldg(p) : 0;
  if (!sh) return w0;
  const uint64_t w1 = (p + 1) < lim ? __ldg(p + 1) : 0;
  return (w0 >> sh) | (w1 << (64 - sh));
}

// Index of the first byte where a[0, n) and b[0, n) differ, or n. 32 bytes
// per step with every load of the step issued before the first compare (a
// per-8-byte loop waits a full load latency per step on long common
// prefixes).
__device__ __forceinline__ uint64_t first_diff(const uint8_t* a, const uint8_t* b, uint64_t n,
                                               const uint8_t* limit) {
  for (uint64_t t = 0; t < n; t += 32) {
    uint64_t x[4], y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool in = t + 8 * u < n;
      x[u] = in ? load8_unaligned(a + t + 8 * u, limit) : 0;
      y[u] = in ? load8_unaligned(b + t + 8 * u, limit) : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t tt = t + 8 * u;
      if (tt >= n) return n;
      const uint64_t d = mask_low_bytes(x[u] ^ y[u], n - tt >= 8 ? 8u : uint32_t(n - tt));
      if (d) return tt + uint64_t(__ffsll((long long)d) - 1) / 8;
    }
  }
  return n;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Whole-warp hash of one cell (same value as hash_bytes). All lanes call it
// with the same (a, len) and all receive the hash.
__device__ __forceinline__ uint64_t warp_hash_bytes(const uint8_t* a, uint64_t len,
                                                    const uint8_t* limit, uint32_t lane) {
  const uint64_t words = (len + 7) / 8;
  uint64_t sum = 0;
  for (uint64_t k = lane; k < words; k += 32) {
    const uint64_t rem = len - 8 * k;
    sum += word_term(mask_low_bytes(load8_unaligned(a + 8 * k, limit), rem >= 8 ? 8u : uint32_t(rem)), k);
  }
  return hash_finish(warp_sum_u64(sum), len);
}

// Whole-warp byte compare: all loads issued before any result is used
// (no early exit), 2 words per lane per step.
__device__ __forceinline__ bool warp_bytes_equal(const uint8_t* a, const uint8_t* b, uint64_t len,
                                                 const uint8_t* limit, uint32_t lane) {
  uint64_t diff = 0;
  const uint64_t words = (len + 7) / 8;
  for (uint64_t k0 = 0; k0 < words; k0 += 64) {
    const uint64_t k1 = k0 + lane, k2 = k0 + 32 + lane;
    uint64_t a1 = 0, b1 = 0, a2 = 0, b2 = 0;
    if (k1 < words) {
      a1 = load8_unaligned(a + 8 * k1, limit);
      b1 = load8_unaligned(b + 8 * k1, limit);
    }
    if (k2 < words) {
      a2 = load8_unaligned(a + 8 * k2, limit);
      b2 = load8_unaligned(b + 8 * k2, limit);
    }
    if (k1 < words) {
      const uint64_t rem = len - 8 * k1;
      const uint32_t take = rem >= 8 ? 8u : uint32_t(rem);
      diff |= mask_low_bytes(a1 ^ b1, take);
    }
    if (k2 < words) {
      const uint64_t rem = len - 8 * k2;
      const uint32_t take = rem >= 8 ? 8u : uint32_t(rem);
      diff |= mask_low_bytes(a2 ^ b2, take);
    }
  }
  return __all_sync(0xffffffffu, diff == 0);
}

__device__ __forceinline__ bool bytes_equal(const uint8_t* a, const uint8_t* b, uint64_t len,
                                            const uint8_t* limit) {
  if (a == b || len == 0) return true;
  WordReader ra(a, limit), rb(b, limit);
  uint64_t left = len;
  while (left) {
    uint32_t take = left >= 8 ? 8u : uint32_t(left);
    uint64_t wa = mask_low_bytes(ra.next(), take);
    uint64_t wb = mask_low_bytes(rb.next(), take);
    if (wa != wb) return false;
    left -= take;
  }
  return true;
}

// ---- TMA bulk copy (cp.async.bulk) + mbarrier helpers (sm_90+/sm_100a) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

typedef unsigned __int128 u128;

}  // namespace po
