// K8 multikey_sort engine: a hand-written onesweep LSD radix sort of
// (u64 key, u32 value) pairs, stable, over key bits [begin_bit, end_bit).
// Replaces cub::DeviceRadixSort in the row-key and string refine rounds
// (refine.cu) and the sharded layout sort (shard.cu): the sorts behind
// ggr.hpp:221-231, 340-350 and objective.hpp:156-166.
//
// Design (one pass per 8-bit digit):
//   * k_radix_hist reads the keys once and builds the digit histograms of
//     every pass (shared-memory atomics; the hardware combines lanes of a
//     warp that add to one bin); the last block to finish turns them into
//     digit offsets;
//   * k_radix_pass: a tile of 256 x 20 items per block (tiles taken in order
//     from an atomic counter). Each warp ranks its 640 items stably (32 at a
//     time: __match_any_sync groups lanes with the same digit; a per-warp
//     shared histogram gives the running offset), the block combines the
//     warps' counts, and one thread per digit finds the digit's count in all
//     earlier tiles by decoupled look-back over (flag, value) status words
//     (aggregate / inclusive prefix), so the whole pass is a single read and
//     a single scatter of the pairs.
// Within a tile the item order is (warp, round, lane) = input order, across
// tiles the look-back follows tile order: equal digits keep input order and
// LSD passes compose into a stable sort.

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "internal.cuh"

namespace po {

namespace {

constexpr int kRadixBits = 8;
constexpr uint32_t kBins = 1u << kRadixBits;
constexpr uint32_t kHistThreads = 256;
constexpr uint32_t kMaxPasses = 8;
// status word of (tile, digit): flag (2 bits: 1 aggregate, 2 inclusive) |
// pass tag (6 bits: words left by an earlier pass read as "not yet") | value
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 56) - 1;
__device__ __forceinline__ unsigned long long tag_of(uint32_t pass) {
  return (unsigned long long)(pass + 1) << 56;
}

// digit of pass p: key bits [begin + 8p, min(begin + 8p + 8, end))
__device__ __forceinline__ uint32_t digit_of(uint64_t k, int shift, int end) {
  const int w = end - shift < kRadixBits ? end - shift : kRadixBits;
  return uint32_t((k >> shift) & ((1ull << w) - 1));
}

// Digit histograms of every pass in one read of the keys; the last block to
// finish turns them into exclusive digit start offsets (hist[p][d]).
__global__ void __launch_bounds__(kHistThreads) k_radix_hist(const uint64_t* __restrict__ keys,
                                                             uint32_t n, int begin, int end,
                                                             int passes, uint32_t* hist,
                                                             uint32_t* done) {
  // two copies of the bins (even / odd warps); lanes of one warp adding to
  // the same bin are combined by the hardware (ATOMS.POPC.INC), so skewed or
  // constant digits cost one shared atomic per warp
  constexpr uint32_t kParts = 2;
  __shared__ uint32_t sh[kParts][kMaxPasses][kBins];
  __shared__ bool s_last;
  for (uint32_t i = threadIdx.x; i < kParts * kMaxPasses * kBins; i += blockDim.x)
    (&sh[0][0][0])[i] = 0;
  __syncthreads();
  auto& mine = sh[(threadIdx.x >> 5) & (kParts - 1)];
  const uint64_t key_mask = end - begin >= 64 ? ~0ull : (1ull << (end - begin)) - 1;
  constexpr uint32_t kKeys = 4;  // loads in flight per thread
  const uint32_t stride = gridDim.x * blockDim.x * kKeys;
  for (uint32_t base = blockIdx.x * blockDim.x * kKeys; base < n; base += stride) {
    uint64_t k[kKeys];
#pragma unroll
    for (uint32_t q = 0; q < kKeys; ++q) {
      const uint32_t i = base + q * blockDim.x + threadIdx.x;
      k[q] = i < n ? keys[i] : 0;
    }
#pragma unroll
    for (uint32_t q = 0; q < kKeys; ++q) {
      if (base + q * blockDim.x + threadIdx.x >= n) break;
      // digits = bytes of the key shifted down to begin (the last one masked)
      const uint64_t kk = (k[q] >> begin) & key_mask;
      const uint32_t lo = uint32_t(kk), hi = uint32_t(kk >> 32);
#pragma unroll
      for (int p = 0; p < int(kMaxPasses); ++p) {
        if (p >= passes) break;
        atomicAdd(&mine[p][(p < 4 ? lo : hi) >> (8 * (p & 3)) & 0xFF], 1u);
      }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < uint32_t(passes) * kBins; i += blockDim.x) {
    uint32_t v = 0;
#pragma unroll
    for (uint32_t c = 0; c < kParts; ++c) v += (&sh[c][0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // exclusive scan of each pass's 256 counts (kHistThreads == kBins)
  const uint32_t t = threadIdx.x;
  for (int p = 0; p < passes; ++p) {
    uint32_t* h = hist + p * kBins;
    uint32_t* sc = sh[0][0];
    const uint32_t c = __ldcg(h + t);
    sc[t] = c;
    __syncthreads();
    for (uint32_t o = 1; o < kBins; o <<= 1) {  // inclusive Hillis-Steele scan
      const uint32_t x = t >= o ? sc[t - o] : 0;
      __syncthreads();
      sc[t] += x;
      __syncthreads();
    }
    h[t] = sc[t] - c;
    __syncthreads();
  }
}

// One LSD pass over tiles of T * IPT items (T threads, T >= 256): shared
// memory = per-warp digit counts + the tile sorted by digit (dynamic).
template <uint32_t T, uint32_t IPT, uint32_t MINB>
__global__ void __launch_bounds__(T, MINB) k_radix_pass(
    const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint64_t* __restrict__ kout,
    uint32_t* __restrict__ vout, uint32_t n, int shift, int end,
    const uint32_t* __restrict__ digit_off, unsigned long long* status, uint32_t* tile_counter,
    uint32_t pass) {
  constexpr uint32_t W = T / 32, TILE = T * IPT;
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* s_key = reinterpret_cast<uint64_t*>(smem);            // TILE
  uint32_t* s_val = reinterpret_cast<uint32_t*>(s_key + TILE);    // TILE
  uint32_t* whist = s_val + TILE;                                 // W * kBins
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_base[kBins];  // global start of the tile's run of each digit
  __shared__ uint32_t s_loc[kBins];   // start of each digit inside the sorted tile
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (uint32_t i = threadIdx.x; i < W * kBins; i += T) whist[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t first = uint64_t(tile) * TILE + uint64_t(w) * (32 * IPT);
  uint64_t k[IPT];
  uint32_t v[IPT], d[IPT], r[IPT];
#pragma unroll
  for (uint32_t q = 0; q < IPT; ++q) {
    const uint64_t i = first + q * 32 + lane;
    const bool valid = i < n;
    k[q] = valid ? kin[i] : 0;
    v[q] = valid ? vin[i] : 0;
    d[q] = valid ? digit_of(k[q], shift, end) : kBins + lane;  // invalid: never matches
  }
  // stable rank inside the warp's items, round by round
  uint32_t* wh = whist + w * kBins;
#pragma unroll
  for (uint32_t q = 0; q < IPT; ++q) {
    const unsigned peers = __match_any_sync(0xffffffffu, d[q]);
    const int leader = __ffs(peers) - 1;
    const uint32_t before = __popc(peers & ((1u << lane) - 1u));
    uint32_t run = 0;
    if (d[q] < kBins && int(lane) == leader) {
      run = wh[d[q]];
      wh[d[q]] = run + __popc(peers);
    }
    run = __shfl_sync(0xffffffffu, run, leader);
    r[q] = run + before;
    __syncwarp();
  }
  __syncthreads();
  // per digit (threads < 256, whole warps): the tile's count and the warps'
  // prefixes; the count is published at once (successors' look-back), then
  // the digit's start in the sorted tile (shuffle scan) and the look-back for
  // its global start
  __shared__ uint32_t s_wsum[kBins / 32];
  const uint32_t dg = threadIdx.x;
  const unsigned long long tag = tag_of(pass);
  unsigned long long* st = status + uint64_t(tile) * kBins + dg;
  uint32_t cnt = 0, inc = 0;
  if (dg < kBins) {
    for (uint32_t x = 0; x < W; ++x) {
      const uint32_t c = whist[x * kBins + dg];
      whist[x * kBins + dg] = cnt;
      cnt += c;
    }
    atomicExch(st, (tile == 0 ? kFlagInc : kFlagAgg) | tag | cnt);
    inc = cnt;
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_wsum[w] = inc;
  }
  __syncthreads();
  if (dg < kBins) {
    uint32_t loc = inc - cnt;
    for (uint32_t x = 0; x < w; ++x) loc += s_wsum[x];
    uint64_t excl = 0;
    if (tile != 0) {
      for (int64_t prev = int64_t(tile) - 1; prev >= 0; --prev) {
        const unsigned long long* ps = status + uint64_t(prev) * kBins + dg;
        unsigned long long x;
        do {
          x = *reinterpret_cast<const volatile unsigned long long*>(ps);
        } while ((x >> 62) == 0 || (x & (0x3Full << 56)) != tag);
        excl += x & kValMask;
        if ((x >> 62) == 2) break;
      }
      atomicExch(st, kFlagInc | tag | (excl + cnt));
    }
    s_loc[dg] = loc;
    s_base[dg] = digit_off[dg] + uint32_t(excl) - loc;  // global = s_base[d] + sorted index
  }
  __syncthreads();
  // place the tile in shared memory sorted by digit, then write it out in
  // order: the runs of one digit go to consecutive global positions
#pragma unroll
  for (uint32_t q = 0; q < IPT; ++q) {
    if (d[q] >= kBins) continue;
    const uint32_t at = s_loc[d[q]] + wh[d[q]] + r[q];
    s_key[at] = k[q];
    s_val[at] = v[q];
  }
  __syncthreads();
  const uint64_t left = uint64_t(n) - uint64_t(tile) * TILE;
  const uint32_t valid_n = left < TILE ? uint32_t(left) : TILE;
  for (uint32_t at = threadIdx.x; at < valid_n; at += T) {
    const uint64_t key = s_key[at];
    const uint32_t pos = s_base[digit_of(key, shift, end)] + at;
    kout[pos] = key;
    vout[pos] = s_val[at];
  }
}

__global__ void k_copy_pairs(const uint64_t* kin, const uint32_t* vin, uint64_t* kout, uint32_t* vout,
                             uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    kout[i] = kin[i];
    vout[i] = vin[i];
  }
}

}  // namespace

namespace {

using PassFn = void (*)(const uint64_t*, const uint32_t*, uint64_t*, uint32_t*, uint32_t, int, int,
                        const uint32_t*, unsigned long long*, uint32_t*, uint32_t);

struct RadixShape {
  const char* name;
  uint32_t threads, ipt;
  PassFn fn;
  size_t smem;
  template <class... A>
  void launch(uint32_t grid, size_t sm, cudaStream_t s, A... a) const {
    const PassFn k_radix_pass = fn;  // profiled under the kernel's name
    PO_LAUNCH(k_radix_pass, grid, threads, sm, s, a...);
  }
};

template <uint32_t T, uint32_t IPT, uint32_t MINB>
RadixShape shape(const char* name) {
  return {name, T, IPT, &k_radix_pass<T, IPT, MINB>, size_t(T) * IPT * 12 + size_t(T / 32) * kBins * 4};
}

// Tile shape of the pass kernel (PO_RADIX_TILE=TxIPT picks another one for
// experiments); its dynamic shared-memory limit is raised once per device.
const RadixShape& radix_shape() {
  static const std::vector<RadixShape> shapes = {
      shape<256, 20, 2>("256x20"), shape<256, 12, 3>("256x12"), shape<384, 12, 2>("384x12"),
      shape<256, 24, 2>("256x24"), shape<512, 8, 2>("512x8")};
  static const size_t pick = [] {
    const char* v = std::getenv("PO_RADIX_TILE");
    for (size_t i = 0; v && i < shapes.size(); ++i)
      if (std::string(v) == shapes[i].name) return i;
    return size_t(0);
  }();
  static std::mutex mu;
  static std::vector<int> ready;
  int dev = 0;
  PO_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(ready.begin(), ready.end(), dev) == ready.end()) {
    PO_CUDA(cudaFuncSetAttribute(shapes[pick].fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(shapes[pick].smem)));
    ready.push_back(dev);
  }
  return shapes[pick];
}

}  // namespace

void radix_sort_pairs(const uint64_t* kin, uint64_t* kout, const uint32_t* vin, uint32_t* vout,
                      uint32_t n, int begin_bit, int end_bit, cudaStream_t s) {
  if (n == 0) return;
  static const bool use_cub = [] {  // PO_RADIX=cub: the library sort (comparison runs)
    const char* v = std::getenv("PO_RADIX");
    return v && std::string(v) == "cub";
  }();
  if (use_cub) {
    ProfScope ps("cub_radix_sort", s);
    size_t tb = 0;
    PO_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, kout, vin, vout, int(n), begin_bit,
                                            end_bit, s));
    DevBuf<uint8_t> tmp(tb, s);
    PO_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, kin, kout, vin, vout, int(n), begin_bit,
                                            end_bit, s));
    return;
  }
  ProfScope ps("radix_sort", s);
  const int bits = end_bit - begin_bit;
  const int passes = bits > 0 ? (bits + kRadixBits - 1) / kRadixBits : 0;
  if (passes == 0) {
    PO_LAUNCH(k_copy_pairs, grid_for(n, 256), 256, 0, s, kin, vin, kout, vout, n);
    return;
  }
  if (passes > int(kMaxPasses)) fail(PO_ERR_ERROR, "internal: radix sort over more than 64 bits");
  const RadixShape& sh = radix_shape();
  const uint32_t tile_items = sh.threads * sh.ipt;
  const uint32_t tiles = (n + tile_items - 1) / tile_items;
  // one workspace, one memset: digit offsets | tile counters + done flag |
  // status words (zeroed once: later passes tell theirs apart by the tag)
  const size_t hist_words = size_t(passes) * kBins + kMaxPasses + 1;
  const size_t status_off = (hist_words * 4 + 255) / 256 * 256;
  DevBuf<uint8_t> ws(status_off + size_t(tiles) * kBins * 8, s);
  ws.zero();
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws.get());
  uint32_t* counters = hist + size_t(passes) * kBins;
  auto* status = reinterpret_cast<unsigned long long*>(ws.get() + status_off);
  PO_LAUNCH(k_radix_hist, std::min<unsigned>(grid_for(n, kHistThreads * 4), kSMs * 4), kHistThreads, 0,
            s, kin, n, begin_bit, end_bit, passes, hist, counters + kMaxPasses);
  // ping-pong so that the last pass lands in (kout, vout)
  DevBuf<uint64_t> ktmp;
  DevBuf<uint32_t> vtmp;
  if (passes > 1) {
    ktmp.alloc(n, s);
    vtmp.alloc(n, s);
  }
  const uint64_t* ksrc = kin;
  const uint32_t* vsrc = vin;
  for (int p = 0; p < passes; ++p) {
    const bool to_out = ((passes - 1 - p) & 1) == 0;
    uint64_t* kd = to_out ? kout : ktmp.get();
    uint32_t* vd = to_out ? vout : vtmp.get();
    sh.launch(tiles, sh.smem, s, ksrc, vsrc, kd, vd, n, begin_bit + kRadixBits * p, end_bit,
              hist + size_t(p) * kBins, status, counters + p, uint32_t(p));
    ksrc = kd;
    vsrc = vd;
  }
}

}  // namespace po
