// Stable merge sort of small records on the device (the K3 small-job string
// sorts: (group, 14-symbol prefix) records whose comparator falls back to the
// string bytes, and the 128-bit round-0 keys). Replaces
// cub::DeviceMergeSort on those calls (ggr.hpp:196, 223-228; objective.hpp
// escaped-order ranks).
//
//   k_msort_tile   a tile of kMsTile records per block: 7 per thread sorted in
//                  registers (odd-even transposition), then log2(256) in-block
//                  merge rounds in shared memory (merge path, ties to the left)
//   k_msort_merge  one pass per doubling of the run width: each block emits
//                  kMsTile outputs of one run pair; the warp finds the block's
//                  two merge-path splits by a 32-way search in global memory,
//                  stages both input ranges in shared memory and every thread
//                  merges its 7 outputs there
// Stability: the register network and every merge take the left element on ties,
// so equal records keep their input order.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace po {

// 7 records per thread: a tile of 24-byte records (1792 x 24 B = 42 KB) fits
// the default shared-memory limit
constexpr uint32_t kMsThreads = 256, kMsItems = 7, kMsTile = kMsThreads * kMsItems;

// Merge path: number of A elements among the first d outputs of the stable
// merge of A[0, la) and B[0, lb).
template <class T, class Less>
__device__ __forceinline__ uint32_t ms_split(const T* A, uint32_t la, const T* B, uint32_t lb,
                                             uint32_t d, const Less& less) {
  uint32_t lo = d > lb ? d - lb : 0, hi = d < la ? d : la;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (less(B[d - 1 - mid], A[mid])) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// The same split found by a whole warp: each round probes 32 candidates at
// once (one dependent global load round per 5 bits of the range).
template <class T, class Less>
__device__ __forceinline__ uint32_t ms_split_warp(const T* A, uint32_t la, const T* B, uint32_t lb,
                                                  uint32_t d, const Less& less, uint32_t lane) {
  uint32_t lo = d > lb ? d - lb : 0, hi = d < la ? d : la;
  // invariant: the split is in [lo, hi]; pred(i) = less(B[d-1-i], A[i]) is
  // monotone (false...false true...true) and the split = first i with pred
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t i = lo + lane * step;
    const bool p = i < hi ? less(B[d - 1 - i], A[i]) : true;
    const unsigned m = __ballot_sync(0xffffffffu, p);
    const uint32_t f = m ? uint32_t(__ffs(m) - 1) : 32u;  // first lane whose probe is true
    const uint32_t nlo = f == 0 ? lo : lo + (f - 1) * step + 1;
    const uint32_t nhi = f == 32 ? hi : (lo + f * step < hi ? lo + f * step : hi);
    lo = nlo;
    hi = nhi;
  }
  const uint32_t i = lo + lane;
  const bool p = i < hi ? less(B[d - 1 - i], A[i]) : true;
  const unsigned m = __ballot_sync(0xffffffffu, p);
  return lo + (m ? uint32_t(__ffs(m) - 1) : 32u);
}

// Sequential stable merge of k outputs starting at split (i, j).
template <class T, class Less, int K>
__device__ __forceinline__ void ms_merge_run(const T* A, uint32_t la, const T* B, uint32_t lb,
                                             uint32_t i, uint32_t j, const Less& less, T (&out)[K],
                                             uint32_t count) {
#pragma unroll
  for (int t = 0; t < K; ++t) {
    if (uint32_t(t) >= count) break;
    const bool takeA = i < la && (j >= lb || !less(B[j], A[i]));
    out[t] = takeA ? A[i] : B[j];
    if (takeA) ++i;
    else ++j;
  }
}

template <class T, class Less>
__global__ void __launch_bounds__(kMsThreads) k_msort_tile(T* data, uint32_t n, Less less) {
  extern __shared__ __align__(16) uint8_t ms_smem[];
  T* sm = reinterpret_cast<T*>(ms_smem);
  const uint64_t base = uint64_t(blockIdx.x) * kMsTile;
  const uint32_t c = uint32_t(n - base < kMsTile ? n - base : kMsTile);
  for (uint32_t k = threadIdx.x; k < c; k += kMsThreads) sm[k] = data[base + k];
  __syncthreads();
  // kMsItems consecutive records per thread, sorted in registers
  T r[kMsItems];
  const uint32_t my0 = threadIdx.x * kMsItems;
  const uint32_t mine = my0 < c ? (c - my0 < kMsItems ? c - my0 : kMsItems) : 0;
#pragma unroll
  for (uint32_t t = 0; t < kMsItems; ++t)
    if (t < mine) r[t] = sm[my0 + t];
  // odd-even transposition network (static indices: registers), swapping
  // only strictly decreasing neighbours: stable
#pragma unroll
  for (uint32_t round = 0; round < kMsItems; ++round) {
#pragma unroll
    for (uint32_t t = round & 1; t + 1 < kMsItems; t += 2) {
      if (t + 1 < mine && less(r[t + 1], r[t])) {
        const T x = r[t];
        r[t] = r[t + 1];
        r[t + 1] = x;
      }
    }
  }
  __syncthreads();
  for (uint32_t t = 0; t < mine; ++t) sm[my0 + t] = r[t];
  __syncthreads();
  for (uint32_t w = kMsItems; w < kMsTile; w *= 2) {
    // this thread's outputs of the merged pair of w-runs it falls in
    const uint32_t start = (my0 / (2 * w)) * (2 * w);
    const uint32_t a0 = start < c ? start : c, a1 = start + w < c ? start + w : c;
    const uint32_t b1 = start + 2 * w < c ? start + 2 * w : c;
    const uint32_t la = a1 - a0, lb = b1 - a1;
    const uint32_t d = my0 - start;
    T o[kMsItems];
    uint32_t cnt = 0;
    if (my0 < c) {
      cnt = mine;
      const uint32_t i = ms_split(sm + a0, la, sm + a1, lb, d, less);
      ms_merge_run<T, Less, kMsItems>(sm + a0, la, sm + a1, lb, i, d - i, less, o, cnt);
    }
    __syncthreads();
    for (uint32_t t = 0; t < cnt; ++t) sm[my0 + t] = o[t];
    __syncthreads();
  }
  for (uint32_t k = threadIdx.x; k < c; k += kMsThreads) data[base + k] = sm[k];
}

template <class T, class Less>
__global__ void __launch_bounds__(kMsThreads) k_msort_merge(const T* __restrict__ src,
                                                            T* __restrict__ dst, uint32_t n,
                                                            uint32_t w, Less less) {
  extern __shared__ __align__(16) uint8_t ms_smem[];
  T* sm = reinterpret_cast<T*>(ms_smem);
  __shared__ uint32_t s_split[2];
  const uint64_t o0 = uint64_t(blockIdx.x) * kMsTile;  // first output of this block
  const uint64_t pair = o0 / (2ull * w);
  const uint64_t start = pair * 2ull * w;
  const uint32_t a0 = uint32_t(start), a1 = uint32_t(start + w < n ? start + w : n);
  const uint32_t b1 = uint32_t(start + 2ull * w < n ? start + 2ull * w : n);
  const uint32_t la = a1 - a0, lb = b1 - a1;
  const uint32_t d0 = uint32_t(o0 - start);
  const uint32_t d1 = d0 + kMsTile < la + lb ? d0 + kMsTile : la + lb;
  const T* A = src + a0;
  const T* B = src + a1;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 2) {
    const uint32_t s = ms_split_warp(A, la, B, lb, warp == 0 ? d0 : d1, less, lane);
    if (lane == 0) s_split[warp] = s;
  }
  __syncthreads();
  const uint32_t i0 = s_split[0], i1 = s_split[1];
  const uint32_t j0 = d0 - i0, j1 = d1 - i1;
  const uint32_t na = i1 - i0, nb = j1 - j0;
  for (uint32_t k = threadIdx.x; k < na; k += kMsThreads) sm[k] = A[i0 + k];
  for (uint32_t k = threadIdx.x; k < nb; k += kMsThreads) sm[na + k] = B[j0 + k];
  __syncthreads();
  const uint32_t my0 = threadIdx.x * kMsItems, total = d1 - d0;
  if (my0 < total) {
    const uint32_t cnt = total - my0 < kMsItems ? total - my0 : kMsItems;
    const uint32_t i = ms_split(sm, na, sm + na, nb, my0, less);
    T o[kMsItems];
    ms_merge_run<T, Less, kMsItems>(sm, na, sm + na, nb, i, my0 - i, less, o, cnt);
    for (uint32_t t = 0; t < cnt; ++t) dst[start + d0 + my0 + t] = o[t];
  }
}

// Stable sort of data[0, n) by less; tmp holds n records. The result is in
// data.
template <class T, class Less>
void stable_merge_sort(T* data, T* tmp, uint32_t n, Less less, cudaStream_t s) {
  if (n <= 1) return;
  static_assert(kMsTile * sizeof(T) + 64 <= 48 * 1024, "tile must fit the default shared memory");
  const size_t smem = size_t(kMsTile) * sizeof(T);
  const uint32_t tiles = (n + kMsTile - 1) / kMsTile;
  PO_LAUNCH((k_msort_tile<T, Less>), tiles, kMsThreads, smem, s, data, n, less);
  T* a = data;
  T* b = tmp;
  for (uint64_t w = kMsTile; w < n; w *= 2) {
    PO_LAUNCH((k_msort_merge<T, Less>), tiles, kMsThreads, smem, s, a, b, n, uint32_t(w), less);
    T* x = a;
    a = b;
    b = x;
  }
  if (a != data) PO_CUDA(cudaMemcpyAsync(data, a, size_t(n) * sizeof(T), cudaMemcpyDeviceToDevice, s));
}

}  // namespace po
