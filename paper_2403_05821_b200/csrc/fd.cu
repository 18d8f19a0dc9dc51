// Functional-dependency checks on the dictionary.
//
// The reference's partition_signature (fd.hpp:56-64) maps row r of field f to
// the first row holding the same value; validate_fds (fd.hpp:66-109) and
// discover_fds (fd.hpp:114-141) only ever compare two signatures row by row
// and look at the first row where they differ. With exact per-column value
// ids (encode(): vid), sig_f[r] = first_row[f][vid[r][f]] — one atomicMin
// pass over the cells — and the comparison of field pairs is one pass over
// the rows (first differing row by atomicMin). The host side (C++ drop-in
// headers, Python API) keeps the reference's control flow, error checks and
// witness rule on top of these results.

#include "internal.cuh"

namespace po {

namespace {

__global__ void k_first_row(const uint32_t* __restrict__ vid, uint64_t n, uint32_t m,
                            const uint64_t* __restrict__ colbase, const uint8_t* __restrict__ used,
                            uint32_t* first) {
  const uint64_t cells = n * m;
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < cells;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t c = uint32_t(t % m);
    if (!used[c]) continue;
    // values only decrease: a row not below the (possibly stale, never
    // smaller) value read skips the atomic — hot values (a two-valued column)
    // otherwise serialise on one address
    uint32_t* f = &first[colbase[c] + vid[t]];
    const uint32_t r = uint32_t(t / m);
    if (*f > r) atomicMin(f, r);
  }
}

__device__ __forceinline__ uint32_t sig_of(const uint32_t* vid, uint32_t m, const uint64_t* colbase,
                                           const uint32_t* first, uint64_t r, int32_t f) {
  return first[colbase[f] + vid[r * m + f]];
}

// first row where the signatures of pair k differ (diff[k] starts at n)
__global__ void k_pair_diff(const uint32_t* __restrict__ vid, uint64_t n, uint32_t m,
                            const uint64_t* __restrict__ colbase, const uint32_t* __restrict__ first,
                            uint32_t np, const int32_t* __restrict__ pa,
                            const int32_t* __restrict__ pb, unsigned long long* diff) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x)
    for (uint32_t k = 0; k < np; ++k) {
      if (r >= *(volatile unsigned long long*)&diff[k]) continue;  // an earlier row already differs
      if (sig_of(vid, m, colbase, first, r, pa[k]) != sig_of(vid, m, colbase, first, r, pb[k]))
        atomicMin(&diff[k], (unsigned long long)r);
    }
}

__global__ void k_pair_witness(const uint32_t* __restrict__ vid, uint64_t n, uint32_t m,
                               const uint64_t* __restrict__ colbase,
                               const uint32_t* __restrict__ first, uint32_t np,
                               const int32_t* __restrict__ pa, const int32_t* __restrict__ pb,
                               const unsigned long long* diff, uint64_t* sa, uint64_t* sb) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  const uint64_t r = diff[k];
  sa[k] = r < n ? sig_of(vid, m, colbase, first, r, pa[k]) : 0;
  sb[k] = r < n ? sig_of(vid, m, colbase, first, r, pb[k]) : 0;
}

}  // namespace

void fd_compare_device(const Encoded& e, const std::vector<int32_t>& pa,
                       const std::vector<int32_t>& pb, std::vector<uint64_t>& first_diff,
                       std::vector<uint64_t>& sig_a, std::vector<uint64_t>& sig_b, cudaStream_t s) {
  const uint32_t np = uint32_t(pa.size());
  const uint64_t n = e.n;
  const uint32_t m = e.m;
  first_diff.assign(np, n);
  sig_a.assign(np, 0);
  sig_b.assign(np, 0);
  if (np == 0 || n == 0) return;
  std::vector<uint8_t> used(m, 0);
  for (uint32_t k = 0; k < np; ++k) {
    if (pa[k] < 0 || pb[k] < 0 || uint32_t(pa[k]) >= m || uint32_t(pb[k]) >= m)
      fail(PO_ERR_SCHEMA, "FD pair names a field outside the schema");
    used[pa[k]] = used[pb[k]] = 1;
  }
  auto d_used = to_device(used, s);
  auto d_pa = to_device(pa, s), d_pb = to_device(pb, s);
  DevBuf<uint32_t> first(e.D, s);
  first.fill_bytes(0xFF);
  PO_LAUNCH(k_first_row, grid_for(n * m, 256), 256, 0, s, e.vid.get(), n, m, e.d_colbase.get(),
            d_used.get(), first.get());
  std::vector<unsigned long long> init(np, n);
  DevBuf<unsigned long long> diff(np, s);
  diff.upload(init.data(), np);
  PO_LAUNCH(k_pair_diff, grid_for(n, 256), 256, 0, s, e.vid.get(), n, m, e.d_colbase.get(),
            first.get(), np, d_pa.get(), d_pb.get(), diff.get());
  DevBuf<uint64_t> d_sa(np, s), d_sb(np, s);
  PO_LAUNCH(k_pair_witness, (np + 127) / 128, 128, 0, s, e.vid.get(), n, m, e.d_colbase.get(),
            first.get(), np, d_pa.get(), d_pb.get(), diff.get(), d_sa.get(), d_sb.get());
  std::vector<unsigned long long> hd(np);
  diff.download(hd.data(), np);
  d_sa.download(sig_a.data(), np);
  d_sb.download(sig_b.data(), np);
  sync(s);
  for (uint32_t k = 0; k < np; ++k) first_diff[k] = hd[k];
}

}  // namespace po
