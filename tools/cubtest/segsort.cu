// Standalone check of cub::DeviceSegmentedSort::StableSortPairs usage.
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 1000000;
  std::mt19937 rng(1);
  std::vector<uint32_t> seg{0};
  while (seg.back() < (uint32_t)n) { uint32_t sz = (argc > 2) ? (2 + rng() % atoi(argv[2])) : ((rng() % 10 == 0) ? 1000 + rng() % 40000 : 2 + rng() % 60); seg.push_back(std::min<uint32_t>(n, seg.back() + sz)); }
  int nseg = seg.size() - 1;
  std::vector<uint64_t> keys(n); std::vector<uint32_t> vals(n);
  for (int i = 0; i < n; ++i) { keys[i] = (argc > 3) ? ((uint64_t)rng() << 32 | rng()) : ((uint64_t)rng() << 32 | rng()) % 5; vals[i] = i; }
  uint64_t *dk, *dk2; uint32_t *dv, *dv2, *ds;
  cudaMalloc(&dk, n*8); cudaMalloc(&dk2, n*8); cudaMalloc(&dv, n*4); cudaMalloc(&dv2, n*4); cudaMalloc(&ds, (nseg+1)*4);
  cudaMemcpy(dk, keys.data(), n*8, cudaMemcpyHostToDevice); cudaMemcpy(dv, vals.data(), n*4, cudaMemcpyHostToDevice);
  cudaMemcpy(ds, seg.data(), (nseg+1)*4, cudaMemcpyHostToDevice);
  size_t tb = 0;
  cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb, dk, dk2, dv, dv2, n, nseg, ds, ds + 1, 0);
  void* tmp; cudaMalloc(&tmp, tb);
  cudaError_t e = cub::DeviceSegmentedSort::StableSortPairs(tmp, tb, dk, dk2, dv, dv2, n, nseg, ds, ds + 1, 0);
  cudaError_t e2 = cudaDeviceSynchronize();
  std::vector<uint64_t> ok(n); std::vector<uint32_t> ov(n);
  cudaMemcpy(ok.data(), dk2, n*8, cudaMemcpyDeviceToHost); cudaMemcpy(ov.data(), dv2, n*4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int s = 0; s < nseg; ++s) {
    std::vector<std::pair<uint64_t,uint32_t>> v;
    for (uint32_t i = seg[s]; i < seg[s+1]; ++i) v.push_back({keys[i], vals[i]});
    std::stable_sort(v.begin(), v.end(), [](auto&a, auto&b){return a.first<b.first;});
    for (uint32_t i = seg[s]; i < seg[s+1]; ++i) if (ok[i] != v[i-seg[s]].first || ov[i] != v[i-seg[s]].second) ++bad;
  }
  printf("n=%d nseg=%d err=%s/%s bad=%ld\n", n, nseg, cudaGetErrorString(e), cudaGetErrorString(e2), bad);
}
