// K9 phc_lcp: Prefix Hit Count of a schedule (objective.hpp:70-99), plus
// the whole-table fixed-order row sort (objective.hpp:154-171) and the
// IEEE-double field rankings (ggr.hpp:59-84, objective.hpp:176-188).

#include <cub/cub.cuh>

#include <algorithm>
#include <numeric>

#include "internal.cuh"

namespace po {

namespace {

// One thread per request i >= first: hit(i) against i-1. Positions are
// evaluated lazily exactly as the reference does, and an out-of-range row or
// field at an evaluated position raises the error flag (std::out_of_range
// from Table::cell's .at(), table.hpp:62-64).
__global__ void k_phc(const uint32_t* __restrict__ vid, const uint64_t* __restrict__ vlen,
                      const uint64_t* __restrict__ colbase, uint64_t n_rows, uint32_t m,
                      uint64_t n_entries, uint64_t first, const uint64_t* rows64,
                      const uint32_t* rows32, const uint64_t* offs, const int32_t* fields,
                      int uniform, unsigned long long* total, int* err) {
  uint64_t local = 0;
  for (uint64_t i = first + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n_entries;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t ra = rows64 ? rows64[i] : rows32[i];
    const uint64_t rb = rows64 ? rows64[i - 1] : rows32[i - 1];
    uint64_t a0, a1, b0, b1;
    if (uniform) {
      a0 = 0;
      a1 = m;
      b0 = 0;
      b1 = m;
    } else if (offs) {
      a0 = offs[i];
      a1 = offs[i + 1];
      b0 = offs[i - 1];
      b1 = a0;
    } else {
      a0 = i * m;
      a1 = a0 + m;
      b0 = a0 - m;
      b1 = a0;
    }
    const uint64_t lim = min(a1 - a0, b1 - b0);
    uint64_t sum = 0;
    for (uint64_t p = 0; p < lim; ++p) {
      const int32_t f = fields[a0 + p];
      if (f != fields[b0 + p]) break;
      if (ra >= n_rows || rb >= n_rows || f < 0 || uint32_t(f) >= m) {
        atomicExch(err, 1);
        break;
      }
      const uint32_t va = vid[ra * m + f];
      if (va != vid[rb * m + f]) break;
      const uint64_t l = vlen[colbase[f] + va];
      sum += l * l;
    }
    local += sum;
  }
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long blk = BR(tmp).Sum((unsigned long long)local);
  if (threadIdx.x == 0 && blk) atomicAdd(total, blk);
}

}  // namespace

__global__ void k_invert(const uint32_t* pos, uint64_t n, uint32_t* perm) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x)
    perm[pos[r]] = uint32_t(r);
}

uint64_t phc_device(const Encoded& e, uint64_t n_entries, const uint64_t* rows64,
                    const uint32_t* rows32, const uint64_t* order_offsets, const int32_t* fields,
                    cudaStream_t s, uint64_t first_entry, bool uniform_order) {
  if (n_entries <= first_entry) return 0;
  DevBuf<unsigned long long> tot(1, s);
  DevBuf<int> err(1, s);
  tot.zero();
  err.zero();
  PO_LAUNCH(k_phc, grid_for(n_entries, 256, 8), 256, 0, s, e.vid.get(), e.vlen.get(),
            e.d_colbase.get(), e.n, e.m, n_entries, first_entry, rows64, rows32, order_offsets,
            fields, uniform_order ? 1 : 0, tot.get(), err.get());
  unsigned long long h = 0;
  int herr = 0;
  tot.download(&h, 1);
  err.download(&herr, 1);
  sync(s);
  if (herr) fail(PO_ERR_OUT_OF_RANGE, "schedule references a row or field outside the table");
  return h;
}

// Keys of a single leaf covering all rows (one field order, escaped ranks),
// packed into 64-bit chunks next to the group id.
FixedOrderSort::FixedOrderSort(const Encoded& e, const std::vector<int>& order, cudaStream_t s)
    : n_(e.n), s_(s) {
  if (n_ == 0) return;
  KeySchedule ks;
  std::vector<std::pair<int, uint8_t>> keys;
  for (int f : order) keys.push_back({f, uint8_t(1)});  // escaped ranks
  // one round-0 group (index 0, start 0); later rounds: start positions < n
  // rounds >= 1 sort inside groups: their chunks may use all 64 bits
  const uint32_t nch = ks.add_leaf(keys, e.card, int(refine_chunk_bits(0)), 64);
  ks.pad();
  std::vector<uint32_t> leaf_chunk_off{0}, leaf_nchunks{nch};
  lco_ = to_device(leaf_chunk_off, s);
  lnc_ = to_device(leaf_nchunks, s);
  cko_ = to_device(ks.chunk_key_off, s);
  cnk_ = to_device(ks.chunk_nkeys, s);
  kf_ = to_device(ks.key_field, s);
  kk_ = to_device(ks.key_kind, s);
  kb_ = to_device(ks.key_bits, s);
  row_leaf_.alloc(n_, s);
  grp_.alloc(n_, s);
  pos_.alloc(n_, s);
  start_.alloc(1, s);
  row_leaf_.zero();
  grp_.zero();
  start_.zero();
  job_.n_items = uint32_t(n_);
  job_.d_grp_init = grp_.get();
  job_.d_grp_start = start_.get();
  job_.n_groups = 1;
  job_.grp_max = uint32_t(n_);
  job_.d_out_pos = pos_.get();
  job_.row_chunk_bits0 = ks.widest0;
  job_.row_chunk_bits = ks.widest;
  RefineKey& K = job_.key;
  K.kind = 2;
  K.m = e.m;
  K.vid = e.vid.get();
  K.colbase = e.d_colbase.get();
  K.row_leaf = row_leaf_.get();
  K.leaf_chunk_off = lco_.get();
  K.leaf_nchunks = lnc_.get();
  K.chunk_key_off = cko_.get();
  K.chunk_nkeys = cnk_.get();
  K.key_field = kf_.get();
  K.key_kind = kk_.get();
  K.key_bits = kb_.get();
}

void FixedOrderSort::finish(uint32_t* d_perm) {
  if (n_) PO_LAUNCH(k_invert, grid_for(n_, 256), 256, 0, s_, pos_.get(), n_, d_perm);
}

void sort_all_rows(const Encoded& e, const std::vector<int>& order, uint32_t* d_perm,
                   cudaStream_t s) {
  FixedOrderSort fs(e, order, s);
  if (e.n == 0) return;
  refine_sort_multi({fs.job()}, s);
  fs.finish(d_perm);
}

// fixed_order_by_hitcount_stats (ggr.hpp:59-84): host IEEE double; this
// translation unit is compiled without FMA contraction (see build flags).
std::vector<int> hitcount_order(uint64_t total_rows, const std::vector<uint64_t>& card,
                                const std::vector<double>& avg, int variant) {
  const size_t k = card.size();
  std::vector<double> score(k, 0.0);
  for (size_t f = 0; f < k; ++f) {
    if (card[f] == 0) continue;
    volatile double ratio = static_cast<double>(total_rows) / static_cast<double>(card[f]);
    volatile double sq = avg[f] * avg[f];
    if (variant == PO_STATS_WEIGHTED) score[f] = sq * (ratio - 1.0);
    else if (variant == PO_STATS_SQUARED) score[f] = sq;
    else score[f] = avg[f] * ratio;
  }
  std::vector<int> idx(k);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return score[a] > score[b]; });
  return idx;
}

// fixed_order_by_stats (objective.hpp:176-188): ASL * rows / cardinality.
std::vector<int> stats_order(uint64_t total_rows, const std::vector<uint64_t>& card,
                             const std::vector<double>& avg) {
  const size_t k = card.size();
  std::vector<double> score(k, 0.0);
  for (size_t f = 0; f < k; ++f) {
    if (card[f] == 0) continue;
    volatile double ratio = static_cast<double>(total_rows) / static_cast<double>(card[f]);
    score[f] = avg[f] * ratio;
  }
  std::vector<int> idx(k);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return score[a] > score[b]; });
  return idx;
}

}  // namespace po
