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
// packed into 64-bit chunks.
void sort_all_rows(const Encoded& e, const std::vector<int>& order, uint32_t* d_perm,
                   cudaStream_t s) {
  const uint64_t n = e.n;
  if (n == 0) return;
  std::vector<uint32_t> chunk_key_off, chunk_nkeys;
  std::vector<int32_t> key_field;
  std::vector<uint8_t> key_kind, key_bits;
  // later rounds use start positions (< n) as group ids
  const int cap_bits = int(refine_chunk_bits(uint32_t(n)));
  int used = cap_bits;
  for (int f : order) {
    int b = bits_for(e.card[f] ? e.card[f] - 1 : 0);
    if (used + b > cap_bits) {
      chunk_key_off.push_back(uint32_t(key_field.size()));
      chunk_nkeys.push_back(0);
      used = 0;
    }
    key_field.push_back(f);
    key_kind.push_back(1);
    key_bits.push_back(uint8_t(b));
    chunk_nkeys.back()++;
    used += b;
  }
  std::vector<uint32_t> leaf_chunk_off{0}, leaf_nchunks{uint32_t(chunk_nkeys.size())};
  if (chunk_nkeys.empty()) {  // keep device arrays non-empty
    chunk_key_off.push_back(0);
    chunk_nkeys.push_back(0);
    key_field.push_back(0);
    key_kind.push_back(1);
    key_bits.push_back(1);
  }
  auto d_lco = to_device(leaf_chunk_off, s), d_lnc = to_device(leaf_nchunks, s);
  auto d_cko = to_device(chunk_key_off, s), d_cnk = to_device(chunk_nkeys, s);
  auto d_kf = to_device(key_field, s);
  auto d_kk = to_device(key_kind, s), d_kb = to_device(key_bits, s);
  DevBuf<uint32_t> row_leaf(n, s), grp(n, s), pos(n, s);
  row_leaf.zero();
  grp.zero();
  RefineKey K;
  K.kind = 2;
  K.m = e.m;
  K.vid = e.vid.get();
  K.esc_rank = e.esc_rank.get();
  K.colbase = e.d_colbase.get();
  K.row_leaf = row_leaf.get();
  K.leaf_chunk_off = d_lco.get();
  K.leaf_nchunks = d_lnc.get();
  K.chunk_key_off = d_cko.get();
  K.chunk_nkeys = d_cnk.get();
  K.key_field = d_kf.get();
  K.key_kind = d_kk.get();
  K.key_bits = d_kb.get();
  refine_sort(uint32_t(n), grp.get(), uint32_t(n), K, pos.get(), s);
  PO_LAUNCH(k_invert, grid_for(n, 256), 256, 0, s, pos.get(), n, d_perm);
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
