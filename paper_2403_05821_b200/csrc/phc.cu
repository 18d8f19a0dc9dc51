// K9 phc_lcp: Prefix Hit Count of a schedule (objective.hpp:70-99), plus
// the whole-table fixed-order row sort (objective.hpp:154-171) and the
// IEEE-double field rankings (ggr.hpp:59-84, objective.hpp:176-188).

#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <map>
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

void phc_device_raw_async(const uint32_t* vid, const uint64_t* vlen, const uint64_t* colbase,
                          uint64_t n_rows, uint32_t m, uint64_t n_entries, const uint64_t* rows64,
                          const uint32_t* rows32, const uint64_t* order_offsets,
                          const int32_t* fields, cudaStream_t s, unsigned long long* d_tot,
                          int* d_err, uint64_t first_entry, bool uniform_order) {
  PO_CUDA(cudaMemsetAsync(d_tot, 0, sizeof(unsigned long long), s));
  PO_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), s));
  if (n_entries <= first_entry) return;
  PO_LAUNCH(k_phc, grid_for(n_entries, 256, 8), 256, 0, s, vid, vlen, colbase, n_rows, m,
            n_entries, first_entry, rows64, rows32, order_offsets, fields, uniform_order ? 1 : 0,
            d_tot, d_err);
}

uint64_t phc_device_raw(const uint32_t* vid, const uint64_t* vlen, const uint64_t* colbase,
                        uint64_t n_rows, uint32_t m, uint64_t n_entries, const uint64_t* rows64,
                        const uint32_t* rows32, const uint64_t* order_offsets,
                        const int32_t* fields, cudaStream_t s, uint64_t first_entry,
                        bool uniform_order) {
  if (n_entries <= first_entry) return 0;
  struct R {
    unsigned long long tot;
    int err, pad;
  };
  DevBuf<R> res(1, s);
  phc_device_raw_async(vid, vlen, colbase, n_rows, m, n_entries, rows64, rows32, order_offsets,
                       fields, s, &res.get()->tot, &res.get()->err, first_entry, uniform_order);
  R h{};
  d2h_sync(&h, res.get(), sizeof(R), s);
  if (h.err) fail(PO_ERR_OUT_OF_RANGE, "schedule references a row or field outside the table");
  return h.tot;
}

uint64_t phc_device(const Encoded& e, uint64_t n_entries, const uint64_t* rows64,
                    const uint32_t* rows32, const uint64_t* order_offsets, const int32_t* fields,
                    cudaStream_t s, uint64_t first_entry, bool uniform_order) {
  return phc_device_raw(e.vid.get(), e.vlen.get(), e.d_colbase.get(), e.n, e.m, n_entries, rows64,
                        rows32, order_offsets, fields, s, first_entry, uniform_order);
}

// PHC of the whole table sorted by one fixed field order, without sorting.
// In a lexicographic order the rows sharing a prefix (v1..vp) are
// contiguous, so the adjacent pairs that hit field p are exactly |G|-1 per
// prefix group G of depth p, each scoring len(v_p)^2:
//   PHC = sum_p sum_{G at depth p} (|G|-1) len(v_p)^2
//       = sum_p ( sum_rows len(v_p(row))^2 - sum_{G at depth p} len(v_p(G))^2 ).
// Prefix groups are refined one field at a time with an exact hash table on
// (group, value id); a group's id is its table slot. Sums wrap mod 2^64 like
// the reference's uint64 accumulator, so the identity holds bit-exactly.
// The row order itself is only materialised when the fallback wins.
namespace {

constexpr unsigned long long kFbEmpty = ~0ull;

__global__ void k_fb_init(const uint32_t* vid, uint64_t n, uint32_t m, uint32_t f, uint32_t* gid) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x)
    gid[r] = vid[r * m + f];
}

// depth 1: value ids are the groups; sum over the column's dictionary of
// (count - 1) * len^2
__global__ void k_fb_first(const uint32_t* count, const uint64_t* vlen, uint64_t card,
                           unsigned long long* acc) {
  unsigned long long local = 0;
  for (uint64_t v = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; v < card;
       v += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t l = vlen[v];
    local += uint64_t(count[v] - 1) * (l * l);
  }
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  const unsigned long long blk = BR(tmp).Sum(local);
  if (threadIdx.x == 0 && blk) atomicAdd(acc, blk);
}

__global__ void k_fb_depth(const uint32_t* vid, uint64_t n, uint32_t m, uint32_t f,
                           const uint64_t* vlen_col, uint32_t* gid, unsigned long long* keys,
                           uint64_t mask, unsigned long long* acc, const unsigned long long* ng_prev,
                           unsigned long long* ng) {
  if (*ng_prev == n) {  // every group a singleton: no deeper hits
    if (blockIdx.x == 0 && threadIdx.x == 0) *ng = n;
    return;
  }
  unsigned long long sum = 0, fresh = 0;
  auto probe = [&](unsigned long long key, unsigned long long sq) -> uint32_t {
    uint64_t slot = fmix64(key) & mask;
    for (;;) {
      unsigned long long k = keys[slot];
      if (k == kFbEmpty) {
        k = atomicCAS(&keys[slot], kFbEmpty, key);
        if (k == kFbEmpty) {  // first row of a new group
          ++fresh;
          sum -= sq;
          break;
        }
      }
      if (k == key) break;
      slot = (slot + 1) & mask;
    }
    sum += sq;
    return uint32_t(slot);
  };
  // two rows per iteration: both rows' gathers are in flight before either
  // probes the table
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n; r += 2 * stride) {
    const uint64_t r2 = r + stride;
    const bool two = r2 < n;
    const uint32_t v = vid[r * m + f];
    const uint32_t v2 = two ? vid[r2 * m + f] : 0u;
    const unsigned long long key = (uint64_t(gid[r]) << 32) | v;
    const unsigned long long key2 = two ? ((uint64_t(gid[r2]) << 32) | v2) : 0ull;
    const uint64_t l = vlen_col[v], l2 = two ? vlen_col[v2] : 0;
    gid[r] = probe(key, l * l);
    if (two) gid[r2] = probe(key2, l2 * l2);
  }
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  const unsigned long long bs = BR(tmp).Sum(sum);
  __syncthreads();
  const unsigned long long bf = BR(tmp).Sum(fresh);
  if (threadIdx.x == 0) {
    if (bs) atomicAdd(acc, bs);
    if (bf) atomicAdd(ng, bf);
  }
}

}  // namespace

namespace {
// sum over the distinct values of (count - 1) * len^2, in double
__global__ void k_fb_bound(const uint32_t* __restrict__ count, const uint64_t* __restrict__ vlen,
                           uint64_t D, double* out) {
  double local = 0;
  for (uint64_t d = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; d < D;
       d += uint64_t(gridDim.x) * blockDim.x) {
    const double l = double(vlen[d]);
    local += double(count[d] - 1) * l * l;
  }
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  const double b = BR(tmp).Sum(local);
  if (threadIdx.x == 0 && b > 0) atomicAdd(out, b);
}
}  // namespace

// The whole-table fallback's PHC is at most sum_f sum_v (count(v) - 1) *
// len(v)^2: at every prefix depth the pairs hitting field f inside groups
// whose last value is v number at most count(v) - 1. When that bound is below
// 2^64 (no wraparound) and not above the recursion's PHC, the fallback cannot
// be strictly better (ggr.hpp:383) and its PHC / sort are skipped. Every term
// is computed in double; the relative error of the sum is below 1e-9.
void fallback_ub_async(const Encoded& e, cudaStream_t s, double* d_ub) {
  PO_CUDA(cudaMemsetAsync(d_ub, 0, sizeof(double), s));
  if (e.D == 0) return;
  PO_LAUNCH(k_fb_bound, grid_for(e.D, 256, 4), 256, 0, s, e.count.get(), e.vlen.get(), e.D, d_ub);
}

bool fallback_bound_prunes(const Encoded& e, double ub, uint64_t phc) {
  if (e.D == 0) return true;
  const double ub_hi = ub * (1.0 + 1e-9) + 1.0;
  return ub_hi < 1.8e19 && ub_hi < double(phc) * (1.0 - 1e-15);
}

bool fallback_cannot_win(const Encoded& e, uint64_t phc, cudaStream_t s) {
  if (e.D == 0) return true;
  DevBuf<double> acc(1, s);
  fallback_ub_async(e, s, acc.get());
  double ub = 0;
  d2h_sync(&ub, acc.get(), sizeof(double), s);
  return fallback_bound_prunes(e, ub, phc);
}

void fixed_order_phc_async(const Encoded& e, const std::vector<int>& order, cudaStream_t s,
                           unsigned long long* d_acc) {
  const uint64_t n = e.n;
  const uint32_t m = e.m;
  PO_CUDA(cudaMemsetAsync(d_acc, 0, sizeof(unsigned long long), s));
  if (n < 2 || order.empty()) return;
  const std::vector<uint64_t>& colbase = e.colbase;
  const int f0 = order[0];
  PO_LAUNCH(k_fb_first, grid_for(e.card[f0], 256, 4), 256, 0, s, e.count.get() + colbase[f0],
            e.vlen.get() + colbase[f0], uint64_t(e.card[f0]), d_acc);
  if (order.size() > 1 && e.card[f0] < n) {
    uint64_t cap = 1;
    while (cap < 2 * n) cap <<= 1;
    if (cap > (1ull << 32)) fail(PO_ERR_SIZE, "table too large for the fallback group table");
    DevBuf<uint32_t> gid = dev_auto<uint32_t>(n, s);
    DevBuf<unsigned long long> keys = dev_auto<unsigned long long>(cap, s);
    DevBuf<unsigned long long> ng(order.size(), s);
    ng.zero();
    const unsigned long long c0 = e.card[f0];
    h2d_async(ng.get(), &c0, sizeof(c0), s);
    PO_LAUNCH(k_fb_init, grid_for(n, 256), 256, 0, s, e.vid.get(), n, m, uint32_t(f0), gid.get());
    for (size_t p = 1; p < order.size(); ++p) {
      const int f = order[p];
      // a unique column splits every group into singletons: no hits from here
      if (e.card[f] == n) break;
      keys.fill_bytes(0xFF);
      PO_LAUNCH(k_fb_depth, grid_for(n, 256, 8), 256, 0, s, e.vid.get(), n, m, uint32_t(f),
                e.vlen.get() + colbase[f], gid.get(), keys.get(), cap - 1, d_acc,
                ng.get() + (p - 1), ng.get() + p);
    }
  }
}

uint64_t fixed_order_phc_device(const Encoded& e, const std::vector<int>& order, cudaStream_t s) {
  if (e.n < 2 || order.empty()) return 0;
  DevBuf<unsigned long long> acc(1, s);
  fixed_order_phc_async(e, order, s, acc.get());
  unsigned long long h = 0;
  d2h_sync(&h, acc.get(), sizeof(h), s);
  return h;
}

namespace {

// Run heads of the tie-break: position q starts a run unless the row before
// it (same leaf) agrees on every ranked key of the leaf. Non-tie leaves:
// every position its own run.
__global__ void k_tie_heads(const uint32_t* perm, uint64_t n, uint32_t m,
                            const uint32_t* __restrict__ vid, const uint32_t* row_leaf,
                            const uint32_t* leaf_off, const int32_t* tie_col,
                            const uint32_t* key_off, const int32_t* key_fields, uint32_t* head) {
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < n;
       q += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = perm[q], l = row_leaf[r];
    bool start = tie_col[l] < 0 || q == leaf_off[l];
    if (!start) {
      const uint32_t rp = perm[q - 1];
      for (uint32_t k = key_off[l]; k < key_off[l + 1]; ++k) {
        const int32_t f = key_fields[k];
        if (vid[uint64_t(rp) * m + f] != vid[uint64_t(r) * m + f]) {
          start = true;
          break;
        }
      }
    }
    head[q] = start ? uint32_t(q) : 0u;
  }
}

struct MaxOp {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const {
    return a > b ? a : b;
  }
};

// run_len[start] of every run (written at its last position)
__global__ void k_run_len(const uint32_t* run, uint64_t n, uint32_t* run_len) {
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < n;
       q += uint64_t(gridDim.x) * blockDim.x)
    if (q + 1 == n || run[q + 1] != run[q]) run_len[run[q]] = uint32_t(q - run[q] + 1);
}

// work of the quadratic long-run ranking: sum of squared long-run lengths
// (and work[1] = the longest run)
__global__ void k_long_work(const uint32_t* run, const uint32_t* run_len, uint64_t n,
                            uint32_t max_short, unsigned long long* work) {
  unsigned long long local = 0, mx = 0;
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < n;
       q += uint64_t(gridDim.x) * blockDim.x)
    if (run[q] == q && run_len[q] > max_short) {
      local += uint64_t(run_len[q]) * run_len[q];
      mx = max(mx, (unsigned long long)run_len[q]);
    }
  for (int o = 16; o; o >>= 1) {
    local += __shfl_down_sync(0xffffffffu, local, o);
    mx = max(mx, __shfl_down_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0 && local) {
    atomicAdd(work, local);
    atomicMax(work + 1, mx);
  }
}

// positions in runs longer than max_short (left to the refine job)
__global__ void k_tie_flags(const uint32_t* run, const uint32_t* run_len, uint64_t n,
                            uint32_t max_short, uint8_t* flag) {
  for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < n;
       q += uint64_t(gridDim.x) * blockDim.x)
    flag[q] = run_len[run[q]] > (max_short > 1 ? max_short : 1);
}

__global__ void k_tie_items(const uint32_t* items, uint32_t nt, const uint32_t* perm,
                            const uint32_t* run, const uint32_t* row_leaf, const int32_t* tie_col,
                            const uint32_t* vid, const uint64_t* colbase, uint32_t m,
                            uint32_t* t_row, uint32_t* t_grp, uint32_t* t_ref) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nt; k += gridDim.x * blockDim.x) {
    const uint32_t q = items[k], r = perm[q];
    const uint32_t c = uint32_t(tie_col[row_leaf[r]]);
    t_row[k] = r;
    t_grp[k] = run[q];
    t_ref[k] = uint32_t(colbase[c] + vid[uint64_t(r) * m + c]);  // the cell's distinct value
  }
}

__global__ void k_tie_scatter(const uint32_t* t_row, const uint32_t* t_pos, uint32_t nt,
                              uint32_t* pos) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nt; k += gridDim.x * blockDim.x)
    pos[t_row[k]] = t_pos[k];
}

}  // namespace

// PO_SHORT_RUN_MAX: longest tied run ranked by direct comparisons (default 32)
uint32_t short_run_max() {
  const char* e = std::getenv("PO_SHORT_RUN_MAX");
  return e && *e ? uint32_t(std::atoi(e)) : 32u;
}

// PO_LONG_RUN_BUDGET: largest sum of squared long-run lengths ranked by
// direct counting (default 2^29, a few tenths of a ms at most); above it a sort.
uint64_t long_run_budget() {
  const char* e = std::getenv("PO_LONG_RUN_BUDGET");
  return e && *e ? uint64_t(std::strtoull(e, nullptr, 10)) : (1ull << 29);
}

// Values of an unranked column are distinct (one per row), so after this
// every tied run is totally ordered, as a sort by the column's escaped rank
// would order it.
void break_unranked_ties(const Encoded& e, const TieSpec& ts, const uint32_t* row_leaf,
                         const uint32_t* d_leaf_off, uint32_t* pos, cudaStream_t s) {
  const uint64_t n = e.n;
  if (n < 2 || !ts.any()) return;
  auto d_tc = to_device(ts.tie_col, s);
  auto d_ko = to_device(ts.key_off, s);
  std::vector<int32_t> kf = ts.key_fields;
  if (kf.empty()) kf.push_back(0);
  auto d_kf = to_device(kf, s);
  DevBuf<uint32_t> perm = dev_auto<uint32_t>(n, s), run = dev_auto<uint32_t>(n, s),
                   items = dev_auto<uint32_t>(n, s);
  PO_LAUNCH(k_invert, grid_for(n, 256), 256, 0, s, pos, n, perm.get());
  timing_mark("ties_setup", s);
  PO_LAUNCH(k_tie_heads, grid_for(n, 256), 256, 0, s, perm.get(), n, e.m, e.vid.get(), row_leaf,
            d_leaf_off, d_tc.get(), d_ko.get(), d_kf.get(), run.get());
  size_t tb = 0;
  PO_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, run.get(), run.get(), MaxOp(), int(n), s));
  {
    DevBuf<uint8_t> tmp(tb, s);
    PO_CUDA(cub::DeviceScan::InclusiveScan(tmp.get(), tb, run.get(), run.get(), MaxOp(), int(n), s));
  }
  // short runs: each position ranks itself against its run (quadratic, no
  // sort); long runs: a kind-1 string refine job
  const uint32_t max_short = short_run_max();
  DevBuf<uint32_t> run_len = dev_auto<uint32_t>(n, s);
  PO_LAUNCH(k_run_len, grid_for(n, 256), 256, 0, s, run.get(), n, run_len.get());
  timing_mark("ties_runs", s);
  const CellStr cs = cell_str(e);
  rank_short_runs(cs, perm.get(), run.get(), run_len.get(), row_leaf, d_tc.get(), n, max_short,
                  pos, s);
  timing_mark("ties_short", s);
  DevBuf<uint8_t> flag(n, s);
  PO_LAUNCH(k_tie_flags, grid_for(n, 256), 256, 0, s, run.get(), run_len.get(), n, max_short,
            flag.get());
  DevBuf<int> nsel(1, s);
  cub::CountingInputIterator<uint32_t> it(0);
  tb = 0;
  PO_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, flag.get(), items.get(), nsel.get(), int(n), s));
  {
    DevBuf<uint8_t> tmp(tb, s);
    PO_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, it, flag.get(), items.get(), nsel.get(),
                                       int(n), s));
  }
  const uint32_t ms = max_short > 1 ? max_short : 1;
  DevBuf<unsigned long long> work(2, s);
  work.zero();
  PO_LAUNCH(k_long_work, grid_for(n, 256), 256, 0, s, run.get(), run_len.get(), n, ms, work.get());
  int hn = 0;
  unsigned long long hw[2] = {0, 0};
  PO_CUDA(cudaMemcpyAsync(&hn, nsel.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  PO_CUDA(cudaMemcpyAsync(hw, work.get(), sizeof(hw), cudaMemcpyDeviceToHost, s));
  sync(s);
  const uint32_t nt = uint32_t(hn);
  if (debug_timing()) {
    std::vector<uint32_t> hr(n), hl(n);
    PO_CUDA(cudaMemcpyAsync(hr.data(), run.get(), n * 4, cudaMemcpyDeviceToHost, s));
    PO_CUDA(cudaMemcpyAsync(hl.data(), run_len.get(), n * 4, cudaMemcpyDeviceToHost, s));
    sync(s);
    std::map<uint32_t, uint64_t> hist;  // log2 bucket -> runs
    uint32_t mx = 0;
    for (uint64_t q = 0; q < n; ++q)
      if (hr[q] == q && hl[q] > 1) {
        hist[31 - __builtin_clz(hl[q])]++;
        mx = std::max(mx, hl[q]);
      }
    fprintf(stderr, "[po ties] %u positions in long runs; max run %u; runs by log2 len:", nt, mx);
    for (auto& kv : hist) fprintf(stderr, " %u:%llu", kv.first, (unsigned long long)kv.second);
    fprintf(stderr, "\n");
  }
  if (nt == 0) return;
  if (hw[0] <= long_run_budget()) {  // quadratic per run, no sort
    rank_long_runs(cs, perm.get(), run.get(), run_len.get(), row_leaf, d_tc.get(), items.get(), nt,
                   n, uint32_t(hw[1]), pos, s);
    return;
  }
  DevBuf<uint32_t> t_row(nt, s), t_grp(nt, s), t_col(nt, s), t_pos(nt, s);
  PO_LAUNCH(k_tie_items, grid_for(nt, 256), 256, 0, s, items.get(), nt, perm.get(), run.get(),
            row_leaf, d_tc.get(), e.vid.get(), e.d_colbase.get(), e.m, t_row.get(), t_grp.get(),
            t_col.get());
  RefineJob tj;
  tj.n_items = nt;
  tj.d_grp_init = t_grp.get();  // run start positions
  tj.grp_max = uint32_t(n);
  tj.key.kind = 1;  // escaped bytes: the order of the column's ranks
  tj.key.arena = e.val_arena;
  tj.key.arena_bytes = e.val_bytes;
  tj.key.str_off = e.val_off.get();
  tj.key.str_len = e.val_len.get();
  tj.key.item_ref = t_col.get();
  tj.d_out_pos = t_pos.get();
  refine_sort_multi({tj}, s);
  PO_LAUNCH(k_tie_scatter, grid_for(nt, 256), 256, 0, s, t_row.get(), t_pos.get(), nt, pos);
}

// Keys of a single leaf covering all rows (one field order, escaped ranks),
// packed into 64-bit chunks next to the group id.
FixedOrderSort::FixedOrderSort(const Encoded& e, const std::vector<int>& order, cudaStream_t s)
    : e_(e), n_(e.n), s_(s) {
  if (n_ == 0) return;
  KeySchedule ks;
  std::vector<std::pair<int, uint8_t>> keys;
  ties_.tie_col.assign(1, -1);
  for (int f : order) {
    if (e.is_unranked(f)) {  // distinct per row: its bytes break the remaining ties
      ties_.tie_col[0] = f;
      break;
    }
    keys.push_back({f, uint8_t(1)});  // escaped ranks
    ties_.key_fields.push_back(f);
  }
  ties_.key_off.push_back(uint32_t(ties_.key_fields.size()));
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
  if (n_) break_unranked_ties(e_, ties_, row_leaf_.get(), start_.get(), pos_.get(), s_);
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
