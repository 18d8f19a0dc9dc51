// Greedy Group Recursion on the GPU (ggr.hpp:135-394), level-synchronous.
//
// The reference recursion (recurse, ggr.hpp:207-314) is processed one tree
// level at a time. Every live node owns a value-group histogram ("table")
// keyed by (column, vid) with the group's row count and one partner-length
// sum per distinct FD partner of the column:
//   * the root table is dense (index colbase[c] + vid) and comes free from
//     the dictionary counts (K2);
//   * a split's rest child inherits its parent's table and subtracts the
//     block rows (decremental histogram: hist(rest) = hist(parent) -
//     hist(block), exact integer arithmetic);
//   * a split's block child gets a fresh hashed table aggregated from its
//     own rows only.
// Per level: K5 argmax_seg (exact u128 rational argmax with the reference's
// total tie order) over every scanning node's table, a host decision per
// node (early stop / split, ggr.hpp:276-301), K6 split (relabel rows), K4
// group_hist aggregation of block rows, and K7 leaf_stats for every node that
// falls back. After the last level the leaves are laid out in DFS order
// (block before rest, ggr.hpp:303-313) and one K8 multikey row sort orders
// every leaf's rows at once; K10 emits the schedule and K9 scores it. The
// whole-table statistics fallback competes last (ggr.hpp:379-387).

#include <optional>
#include <cub/cub.cuh>
#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>

#include "comm.cuh"
#include "internal.cuh"

namespace cg = cooperative_groups;

namespace po {

namespace {

// ---------------------------------------------------------------------------
// tables
// ---------------------------------------------------------------------------
struct TDesc {
  unsigned long long* keys;  // hashed: (c+1)<<32 | vid, 0 = empty; null for dense
  uint32_t* cnt;
  unsigned long long* psum;  // cap * K
  uint64_t cap;
  uint32_t dense;
  uint32_t pad;
};

struct HTable {
  bool dense = false;
  uint64_t cap = 0;
  unsigned long long* keys = nullptr;
  uint32_t* cnt = nullptr;
  unsigned long long* psum = nullptr;
  std::shared_ptr<DevBuf<uint8_t>> mem;  // backing allocation (shared by a level's tables)
  TDesc desc() const { return TDesc{keys, cnt, psum, cap, dense ? 1u : 0u, 0u}; }
};

// The hashed tables ts (cap set) carved out of ONE zeroed allocation: a
// level's new tables cost one cudaMallocAsync and one memset instead of three
// of each per table (host launch overhead between the level's syncs).
void alloc_tables(const std::vector<HTable*>& ts, uint32_t K, cudaStream_t s) {
  if (ts.empty()) return;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  size_t total = 0;
  for (const HTable* t : ts) total += al(t->cap * 8) + al(t->cap * 4) + (K ? al(t->cap * K * 8) : 0);
  auto mem = std::make_shared<DevBuf<uint8_t>>(total, s);
  {
    ProfScope ps("memset_tables", s);
    mem->zero();
  }
  uint8_t* p = mem->get();
  for (HTable* t : ts) {
    t->keys = reinterpret_cast<unsigned long long*>(p);
    p += al(t->cap * 8);
    t->cnt = reinterpret_cast<uint32_t*>(p);
    p += al(t->cap * 4);
    if (K) {
      t->psum = reinterpret_cast<unsigned long long*>(p);
      p += al(t->cap * K * 8);
    }
    t->mem = mem;
  }
}

__device__ __forceinline__ uint64_t tkey_hash(unsigned long long k) { return fmix64(k); }

__device__ __forceinline__ uint64_t tbl_insert(const TDesc& t, unsigned long long key) {
  uint64_t s = tkey_hash(key) & (t.cap - 1);
  for (;;) {
    unsigned long long k = t.keys[s];
    if (k == key) return s;
    if (k == 0) {
      unsigned long long prev = atomicCAS(&t.keys[s], 0ull, key);
      if (prev == 0 || prev == key) return s;
    }
    s = (s + 1) & (t.cap - 1);
  }
}

__device__ __forceinline__ uint64_t tbl_find(const TDesc& t, unsigned long long key) {
  uint64_t s = tkey_hash(key) & (t.cap - 1);
  for (;;) {
    unsigned long long k = t.keys[s];
    if (k == key || k == 0) return s;  // 0 cannot happen for a present key
    s = (s + 1) & (t.cap - 1);
  }
}

__device__ __forceinline__ uint32_t col_of_dense(const uint64_t* colbase, uint32_t m, uint64_t e) {
  uint32_t lo = 0, hi = m;  // largest c with colbase[c] <= e
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (colbase[mid] <= e) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Decodes table entry e into (column, vid); false when the slot is empty.
__device__ __forceinline__ bool decode_entry(const TDesc& t, const uint64_t* colbase, uint32_t m,
                                             uint64_t e, uint32_t& c, uint32_t& v) {
  if (t.dense) {
    c = col_of_dense(colbase, m, e);
    v = uint32_t(e - colbase[c]);
    return true;
  }
  unsigned long long k = t.keys[e];
  if (!k) return false;
  c = uint32_t(k >> 32) - 1;
  v = uint32_t(k);
  return true;
}

__device__ __forceinline__ bool mask_has(const uint32_t* mask, uint32_t c) {
  return (mask[c >> 5] >> (c & 31)) & 1u;
}

// ---------------------------------------------------------------------------
// K5 argmax_seg
// ---------------------------------------------------------------------------
struct Cand {
  u128 numer;
  uint64_t count;  // 0 = no candidate
  uint32_t col;
  uint32_t vid;
  uint64_t ties;   // entries sharing this (score, count, column) key
  uint64_t pad;
};

// Candidate::better_than (ggr.hpp:189-197) up to its last criterion: exact
// rational compare of numer/count via u128 cross products (wrapping exactly
// like the reference), then larger count, then lower column. Entries equal on
// that key are merged and counted; the final tie-break — smaller raw bytes —
// is resolved afterwards on the tied values only (vids are ranks in the
// escaped order, not in raw-byte order). The merge is associative and
// commutative, so any reduction order gives the same result.
__host__ __device__ __forceinline__ Cand merge(const Cand& a, const Cand& b) {
  if (a.count == 0) return b;
  if (b.count == 0) return a;
  const u128 l = a.numer * u128(b.count), r = b.numer * u128(a.count);
  if (l != r) return l > r ? a : b;
  if (a.count != b.count) return a.count > b.count ? a : b;
  if (a.col != b.col) return a.col < b.col ? a : b;
  Cand c = a;
  c.ties = a.ties + b.ties;
  c.vid = a.vid < b.vid ? a.vid : b.vid;
  return c;
}

__device__ __forceinline__ bool same_key(const Cand& a, const Cand& b) {
  return a.count == b.count && a.col == b.col && a.numer == b.numer;
}

__device__ __forceinline__ Cand shfl_cand(const Cand& a, int delta) {
  Cand o;
  uint64_t lo = uint64_t(a.numer), hi = uint64_t(a.numer >> 64);
  lo = __shfl_down_sync(0xffffffffu, lo, delta);
  hi = __shfl_down_sync(0xffffffffu, hi, delta);
  o.numer = (u128(hi) << 64) | lo;
  o.count = __shfl_down_sync(0xffffffffu, a.count, delta);
  o.col = __shfl_down_sync(0xffffffffu, a.col, delta);
  o.vid = __shfl_down_sync(0xffffffffu, a.vid, delta);
  o.ties = __shfl_down_sync(0xffffffffu, a.ties, delta);
  o.pad = 0;
  return o;
}

struct ScanSlot {
  TDesc t;
  uint32_t mask_off;  // into level colmask words
  uint32_t w_off;     // into level partner weights (m*K per slot)
};

struct WorkItem {
  uint32_t slot;
  uint32_t col;  // dense tables: the one column of [lo, hi); hashed: kAnyCol
  uint64_t lo, hi;
};

constexpr uint32_t kAnyCol = 0xFFFFFFFFu;

// A slot's scan of one table (or one dense column) as consecutive work items
// of kWorkChunk entries; first = the item number of its first item.
struct WorkSeg {
  uint32_t slot, col;
  uint64_t lo, hi;
  uint32_t first, pad;
};
constexpr uint64_t kWorkChunk = 2048;

// This block's work item: the last segment with first <= blockIdx.x.
__device__ __forceinline__ WorkItem work_at(const WorkSeg* __restrict__ segs, uint32_t nseg) {
  uint32_t lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) / 2;
    if (segs[mid].first <= blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const WorkSeg& g = segs[lo];
  const uint64_t a = g.lo + uint64_t(blockIdx.x - g.first) * kWorkChunk;
  return WorkItem{g.slot, g.col, a, a + kWorkChunk < g.hi ? a + kWorkChunk : g.hi};
}

__device__ __forceinline__ bool decode_work(const WorkItem& w, const TDesc& t,
                                            const uint64_t* colbase, uint32_t m, uint64_t e,
                                            uint32_t& c, uint32_t& v) {
  if (w.col != kAnyCol) {
    c = w.col;
    v = uint32_t(e - colbase[c]);
    return true;
  }
  return decode_entry(t, colbase, m, e, c, v);
}

constexpr int kArgBlock = 256;

// Sharded solve: which rank scans an entry of a replicated table. Dense
// tables have the same layout on every rank: whole work items are dealt out
// (item i to rank i % nparts, the others skip it without reading it). A
// hashed table holds the same keys on every rank but at slot positions that
// depend on the insertion order, so its entries are dealt out by identity:
// (colbase[c] + vid) % nparts.
__device__ __forceinline__ bool item_skipped(const TDesc& t, uint32_t part, uint32_t nparts) {
  return nparts > 1 && t.dense && blockIdx.x % nparts != part;
}
__device__ __forceinline__ bool entry_skipped(const TDesc& t, const uint64_t* colbase, uint32_t c,
                                              uint32_t v, uint32_t part, uint32_t nparts) {
  return nparts > 1 && !t.dense && (colbase[c] + v) % nparts != part;
}

template <int MINB>
__global__ void __launch_bounds__(kArgBlock, MINB) k_argmax(
    const WorkSeg* __restrict__ work, uint32_t nwseg, const ScanSlot* __restrict__ slots,
    const uint32_t* __restrict__ masks, const uint32_t* __restrict__ weights,
    const uint64_t* __restrict__ colbase, const uint64_t* __restrict__ vlen, uint32_t m,
    uint32_t K, Cand* partial, unsigned long long* partial_cands, uint32_t part, uint32_t nparts) {
  // sharded solve: the replicated tables' work items are split over the
  // ranks (item i on rank i % nparts); the per-slot results are merged
  // across ranks afterwards (merge is associative and commutative)
  const WorkItem w = work_at(work, nwseg);
  const ScanSlot sl = slots[w.slot];
  if (item_skipped(sl.t, part, nparts)) {
    if (threadIdx.x == 0) {
      partial[blockIdx.x] = Cand{};
      partial_cands[blockIdx.x] = 0;
    }
    return;
  }
  const uint32_t* mask = masks + sl.mask_off;
  const uint32_t* wt = weights + sl.w_off;
  Cand best{};
  unsigned long long ncand = 0;
  for (uint64_t e = w.lo + threadIdx.x; e < w.hi; e += blockDim.x) {
    uint32_t c, v;
    if (!decode_work(w, sl.t, colbase, m, e, c, v)) continue;
    const uint32_t cnt = sl.t.cnt[e];
    if (cnt == 0 || !mask_has(mask, c) || entry_skipped(sl.t, colbase, c, v, part, nparts)) continue;
    ++ncand;
    const uint64_t vl = vlen[colbase[c] + v];
    uint64_t ptot = 0;
    for (uint32_t k = 0; k < K; ++k)
      if (wt[c * K + k]) ptot += uint64_t(wt[c * K + k]) * sl.t.psum[e * K + k];
    // hitcount numerator (ggr.hpp:261-266)
    Cand cd;
    cd.numer = (u128(vl) * vl * cnt + ptot) * u128(cnt - 1);
    cd.count = cnt;
    cd.col = c;
    cd.vid = v;
    cd.ties = 1;
    cd.pad = 0;
    best = merge(best, cd);
  }
  // block reduction (any order: merge is associative and commutative)
  for (int d = 16; d > 0; d >>= 1) {
    best = merge(best, shfl_cand(best, d));
    ncand += __shfl_down_sync(0xffffffffu, ncand, d);
  }
  __shared__ Cand sb[kArgBlock / 32];
  __shared__ unsigned long long sc[kArgBlock / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    sb[wid] = best;
    sc[wid] = ncand;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Cand b = sb[0];
    unsigned long long n = sc[0];
    for (int i = 1; i < kArgBlock / 32; ++i) {
      b = merge(b, sb[i]);
      n += sc[i];
    }
    partial[blockIdx.x] = b;
    partial_cands[blockIdx.x] = n;
  }
}

// Every entry of a tied slot whose (score, count, column) key equals the
// slot's best: its value is appended to the slot's segment for the raw-byte
// tie-break (ggr.hpp:196).
__global__ void k_collect_ties(const WorkSeg* __restrict__ work, uint32_t nwseg, const ScanSlot* __restrict__ slots,
                               const uint32_t* __restrict__ masks,
                               const uint32_t* __restrict__ weights,
                               const uint64_t* __restrict__ colbase,
                               const uint64_t* __restrict__ vlen, uint32_t m, uint32_t K,
                               const Cand* __restrict__ best, const int32_t* __restrict__ tie_group,
                               const uint32_t* __restrict__ tie_off, uint32_t* cursor,
                               uint32_t* t_ref, uint32_t* t_vid, uint32_t* t_grp) {
  const WorkItem w = work_at(work, nwseg);
  const int32_t g = tie_group[w.slot];
  if (g < 0) return;
  const ScanSlot sl = slots[w.slot];
  const uint32_t* mask = masks + sl.mask_off;
  const uint32_t* wt = weights + sl.w_off;
  const Cand b = best[w.slot];
  for (uint64_t e = w.lo + threadIdx.x; e < w.hi; e += blockDim.x) {
    uint32_t c, v;
    if (!decode_work(w, sl.t, colbase, m, e, c, v)) continue;
    const uint32_t cnt = sl.t.cnt[e];
    if (cnt != b.count || c != b.col || !mask_has(mask, c)) continue;
    const uint64_t vl = vlen[colbase[c] + v];
    uint64_t ptot = 0;
    for (uint32_t k = 0; k < K; ++k)
      if (wt[c * K + k]) ptot += uint64_t(wt[c * K + k]) * sl.t.psum[e * K + k];
    if ((u128(vl) * vl * cnt + ptot) * u128(cnt - 1) != b.numer) continue;
    const uint32_t at = tie_off[g] + atomicAdd(&cursor[g], 1u);
    t_ref[at] = uint32_t(colbase[c] + v);
    t_vid[at] = v;
    t_grp[at] = uint32_t(g);
  }
}

// After the raw-byte sort of each tie group: the value at the group's first
// position is the smallest.
__global__ void k_pick_min(const uint32_t* pos, const uint32_t* t_grp, const uint32_t* t_vid,
                           const uint32_t* tie_off, uint32_t total, uint32_t* min_vid) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x)
    if (pos[i] == tie_off[t_grp[i]]) min_vid[t_grp[i]] = t_vid[i];
}

// Rows of single-column leaves (ggr.hpp:221-231), for their raw-byte sort.
__global__ void k_raw1_flags(const uint32_t* row_leaf, uint64_t n, const int32_t* leaf_raw1_col,
                             uint8_t* flags) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x)
    flags[r] = leaf_raw1_col[row_leaf[r]] >= 0 ? 1 : 0;
}

__global__ void k_raw1_items(const uint32_t* rows, uint32_t cnt, const uint32_t* row_leaf,
                             const int32_t* leaf_raw1_col, const uint32_t* vid,
                             const uint64_t* colbase, uint32_t m, uint32_t* grp, uint32_t* ref) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x) {
    const uint32_t r = rows[k];
    const uint32_t l = row_leaf[r];
    const uint32_t c = uint32_t(leaf_raw1_col[l]);
    grp[k] = l;
    ref[k] = uint32_t(colbase[c] + vid[uint64_t(r) * m + c]);  // the cell's distinct value
  }
}

__global__ void k_raw1_scatter(const uint32_t* rows, const uint32_t* raw_pos, uint32_t cnt,
                               uint32_t* pos) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x)
    pos[rows[k]] = raw_pos[k];
}

// Sharded solve: tie-break by the global raw-byte rank (rv, per global dense
// index): per tie group the entry with the smallest (raw rank, vid).
__global__ void k_tie_min_raw(const WorkSeg* __restrict__ work, uint32_t nwseg, const ScanSlot* __restrict__ slots,
                              const uint32_t* __restrict__ masks,
                              const uint32_t* __restrict__ weights,
                              const uint64_t* __restrict__ colbase,
                              const uint64_t* __restrict__ vlen, uint32_t m, uint32_t K,
                              const Cand* __restrict__ best, const int32_t* __restrict__ tie_group,
                              const uint32_t* __restrict__ rv, unsigned long long* minkey,
                              uint32_t part, uint32_t nparts) {
  const WorkItem w = work_at(work, nwseg);
  const int32_t g = tie_group[w.slot];
  if (g < 0) return;
  const ScanSlot sl = slots[w.slot];
  if (item_skipped(sl.t, part, nparts)) return;
  const uint32_t* mask = masks + sl.mask_off;
  const uint32_t* wt = weights + sl.w_off;
  const Cand b = best[w.slot];
  for (uint64_t e = w.lo + threadIdx.x; e < w.hi; e += blockDim.x) {
    uint32_t c, v;
    if (!decode_work(w, sl.t, colbase, m, e, c, v)) continue;
    const uint32_t cnt = sl.t.cnt[e];
    if (cnt != b.count || c != b.col || !mask_has(mask, c) ||
        entry_skipped(sl.t, colbase, c, v, part, nparts))
      continue;
    const uint64_t vl = vlen[colbase[c] + v];
    uint64_t ptot = 0;
    for (uint32_t k = 0; k < K; ++k)
      if (wt[c * K + k]) ptot += uint64_t(wt[c * K + k]) * sl.t.psum[e * K + k];
    if ((u128(vl) * vl * cnt + ptot) * u128(cnt - 1) != b.numer) continue;
    atomicMin(&minkey[g], (uint64_t(rv[colbase[c] + v]) << 32) | v);
  }
}

// One block per scanning node: reduce its per-chunk partials.
__global__ void __launch_bounds__(kArgBlock) k_argmax_final(
    const Cand* partial, const unsigned long long* partial_cands, const uint32_t* slot_work_off,
    Cand* out, unsigned long long* out_cands) {
  const uint32_t s = blockIdx.x;
  Cand b{};
  unsigned long long n = 0;
  for (uint32_t i = slot_work_off[s] + threadIdx.x; i < slot_work_off[s + 1]; i += blockDim.x) {
    b = merge(b, partial[i]);
    n += partial_cands[i];
  }
  for (int d = 16; d > 0; d >>= 1) {
    b = merge(b, shfl_cand(b, d));
    n += __shfl_down_sync(0xffffffffu, n, d);
  }
  __shared__ Cand sb[kArgBlock / 32];
  __shared__ unsigned long long sc[kArgBlock / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    sb[wid] = b;
    sc[wid] = n;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kArgBlock / 32; ++i) {
      sb[0] = merge(sb[0], sb[i]);
      sc[0] += sc[i];
    }
    out[s] = sb[0];
    out_cands[s] = sc[0];
  }
}

// Per-slot results of every rank ([rank][slot] Cands then [rank][slot]
// candidate counts) merged into the first rank's rows.
__global__ void k_merge_ranks(Cand* all_best, unsigned long long* all_cands, uint32_t nslots,
                              uint32_t nranks) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nslots; i += gridDim.x * blockDim.x) {
    Cand b = all_best[i];
    unsigned long long n = all_cands[i];
    for (uint32_t r = 1; r < nranks; ++r) {
      b = merge(b, all_best[size_t(r) * nslots + i]);
      n += all_cands[size_t(r) * nslots + i];
    }
    all_best[i] = b;
    all_cands[i] = n;
  }
}

__global__ void k_complement_u64(unsigned long long* x, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = ~x[i];
}

// ---------------------------------------------------------------------------
// K6 split: relabel rows of split nodes and collect block rows
// ---------------------------------------------------------------------------
struct SplitD {
  TDesc tB;           // new table of the block child (keys null: not needed)
  TDesc tP;           // parent table to decrement for the rest child (cnt null: not needed)
  uint32_t mask_off;  // parent columns
  uint32_t col, vid;
  uint32_t block_id, rest_id;
  uint32_t need_rows;
};

// Split lookup by binary search over the level's split nodes (ascending
// node ids), staged in shared memory when they fit.
constexpr uint32_t kRelabelSmem = 4096;
constexpr uint32_t kRelabelBlock = 256;  // k_relabel block size (one table slot per thread)

__global__ void k_relabel(uint32_t* node_of_row, uint64_t n, const int32_t* split_of_node,
                          uint32_t node_lo, uint32_t lut_n, const SplitD* sp, const uint32_t* vid,
                          uint32_t m, uint32_t* cursor, const uint64_t* seg_off,
                          uint32_t* blockrows) {
  // split_of_node[node - node_lo]: this level's split index of a node (-1:
  // not split), staged in shared memory when it fits
  extern __shared__ int32_t s_lut[];
  __shared__ int32_t s_key[kRelabelBlock];
  __shared__ uint32_t s_cnt[kRelabelBlock], s_base[kRelabelBlock];
  s_key[threadIdx.x] = -1;
  s_cnt[threadIdx.x] = 0;
  const uint32_t lane = threadIdx.x & 31;
  const bool staged = lut_n <= kRelabelSmem;
  if (staged)
    for (uint32_t i = threadIdx.x; i < lut_n; i += blockDim.x) s_lut[i] = split_of_node[i];
  __syncthreads();
  const int32_t* tab = staged ? s_lut : split_of_node;
  for (uint64_t base = blockIdx.x * uint64_t(blockDim.x); base < n;
       base += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = base + threadIdx.x;
    int32_t j = -1;
    bool inb = false;
    if (r < n) {
      const uint32_t node = node_of_row[r];
      const uint32_t k = node - node_lo;  // wraps for nodes below node_lo
      if (k < lut_n) j = tab[k];
      if (j >= 0) {
        const SplitD& d = sp[j];
        inb = vid[r * m + d.col] == d.vid;
        node_of_row[r] = inb ? d.block_id : d.rest_id;
        if (!d.need_rows) inb = false;
      }
    }
    // Append of block rows to their split's segment, aggregated per warp
    // (__match_any_sync) and then per block (a shared table keyed by split):
    // one global atomic per split per block instead of one per warp — the
    // rows of a level's large splits otherwise serialise on its cursor.
    const unsigned active = __ballot_sync(0xffffffffu, inb);
    unsigned peers = 0;
    int leader = 0;
    uint32_t slot = 0, off = 0;
    if (inb) {
      peers = __match_any_sync(active, j);
      leader = __ffs(peers) - 1;
      if (int(lane) == leader) {
        slot = uint32_t(j) & (kRelabelBlock - 1);
        for (;;) {  // at most kRelabelBlock distinct splits per block: never full
          const int32_t prev = atomicCAS(&s_key[slot], -1, j);
          if (prev == -1 || prev == j) break;
          slot = (slot + 1) & (kRelabelBlock - 1);
        }
        off = atomicAdd(&s_cnt[slot], uint32_t(__popc(peers)));
      }
    }
    __syncthreads();
    {
      const int32_t key = s_key[threadIdx.x];
      if (key >= 0) s_base[threadIdx.x] = atomicAdd(&cursor[key], s_cnt[threadIdx.x]);
    }
    __syncthreads();
    if (inb) {
      uint32_t basepos = int(lane) == leader ? s_base[slot] + off : 0u;
      basepos = __shfl_sync(peers, basepos, leader);
      const uint32_t rank = __popc(peers & ((1u << lane) - 1));
      blockrows[seg_off[j] + basepos + rank] = uint32_t(r);
    }
    __syncthreads();
    s_key[threadIdx.x] = -1;
    s_cnt[threadIdx.x] = 0;
  }
}

// ---------------------------------------------------------------------------
// K4 group_hist: block-row aggregation into the block child's table and
// decrement of the parent's table (inherited by the rest child)
// ---------------------------------------------------------------------------
// One (split, column) pair of a level's aggregation: the block rows [lo, hi)
// of the split's segment, cut into kAggRows-row tasks; first = the task
// number of its first task (exclusive prefix over the level's segments).
struct AggSeg {
  uint32_t split;  // index into this level's SplitD array
  uint32_t col;
  uint32_t to_b;   // add into the block child's table (col is one of its columns)
  uint32_t to_p;   // subtract from the parent's table (kept by the rest child)
  uint64_t lo, hi;
  uint32_t first, pad;
};

constexpr int kAggBlock = 256;
constexpr uint64_t kAggRows = 2 * kAggBlock;

// Host: append (split, col) over rows [lo, hi); returns the tasks added.
inline uint32_t add_agg_seg(std::vector<AggSeg>& v, uint32_t& ntask, uint32_t split, uint32_t col,
                            uint32_t to_b, uint32_t to_p, uint64_t lo, uint64_t hi) {
  if (hi <= lo) return 0;
  const uint32_t t = uint32_t((hi - lo + kAggRows - 1) / kAggRows);
  v.push_back(AggSeg{split, col, to_b, to_p, lo, hi, ntask, 0});
  ntask += t;
  return t;
}

// One block per (split, column, row range). Lanes of a warp hold consecutive
// block rows of ONE column, so equal values inside a warp are merged with
// __match_any_sync / a labeled-partition reduction before the table atomics
// (low-cardinality columns and the split column itself collapse to one
// atomic per warp).
template <int MINB>
__global__ void __launch_bounds__(kAggBlock, MINB) k_aggregate(
    const AggSeg* __restrict__ segs, uint32_t nseg, const uint32_t* __restrict__ blockrows,
    const SplitD* __restrict__ sp, const uint32_t* __restrict__ vid,
    const uint64_t* __restrict__ vlen, const uint64_t* __restrict__ colbase, uint32_t m,
    uint32_t K, const int32_t* __restrict__ dpart, const uint32_t* __restrict__ npart) {
  // this block's task: the last segment with first <= blockIdx.x
  __shared__ uint32_t s_seg;
  if (threadIdx.x == 0) {
    uint32_t lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) / 2;
      if (segs[mid].first <= blockIdx.x) lo = mid;
      else hi = mid - 1;
    }
    s_seg = lo;
  }
  __syncthreads();
  struct {
    uint32_t split, col, to_b, to_p;
    uint64_t lo, hi;
  } tk;
  {
    const AggSeg& g = segs[s_seg];
    tk.split = g.split;
    tk.col = g.col;
    tk.to_b = g.to_b;
    tk.to_p = g.to_p;
    tk.lo = g.lo + uint64_t(blockIdx.x - g.first) * kAggRows;
    tk.hi = tk.lo + kAggRows < g.hi ? tk.lo + kAggRows : g.hi;
  }
  const SplitD& d = sp[tk.split];
  const uint32_t c = tk.col;
  const uint32_t np = npart[c];
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t base = tk.lo; base < tk.hi; base += kAggBlock) {
    const uint64_t q = base + threadIdx.x;
    const bool valid = q < tk.hi;
    uint32_t r = 0, v = 0xFFFFFFFFu;
    if (valid) {
      r = blockrows[q];
      v = vid[uint64_t(r) * m + c];
    }
    const unsigned grp = __match_any_sync(0xffffffffu, v);
    const int leader = __ffs(grp) - 1;
    const bool lead = valid && int(lane) == leader;
    const unsigned long long key = (uint64_t(c + 1) << 32) | v;
    uint64_t sb = 0, spn = 0;
    if (lead) {
      const uint32_t cnt = __popc(grp);
      if (tk.to_b) {
        sb = tbl_insert(d.tB, key);
        atomicAdd(&d.tB.cnt[sb], cnt);
      }
      if (tk.to_p) {
        spn = d.tP.dense ? colbase[c] + v : tbl_find(d.tP, key);
        atomicSub(&d.tP.cnt[spn], cnt);
      }
    }
    for (uint32_t k = 0; k < np; ++k) {  // FD partner lengths, summed per group
      const int32_t p = dpart[c * K + k];
      unsigned long long l = valid ? vlen[colbase[p] + vid[uint64_t(r) * m + p]] : 0ull;
      auto g = cg::labeled_partition(cg::tiled_partition<32>(cg::this_thread_block()), v);
      l = cg::reduce(g, l, cg::plus<unsigned long long>());
      if (lead) {
        if (tk.to_b) atomicAdd(&d.tB.psum[sb * K + k], l);
        if (tk.to_p) atomicAdd(&d.tP.psum[spn * K + k], 0ull - l);
      }
    }
  }
}

// Unique columns (one distinct value per row, single GPU) are never scanned
// and get no table entries; a node keeps only its length sum per unique
// column (usum[node * U + u]) for the leaf statistics. k_unique_sums adds
// the block rows' lengths of split j (one task per AggSeg chunk); its last
// block sets block = that sum and rest = parent - block.
__global__ void k_unique_sums(const AggSeg* __restrict__ segs, uint32_t nseg,
                              const uint32_t* __restrict__ blockrows,
                              const uint32_t* __restrict__ vid, const uint64_t* __restrict__ vlen,
                              const uint64_t* __restrict__ colbase, uint32_t m,
                              const int32_t* __restrict__ uidx, uint32_t U, unsigned long long* ublk,
                              const SplitD* __restrict__ sp, const uint32_t* __restrict__ parent,
                              uint32_t ns, unsigned long long* usum, uint32_t* done) {
  __shared__ bool s_last;
  if (nseg) {
    uint32_t lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) / 2;
      if (segs[mid].first <= blockIdx.x) lo = mid;
      else hi = mid - 1;
    }
    const AggSeg& g = segs[lo];
    const uint64_t a = g.lo + uint64_t(blockIdx.x - g.first) * kAggRows;
    const uint64_t b = a + kAggRows < g.hi ? a + kAggRows : g.hi;
    const uint32_t c = g.col;
    unsigned long long sum = 0;
    for (uint64_t q = a + threadIdx.x; q < b; q += blockDim.x) {
      const uint32_t r = blockrows[q];
      sum += vlen[colbase[c] + vid[uint64_t(r) * m + c]];
    }
    sum = warp_sum_u64(sum);
    if ((threadIdx.x & 31) == 0 && sum)
      atomicAdd(&ublk[uint64_t(g.split) * U + uint32_t(uidx[c])], sum);
  }
  // the last block to finish sets the children's sums: block = the block
  // rows' sum, rest = parent - block
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (uint32_t t = threadIdx.x; t < ns * U; t += blockDim.x) {
    const uint32_t j = t / U, u = t - j * U;
    const unsigned long long blk = __ldcg(&ublk[t]);
    usum[uint64_t(sp[j].block_id) * U + u] = blk;
    usum[uint64_t(sp[j].rest_id) * U + u] = usum[uint64_t(parent[j]) * U + u] - blk;
  }
}

// Leaf statistics of the unique columns: distinct count = leaf size, length
// sum from usum (k_leaf_stats leaves these (leaf, column) slots at zero).
__global__ void k_unique_leaf_stats(const uint32_t* __restrict__ leaf_node,
                                    const unsigned long long* __restrict__ leaf_size, uint32_t nleaf,
                                    const int32_t* __restrict__ ucol, uint32_t U, uint32_t m,
                                    const unsigned long long* __restrict__ usum,
                                    unsigned long long* card, unsigned long long* tot) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nleaf * U; t += gridDim.x * blockDim.x) {
    const uint32_t i = t / U, u = t - i * U;
    const uint32_t c = uint32_t(ucol[u]);
    card[uint64_t(i) * m + c] = leaf_size[i];
    tot[uint64_t(i) * m + c] = usum[uint64_t(leaf_node[i]) * U + u];
  }
}

// Sharded solve: this rank's block-row aggregate of split j (a private
// table) as records [key][split<<32 | count][K partner sums].
__global__ void k_compact_contrib(TDesc t, uint32_t j, uint32_t K, uint64_t* out,
                                  unsigned long long* cursor) {
  const uint32_t lane = threadIdx.x & 31;
  // t.cap is a power of two >= 64 and the grid a multiple of 32 threads, so a
  // warp stays converged through the loop (warp-aggregated cursor)
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < t.cap;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const unsigned long long key = t.keys[e];
    const unsigned has = __ballot_sync(0xffffffffu, key != 0);
    unsigned long long base = 0;
    if (lane == 0 && has) base = atomicAdd(cursor, (unsigned long long)__popc(has));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (!key) continue;
    uint64_t* r = out + (base + __popc(has & ((1u << lane) - 1))) * (2 + K);
    r[0] = key;
    r[1] = (uint64_t(j) << 32) | t.cnt[e];
    for (uint32_t k = 0; k < K; ++k) r[2 + k] = t.psum[e * K + k];
  }
}

// Every rank's contributions into the replicated tables: add to the block
// child's table (columns outside the block columns) and subtract from the
// parent's table kept by the rest child — the same updates k_aggregate
// makes from the rows themselves on one GPU.
__global__ void k_apply_contrib(uint64_t E, const uint64_t* __restrict__ recs, uint32_t K,
                                const SplitD* __restrict__ sp, const uint32_t* __restrict__ bmask,
                                uint32_t W, const uint64_t* __restrict__ colbase) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < E;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t* r = recs + i * (2 + K);
    const unsigned long long key = r[0];
    const uint32_t j = uint32_t(r[1] >> 32), cnt = uint32_t(r[1]);
    const uint32_t c = uint32_t(key >> 32) - 1, v = uint32_t(key);
    const SplitD& d = sp[j];
    if (d.tB.keys && !((bmask[j * W + (c >> 5)] >> (c & 31)) & 1u)) {
      const uint64_t sb = tbl_insert(d.tB, key);
      atomicAdd(&d.tB.cnt[sb], cnt);
      for (uint32_t k = 0; k < K; ++k) atomicAdd(&d.tB.psum[sb * K + k], (unsigned long long)r[2 + k]);
    }
    if (d.tP.cnt) {
      const uint64_t spn = d.tP.dense ? colbase[c] + v : tbl_find(d.tP, key);
      atomicSub(&d.tP.cnt[spn], cnt);
      for (uint32_t k = 0; k < K; ++k) atomicAdd(&d.tP.psum[spn * K + k], 0ull - r[2 + k]);
    }
  }
}

// ---- debug consistency checks (PO_DEBUG_CHECKS=1) ----
__global__ void k_dbg_node_hist(const uint32_t* node_of_row, uint64_t n, uint32_t nnodes,
                                unsigned long long* hist) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t nd = node_of_row[r];
    atomicAdd(&hist[nd < nnodes ? nd : nnodes], 1ull);
  }
}

__global__ void k_dbg_perm(const uint32_t* pos, uint64_t n, unsigned* seen, unsigned long long* bad) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t p = pos[r];
    if (p >= n || atomicAdd(&seen[p], 1u) != 0) atomicAdd(bad, 1ull);
  }
}


// Root partner sums: psum[colbase[c]+vid(r,c)][k] += len(r, partner k of c).
// A warp takes 32 consecutive rows of one column that has partners; lanes
// holding the same value add their partner lengths first (labeled partition)
// and one lane per value issues the atomic (a Zipf-hot value otherwise
// serialises on one address: C3's movie_title).
__global__ void k_root_psum(const uint32_t* vid, uint64_t n, uint32_t m, uint32_t K,
                            const int32_t* dpart, const uint32_t* npart, const uint64_t* vlen,
                            const uint64_t* colbase, unsigned long long* psum) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t ntiles = (n + 31) / 32;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  auto tile32 = cg::tiled_partition<32>(cg::this_thread_block());
  for (uint64_t w = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; w < ntiles * m;
       w += nwarps) {
    const uint32_t c = uint32_t(w % m);
    const uint32_t np = npart[c];
    if (!np) continue;  // warp-uniform
    const uint64_t r = (w / m) * 32 + lane;
    const bool valid = r < n;
    const uint32_t v = valid ? vid[r * m + c] : 0xFFFFFFFFu;
    auto g = cg::labeled_partition(tile32, v);
    const uint64_t e = colbase[c] + v;
    for (uint32_t k = 0; k < np; ++k) {
      const int32_t p = dpart[c * K + k];
      const unsigned long long l =
          valid ? (unsigned long long)vlen[colbase[p] + vid[r * m + p]] : 0ull;
      const unsigned long long sum = cg::reduce(g, l, cg::plus<unsigned long long>());
      if (valid && g.thread_rank() == 0) atomicAdd(&psum[e * K + k], sum);
    }
  }
}

// ---------------------------------------------------------------------------
// K7 leaf_stats: per (leaf, column) distinct count and length sum
// ---------------------------------------------------------------------------
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_leaf_stats(
    const WorkSeg* work, uint32_t nwseg, const ScanSlot* slots, const uint32_t* masks, const uint64_t* colbase,
    const uint64_t* vlen, uint32_t m, unsigned long long* card, unsigned long long* tot,
    uint32_t part, uint32_t nparts) {
  extern __shared__ unsigned long long sh[];  // [2*m] for hashed tables with small m
  const WorkItem w = work_at(work, nwseg);
  const ScanSlot sl = slots[w.slot];
  if (item_skipped(sl.t, part, nparts)) return;  // sharded: dealt to another rank
  const uint32_t* mask = masks + sl.mask_off;
  if (w.col != kAnyCol) {
    // dense table, one column: per-thread sums, one atomic pair per block
    const uint32_t c = w.col;
    unsigned long long k = 0, l = 0;
    for (uint64_t e = w.lo + threadIdx.x; e < w.hi; e += blockDim.x) {
      const uint32_t cnt = sl.t.cnt[e];
      if (cnt) {
        ++k;
        l += uint64_t(cnt) * vlen[e];
      }
    }
    typedef cub::BlockReduce<unsigned long long, 256> BR;
    __shared__ typename BR::TempStorage t1, t2;
    k = BR(t1).Sum(k);
    l = BR(t2).Sum(l);
    if (threadIdx.x == 0 && k) {
      atomicAdd(&card[uint64_t(w.slot) * m + c], k);
      atomicAdd(&tot[uint64_t(w.slot) * m + c], l);
    }
    return;
  }
  const bool priv = m <= 2048;
  if (priv)
    for (uint32_t c = threadIdx.x; c < 2 * m; c += blockDim.x) sh[c] = 0;
  __syncthreads();
  // hashed table: entries of mixed columns; lanes with the same column are
  // merged per warp before the shared-memory atomics
  for (uint64_t base = w.lo; base < w.hi; base += blockDim.x) {
    const uint64_t e = base + threadIdx.x;
    uint32_t c = 0xFFFFFFFFu, v = 0;
    unsigned long long l = 0;
    if (e < w.hi && decode_entry(sl.t, colbase, m, e, c, v)) {
      const uint32_t cnt = sl.t.cnt[e];
      if (cnt == 0 || !mask_has(mask, c) || entry_skipped(sl.t, colbase, c, v, part, nparts))
        c = 0xFFFFFFFFu;
      else l = uint64_t(cnt) * vlen[colbase[c] + v];
    } else {
      c = 0xFFFFFFFFu;
    }
    const unsigned grp = __match_any_sync(0xffffffffu, c);
    auto g = cg::labeled_partition(cg::tiled_partition<32>(cg::this_thread_block()), c);
    l = cg::reduce(g, l, cg::plus<unsigned long long>());
    if (c != 0xFFFFFFFFu && int(threadIdx.x & 31) == __ffs(grp) - 1) {
      const unsigned long long k = __popc(grp);
      if (priv) {
        atomicAdd(&sh[c], k);
        atomicAdd(&sh[m + c], l);
      } else {
        atomicAdd(&card[uint64_t(w.slot) * m + c], k);
        atomicAdd(&tot[uint64_t(w.slot) * m + c], l);
      }
    }
  }
  if (priv) {
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < m; c += blockDim.x)
      if (sh[c]) {
        atomicAdd(&card[uint64_t(w.slot) * m + c], sh[c]);
        atomicAdd(&tot[uint64_t(w.slot) * m + c], sh[m + c]);
      }
  }
}

// ---------------------------------------------------------------------------
// layout + emit
// ---------------------------------------------------------------------------
__global__ void k_row_leaf(const uint32_t* node_of_row, uint64_t n, const uint32_t* node_leaf,
                           const uint32_t* leaf_off, uint32_t* row_leaf, uint32_t* grp) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t l = node_leaf[node_of_row[r]];
    row_leaf[r] = l;
    grp[r] = leaf_off[l];
  }
}

__global__ void k_emit(const uint32_t* pos, uint64_t n, uint32_t* rows_out) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x)
    rows_out[pos[r]] = uint32_t(r);
}

// Field orders in schedule order, one thread per output entry (coalesced
// writes; the row's leaf order is a small cached table).
__global__ void k_emit_orders(const uint32_t* rows, uint64_t n, uint32_t m,
                              const uint32_t* row_leaf, const int32_t* leaf_orders,
                              int32_t* orders_out) {
  const uint64_t total = n * m;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t p = i / m;
    const uint32_t f = uint32_t(i - p * m);
    orders_out[i] = leaf_orders[uint64_t(row_leaf[rows[p]]) * m + f];
  }
}

// CSR field orders (repeated FD pairs): thread per schedule position.
__global__ void k_emit_orders_csr(const uint32_t* rows, uint64_t n, const uint32_t* row_leaf,
                                  const int32_t* leaf_fields, const uint32_t* leaf_fields_off,
                                  const uint32_t* leaf_width, const uint64_t* leaf_base,
                                  const uint32_t* leaf_pos, uint64_t total, uint64_t* offsets,
                                  int32_t* fields) {
  for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < n;
       p += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t l = row_leaf[rows[p]];
    const uint32_t w = leaf_width[l];
    const uint64_t at = leaf_base[l] + (p - leaf_pos[l]) * uint64_t(w);
    offsets[p] = at;
    for (uint32_t j = 0; j < w; ++j) fields[at + j] = leaf_fields[leaf_fields_off[l] + j];
    if (p + 1 == n) offsets[n] = total;
  }
}

__global__ void k_tile_order(const int32_t* order, uint64_t n, uint32_t m, int32_t* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n * m;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = order[i % m];
}

__global__ void k_iota_u32(uint32_t* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    a[i] = uint32_t(i);
}

// ---------------------------------------------------------------------------
// host-side tree
// ---------------------------------------------------------------------------
enum Kind { SCAN, EMPTY, ROWID, SINGLE, RAW1, FALLBACK, SPLIT };

struct Node {
  uint64_t size = 0;
  std::vector<int> cols;  // ascending schema order (ggr.hpp:177, 292-296)
  uint64_t rd = 0, cd = 0, depth = 0;
  int kind = SCAN;
  std::shared_ptr<HTable> table;
  std::vector<int> block_cols;  // SPLIT: [best.col] + active partners
  int block_child = -1, rest_child = -1;
  std::vector<int> leaf_order;  // FALLBACK: stats-ranked order
};

int classify(const Node& nd, const po_ggr_config& cfg) {
  // base cases then depth gate, in the reference's order (ggr.hpp:213-234)
  if (nd.size == 0) return EMPTY;
  if (nd.cols.empty()) return ROWID;
  if (nd.size == 1) return SINGLE;
  if (nd.cols.size() == 1) return RAW1;
  if (nd.rd > cfg.row_recursion_depth || nd.cd > cfg.column_recursion_depth) return FALLBACK;
  return SCAN;
}


bool debug_checks() {
  static const bool on = [] {
    const char* v = std::getenv("PO_DEBUG_CHECKS");
    return v && *v && *v != '0';
  }();
  return on;
}

struct Level {
  std::vector<ScanSlot> slots;
  std::vector<uint32_t> masks;
  std::vector<uint32_t> weights;
  std::vector<WorkSeg> work;
  uint32_t nitems = 0;  // work items (blocks) over all segments
  std::vector<uint32_t> slot_work_off{0};
};

// Per-level device upload: every small array of a level in one H2D copy.
struct Pack {
  std::vector<uint8_t> host;
  template <class T>
  size_t add(const std::vector<T>& v) {
    size_t off = (host.size() + 15) & ~size_t(15);
    host.resize(off + std::max<size_t>(1, v.size()) * sizeof(T), 0);
    if (!v.empty()) std::memcpy(host.data() + off, v.data(), v.size() * sizeof(T));
    return off;
  }
};

}  // namespace

// Occupancy of the level kernels: min blocks per SM of k_argmax (8: 32
// registers), k_aggregate (6: 40) and k_leaf_stats (1), measured with
// tools/level_minb_sweep.sh (C4 20M-row argmax 2.07 -> 1.29 ms per call,
// C3 0.30 -> 0.27); PO_LEVEL_MINB=a,b,c picks others (experiments).
static int level_minb(int which) {
  static const std::vector<int> v = [] {
    std::vector<int> r{8, 6, 1};
    const char* e = std::getenv("PO_LEVEL_MINB");
    if (e && *e) sscanf(e, "%d,%d,%d", &r[0], &r[1], &r[2]);
    return r;
  }();
  return v[which];
}
#define PO_MINB_SWITCH(which, K, grid, block, smem, s, ...)                  \
  do {                                                                     \
    switch (level_minb(which)) {                                           \
      case 4: PO_LAUNCH((K<4>), grid, block, smem, s, __VA_ARGS__); break; \
      case 6: PO_LAUNCH((K<6>), grid, block, smem, s, __VA_ARGS__); break; \
      case 8: PO_LAUNCH((K<8>), grid, block, smem, s, __VA_ARGS__); break; \
      default: PO_LAUNCH((K<1>), grid, block, smem, s, __VA_ARGS__); break; \
    }                                                                      \
  } while (0)
#define PO_ARGMAX(grid, ...) PO_MINB_SWITCH(0, k_argmax, grid, __VA_ARGS__)
#define PO_AGG(grid, ...) PO_MINB_SWITCH(1, k_aggregate, grid, __VA_ARGS__)
#define PO_LEAFSTATS(grid, ...) PO_MINB_SWITCH(2, k_leaf_stats, grid, __VA_ARGS__)

void ggr_device(const Encoded& e, const std::vector<std::vector<int>>& fd_groups,
                const po_ggr_config& cfg, uint32_t* d_rows, int32_t* d_orders, GgrOutput& out,
                cudaStream_t s, DistCtx* dist) {
  const uint64_t n = e.n;  // rows held here (all of them on one GPU)
  const uint32_t m = e.m;
  const uint64_t ng = dist ? dist->n_global : n;  // rows of the whole table
  out = GgrOutput{};
  out.stats.recursive_calls = 1;  // the root call (ggr.hpp:210)
  if (ng == 0) return;
  if (m == 0) {  // every row, ascending, no fields (ggr.hpp:214-219)
    if (dist) fail(PO_ERR_ERROR, "internal: sharded solve with no fields");
    PO_LAUNCH(k_iota_u32, grid_for(n, 256), 256, 0, s, d_rows, n);
    return;
  }

  // Whole-table fallback competitor (ggr.hpp:379-387), single GPU: its order
  // comes from the global stats and its PHC and pruning bound need only the
  // dictionary, so both are queued now on a side stream and run while the
  // level loop's host round trips leave the device idle; the end of the call
  // reads them together with the recursion's PHC in one transfer.
  static const bool early_fb_on = [] {  // PO_EARLY_FALLBACK=0: at the end, on s
    const char* v = std::getenv("PO_EARLY_FALLBACK");
    return !(v && *v == '0');
  }();
  const bool early_fb = early_fb_on && !dist && !debug_checks();
  std::vector<int> fb_order;
  DevBuf<unsigned long long> fbres;  // [fallback phc][bound (double)][phc][out-of-range flag]
  struct FbJoin {  // the call's stream waits for the side stream on every exit
    cudaStream_t s;
    cudaEvent_t ev = nullptr;
    ~FbJoin() {
      if (ev) {
        cudaStreamWaitEvent(s, ev, 0);
        cudaEventDestroy(ev);
      }
    }
  } fb_join{s};
  if (early_fb) {
    std::vector<double> avg(m);
    for (uint32_t c = 0; c < m; ++c)
      avg[c] = static_cast<double>(e.total_len[c]) / static_cast<double>(ng);
    fb_order = hitcount_order(ng, e.card, avg, cfg.stats_variant);
    fbres.alloc(4, s);
    cudaStream_t a = aux_stream();
    cudaEvent_t ready;
    PO_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    PO_CUDA(cudaEventRecord(ready, s));
    PO_CUDA(cudaStreamWaitEvent(a, ready, 0));
    PO_CUDA(cudaEventDestroy(ready));
    fallback_ub_async(e, a, reinterpret_cast<double*>(fbres.get() + 1));
    fixed_order_phc_async(e, fb_order, a, fbres.get());
    PO_CUDA(cudaEventCreateWithFlags(&fb_join.ev, cudaEventDisableTiming));
    PO_CUDA(cudaEventRecord(fb_join.ev, a));
  }

  // FD partners (ggr.hpp:154-164): per field, the other members of every
  // group holding it, each group's members in ascending order.
  std::vector<std::vector<int>> partners(m);
  if (cfg.use_fds) {
    for (const auto& g : fd_groups) {
      std::vector<int> mem = g;
      for (int f : mem)
        if (f < 0 || f >= int(m)) fail(PO_ERR_SCHEMA, "FD group names a field outside the schema");
      std::sort(mem.begin(), mem.end());
      for (int f : mem)
        for (int o : mem)
          if (o != f) partners[f].push_back(o);
    }
  }
  // Groups may share members: a partner then appears several times in
  // partners_[f] and the reference counts its length once per appearance
  // (ggr.hpp:252-255) and emits it once per appearance in the block prefix
  // (ggr.hpp:280-282, 303-309). Partner sums are kept per distinct partner
  // (dpart) and weighted by the multiplicity (dmult).
  uint32_t K = 0;
  std::vector<std::vector<int>> dpart(m);
  std::vector<std::vector<uint32_t>> dmult(m);
  for (uint32_t c = 0; c < m; ++c) {
    std::vector<int> u = partners[c];
    std::sort(u.begin(), u.end());
    for (size_t i = 0; i < u.size();) {
      size_t j = i;
      while (j < u.size() && u[j] == u[i]) ++j;
      dpart[c].push_back(u[i]);
      dmult[c].push_back(uint32_t(j - i));
      i = j;
    }
    K = std::max<uint32_t>(K, uint32_t(dpart[c].size()));
  }
  std::vector<int32_t> h_dpart(std::max<size_t>(1, size_t(m) * K), 0);
  std::vector<uint32_t> h_npart(m, 0);
  for (uint32_t c = 0; c < m; ++c) {
    h_npart[c] = uint32_t(dpart[c].size());
    for (size_t k = 0; k < dpart[c].size(); ++k) h_dpart[c * K + k] = dpart[c][k];
  }
  auto d_dpart = to_device(h_dpart, s);
  auto d_npart = to_device(h_npart, s);
  const uint32_t W = (m + 31) / 32;
  const uint64_t* colbase = e.d_colbase.get();
  const uint64_t* vlen = e.vlen.get();

  // Tree state.
  std::vector<Node> nodes;
  nodes.reserve(1024);
  {
    Node root;
    root.size = ng;
    root.cols.resize(m);
    std::iota(root.cols.begin(), root.cols.end(), 0);
    root.kind = classify(root, cfg);
    nodes.push_back(std::move(root));
  }
  DevBuf<uint32_t> node_of_row = dev_auto<uint32_t>(n, s);
  node_of_row.zero();

  // Work items over a node's table: dense tables are cut at column
  // boundaries (only the node's active columns), hashed ones in plain chunks.
  auto add_work = [&](Level& lv, uint32_t slot, const HTable& t, const std::vector<int>& cols) {
    auto seg = [&](uint32_t col, uint64_t lo, uint64_t hi) {
      if (hi <= lo) return;
      lv.work.push_back(WorkSeg{slot, col, lo, hi, lv.nitems, 0});
      lv.nitems += uint32_t((hi - lo + kWorkChunk - 1) / kWorkChunk);
    };
    if (t.dense) {
      for (int c : cols) seg(uint32_t(c), e.colbase[c], e.colbase[c + 1]);
    } else {
      seg(kAnyCol, 0, t.cap);
    }
  };
  auto col_mask = [&](const std::vector<int>& cols, std::vector<uint32_t>& dst) {
    uint32_t off = uint32_t(dst.size());
    dst.resize(dst.size() + W, 0);
    for (int c : cols) dst[off + (uint32_t(c) >> 5)] |= 1u << (uint32_t(c) & 31);
    return off;
  };

  // Root table: dense over all distinct values.
  if (nodes[0].kind == SCAN || nodes[0].kind == FALLBACK) {
    auto t = std::make_shared<HTable>();
    t->dense = true;
    t->cap = e.D;
    t->mem = std::make_shared<DevBuf<uint8_t>>(e.D * 4 + 256 + (K ? e.D * K * 8 : 0), s);
    t->cnt = reinterpret_cast<uint32_t*>(t->mem->get());
    if (K) t->psum = reinterpret_cast<unsigned long long*>(t->mem->get() + ((e.D * 4 + 255) & ~uint64_t(255)));
    PO_CUDA(cudaMemcpyAsync(t->cnt, e.count.get(), e.D * sizeof(uint32_t),
                            cudaMemcpyDeviceToDevice, s));
    if (K) {
      PO_CUDA(cudaMemsetAsync(t->psum, 0, e.D * K * 8, s));
      PO_LAUNCH(k_root_psum, grid_for(n * m, 256), 256, 0, s, e.vid.get(), n, m, K, d_dpart.get(),
                d_npart.get(), vlen, colbase, t->psum);
      if (dist) dist->comm->allreduce(t->psum, e.D * K, CDtype::U64, COp::Sum, s);
    }
    nodes[0].table = t;
  }

  // Unique columns (single GPU): no table entries, length sums per node
  // (k_unique_sums / k_unique_leaf_stats)
  std::vector<int> ucols;
  std::vector<int32_t> uidx(m, -1);
  if (!dist)
    for (uint32_t c = 0; c < m; ++c)
      if (e.card[c] == ng && ng > 1) {
        uidx[c] = int32_t(ucols.size());
        ucols.push_back(int(c));
      }
  const uint32_t U = uint32_t(ucols.size());
  DevBuf<int32_t> d_uidx, d_ucol;
  DevBuf<unsigned long long> usum;  // [node][U]
  if (U) {
    d_uidx = to_device(uidx, s);
    d_ucol = to_device(std::vector<int32_t>(ucols.begin(), ucols.end()), s);
    usum.alloc(size_t(64) * U, s);
    std::vector<unsigned long long> root(U);
    for (uint32_t u = 0; u < U; ++u) root[u] = e.total_len[ucols[u]];
    usum.upload(root.data(), U);
  }
  auto grow_usum = [&](size_t nodes_n) {  // keeps the sums of existing nodes
    if (!U || usum.size() >= nodes_n * U) return;
    DevBuf<unsigned long long> nb(std::max(nodes_n, usum.size() / U * 2) * U, s);
    PO_CUDA(cudaMemcpyAsync(nb.get(), usum.get(), usum.size() * sizeof(unsigned long long),
                            cudaMemcpyDeviceToDevice, s));
    usum = std::move(nb);
  };


  // per-level scratch, grown only (stream order makes the reuse safe: a
  // level's copies and kernels queue behind the previous level's kernels)
  DevBuf<uint8_t> pack_dev;
  auto grow = [&](auto& buf, size_t n) {
    if (buf.size() < n) buf.alloc(std::max(n, 2 * buf.size()), s);
  };
  auto upload = [&](Pack& pk) -> uint8_t* {
    grow(pack_dev, pk.host.size());
    pack_dev.upload(pk.host.data(), pk.host.size());
    return pack_dev.get();
  };
  DevBuf<Cand> partial;
  DevBuf<unsigned long long> pcands;
  DevBuf<uint8_t> res;

  // Leaf statistics -> stats-ranked field order of a fallback leaf
  // (ggr.hpp:319-338). hc/ht: per (leaf slot, column) distinct count and
  // length sum.
  auto finish_leaves = [&](const std::vector<int>& leaves, const unsigned long long* hc,
                           const unsigned long long* ht) {
    for (size_t i = 0; i < leaves.size(); ++i) {
      Node& nd = nodes[leaves[i]];
      std::vector<uint64_t> cc(nd.cols.size());
      std::vector<double> avg(nd.cols.size());
      for (size_t k = 0; k < nd.cols.size(); ++k) {
        cc[k] = hc[i * m + nd.cols[k]];
        avg[k] = static_cast<double>(ht[i * m + nd.cols[k]]) / static_cast<double>(nd.size);
      }
      std::vector<int> local = hitcount_order(nd.size, cc, avg, cfg.stats_variant);
      nd.leaf_order.clear();
      for (int li : local) nd.leaf_order.push_back(nd.cols[li]);
      nd.table.reset();
    }
  };

  std::vector<int> frontier, pending;  // pending: fallback leaves awaiting stats
  if (nodes[0].kind == SCAN) frontier.push_back(0);
  else if (nodes[0].kind == FALLBACK) pending.push_back(0);

  while (!frontier.empty() || !pending.empty()) {
    // ---- one GPU pass per level: K5 argmax over the frontier, K7 leaf
    // statistics of the leaves created by the previous level, one D2H ----
    std::optional<HostScope> hs_build(std::in_place, "lvl_build");
    Level L, S;
    std::vector<uint64_t> unique_groups(frontier.size(), 0);
    for (size_t i = 0; i < frontier.size(); ++i) {
      const Node& nd = nodes[frontier[i]];
      ScanSlot sl;
      sl.t = nd.table->desc();
      // Columns whose values are all distinct (card == n) hold one row per
      // group in every node: their groups score 0 and can never be chosen
      // over a positive score (ggr.hpp:263-266), so they are not scanned —
      // their |node| groups are added to candidates_examined directly.
      std::vector<int> scan_cols;
      for (int c : nd.cols)
        if (e.card[c] == ng) unique_groups[i] += nd.size;
        else scan_cols.push_back(c);
      sl.mask_off = col_mask(scan_cols, L.masks);
      sl.w_off = uint32_t(L.weights.size());
      L.weights.resize(L.weights.size() + size_t(m) * std::max<uint32_t>(K, 1), 0);
      std::vector<char> act(m, 0);
      for (int c : nd.cols) act[c] = 1;
      for (uint32_t c = 0; c < m; ++c)
        for (size_t k = 0; k < dpart[c].size(); ++k)
          if (act[dpart[c][k]]) L.weights[sl.w_off + c * K + k] = dmult[c][k];
      L.slots.push_back(sl);
      add_work(L, uint32_t(i), *nd.table, scan_cols);
      L.slot_work_off.push_back(L.nitems);
    }
    for (size_t i = 0; i < pending.size(); ++i) {
      const Node& nd = nodes[pending[i]];
      ScanSlot sl;
      sl.t = nd.table->desc();
      sl.mask_off = col_mask(nd.cols, S.masks);
      sl.w_off = 0;
      S.slots.push_back(sl);
      add_work(S, uint32_t(i), *nd.table, nd.cols);
    }
    const uint32_t nslots = uint32_t(L.slots.size());
    const size_t nleaf = pending.size();
    Pack pk;
    const size_t o_slots = pk.add(L.slots), o_masks = pk.add(L.masks), o_w = pk.add(L.weights);
    const size_t o_work = pk.add(L.work), o_swo = pk.add(L.slot_work_off);
    const size_t o_sslots = pk.add(S.slots), o_smasks = pk.add(S.masks), o_swork = pk.add(S.work);
    std::vector<uint32_t> uln;
    std::vector<unsigned long long> ulsz;
    if (U)
      for (int id : pending) {
        uln.push_back(uint32_t(id));
        ulsz.push_back(nodes[id].size);
      }
    const size_t o_uln = pk.add(uln), o_ulsz = pk.add(ulsz);
    uint8_t* dp = upload(pk);
    grow(partial, std::max<size_t>(1, L.nitems));
    grow(pcands, std::max<size_t>(1, L.nitems));
    // results: [best Cand x nslots][ncand u64 x nslots][card u64 x nleaf*m][tot u64 x nleaf*m]
    const size_t res_bytes = nslots * (sizeof(Cand) + 8) + 2 * nleaf * m * 8;
    grow(res, std::max<size_t>(16, res_bytes));
    Cand* d_best = reinterpret_cast<Cand*>(res.get());
    auto* d_ncand = reinterpret_cast<unsigned long long*>(res.get() + nslots * sizeof(Cand));
    auto* d_card = d_ncand + nslots;
    auto* d_tot = d_card + nleaf * m;
    if (nleaf) PO_CUDA(cudaMemsetAsync(d_card, 0, 2 * nleaf * m * 8, s));
    hs_build.reset();
    // sharded solve: every rank scans its share of the replicated tables'
    // work items; results merged across ranks below
    static const bool partition = [] {  // PO_DIST_PARTITION=0: every rank scans everything
      const char* v = std::getenv("PO_DIST_PARTITION");
      return !(v && *v == '0');
    }();
    const uint32_t nparts = dist && partition ? uint32_t(dist->comm->size()) : 1u;
    const uint32_t part = dist && partition ? uint32_t(dist->comm->rank()) : 0u;
    if (nslots) {
      PO_ARGMAX(L.nitems, kArgBlock, 0, s,
                reinterpret_cast<WorkSeg*>(dp + o_work), uint32_t(L.work.size()), reinterpret_cast<ScanSlot*>(dp + o_slots),
                reinterpret_cast<uint32_t*>(dp + o_masks), reinterpret_cast<uint32_t*>(dp + o_w),
                colbase, vlen, m, K, partial.get(), pcands.get(), part, nparts);
      PO_LAUNCH(k_argmax_final, nslots, kArgBlock, 0, s, partial.get(), pcands.get(),
                reinterpret_cast<uint32_t*>(dp + o_swo), d_best, d_ncand);
    }
    if (nleaf)
      PO_LEAFSTATS(S.nitems, 256, m <= 2048 ? 16 * m : 0, s,
                reinterpret_cast<WorkSeg*>(dp + o_swork), uint32_t(S.work.size()), reinterpret_cast<ScanSlot*>(dp + o_sslots),
                reinterpret_cast<uint32_t*>(dp + o_smasks), colbase, vlen, m, d_card, d_tot, part,
                nparts);
    if (nleaf && U)
      PO_LAUNCH(k_unique_leaf_stats, grid_for(nleaf * U, 128), 128, 0, s,
                reinterpret_cast<uint32_t*>(dp + o_uln), reinterpret_cast<unsigned long long*>(dp + o_ulsz),
                uint32_t(nleaf), d_ucol.get(), U, m, usum.get(), d_card, d_tot);
    if (nparts > 1) {
      if (nslots) {
        DevBuf<Cand> ab(size_t(nslots) * nparts, s);
        DevBuf<unsigned long long> ac(size_t(nslots) * nparts, s);
        dist->comm->allgather(d_best, ab.get(), nslots * sizeof(Cand), s);
        dist->comm->allgather(d_ncand, ac.get(), nslots * 8, s);
        PO_LAUNCH(k_merge_ranks, grid_for(nslots, 128), 128, 0, s, ab.get(), ac.get(), nslots, nparts);
        PO_CUDA(cudaMemcpyAsync(d_best, ab.get(), nslots * sizeof(Cand), cudaMemcpyDeviceToDevice, s));
        PO_CUDA(cudaMemcpyAsync(d_ncand, ac.get(), nslots * 8, cudaMemcpyDeviceToDevice, s));
      }
      if (nleaf) dist->comm->allreduce(d_card, 2 * nleaf * m, CDtype::U64, COp::Sum, s);
    }
    std::vector<uint8_t> hres(std::max<size_t>(16, res_bytes));
    d2h_sync(hres.data(), res.get(), res_bytes, s);
    std::vector<Cand> hbest(nslots);
    if (nslots) std::memcpy(hbest.data(), hres.data(), nslots * sizeof(Cand));
    const unsigned long long* hn =
        reinterpret_cast<const unsigned long long*>(hres.data() + nslots * sizeof(Cand));
    finish_leaves(pending, hn + nslots, hn + nslots + nleaf * m);
    pending.clear();
    if (frontier.empty()) break;

    // ---- raw-byte tie-break among candidates equal on (score, count,
    // column) (ggr.hpp:196), only for nodes that will split ----
    {
      std::vector<int32_t> tie_group(std::max<uint32_t>(nslots, 1), -1);
      std::vector<uint32_t> tie_off{0}, tie_slot;
      for (uint32_t i = 0; i < nslots; ++i) {
        const Cand& b = hbest[i];
        const bool stops = b.count == 0 || b.numer == 0 ||
                           b.numer < u128(cfg.hitcount_stop_threshold) * u128(b.count);
        if (stops || b.ties <= 1) continue;
        tie_group[i] = int32_t(tie_slot.size());
        tie_slot.push_back(i);
        tie_off.push_back(tie_off.back() + uint32_t(b.ties));
      }
      if (!tie_slot.empty() && dist) {
        const uint32_t nt = uint32_t(tie_slot.size());
        const uint32_t* rv = dist->raw_ranks();
        auto d_tg = to_device(tie_group, s);
        DevBuf<unsigned long long> mk(nt, s);
        mk.fill_bytes(0xFF);
        PO_LAUNCH(k_tie_min_raw, L.nitems, kArgBlock, 0, s,
                  reinterpret_cast<WorkSeg*>(dp + o_work), uint32_t(L.work.size()), reinterpret_cast<ScanSlot*>(dp + o_slots),
                  reinterpret_cast<uint32_t*>(dp + o_masks), reinterpret_cast<uint32_t*>(dp + o_w),
                  colbase, vlen, m, K, d_best, d_tg.get(), rv, mk.get(), part, nparts);
        if (nparts > 1) {  // min over the ranks' shares = ~max(~x)
          PO_LAUNCH(k_complement_u64, grid_for(nt, 128), 128, 0, s, mk.get(), nt);
          dist->comm->allreduce(mk.get(), nt, CDtype::U64, COp::Max, s);
          PO_LAUNCH(k_complement_u64, grid_for(nt, 128), 128, 0, s, mk.get(), nt);
        }
        std::vector<unsigned long long> hm(nt);
        d2h_sync(hm.data(), mk.get(), (nt) * sizeof(*mk.get()), s);
        for (uint32_t g = 0; g < nt; ++g) hbest[tie_slot[g]].vid = uint32_t(hm[g]);
      } else if (!tie_slot.empty()) {
        const uint32_t ng = uint32_t(tie_slot.size()), total = tie_off.back();
        auto d_tg = to_device(tie_group, s);
        auto d_toff = to_device(tie_off, s);
        DevBuf<uint32_t> cursor(ng, s), t_ref(total, s), t_vid(total, s), t_grp(total, s),
            t_pos(total, s), min_vid(ng, s);
        cursor.zero();
        PO_LAUNCH(k_collect_ties, L.nitems, kArgBlock, 0, s,
                  reinterpret_cast<WorkSeg*>(dp + o_work), uint32_t(L.work.size()), reinterpret_cast<ScanSlot*>(dp + o_slots),
                  reinterpret_cast<uint32_t*>(dp + o_masks), reinterpret_cast<uint32_t*>(dp + o_w),
                  colbase, vlen, m, K, d_best, d_tg.get(), d_toff.get(), cursor.get(),
                  t_ref.get(), t_vid.get(), t_grp.get());
        RefineJob tj;
        tj.n_items = total;
        tj.d_grp_init = t_grp.get();
        tj.d_grp_start = d_toff.get();
        tj.n_groups = ng;
        tj.grp_max = total;
        tj.key.kind = 0;  // raw bytes
        tj.key.arena = e.val_arena;
        tj.key.arena_bytes = e.val_bytes;
        tj.key.str_off = e.val_off.get();
        tj.key.str_len = e.val_len.get();
        tj.key.item_ref = t_ref.get();
        tj.d_out_pos = t_pos.get();
        refine_sort_multi({tj}, s);
        PO_LAUNCH(k_pick_min, grid_for(total, 256), 256, 0, s, t_pos.get(), t_grp.get(),
                  t_vid.get(), d_toff.get(), total, min_vid.get());
        std::vector<uint32_t> hmin(ng);
        d2h_sync(hmin.data(), min_vid.get(), (ng) * sizeof(*min_vid.get()), s);
        for (uint32_t g = 0; g < ng; ++g) hbest[tie_slot[g]].vid = hmin[g];
      }
    }

    // ---- host decisions (ggr.hpp:276-301) ----
    std::optional<HostScope> hs_dec(std::in_place, "lvl_decide");
    std::vector<int> next;
    struct SplitH {
      int node;
      SplitD d;
    };
    std::vector<SplitH> splits;
    std::vector<HTable*> new_tables;  // block children's tables of this level
    if (debug_timing()) {
      unsigned long long sh = 0, st = 0;
      for (uint32_t i = 0; i < nslots; ++i) {
        sh += hn[i];
        st += hbest[i].ties;
      }
      fprintf(stderr, "[po level] rank %d slots %u work %zu cands %llu ties %llu\n",
              dist ? dist->comm->rank() : 0, nslots, size_t(L.nitems), sh, st);
    }
    for (uint32_t i = 0; i < nslots; ++i) {
      const int id = frontier[i];
      out.stats.candidates_examined += hn[i] + unique_groups[i];
      const Cand& b = hbest[i];
      if (b.count == 0 || b.numer == 0 ||
          b.numer < u128(cfg.hitcount_stop_threshold) * u128(b.count)) {
        nodes[id].kind = FALLBACK;  // early stop: statistics fallback
        pending.push_back(id);
        continue;
      }
      Node& P = nodes[id];
      P.kind = SPLIT;
      std::vector<char> act(m, 0);
      for (int c : P.cols) act[c] = 1;
      P.block_cols = {int(b.col)};
      for (int o : partners[b.col])
        if (act[o]) P.block_cols.push_back(o);
      Node B, R;
      B.size = b.count;
      for (int c : P.cols)
        if (std::find(P.block_cols.begin(), P.block_cols.end(), c) == P.block_cols.end())
          B.cols.push_back(c);
      B.rd = P.rd;
      B.cd = P.cd + 1;
      B.depth = P.depth + 1;
      R.size = P.size - b.count;
      R.cols = P.cols;
      R.rd = P.rd + 1;
      R.cd = P.cd;
      R.depth = P.depth + 1;
      B.kind = classify(B, cfg);
      R.kind = classify(R, cfg);
      out.stats.recursive_calls += 2;
      out.stats.max_depth = std::max<uint64_t>(out.stats.max_depth, P.depth + 1);
      const bool needB = B.kind == SCAN || B.kind == FALLBACK;
      const bool needR = R.kind == SCAN || R.kind == FALLBACK;
      SplitD d{};
      d.mask_off = 0;
      d.col = b.col;
      d.vid = b.vid;
      if (needB) {
        // entries <= sum over the parent's columns of min(card, |B|)
        uint64_t bound = 0;
        for (int c : P.cols)
          if (uidx[c] < 0) bound += std::min<uint64_t>(e.card[c], B.size);
        uint64_t cap = 64;
        while (cap < bound + bound / 2) cap <<= 1;
        auto t = std::make_shared<HTable>();
        t->cap = cap;  // memory: alloc_tables after the level's decisions
        B.table = t;
        new_tables.push_back(t.get());
      }
      if (needR) {
        R.table = P.table;
        d.tP = P.table->desc();
      }
      d.need_rows = (needB || needR) ? 1u : 0u;
      P.table.reset();
      const int bid = int(nodes.size());
      P.block_child = bid;
      P.rest_child = bid + 1;
      d.block_id = uint32_t(bid);
      d.rest_id = uint32_t(bid + 1);
      splits.push_back({id, d});
      nodes.push_back(std::move(B));
      nodes.push_back(std::move(R));
      for (int ch : {bid, bid + 1}) {
        if (nodes[ch].kind == SCAN) next.push_back(ch);
        else if (nodes[ch].kind == FALLBACK) pending.push_back(ch);
      }
    }

    hs_dec.reset();
    alloc_tables(new_tables, K, s);
    HostScope hs_split("lvl_split");
    for (SplitH& sh : splits)
      if (nodes[sh.d.block_id].table) sh.d.tB = nodes[sh.d.block_id].table->desc();

    // ---- K6 split + K4 aggregation ----
    if (!splits.empty()) {
      const uint32_t ns = uint32_t(splits.size());
      std::sort(splits.begin(), splits.end(),
                [](const SplitH& a, const SplitH& b) { return a.node < b.node; });
      std::vector<SplitD> hsp(ns);
      std::vector<uint64_t> seg(ns + 1, 0);
      std::vector<uint32_t> split_nodes(ns);
      std::vector<AggSeg> tasks, usegs;
      uint32_t ntask = 0, nutask = 0;
      for (uint32_t j = 0; j < ns; ++j) {
        hsp[j] = splits[j].d;
        split_nodes[j] = uint32_t(splits[j].node);
        const uint64_t rows = hsp[j].need_rows ? nodes[hsp[j].block_id].size : 0;
        seg[j + 1] = seg[j] + rows;
        if (!rows) continue;
        const Node& P = nodes[splits[j].node];
        const Node& B = nodes[hsp[j].block_id];
        std::vector<char> inB(m, 0);
        for (int c : B.cols) inB[c] = 1;
        for (int c : P.cols) {
          if (uidx[c] >= 0) {  // length sum of the block rows only
            add_agg_seg(usegs, nutask, j, uint32_t(c), 0u, 0u, seg[j], seg[j + 1]);
            continue;
          }
          const uint32_t to_b = (hsp[j].tB.keys && inB[c]) ? 1u : 0u;
          const uint32_t to_p = hsp[j].tP.cnt ? 1u : 0u;
          if (!to_b && !to_p) continue;
          add_agg_seg(tasks, ntask, j, uint32_t(c), to_b, to_p, seg[j], seg[j + 1]);
        }
      }
      // dense node -> split index table over this level's node id range
      const uint32_t node_lo = split_nodes.front();
      const uint32_t lut_n = split_nodes.back() - node_lo + 1;
      std::vector<int32_t> lut(lut_n, -1);
      for (uint32_t j = 0; j < ns; ++j) lut[split_nodes[j] - node_lo] = int32_t(j);
      Pack sp;
      const size_t o_sp = sp.add(hsp), o_seg = sp.add(seg), o_sn = sp.add(lut);
      const size_t o_tasks = sp.add(tasks);
      const size_t o_cursor = sp.add(std::vector<uint32_t>(ns, 0u));
      const size_t o_usegs = sp.add(usegs), o_parent = sp.add(split_nodes);
      const size_t o_ublk = sp.add(std::vector<unsigned long long>(size_t(ns) * U, 0ull));
      const size_t o_udone = sp.add(std::vector<uint32_t>(1, 0u));
      uint8_t* ds = upload(sp);
      auto* d_sp = reinterpret_cast<SplitD*>(ds + o_sp);
      auto* d_seg = reinterpret_cast<uint64_t*>(ds + o_seg);
      auto* d_lut = reinterpret_cast<int32_t*>(ds + o_sn);
      auto* d_cursor = reinterpret_cast<uint32_t*>(ds + o_cursor);
      DevBuf<uint32_t> blockrows(std::max<uint64_t>(1, seg[ns]), s);
      PO_LAUNCH(k_relabel, grid_for(n, kRelabelBlock), kRelabelBlock,
                lut_n <= kRelabelSmem ? lut_n * 4 : 0, s,
                node_of_row.get(), n, d_lut, node_lo, lut_n, d_sp, e.vid.get(), m, d_cursor,
                d_seg, blockrows.get());
      if (!dist && !tasks.empty())
        PO_AGG(ntask, kAggBlock, 0, s, reinterpret_cast<AggSeg*>(ds + o_tasks),
                  uint32_t(tasks.size()), blockrows.get(), d_sp, e.vid.get(),
                  vlen, colbase, m, K, d_dpart.get(), d_npart.get());
      if (U) {
        grow_usum(nodes.size());
        auto* d_ublk = reinterpret_cast<unsigned long long*>(ds + o_ublk);
        PO_LAUNCH(k_unique_sums, std::max<uint32_t>(nutask, 1), kAggBlock, 0, s,
                  reinterpret_cast<AggSeg*>(ds + o_usegs), uint32_t(usegs.size()), blockrows.get(),
                  e.vid.get(), vlen, colbase, m, d_uidx.get(), U, d_ublk, d_sp,
                  reinterpret_cast<uint32_t*>(ds + o_parent), ns, usum.get(),
                  reinterpret_cast<uint32_t*>(ds + o_udone));
      }
      if (dist) {
        // this rank's block rows -> private tables -> contributions, all-gathered
        // and applied to the replicated child / parent tables
        std::vector<uint32_t> lcnt(ns);
        PO_CUDA(cudaMemcpyAsync(lcnt.data(), d_cursor, ns * 4, cudaMemcpyDeviceToHost, s));
        sync(s);
        std::vector<std::unique_ptr<HTable>> priv(ns);
        std::vector<SplitD> hsp2(hsp);
        std::vector<AggSeg> tasks2;
        uint32_t ntask2 = 0;
        std::vector<uint32_t> bmask(size_t(ns) * W, 0);
        uint64_t max_entries = 0;
        for (uint32_t j = 0; j < ns; ++j) {
          const Node& P = nodes[splits[j].node];
          for (int c : P.block_cols) bmask[size_t(j) * W + (uint32_t(c) >> 5)] |= 1u << (uint32_t(c) & 31);
          hsp2[j].tP = TDesc{};
          if (!hsp[j].need_rows || !lcnt[j]) continue;
          uint64_t bound = 0;
          for (int c : P.cols) bound += std::min<uint64_t>(e.card[c], lcnt[j]);
          uint64_t cap = 64;
          while (cap < bound + bound / 2) cap <<= 1;
          auto t = std::make_unique<HTable>();
          t->cap = cap;
          alloc_tables({t.get()}, K, s);
          hsp2[j].tB = t->desc();
          priv[j] = std::move(t);
          max_entries += bound;
          for (int c : P.cols)
            add_agg_seg(tasks2, ntask2, j, uint32_t(c), 1u, 0u, seg[j], seg[j] + lcnt[j]);
        }
        Pack p2;
        const size_t o_sp2 = p2.add(hsp2), o_t2 = p2.add(tasks2), o_bm = p2.add(bmask);
        DevBuf<uint8_t> dev2(p2.host.size(), s);
        dev2.upload(p2.host.data(), p2.host.size());
        if (!tasks2.empty())
          PO_AGG(ntask2, kAggBlock, 0, s,
                    reinterpret_cast<AggSeg*>(dev2.get() + o_t2), uint32_t(tasks2.size()),
                    blockrows.get(),
                    reinterpret_cast<SplitD*>(dev2.get() + o_sp2), e.vid.get(), vlen, colbase, m,
                    K, d_dpart.get(), d_npart.get());
        const uint32_t RW = 2 + K;
        DevBuf<uint64_t> contrib(std::max<uint64_t>(1, max_entries) * RW, s);
        DevBuf<unsigned long long> ccur(1, s);
        ccur.zero();
        for (uint32_t j = 0; j < ns; ++j)
          if (priv[j])
            PO_LAUNCH(k_compact_contrib, grid_for(priv[j]->cap, 256), 256, 0, s, priv[j]->desc(), j,
                      K, contrib.get(), ccur.get());
        unsigned long long El = 0;
        d2h_sync(&El, ccur.get(), (1) * sizeof(*ccur.get()), s);
        priv.clear();
        const std::vector<uint64_t> Es = dist->comm->allgather_host({uint64_t(El)}, s);
        std::vector<uint64_t> rbytes(Es.size());
        uint64_t Et = 0;
        for (size_t r = 0; r < Es.size(); ++r) {
          rbytes[r] = Es[r] * RW * 8;
          Et += Es[r];
        }
        DevBuf<uint64_t> allc(std::max<uint64_t>(1, Et) * RW, s);
        dist->comm->allgatherv(contrib.get(), allc.get(), rbytes, s);
        PO_LAUNCH(k_apply_contrib, grid_for(Et, 256), 256, 0, s, Et, allc.get(), K, d_sp,
                  reinterpret_cast<uint32_t*>(dev2.get() + o_bm), W, colbase);
        sync(s);
      }
    }
    if (debug_checks() && !dist) {
      DevBuf<unsigned long long> hist(nodes.size() + 1, s);
      hist.zero();
      PO_LAUNCH(k_dbg_node_hist, grid_for(n, 256), 256, 0, s, node_of_row.get(), n,
                uint32_t(nodes.size()), hist.get());
      std::vector<unsigned long long> hh(nodes.size() + 1);
      d2h_sync(hh.data(), hist.get(), (hh.size()) * sizeof(*hist.get()), s);
      for (size_t id = 0; id < nodes.size(); ++id) {
        const Node& nd = nodes[id];
        const bool live = nd.kind != SPLIT;
        if (live && hh[id] != nd.size)
          fprintf(stderr, "[po debug] level: node %zu kind %d size %llu but %llu rows labelled\n",
                  id, nd.kind, (unsigned long long)nd.size, hh[id]);
        if (!live && hh[id])
          fprintf(stderr, "[po debug] split node %zu still labels %llu rows\n", id, hh[id]);
      }
      if (hh[nodes.size()]) fprintf(stderr, "[po debug] %llu rows with invalid node\n", hh[nodes.size()]);
    }
    timing_mark("levels", s);
    frontier.swap(next);
  }


  // ---- layout: leaves in DFS order, block subtree first ----
  std::vector<int> leaf_nodes;
  std::vector<std::vector<int>> leaf_full_order;
  std::vector<uint32_t> node_leaf(nodes.size(), 0);
  {
    struct Frame {
      int id;
      std::vector<int> prefix;
    };
    std::vector<Frame> stack;
    stack.push_back({0, {}});
    while (!stack.empty()) {
      Frame f = std::move(stack.back());
      stack.pop_back();
      const Node& nd = nodes[f.id];
      if (nd.kind == SPLIT) {
        std::vector<int> bp = f.prefix;
        bp.insert(bp.end(), nd.block_cols.begin(), nd.block_cols.end());
        stack.push_back({nd.rest_child, f.prefix});  // popped after the block subtree
        stack.push_back({nd.block_child, std::move(bp)});
        continue;
      }
      if (nd.kind == EMPTY) continue;
      std::vector<int> full = f.prefix;
      if (nd.kind == FALLBACK) full.insert(full.end(), nd.leaf_order.begin(), nd.leaf_order.end());
      else full.insert(full.end(), nd.cols.begin(), nd.cols.end());
      if (full.size() < m) fail(PO_ERR_ERROR, "internal: leaf field order misses fields");
      node_leaf[f.id] = uint32_t(leaf_nodes.size());
      leaf_nodes.push_back(f.id);
      leaf_full_order.push_back(std::move(full));
    }
  }
  const uint32_t nleaves = uint32_t(leaf_nodes.size());
  std::vector<uint32_t> leaf_off(nleaves, 0), leaf_chunk_off(nleaves), leaf_nchunks(nleaves);
  // repeated FD pairs make some field orders longer than m: CSR output
  bool csr = false;
  for (const auto& fo : leaf_full_order) csr |= fo.size() != m;
  if (csr && dist)
    fail(PO_ERR_SCHEMA, "sharded ggr: FD groups repeating a field pair are not supported");
  std::vector<int32_t> h_leaf_orders(csr ? 0 : size_t(nleaves) * m);
  KeySchedule ks;
  TieSpec ties;
  // round 0 groups the rows by leaf index; later rounds by start position
  const int cap0 = int(refine_chunk_bits(nleaves ? nleaves - 1 : 0));
  const int cap = 64;  // rounds >= 1 sort inside groups: the chunk alone
  uint64_t off = 0;
  for (uint32_t l = 0; l < nleaves; ++l) {
    const Node& nd = nodes[leaf_nodes[l]];
    leaf_off[l] = uint32_t(off);
    off += nd.size;
    if (!csr)
      std::copy(leaf_full_order[l].begin(), leaf_full_order[l].end(),
                h_leaf_orders.begin() + size_t(l) * m);
    // sort keys of the leaf
    std::vector<std::pair<int, uint8_t>> keys;  // (field, kind)
    // single-column leaves are ordered by raw bytes in a separate string job
    ties.tie_col.push_back(-1);
    if (nd.kind == FALLBACK)  // fragment keys (ggr.hpp:340-350)
      for (int f : nd.leaf_order) {
        if (e.is_unranked(f)) {  // distinct per row: break_unranked_ties
          ties.tie_col.back() = f;
          break;
        }
        keys.push_back({f, uint8_t(1)});
      }
    if (ties.tie_col.back() >= 0)
      for (const auto& k : keys) ties.key_fields.push_back(k.first);
    ties.key_off.push_back(uint32_t(ties.key_fields.size()));
    leaf_chunk_off[l] = uint32_t(ks.chunk_nkeys.size());
    leaf_nchunks[l] = ks.add_leaf(keys, e.card, cap0, cap);
  }
  if (off != ng) fail(PO_ERR_ERROR, "internal: leaves do not cover the table");
  if (dist) {
    // distributed layout: leaf order, leaf keys, global row id (ggr.hpp:303-350)
    std::vector<LeafKeys> lk(nleaves);
    for (uint32_t l = 0; l < nleaves; ++l) {
      const Node& nd = nodes[leaf_nodes[l]];
      lk[l].full_order = leaf_full_order[l];
      if (nd.kind == FALLBACK) {
        lk[l].kind = 1;
        lk[l].fields = nd.leaf_order;
      } else if (nd.kind == RAW1) {
        lk[l].kind = 2;
        lk[l].fields = {nd.cols[0]};
      }
    }
    auto d_node_leaf = to_device(node_leaf, s);
    auto d_leaf_off = to_device(leaf_off, s);
    DevBuf<uint32_t> row_leaf(n, s), grp(n, s);
    PO_LAUNCH(k_row_leaf, grid_for(n, 256), 256, 0, s, node_of_row.get(), n, d_node_leaf.get(),
              d_leaf_off.get(), row_leaf.get(), grp.get());
    out.phc = dist_layout(*dist, e, row_leaf.get(), lk, s);
    timing_mark("dist_layout", s);
    // whole-table fallback competition (ggr.hpp:379-387) from global stats;
    // the bound uses the replicated counts, so every rank decides alike
    if (fallback_cannot_win(e, out.phc, s)) {
      timing_mark("dist_fallback_bound", s);
      sync(s);
      return;
    }
    std::vector<double> avg(m);
    for (uint32_t c = 0; c < m; ++c)
      avg[c] = static_cast<double>(e.total_len[c]) / static_cast<double>(ng);
    const std::vector<int> fb_order = hitcount_order(ng, e.card, avg, cfg.stats_variant);
    DistCtx fb;
    fb.comm = dist->comm;
    fb.n_global = ng;
    fb.row_offset = dist->row_offset;
    fb.raw_ranks = dist->raw_ranks;
    row_leaf.zero();
    LeafKeys one;
    one.kind = 1;
    one.fields = fb_order;
    one.full_order = fb_order;
    const uint64_t fb_phc = dist_layout(fb, e, row_leaf.get(), {one}, s);
    if (fb_phc > out.phc) {  // replace only when strictly better (ggr.hpp:383)
      dist->slice_offset = fb.slice_offset;
      dist->slice_count = fb.slice_count;
      dist->rows = std::move(fb.rows);
      dist->orders = std::move(fb.orders);
      out.phc = fb_phc;
    }
    timing_mark("dist_fallback", s);
    sync(s);
    return;
  }
  ks.pad();
  const auto& chunk_key_off = ks.chunk_key_off;
  const auto& chunk_nkeys = ks.chunk_nkeys;
  const auto& key_field = ks.key_field;
  const auto& key_kind = ks.key_kind;
  const auto& key_bits = ks.key_bits;
  auto d_node_leaf = to_device(node_leaf, s);
  auto d_leaf_off = to_device(leaf_off, s);
  auto d_lco = to_device(leaf_chunk_off, s), d_lnc = to_device(leaf_nchunks, s);
  auto d_cko = to_device(chunk_key_off, s), d_cnk = to_device(chunk_nkeys, s);
  auto d_kf = to_device(key_field, s);
  auto d_kk = to_device(key_kind, s), d_kb = to_device(key_bits, s);
  auto d_leaf_orders = to_device(h_leaf_orders, s);
  DevBuf<uint32_t> row_leaf = dev_auto<uint32_t>(n, s), grp = dev_auto<uint32_t>(n, s),
                   pos = dev_auto<uint32_t>(n, s);
  PO_LAUNCH(k_row_leaf, grid_for(n, 256), 256, 0, s, node_of_row.get(), n, d_node_leaf.get(),
            d_leaf_off.get(), row_leaf.get(), grp.get());
  RefineKey RK;
  RK.kind = 2;
  RK.m = m;
  RK.vid = e.vid.get();
  RK.colbase = colbase;
  RK.row_leaf = row_leaf.get();
  RK.leaf_chunk_off = d_lco.get();
  RK.leaf_nchunks = d_lnc.get();
  RK.chunk_key_off = d_cko.get();
  RK.chunk_nkeys = d_cnk.get();
  RK.key_field = d_kf.get();
  RK.key_kind = d_kk.get();
  RK.key_bits = d_kb.get();
  timing_mark("layout", s);
  if (debug_timing()) {  // rows per leaf kind and key width of the leaf sort
    uint64_t rows_by_kind[8] = {0};
    uint32_t leaves_by_kind[8] = {0};
    for (uint32_t l = 0; l < nleaves; ++l) {
      const Node& nd = nodes[leaf_nodes[l]];
      rows_by_kind[nd.kind] += nd.size;
      leaves_by_kind[nd.kind]++;
    }
    fprintf(stderr, "[po leaves] %u leaves; rows/leaves by kind:", nleaves);
    const char* kn[] = {"scan", "empty", "rowid", "single", "raw1", "fallback", "split"};
    for (int k = 0; k < 7; ++k)
      if (leaves_by_kind[k])
        fprintf(stderr, " %s %llu/%u", kn[k], (unsigned long long)rows_by_kind[k], leaves_by_kind[k]);
    fprintf(stderr, "; chunk bits round0 %u later %u\n", ks.widest0, ks.widest);
  }
  RefineJob leaf_job;
  leaf_job.n_items = uint32_t(n);
  leaf_job.d_grp_init = row_leaf.get();  // round 0: leaf index
  leaf_job.d_grp_start = d_leaf_off.get();
  leaf_job.n_groups = nleaves;
  leaf_job.grp_max = uint32_t(n);
  leaf_job.key = RK;
  leaf_job.d_out_pos = pos.get();
  leaf_job.row_chunk_bits0 = ks.widest0;
  leaf_job.row_chunk_bits = ks.widest;
  // single-column leaves (ggr.hpp:221-231): their rows, ascending row id, are
  // sorted by the raw bytes of the one column; positions overwrite the main
  // job's (which leaves them in row order)
  std::vector<int32_t> leaf_raw1_col(std::max<uint32_t>(nleaves, 1), -1);
  bool any_raw1 = false;
  for (uint32_t l = 0; l < nleaves; ++l)
    if (nodes[leaf_nodes[l]].kind == RAW1) {
      leaf_raw1_col[l] = nodes[leaf_nodes[l]].cols[0];
      any_raw1 = true;
    }
  DevBuf<uint32_t> raw_rows, raw_grp, raw_col, raw_pos;
  uint32_t n_raw = 0;
  std::vector<RefineJob> sort_jobs{leaf_job};
  if (any_raw1) {
    auto d_lrc = to_device(leaf_raw1_col, s);
    DevBuf<uint8_t> flags(n, s);
    PO_LAUNCH(k_raw1_flags, grid_for(n, 256), 256, 0, s, row_leaf.get(), n, d_lrc.get(),
              flags.get());
    raw_rows.alloc(n, s);
    DevBuf<int> nsel(1, s);
    cub::CountingInputIterator<uint32_t> it(0);
    size_t tb = 0;
    PO_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, flags.get(), raw_rows.get(), nsel.get(),
                                       int(n), s));
    DevBuf<uint8_t> tmp(tb, s);
    PO_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, it, flags.get(), raw_rows.get(), nsel.get(),
                                       int(n), s));
    int hn1 = 0;
    d2h_sync(&hn1, nsel.get(), (1) * sizeof(*nsel.get()), s);
    n_raw = uint32_t(hn1);
    raw_grp.alloc(n_raw, s);
    raw_col.alloc(n_raw, s);
    raw_pos.alloc(n_raw, s);
    PO_LAUNCH(k_raw1_items, grid_for(n_raw, 256), 256, 0, s, raw_rows.get(), n_raw, row_leaf.get(),
              d_lrc.get(), e.vid.get(), colbase, m, raw_grp.get(), raw_col.get());
    RefineJob rj;
    rj.n_items = n_raw;
    rj.d_grp_init = raw_grp.get();
    rj.d_grp_start = d_leaf_off.get();
    rj.n_groups = nleaves;
    rj.grp_max = uint32_t(n);
    rj.key.kind = 0;  // raw bytes
    rj.key.arena = e.val_arena;
    rj.key.arena_bytes = e.val_bytes;
    rj.key.str_off = e.val_off.get();
    rj.key.str_len = e.val_len.get();
    rj.key.item_ref = raw_col.get();  // distinct value of each item's cell
    rj.d_out_pos = raw_pos.get();
    sort_jobs.push_back(rj);
  }
  refine_sort_multi(sort_jobs, s);
  if (n_raw)
    PO_LAUNCH(k_raw1_scatter, grid_for(n_raw, 256), 256, 0, s, raw_rows.get(), raw_pos.get(), n_raw,
              pos.get());
  timing_mark("leaf_sort", s);
  if (ties.any()) {
    break_unranked_ties(e, ties, row_leaf.get(), d_leaf_off.get(), pos.get(), s);
    timing_mark("leaf_ties", s);
  }
  if (debug_checks()) {
    DevBuf<unsigned> seen(n, s);
    DevBuf<unsigned long long> bad(1, s);
    seen.zero();
    bad.zero();
    PO_LAUNCH(k_dbg_perm, grid_for(n, 256), 256, 0, s, pos.get(), n, seen.get(), bad.get());
    unsigned long long hb = 0;
    d2h_sync(&hb, bad.get(), (1) * sizeof(*bad.get()), s);
    if (hb) fprintf(stderr, "[po debug] leaf sort positions: %llu collisions/out of range\n", hb);
  }
  PO_LAUNCH(k_emit, grid_for(n, 256), 256, 0, s, pos.get(), n, d_rows);
  if (!csr) {
    PO_LAUNCH(k_emit_orders, grid_for(n * m, 256), 256, 0, s, d_rows, n, m, row_leaf.get(),
              d_leaf_orders.get(), d_orders);
    if (early_fb)
      phc_device_raw_async(e.vid.get(), e.vlen.get(), e.d_colbase.get(), e.n, e.m, n, nullptr, d_rows,
                           nullptr, d_orders, s, fbres.get() + 2,
                           reinterpret_cast<int*>(fbres.get() + 3));
    else
      out.phc = phc_device(e, n, nullptr, d_rows, nullptr, d_orders, s);
  } else {
    // leaf l's rows hold positions [leaf_off[l], + size) and each takes
    // |full order of l| fields: CSR offsets per position
    std::vector<int32_t> lf;
    std::vector<uint32_t> lf_off(nleaves + 1, 0), lw(nleaves);
    std::vector<uint64_t> lbase(nleaves);
    uint64_t total = 0;
    for (uint32_t l = 0; l < nleaves; ++l) {
      lf.insert(lf.end(), leaf_full_order[l].begin(), leaf_full_order[l].end());
      lf_off[l + 1] = uint32_t(lf.size());
      lw[l] = uint32_t(leaf_full_order[l].size());
      lbase[l] = total;
      total += nodes[leaf_nodes[l]].size * lw[l];
    }
    auto d_lf = to_device(lf, s);
    auto d_lf_off = to_device(lf_off, s);
    auto d_lw = to_device(lw, s);
    auto d_lbase = to_device(lbase, s);
    auto d_loff = to_device(leaf_off, s);
    out.csr = true;
    out.csr_total = total;
    out.csr_offsets.alloc(n + 1, s);
    out.csr_fields.alloc(std::max<uint64_t>(total, 1), s);
    PO_LAUNCH(k_emit_orders_csr, grid_for(n, 256), 256, 0, s, d_rows, n, row_leaf.get(), d_lf.get(),
              d_lf_off.get(), d_lw.get(), d_lbase.get(), d_loff.get(), total,
              out.csr_offsets.get(), out.csr_fields.get());
    if (early_fb)
      phc_device_raw_async(e.vid.get(), e.vlen.get(), e.d_colbase.get(), e.n, e.m, n, nullptr, d_rows,
                           out.csr_offsets.get(), out.csr_fields.get(), s, fbres.get() + 2,
                           reinterpret_cast<int*>(fbres.get() + 3));
    else
      out.phc = phc_device(e, n, nullptr, d_rows, out.csr_offsets.get(), out.csr_fields.get(), s);
  }
  timing_mark("emit_phc", s);

  // ---- whole-table fallback competition (ggr.hpp:379-387) ----
  uint64_t fb_phc = 0;
  if (early_fb) {
    PO_CUDA(cudaStreamWaitEvent(s, fb_join.ev, 0));
    unsigned long long h[4];
    d2h_sync(h, fbres.get(), sizeof(h), s);
    int err = 0;
    std::memcpy(&err, &h[3], sizeof(err));
    if (err) fail(PO_ERR_OUT_OF_RANGE, "schedule references a row or field outside the table");
    out.phc = n > 1 ? h[2] : 0;
    double ub = 0;
    std::memcpy(&ub, &h[1], sizeof(ub));
    if (fallback_bound_prunes(e, ub, out.phc)) return;
    fb_phc = n > 1 ? h[0] : 0;
  } else {
    if (!debug_checks() && fallback_cannot_win(e, out.phc, s)) {
      timing_mark("fallback_bound", s);
      return;
    }
    std::vector<double> avg(m);
    for (uint32_t c = 0; c < m; ++c)
      avg[c] = static_cast<double>(e.total_len[c]) / static_cast<double>(ng);
    fb_order = hitcount_order(ng, e.card, avg, cfg.stats_variant);
    fb_phc = fixed_order_phc_device(e, fb_order, s);  // prefix groups, no sort
  }
  timing_mark("fallback_phc", s);
  std::vector<int32_t> fo(fb_order.begin(), fb_order.end());
  auto d_fo = to_device(fo, s);
  if (debug_checks()) {  // the prefix-group PHC against the materialised sort
    DevBuf<uint32_t> perm(n, s);
    sort_all_rows(e, fb_order, perm.get(), s);
    const uint64_t chk = phc_device(e, n, nullptr, perm.get(), nullptr, d_fo.get(), s, 1, true);
    if (chk != fb_phc)
      fprintf(stderr, "[po debug] fallback phc %llu but the sorted order scores %llu\n",
              (unsigned long long)fb_phc, (unsigned long long)chk);
  }
  if (fb_phc > out.phc) {  // replace only when strictly better (ggr.hpp:383)
    sort_all_rows(e, fb_order, d_rows, s);
    PO_LAUNCH(k_tile_order, grid_for(n * m, 256), 256, 0, s, d_fo.get(), n, m, d_orders);
    out.phc = fb_phc;
    out.csr = false;  // every order is the fallback's m fields
    out.csr_offsets.release();
    out.csr_fields.release();
  }
  // no sync: the outputs are stream-ordered on s and every caller
  // synchronises after delivering them
}

}  // namespace po
