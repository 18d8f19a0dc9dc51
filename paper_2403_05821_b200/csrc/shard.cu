// Row-sharded GGR over 1..N GPUs.
//
// Rows are range-partitioned: rank r holds rows [row_offset, row_offset+n_r)
// of the table. The solve is the single-GPU level-synchronous GGR
// (ggr.cu) with three distributed pieces:
//
//  1. Global dictionary (this file, `global_ranks`). Every rank encodes its
//     rows locally (K1/K2: the byte-bound hash + exact dictionary pass, the
//     dominant HBM traffic, fully parallel). The local distinct values are
//     then sample-sorted across ranks in escaped fragment-key order
//     (scoring.hpp:33-69): sampled splitters, one all-to-all of (column,
//     bytes) per distinct value to the owner of its key range, an exact
//     merge + dedup at the owner (the refine sort and a byte compare of
//     neighbours), and the global rank sent back. Equal values always meet
//     at one owner, so ids are exact regardless of hash collisions. The raw
//     byte order (candidate ties ggr.hpp:196, single-column leaves
//     ggr.hpp:221-231) is ranked the same way, on first use only.
//  2. Replicated value-group tables. The root histogram is the global value
//     count (an allreduce of scattered local counts, plus an allreduce of
//     the FD partner-length sums); per level, every rank aggregates ITS block
//     rows into a private table, the compacted (column, value, count,
//     partner sums) contributions are all-gathered and applied to the
//     replicated child/parent tables. All sums are integers, so every rank
//     holds bit-identical tables and takes identical decisions
//     (ggr.hpp:239-301) without further communication.
//  3. Distributed layout (`dist_layout`). Each row gets one packed key
//     (leaf in DFS order, leaf sort keys, global row id) — a total order
//     equal to the single-GPU leaf sort (ggr.hpp:303-350); a sample sort
//     with one all-to-all of row records leaves rank r with a contiguous
//     slice of the schedule. PHC (objective.hpp:94-99) is the sum of the
//     slices' PHC plus one boundary pair per rank (the previous non-empty
//     rank's last request), allreduced.
// The whole-table fallback (ggr.hpp:379-387) is laid out and scored the same
// way from global statistics.

#include <cub/cub.cuh>

#include <algorithm>
#include <mutex>
#include <numeric>

#include "comm.cuh"
#include "internal.cuh"

namespace po {

namespace {

// ---------------------------------------------------------------------------
// byte orders: 0 = raw (unsigned bytes, shorter prefix first), 1 = escaped
// fragment key (json_escape(v) + '"')
// ---------------------------------------------------------------------------
__constant__ uint16_t c_code[2][257];
uint16_t h_code[2][257];
std::mutex g_code_mu;
bool g_code_ready = false;

void ensure_codes() {
  std::lock_guard<std::mutex> lk(g_code_mu);
  if (g_code_ready) return;
  for (int b = 0; b < 256; ++b) h_code[0][b] = uint16_t(b + 2);
  h_code[0][256] = 1;
  esc_code_table(h_code[1]);
  PO_CUDA(cudaMemcpyToSymbol(c_code, h_code, sizeof(h_code)));
  g_code_ready = true;
}

template <class Code>
__host__ __device__ __forceinline__ int cmp_bytes(const Code* code, const uint8_t* a, uint64_t la,
                                                  const uint8_t* b, uint64_t lb) {
  const uint64_t n = la < lb ? la : lb;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t x = code[a[i]], y = code[b[i]];
    if (x != y) return x < y ? -1 : 1;
  }
  if (la == lb) return 0;
  const uint32_t x = la == n ? code[256] : code[a[n]];
  const uint32_t y = lb == n ? code[256] : code[b[n]];
  return x < y ? -1 : 1;
}

// Local distinct values: item i (dense index colbase[c] + vid) is the cell
// (rep_row[i], icol[i]) of the local table.
struct LocalDict {
  const uint8_t* arena;
  const uint64_t* val_off;
  const uint32_t* val_len;
  const uint32_t* icol;  // column of each local distinct value
  __device__ __forceinline__ void str(uint32_t i, const uint8_t*& p, uint64_t& len) const {
    p = arena + val_off[i];
    len = val_len[i];
  }
};

constexpr uint32_t kSampleBytes = 56;
struct SampleRec {
  uint32_t col;  // 0xFFFFFFFF: no sample
  uint32_t len;
  uint8_t b[kSampleBytes];
};

__global__ void k_item_col(uint64_t D, const uint64_t* colbase, uint32_t m, uint32_t* icol) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < D;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t lo = 0, hi = m;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (colbase[mid] <= i) lo = mid;
      else hi = mid;
    }
    icol[i] = lo;
  }
}

__global__ void k_pack_samples(uint32_t S, uint64_t D, const uint32_t* ord, LocalDict d,
                               SampleRec* out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < S; j += gridDim.x * blockDim.x) {
    SampleRec r{};
    if (D == 0) {
      r.col = 0xFFFFFFFFu;
    } else {
      const uint64_t k = ((2 * uint64_t(j) + 1) * D) / (2 * uint64_t(S));
      const uint32_t i = ord ? ord[k] : uint32_t(k);
      const uint8_t* p;
      uint64_t len;
      d.str(i, p, len);
      r.col = d.icol[i];
      r.len = uint32_t(len < kSampleBytes ? len : kSampleBytes);
      for (uint32_t t = 0; t < r.len; ++t) r.b[t] = p[t];
    }
    out[j] = r;
  }
}

// bounds[j] = first sorted position whose (column, bytes) >= splitter j
__global__ void k_split_search(uint32_t nsp, const SampleRec* sp, uint64_t D, const uint32_t* ord,
                               LocalDict d, int kind, uint64_t* bounds) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nsp) return;
  const SampleRec s = sp[j];
  uint64_t lo = 0, hi = D;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    const uint32_t i = ord ? ord[mid] : uint32_t(mid);
    const uint32_t c = d.icol[i];
    bool less;
    if (c != s.col) {
      less = c < s.col;
    } else {
      const uint8_t* p;
      uint64_t len;
      d.str(i, p, len);
      less = cmp_bytes(c_code[kind], p, len, s.b, s.len) < 0;
    }
    if (less) lo = mid + 1;
    else hi = mid;
  }
  bounds[j] = lo;
}

__global__ void k_sorted_lens(uint64_t D, const uint32_t* ord, LocalDict d, uint64_t* lens) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < D;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint8_t* p;
    uint64_t len;
    d.str(ord ? ord[k] : uint32_t(k), p, len);
    lens[k] = len;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) lens[D] = 0;
}

// One warp per value (in sorted order): (column, length) record + bytes.
__global__ void k_pack_values(uint64_t D, const uint32_t* ord, LocalDict d, const uint64_t* boff,
                              const uint8_t* lim, uint2* meta, uint8_t* bytes) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t k = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; k < D; k += warps) {
    const uint32_t i = ord ? ord[k] : uint32_t(k);
    const uint8_t* p;
    uint64_t len;
    d.str(i, p, len);
    if (lane == 0) meta[k] = make_uint2(d.icol[i], uint32_t(len));
    uint8_t* dst = bytes + boff[k];
    // aligned 8-byte stores for the destination words fully inside the value
    // (other values share the edge words: bytes there)
    const uintptr_t da = reinterpret_cast<uintptr_t>(dst);
    const uint64_t head = std::min<uint64_t>(len, (8 - (da & 7)) & 7);
    const uint64_t body = (len - head) & ~uint64_t(7);
    if (lane < head) dst[lane] = p[lane];
    uint64_t* dw = reinterpret_cast<uint64_t*>(dst + head);
    for (uint64_t t = 8 * lane; t < body; t += 256) dw[t >> 3] = load8_unaligned(p + head + t, lim);
    for (uint64_t t = head + body + lane; t < len; t += 32) dst[t] = p[t];
  }
}

__global__ void k_gather_u64(const uint64_t* src, const uint64_t* idx, uint32_t n, uint64_t* out) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) out[j] = src[idx[j]];
}

// owner side ----------------------------------------------------------------
// The owner receives one run per source rank (run r = items [ro[r], ro[r+1])),
// each sorted by (column, byte order). Merged position of an item = its index
// in its run + the number of items of every other run that precede it (equal
// values: runs of lower rank first), so no re-sort is needed.
__global__ void k_meta_lens(uint64_t R, const uint2* meta, uint64_t* lens) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < R;
       i += uint64_t(gridDim.x) * blockDim.x)
    lens[i] = meta[i].y;
  if (blockIdx.x == 0 && threadIdx.x == 0) lens[R] = 0;
}

// Byte-order compare 8 bytes per step: the first differing byte comes from
// the lowest set byte of x ^ y (little-endian words), then its order code
// decides; a proper prefix compares the end code against the next byte.
__device__ __forceinline__ int cmp_bytes_w(int kind, const uint8_t* a, uint64_t la,
                                           const uint8_t* b, uint64_t lb, const uint8_t* lim) {
  const uint16_t* code = c_code[kind];
  const uint64_t n = la < lb ? la : lb;
  for (uint64_t i = 0; i < n; i += 8) {
    const uint64_t x = load8_unaligned(a + i, lim), y = load8_unaligned(b + i, lim);
    const uint64_t d = mask_low_bytes(x ^ y, n - i >= 8 ? 8u : uint32_t(n - i));
    if (d) {
      const uint32_t sh = uint32_t(__ffsll((long long)d) - 1) & ~7u;
      const uint32_t ca = code[(x >> sh) & 0xFF], cb = code[(y >> sh) & 0xFF];
      return ca < cb ? -1 : 1;
    }
  }
  if (la == lb) return 0;
  const uint32_t x = la == n ? code[256] : code[a[n]];
  const uint32_t y = lb == n ? code[256] : code[b[n]];
  return x < y ? -1 : 1;
}

__global__ void k_meta_col(uint64_t R, const uint2* __restrict__ meta, uint32_t* col) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < R;
       i += uint64_t(gridDim.x) * blockDim.x)
    col[i] = meta[i].x;
}

// new[k] = sorted value k differs from value k-1 (column or bytes)
__global__ void k_new_flags(uint64_t R, const uint32_t* perm, const uint2* meta,
                            const uint64_t* offs, const uint8_t* bytes, const uint8_t* lim,
                            uint32_t* flags) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < R;
       k += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t f = 1;
    if (k > 0) {
      const uint32_t a = perm[k], b = perm[k - 1];
      const uint2 ma = meta[a], mb = meta[b];
      if (ma.x == mb.x && ma.y == mb.y) {
        f = cmp_bytes_w(0, bytes + offs[a], ma.y, bytes + offs[b], mb.y, lim) != 0;
      }
    }
    flags[k] = f;
  }
}

// per column: number of distinct values the owner holds
__global__ void k_col_dcount(uint32_t m, const uint32_t* cstart, const uint32_t* u, uint64_t* dc) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  const uint32_t a = cstart[c], b = cstart[c + 1];
  dc[c] = b > a ? uint64_t(u[b - 1] - u[a] + 1) : 0;
}

__global__ void k_rank_out(uint64_t R, const uint32_t* pos, const uint2* meta, const uint32_t* u,
                           const uint32_t* cstart, const uint64_t* gstart, uint32_t* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < R;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t c = meta[i].x;
    out[i] = uint32_t(gstart[c] + (u[pos[i]] - u[cstart[c]]));
  }
}

__global__ void k_local_ranks(uint64_t D, const uint32_t* ord, const uint32_t* icol,
                              const uint64_t* colbase, uint32_t* out) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < D;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t i = ord ? ord[k] : uint32_t(k);
    out[i] = uint32_t(k - colbase[icol[i]]);
  }
}

__global__ void k_scatter_back(uint64_t D, const uint32_t* ord, const uint32_t* recv, uint32_t* out) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < D;
       k += uint64_t(gridDim.x) * blockDim.x)
    out[ord ? ord[k] : uint32_t(k)] = recv[k];
}

// global dictionary arrays -------------------------------------------------
__global__ void k_remap_vid(uint64_t cells, uint32_t m, const uint32_t* vid, const uint64_t* lcb,
                            const uint32_t* grank, uint32_t* gvid) {
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < cells;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t c = uint32_t(t % m);
    gvid[t] = grank[lcb[c] + vid[t]];
  }
}

__global__ void k_scatter_dict(uint64_t D, const uint32_t* icol, const uint32_t* grank,
                               const uint64_t* gcb, const uint32_t* cnt, const uint64_t* vlen,
                               uint32_t* gcnt, unsigned long long* gvlen) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < D;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t g = gcb[icol[i]] + grank[i];
    gcnt[g] = cnt[i];
    gvlen[g] = vlen[i];
  }
}

__global__ void k_scatter_u32(uint64_t D, const uint32_t* icol, const uint32_t* grank,
                              const uint64_t* gcb, const uint32_t* val, uint32_t* out) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < D;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[gcb[icol[i]] + grank[i]] = val[i];
}

void inclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
  if (!n) return;
  size_t tb = 0;
  PO_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out, int64_t(n), s));
  DevBuf<uint8_t> tmp(tb, s);
  ProfScope ps("cub_scan", s);
  PO_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tb, in, out, int64_t(n), s));
}

// Global rank (within its column, in byte order `kind`) of every local
// distinct value of L; card_g receives the global distinct count per column.
DevBuf<uint32_t> global_ranks(Comm& comm, const Encoded& L, const uint32_t* d_icol, int kind,
                              std::vector<uint64_t>& card_g, cudaStream_t s) {
  ensure_codes();
  const int N = comm.size();
  const uint32_t m = L.m;
  const uint64_t D = L.D;
  LocalDict ld{L.val_arena, L.val_off.get(), L.val_len.get(), d_icol};

  // local order of the distinct values in `kind` (escaped: the vid order)
  DevBuf<uint32_t> ord;
  if (kind == 0 && D) {
    std::vector<uint32_t> cb32(m);
    for (uint32_t c = 0; c < m; ++c) cb32[c] = uint32_t(L.colbase[c]);
    auto d_cb32 = to_device(cb32, s);
    DevBuf<uint32_t> pos(D, s);
    RefineJob j;
    j.n_items = uint32_t(D);
    j.d_grp_init = d_icol;
    j.d_grp_start = d_cb32.get();
    j.n_groups = m;
    j.grp_max = uint32_t(D);
    j.key.kind = 0;
    j.key.arena = L.val_arena;
    j.key.arena_bytes = L.val_bytes;
    j.key.str_off = L.val_off.get();
    j.key.str_len = L.val_len.get();
    j.d_out_pos = pos.get();
    refine_sort_multi({j}, s);
    ord.alloc(D, s);
    PO_LAUNCH(k_invert, grid_for(D, 256), 256, 0, s, pos.get(), D, ord.get());
  }
  const uint32_t* d_ord = ord.get();

  if (N == 1) {  // one rank: the local order is the global order
    card_g = L.card;
    DevBuf<uint32_t> grank(D, s);
    PO_LAUNCH(k_local_ranks, grid_for(D, 256), 256, 0, s, D, d_ord, d_icol, L.d_colbase.get(),
              grank.get());
    return grank;
  }

  // splitters from regular samples of every rank
  constexpr uint32_t S = 128;
  DevBuf<SampleRec> smp(S, s), all(size_t(S) * N, s);
  PO_LAUNCH(k_pack_samples, 1, 128, 0, s, S, D, d_ord, ld, smp.get());
  comm.allgather(smp.get(), all.get(), S * sizeof(SampleRec), s);
  std::vector<SampleRec> hs(size_t(S) * N);
  all.download(hs.data(), hs.size());
  sync(s);
  std::vector<SampleRec> valid;
  for (const auto& r : hs)
    if (r.col != 0xFFFFFFFFu) valid.push_back(r);
  const uint16_t* hc = h_code[kind];
  std::sort(valid.begin(), valid.end(), [&](const SampleRec& a, const SampleRec& b) {
    if (a.col != b.col) return a.col < b.col;
    return cmp_bytes(hc, a.b, a.len, b.b, b.len) < 0;
  });
  std::vector<uint64_t> bounds(N + 1, 0);
  bounds[N] = D;
  if (N > 1) {
    std::vector<SampleRec> sp(N - 1);
    for (int j = 1; j < N; ++j)
      sp[j - 1] = valid.empty() ? SampleRec{0xFFFFFFFFu, 0, {}} : valid[(size_t(j) * valid.size()) / N];
    auto d_sp = to_device(sp, s);
    DevBuf<uint64_t> d_b(N - 1, s);
    PO_LAUNCH(k_split_search, 1, 32, 0, s, uint32_t(N - 1), d_sp.get(), D, d_ord, ld, kind,
              d_b.get());
    d_b.download(bounds.data() + 1, N - 1);
    sync(s);
  }

  // pack (column, length) + bytes in sorted order; per-destination sizes
  DevBuf<uint64_t> lens(D + 1, s), boff(D + 1, s);
  PO_LAUNCH(k_sorted_lens, grid_for(D + 1, 256), 256, 0, s, D, d_ord, ld, lens.get());
  exclusive_scan_u64(lens.get(), boff.get(), D + 1, s);
  std::vector<uint64_t> bb(N + 1, 0);
  {
    auto d_idx = to_device(bounds, s);
    DevBuf<uint64_t> d_bb(N + 1, s);
    PO_LAUNCH(k_gather_u64, 1, 64, 0, s, boff.get(), d_idx.get(), uint32_t(N + 1), d_bb.get());
    d_bb.download(bb.data(), N + 1);
    sync(s);
  }
  DevBuf<uint2> meta(D, s);
  DevBuf<uint8_t> sbytes(bb[N], s);
  PO_LAUNCH(k_pack_values, grid_for(D * 32, 256), 256, 0, s, D, d_ord, ld, boff.get(),
            L.val_arena + L.val_bytes, meta.get(),
            sbytes.get());
  std::vector<uint64_t> s_items(N), s_bytes(N), s_meta(N);
  for (int r = 0; r < N; ++r) {
    s_items[r] = bounds[r + 1] - bounds[r];
    s_meta[r] = s_items[r] * sizeof(uint2);
    s_bytes[r] = bb[r + 1] - bb[r];
  }
  // per destination: items, bytes and items per column (the sorted order
  // groups columns: column c holds positions [colbase[c], colbase[c+1]))
  const size_t W = 2 + size_t(m);
  std::vector<uint64_t> both(W * N, 0);
  for (int r = 0; r < N; ++r) {
    both[size_t(r) * W] = s_items[r];
    both[size_t(r) * W + 1] = s_bytes[r];
    for (uint32_t c = 0; c < m; ++c) {
      const uint64_t lo = std::max(bounds[r], L.colbase[c]);
      const uint64_t hi = std::min(bounds[r + 1], L.colbase[c + 1]);
      both[size_t(r) * W + 2 + c] = hi > lo ? hi - lo : 0;
    }
  }
  const std::vector<uint64_t> allc = comm.allgather_host(both, s);  // [src][dst][W]
  std::vector<uint64_t> r_items(N), r_meta(N), r_bytes(N);
  std::vector<uint32_t> cstart(m + 1, 0);
  uint64_t R = 0, RB = 0;
  for (int r = 0; r < N; ++r) {
    const uint64_t* e = &allc[(size_t(r) * N + comm.rank()) * W];
    r_items[r] = e[0];
    r_bytes[r] = e[1];
    r_meta[r] = r_items[r] * sizeof(uint2);
    R += r_items[r];
    RB += r_bytes[r];
    for (uint32_t c = 0; c < m; ++c) cstart[c + 1] += uint32_t(e[2 + c]);
  }
  for (uint32_t c = 0; c < m; ++c) cstart[c + 1] += cstart[c];  // merged column starts
  DevBuf<uint2> rmeta(R, s);
  DevBuf<uint8_t> rbytes(RB, s);
  comm.alltoallv(meta.get(), s_meta, rmeta.get(), r_meta, s);
  comm.alltoallv(sbytes.get(), s_bytes, rbytes.get(), r_bytes, s);
  meta.release();
  sbytes.release();

  // owner: exact merge of the received runs, dedup, ranks within the column
  std::vector<uint64_t> dcount(m, 0);
  DevBuf<uint32_t> rrank(R, s);
  DevBuf<uint32_t> u;
  DevBuf<uint32_t> d_cstart;
  DevBuf<uint32_t> pos;
  if (R) {
    DevBuf<uint64_t> rlens(R + 1, s), roffs(R + 1, s);
    PO_LAUNCH(k_meta_lens, grid_for(R + 1, 256), 256, 0, s, R, rmeta.get(), rlens.get());
    exclusive_scan_u64(rlens.get(), roffs.get(), R + 1, s);
    d_cstart = to_device(cstart, s);
    pos.alloc(R, s);
    // the received runs merged by one exact string sort: groups = columns
    // (placed at their merged starts), string order of `kind` inside, equal
    // strings in input order = lower source rank first. (A binary search of
    // every item in every other run cost ~7 ms per rank at N = 8 on C4 rows:
    // O(R N log R) string compares.)
    {
      DevBuf<uint32_t> col(R, s);
      PO_LAUNCH(k_meta_col, grid_for(R, 256), 256, 0, s, R, rmeta.get(), col.get());
      RefineJob j;
      j.n_items = uint32_t(R);
      j.d_grp_init = col.get();
      j.d_grp_start = d_cstart.get();
      j.n_groups = m;
      j.grp_max = uint32_t(R - 1);
      j.key.kind = kind;
      j.key.arena = rbytes.get();
      j.key.arena_bytes = RB;
      j.key.str_off = roffs.get();
      j.key.skip = 0;
      j.d_out_pos = pos.get();
      refine_sort_multi({j}, s);
    }
    DevBuf<uint32_t> perm(R, s), flags(R, s);
    PO_LAUNCH(k_invert, grid_for(R, 256), 256, 0, s, pos.get(), R, perm.get());
    PO_LAUNCH(k_new_flags, grid_for(R, 256), 256, 0, s, R, perm.get(), rmeta.get(), roffs.get(),
              rbytes.get(), rbytes.get() + RB, flags.get());
    rbytes.release();
    u.alloc(R, s);
    inclusive_scan_u32(flags.get(), u.get(), R, s);
    DevBuf<uint64_t> d_dc(m, s);
    PO_LAUNCH(k_col_dcount, (m + 127) / 128, 128, 0, s, m, d_cstart.get(), u.get(), d_dc.get());
    d_dc.download(dcount.data(), m);
    sync(s);
  }
  const std::vector<uint64_t> alld = comm.allgather_host(dcount, s);  // [rank][col]
  card_g.assign(m, 0);
  std::vector<uint64_t> gstart(m, 0);
  for (int r = 0; r < N; ++r)
    for (uint32_t c = 0; c < m; ++c) {
      if (r < comm.rank()) gstart[c] += alld[size_t(r) * m + c];
      card_g[c] += alld[size_t(r) * m + c];
    }
  if (R) {
    auto d_gstart = to_device(gstart, s);
    PO_LAUNCH(k_rank_out, grid_for(R, 256), 256, 0, s, R, pos.get(), rmeta.get(), u.get(),
              d_cstart.get(), d_gstart.get(), rrank.get());
  }
  // ranks back to the values' sources (reverse of the value exchange)
  std::vector<uint64_t> sb4(N), rb4(N);
  for (int r = 0; r < N; ++r) {
    sb4[r] = r_items[r] * 4;
    rb4[r] = s_items[r] * 4;
  }
  DevBuf<uint32_t> back(D, s), grank(D, s);
  comm.alltoallv(rrank.get(), sb4, back.get(), rb4, s);
  PO_LAUNCH(k_scatter_back, grid_for(D, 256), 256, 0, s, D, d_ord, back.get(), grank.get());
  return grank;
}

// ---------------------------------------------------------------------------
// distributed row layout: records [W key words][row u64][leaf u32][pad u32]
// [m gvid u32], padded to 8 bytes; key words most significant first
// ---------------------------------------------------------------------------
struct RecFmt {
  uint32_t W;       // key words
  uint32_t stride;  // u64 words per record
  uint32_t m;
};

__device__ __forceinline__ void put_bits(uint64_t* w, uint32_t& pos, uint64_t v, uint32_t nb) {
  while (nb) {
    const uint32_t room = 64 - (pos & 63);
    const uint32_t take = nb < room ? nb : room;
    const uint64_t chunk = (take == 64 ? v : (v >> (nb - take))) & (take == 64 ? ~0ull : ((1ull << take) - 1));
    w[pos >> 6] |= room - take == 64 ? 0 : (chunk << (room - take));
    pos += take;
    nb -= take;
  }
}

struct KeyPlan {
  const int32_t* leaf_kind;
  const uint32_t* leaf_key_off;
  const uint32_t* leaf_nkeys;
  const int32_t* key_field;
  const uint8_t* key_bits;
  uint32_t Lb, Kb, Rb;
};

__global__ void k_row_recs(uint64_t n, RecFmt f, const uint32_t* gvid, const uint32_t* row_leaf,
                           KeyPlan P, const uint32_t* rvid, const uint64_t* colbase,
                           uint64_t row_offset, uint64_t* recs) {
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n;
       r += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t* rec = recs + r * f.stride;
    uint64_t w[8];
    for (uint32_t i = 0; i < f.W; ++i) w[i] = 0;
    const uint32_t leaf = row_leaf[r];
    uint32_t pos = 0;
    put_bits(w, pos, leaf, P.Lb);
    const int kind = P.leaf_kind[leaf];
    const uint32_t k0 = P.leaf_key_off[leaf], nk = P.leaf_nkeys[leaf];
    const uint32_t* vr = gvid + r * f.m;
    uint32_t used = 0;
    for (uint32_t k = 0; k < nk; ++k) {
      const int32_t fld = P.key_field[k0 + k];
      const uint32_t b = P.key_bits[k0 + k];
      uint64_t v = vr[fld];
      if (kind == 2) v = rvid[colbase[fld] + v];
      put_bits(w, pos, v, b);
      used += b;
    }
    pos += P.Kb - used;
    const uint64_t grow = row_offset + r;
    put_bits(w, pos, grow, P.Rb);
    for (uint32_t i = 0; i < f.W; ++i) rec[i] = w[i];
    rec[f.W] = grow;
    rec[f.W + 1] = leaf;
    uint32_t* g = reinterpret_cast<uint32_t*>(rec + f.W + 2);
    for (uint32_t c = 0; c < f.m; ++c) g[c] = vr[c];
  }
}

__global__ void k_key_word(uint64_t n, const uint64_t* recs, uint32_t stride, uint32_t w,
                           const uint32_t* perm, uint64_t* keys) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    keys[i] = recs[uint64_t(perm ? perm[i] : uint32_t(i)) * stride + w];
}

// merged position of record i among the owner's N sorted runs (keys unique)
__global__ void k_merge_pos_rec(uint64_t R, int N, const uint64_t* ro, const uint64_t* recs,
                                RecFmt f, uint32_t* pos) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < R;
       i += uint64_t(gridDim.x) * blockDim.x) {
    int r = 0;
    while (i >= ro[r + 1]) ++r;
    const uint64_t* key = recs + i * f.stride;
    uint64_t p = i - ro[r];
    for (int q = 0; q < N; ++q) {
      if (q == r) continue;
      uint64_t lo = ro[q], hi = ro[q + 1];
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        const uint64_t* a = recs + mid * f.stride;
        int c = 0;
        for (uint32_t w = 0; w < f.W && !c; ++w)
          if (a[w] != key[w]) c = a[w] < key[w] ? -1 : 1;
        if (c < 0) lo = mid + 1;
        else hi = mid;
      }
      p += lo - ro[q];
    }
    pos[i] = uint32_t(p);
  }
}

__global__ void k_scatter_recs(uint64_t n, const uint64_t* recs, uint32_t stride, const uint32_t* pos,
                               uint64_t* out) {
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < n * stride;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = t / stride, k = t - i * stride;
    out[uint64_t(pos[i]) * stride + k] = recs[t];
  }
}

__global__ void k_gather_recs(uint64_t n, const uint64_t* recs, uint32_t stride, const uint32_t* perm,
                              uint64_t* out) {
  for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < n * stride;
       t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t i = t / stride, k = t - i * stride;
    out[t] = recs[uint64_t(perm[i]) * stride + k];
  }
}

__global__ void k_iota32(uint32_t* a, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    a[i] = uint32_t(i);
}

__global__ void k_iota64(uint64_t* a, uint64_t n, uint64_t base) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    a[i] = base + i;
}

// Stable LSD sort of records by their W key words; result in `out`.
void sort_recs(const uint64_t* recs, uint64_t n, const RecFmt& f, uint32_t key_bits,
               DevBuf<uint64_t>& out, cudaStream_t s) {
  out.alloc(n * f.stride, s);
  if (!n) return;
  DevBuf<uint64_t> k0(n, s), k1(n, s);
  DevBuf<uint32_t> p0(n, s), p1(n, s);
  PO_LAUNCH(k_iota32, grid_for(n, 256), 256, 0, s, p0.get(), n);
  for (int w = int(f.W) - 1; w >= 0; --w) {
    PO_LAUNCH(k_key_word, grid_for(n, 256), 256, 0, s, n, recs, f.stride, uint32_t(w), p0.get(),
              k0.get());
    // keys are packed from the top: the last word's low bits are padding
    const int begin = w == int(f.W) - 1 ? int(64 * f.W - key_bits) : 0;
    radix_sort_pairs(k0.get(), k1.get(), p0.get(), p1.get(), uint32_t(n), begin, 64, s);
    std::swap(p0, p1);
  }
  PO_LAUNCH(k_gather_recs, grid_for(n * f.stride, 256), 256, 0, s, n, recs, f.stride, p0.get(),
            out.get());
}

__global__ void k_row_samples(uint32_t S, uint64_t n, const uint64_t* sorted, RecFmt f,
                              uint64_t* out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < S; j += gridDim.x * blockDim.x) {
    uint64_t* o = out + uint64_t(j) * (f.W + 1);
    if (n == 0) {
      o[0] = 0;
      continue;
    }
    const uint64_t k = ((2 * uint64_t(j) + 1) * n) / (2 * uint64_t(S));
    o[0] = 1;
    for (uint32_t i = 0; i < f.W; ++i) o[1 + i] = sorted[k * f.stride + i];
  }
}

__global__ void k_row_split(uint32_t nsp, const uint64_t* sp, uint64_t n, const uint64_t* sorted,
                            RecFmt f, uint64_t* bounds) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nsp) return;
  const uint64_t* key = sp + uint64_t(j) * f.W;
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    const uint64_t* a = sorted + mid * f.stride;
    int c = 0;
    for (uint32_t i = 0; i < f.W && !c; ++i)
      if (a[i] != key[i]) c = a[i] < key[i] ? -1 : 1;
    if (c < 0) lo = mid + 1;
    else hi = mid;
  }
  bounds[j] = lo;
}

__global__ void k_emit_slice(uint64_t R, const uint64_t* recs, RecFmt f, const int32_t* leaf_orders,
                             uint64_t* rows, int32_t* orders, uint32_t* vid) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < R;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t* rec = recs + i * f.stride;
    rows[i] = rec[f.W];
    const int32_t* lo = leaf_orders + rec[f.W + 1] * f.m;
    const uint32_t* g = reinterpret_cast<const uint32_t*>(rec + f.W + 2);
    for (uint32_t c = 0; c < f.m; ++c) {
      orders[i * f.m + c] = lo[c];
      vid[i * f.m + c] = g[c];
    }
  }
}

}  // namespace

uint64_t dist_layout(DistCtx& dc, const Encoded& G, const uint32_t* d_row_leaf,
                     const std::vector<LeafKeys>& leaves, cudaStream_t s) {
  Comm& comm = *dc.comm;
  const int N = comm.size();
  const uint64_t n = G.n;
  const uint32_t m = G.m;
  const uint32_t nleaves = uint32_t(leaves.size());
  // key plan: leaf index, leaf keys padded to the widest leaf, global row id
  std::vector<int32_t> leaf_kind(std::max<uint32_t>(1, nleaves), 0);
  std::vector<uint32_t> leaf_key_off(std::max<uint32_t>(1, nleaves), 0), leaf_nkeys(leaf_key_off);
  std::vector<int32_t> key_field;
  std::vector<uint8_t> key_bits;
  std::vector<int32_t> leaf_orders(size_t(std::max<uint32_t>(1, nleaves)) * m, 0);
  uint32_t Kb = 0;
  bool need_raw = false;
  for (uint32_t l = 0; l < nleaves; ++l) {
    const LeafKeys& lk = leaves[l];
    leaf_kind[l] = lk.kind;
    leaf_key_off[l] = uint32_t(key_field.size());
    uint32_t used = 0;
    if (lk.kind != 0)
      for (int f : lk.fields) {
        key_field.push_back(f);
        const uint8_t b = uint8_t(bits_for(G.card[f] ? G.card[f] - 1 : 0));
        key_bits.push_back(b);
        used += b;
      }
    leaf_nkeys[l] = uint32_t(key_field.size()) - leaf_key_off[l];
    Kb = std::max(Kb, used);
    if (lk.kind == 2) need_raw = true;
    std::copy(lk.full_order.begin(), lk.full_order.end(), leaf_orders.begin() + size_t(l) * m);
  }
  if (key_field.empty()) {
    key_field.push_back(0);
    key_bits.push_back(1);
  }
  const uint32_t Lb = uint32_t(bits_for(nleaves ? nleaves - 1 : 0));
  const uint32_t Rb = uint32_t(bits_for(dc.n_global ? dc.n_global - 1 : 0));
  const uint32_t T = Lb + Kb + Rb;
  RecFmt f;
  f.W = (T + 63) / 64;
  if (f.W > 8) fail(PO_ERR_SIZE, "sharded layout: sort key wider than 512 bits");
  f.m = m;
  f.stride = f.W + 2 + (m + 1) / 2;
  const uint32_t* rvid = need_raw ? dc.raw_ranks() : nullptr;

  auto d_lkind = to_device(leaf_kind, s);
  auto d_lko = to_device(leaf_key_off, s), d_lnk = to_device(leaf_nkeys, s);
  auto d_kf = to_device(key_field, s);
  auto d_kb = to_device(key_bits, s);
  auto d_lord = to_device(leaf_orders, s);
  KeyPlan P{d_lkind.get(), d_lko.get(), d_lnk.get(), d_kf.get(), d_kb.get(), Lb, Kb, Rb};

  DevBuf<uint64_t> recs(n * f.stride, s), sorted;
  PO_LAUNCH(k_row_recs, grid_for(n, 256), 256, 0, s, n, f, G.vid.get(), d_row_leaf, P, rvid,
            G.d_colbase.get(), dc.row_offset, recs.get());
  sort_recs(recs.get(), n, f, T, sorted, s);
  recs.release();

  // sample sort: splitters from regular samples of every rank's sorted keys
  constexpr uint32_t S = 256;
  std::vector<uint64_t> bounds(N + 1, 0);
  bounds[N] = n;
  if (N > 1) {
    DevBuf<uint64_t> smp(size_t(S) * (f.W + 1), s), all(size_t(S) * (f.W + 1) * N, s);
    PO_LAUNCH(k_row_samples, 1, 256, 0, s, S, n, sorted.get(), f, smp.get());
    comm.allgather(smp.get(), all.get(), size_t(S) * (f.W + 1) * 8, s);
    std::vector<uint64_t> hs(size_t(S) * (f.W + 1) * N);
    all.download(hs.data(), hs.size());
    sync(s);
    std::vector<const uint64_t*> valid;
    for (size_t j = 0; j < size_t(S) * N; ++j)
      if (hs[j * (f.W + 1)]) valid.push_back(&hs[j * (f.W + 1) + 1]);
    std::sort(valid.begin(), valid.end(), [&](const uint64_t* a, const uint64_t* b) {
      return std::lexicographical_compare(a, a + f.W, b, b + f.W);
    });
    std::vector<uint64_t> sp(size_t(N - 1) * f.W, ~0ull);
    if (!valid.empty())
      for (int j = 1; j < N; ++j)
        std::copy(valid[(size_t(j) * valid.size()) / N], valid[(size_t(j) * valid.size()) / N] + f.W,
                  sp.begin() + size_t(j - 1) * f.W);
    auto d_sp = to_device(sp, s);
    DevBuf<uint64_t> d_b(N - 1, s);
    PO_LAUNCH(k_row_split, 1, 32, 0, s, uint32_t(N - 1), d_sp.get(), n, sorted.get(), f, d_b.get());
    d_b.download(bounds.data() + 1, N - 1);
    sync(s);
  }
  std::vector<uint64_t> sb(N);
  for (int r = 0; r < N; ++r) sb[r] = (bounds[r + 1] - bounds[r]) * f.stride * 8;
  const std::vector<uint64_t> rb = comm.exchange_counts(sb, s);
  uint64_t R = 0;
  for (int r = 0; r < N; ++r) R += rb[r] / (f.stride * 8);
  DevBuf<uint64_t> fin(R * f.stride, s);
  if (N == 1) {
    fin = std::move(sorted);
  } else {
    DevBuf<uint64_t> mine(R * f.stride, s);
    comm.alltoallv(sorted.get(), sb, mine.get(), rb, s);
    sorted.release();
    std::vector<uint64_t> ro(N + 1, 0);
    for (int r = 0; r < N; ++r) ro[r + 1] = ro[r] + rb[r] / (f.stride * 8);
    auto d_ro = to_device(ro, s);
    DevBuf<uint32_t> pos(R, s);
    PO_LAUNCH(k_merge_pos_rec, grid_for(R, 256), 256, 0, s, R, N, d_ro.get(), mine.get(), f,
              pos.get());
    PO_LAUNCH(k_scatter_recs, grid_for(R * f.stride, 256), 256, 0, s, R, mine.get(), f.stride,
              pos.get(), fin.get());
  }

  // slice position
  const std::vector<uint64_t> counts = comm.allgather_host({R}, s);
  dc.slice_offset = 0;
  for (int r = 0; r < comm.rank(); ++r) dc.slice_offset += counts[r];
  dc.slice_count = R;
  dc.rows.alloc(R, s);
  dc.orders.alloc((R + 1) * m, s);
  DevBuf<uint32_t> vid_s((R + 1) * m, s);
  PO_LAUNCH(k_emit_slice, grid_for(R, 256), 256, 0, s, R, fin.get(), f, d_lord.get(), dc.rows.get(),
            dc.orders.get() + m, vid_s.get() + m);

  // boundary request: the previous non-empty rank's last entry
  std::vector<uint64_t> last(2 + m, 0);
  if (R) {
    std::vector<uint64_t> rec(f.stride);
    PO_CUDA(cudaMemcpyAsync(rec.data(), fin.get() + (R - 1) * f.stride, f.stride * 8,
                            cudaMemcpyDeviceToHost, s));
    sync(s);
    last[0] = 1;
    last[1] = rec[f.W + 1];
    const uint32_t* g = reinterpret_cast<const uint32_t*>(rec.data() + f.W + 2);
    for (uint32_t c = 0; c < m; ++c) last[2 + c] = g[c];
  }
  const std::vector<uint64_t> lasts = comm.allgather_host(last, s);
  int prev = -1;
  for (int r = comm.rank() - 1; r >= 0; --r)
    if (lasts[size_t(r) * (2 + m)]) {
      prev = r;
      break;
    }
  uint64_t local = 0;
  if (R) {
    if (prev >= 0) {
      const uint64_t* e = &lasts[size_t(prev) * (2 + m)];
      std::vector<uint32_t> v(m);
      for (uint32_t c = 0; c < m; ++c) v[c] = uint32_t(e[2 + c]);
      vid_s.upload(v.data(), m);
      PO_CUDA(cudaMemcpyAsync(dc.orders.get(), d_lord.get() + e[1] * m, m * sizeof(int32_t),
                              cudaMemcpyDeviceToDevice, s));
    }
    DevBuf<uint32_t> idx(R + 1, s);
    PO_LAUNCH(k_iota32, grid_for(R + 1, 256), 256, 0, s, idx.get(), R + 1);
    local = phc_device_raw(vid_s.get(), G.vlen.get(), G.d_colbase.get(), R + 1, m, R + 1, nullptr,
                           idx.get(), nullptr, dc.orders.get(), s, prev >= 0 ? 1 : 2);
  }
  return comm.allreduce_host({local}, COp::Sum, s)[0];
}

void ggr_sharded(Comm& comm, const DeviceTable& t, int tok, int scoring,
                 const std::vector<std::vector<int>>& fd_groups, const po_ggr_config& cfg,
                 DistCtx& dc, GgrOutput& out, cudaStream_t s) {
  const int N = comm.size();
  const uint32_t m = t.m;
  const std::vector<uint64_t> shape = comm.allgather_host({t.n, m}, s);
  uint64_t ng = 0, off = 0;
  for (int r = 0; r < N; ++r) {
    if (shape[2 * r + 1] != m) fail(PO_ERR_SCHEMA, "shards disagree on the number of fields");
    if (r < comm.rank()) off += shape[2 * r];
    ng += shape[2 * r];
  }
  if (ng * uint64_t(m) >= (uint64_t(1) << 32) || ng >= 0xFFFFFFFFull)
    fail(PO_ERR_SIZE, "table too large (rows*fields must be < 2^32)");
  dc.comm = &comm;
  dc.n_global = ng;
  dc.row_offset = off;
  out = GgrOutput{};
  out.stats.recursive_calls = 1;
  if (ng == 0) {
    dc.slice_offset = 0;
    dc.slice_count = 0;
    return;
  }
  if (m == 0) {  // every row, ascending, no fields (ggr.hpp:214-219)
    dc.slice_offset = off;
    dc.slice_count = t.n;
    dc.rows.alloc(t.n, s);
    dc.orders.alloc(1, s);
    PO_LAUNCH(k_iota64, grid_for(t.n, 256), 256, 0, s, dc.rows.get(), t.n, off);
    return;
  }
  Encoded L;
  encode(t, tok, scoring, s, L, debug_hash_bits());
  timing_mark("local_encode", s);
  DevBuf<uint32_t> icol(L.D, s);
  PO_LAUNCH(k_item_col, grid_for(L.D, 256), 256, 0, s, L.D, L.d_colbase.get(), m, icol.get());

  // global escaped-order ids
  Encoded G;
  DevBuf<uint32_t> grank = global_ranks(comm, L, icol.get(), 1, G.card, s);
  timing_mark("global_dict", s);
  G.n = t.n;
  G.m = m;
  G.colbase.assign(m + 1, 0);
  for (uint32_t c = 0; c < m; ++c) G.colbase[c + 1] = G.colbase[c] + G.card[c];
  G.D = G.colbase[m];
  G.d_colbase = to_device(G.colbase, s);
  G.vid.alloc(t.n * m, s);
  PO_LAUNCH(k_remap_vid, grid_for(t.n * m, 256), 256, 0, s, t.n * m, m, L.vid.get(),
            L.d_colbase.get(), grank.get(), G.vid.get());
  G.count.alloc(G.D, s);
  G.count.zero();
  G.vlen.alloc(G.D, s);
  G.vlen.zero();
  PO_LAUNCH(k_scatter_dict, grid_for(L.D, 256), 256, 0, s, L.D, icol.get(), grank.get(),
            G.d_colbase.get(), L.count.get(), L.vlen.get(), G.count.get(),
            reinterpret_cast<unsigned long long*>(G.vlen.get()));
  comm.allreduce(G.count.get(), G.D, CDtype::U32, COp::Sum, s);
  comm.allreduce(G.vlen.get(), G.D, CDtype::U64, COp::Max, s);
  G.total_len = comm.allreduce_host(L.total_len, COp::Sum, s);
  timing_mark("global_arrays", s);

  // raw-byte ranks, built on first use
  DevBuf<uint32_t> rvid;
  bool have_raw = false;
  dc.raw_ranks = [&]() -> const uint32_t* {
    if (!have_raw) {
      std::vector<uint64_t> card_raw;
      DevBuf<uint32_t> rr = global_ranks(comm, L, icol.get(), 0, card_raw, s);
      rvid.alloc(G.D, s);
      rvid.zero();
      PO_LAUNCH(k_scatter_u32, grid_for(L.D, 256), 256, 0, s, L.D, icol.get(), grank.get(),
                G.d_colbase.get(), rr.get(), rvid.get());
      comm.allreduce(rvid.get(), G.D, CDtype::U32, COp::Max, s);
      have_raw = true;
    }
    return rvid.get();
  };
  ggr_device(G, fd_groups, cfg, nullptr, nullptr, out, s, &dc);
  dc.raw_ranks = nullptr;
  timing_mark("ggr", s);
}

}  // namespace po
