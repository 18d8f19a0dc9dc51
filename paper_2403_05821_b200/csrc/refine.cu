// Segmented refinement sort: the engine behind K3 rank_sort (distinct values
// in raw-byte and escaped-fragment order) and K8 multikey_sort (leaf row
// sorts of the statistics fallback, objective.hpp:154-171 / ggr.hpp:340-350,
// and the raw single-column base case, ggr.hpp:221-231).
//
// MSD by key chunks: each round stable-radix-sorts the still-unresolved items
// on one 64-bit word (group << chunk_bits | chunk) — group ids are final
// start positions, so every group keeps a contiguous range of output slots —
// then splits groups where the chunk changes. Most items resolve after one or
// two rounds, so later rounds touch only the long shared prefixes.

#include <cub/cub.cuh>

#include <cstdlib>

#include "internal.cuh"

namespace po {

namespace {

__constant__ uint16_t c_esc_code[257];  // byte -> code in escaped order; [256] = end

constexpr uint16_t kRawEnd = 1;  // raw codes: end = 1, byte b = b + 2

__device__ __forceinline__ uint32_t end_code(const RefineKey& K) {
  return K.kind == 0 ? kRawEnd : c_esc_code[256];
}

// Chunk k of a string: nsym 9-bit symbols (bytes nsym*k .. nsym*k+nsym-1,
// the end marker at position len, zero padding after). Raw order: end <
// every byte (a prefix sorts first). Escaped order: the code of each byte is
// the rank of its json_escape expansion and the end marker is the closing
// '"' (0x22) of the fragment, so comparing code strings == comparing escaped
// fragment keys (the expansions are prefix-free).
__device__ __forceinline__ uint64_t string_chunk(const RefineKey& K, uint32_t item, uint32_t k) {
  const uint64_t i = uint64_t(K.item_cell_row[item]) * K.m + K.item_col[item];
  const uint64_t o0 = K.offsets[i];
  const uint64_t len = K.offsets[i + 1] - o0;
  const uint8_t* p = K.arena + o0;
  const uint32_t nsym = K.chunk_bits / 9;
  uint64_t chunk = 0;
  const uint64_t base = uint64_t(k) * nsym;
  for (uint32_t j = 0; j < nsym; ++j) {
    const uint64_t pos = base + j;
    uint32_t code;
    if (pos < len) {
      const uint8_t b = p[pos];
      code = K.kind == 0 ? uint32_t(b) + 2 : c_esc_code[b];
    } else {
      code = pos == len ? end_code(K) : 0;
    }
    chunk = (chunk << 9) | code;
  }
  return chunk;
}

__device__ __forceinline__ bool string_terminal(const RefineKey& K, uint64_t chunk) {
  const uint32_t nsym = K.chunk_bits / 9;
  const uint32_t e = end_code(K);
  for (uint32_t j = 0; j < nsym; ++j)
    if (((chunk >> (9 * j)) & 511u) == e) return true;
  return false;
}

// Chunk k of a row: the packed ranks of its leaf's k-th key group.
__device__ __forceinline__ uint64_t row_chunk(const RefineKey& K, uint32_t row, uint32_t k) {
  const uint32_t leaf = K.row_leaf[row];
  if (k >= K.leaf_nchunks[leaf]) return 0;
  const uint32_t ch = K.leaf_chunk_off[leaf] + k;
  const uint32_t k0 = K.chunk_key_off[ch], nk = K.chunk_nkeys[ch];
  uint64_t chunk = 0;
  for (uint32_t j = 0; j < nk; ++j) {
    const int32_t f = K.key_field[k0 + j];
    const uint32_t v = K.vid[uint64_t(row) * K.m + f];
    const uint32_t rank = K.key_kind[k0 + j] == 0 ? v : K.esc_rank[K.colbase[f] + v];
    chunk = (chunk << K.key_bits[k0 + j]) | rank;
  }
  return chunk;
}

__device__ __forceinline__ bool row_terminal(const RefineKey& K, uint32_t row, uint32_t k) {
  return k + 1 >= K.leaf_nchunks[K.row_leaf[row]];
}

__global__ void k_build_keys(const uint32_t* items, const uint32_t* grp, uint32_t A, uint32_t k,
                             RefineKey K, uint64_t* keys) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x) {
    const uint64_t chunk = K.kind == 2 ? row_chunk(K, items[i], k) : string_chunk(K, items[i], k);
    keys[i] = (uint64_t(grp[i]) << K.chunk_bits) | chunk;
  }
}

// Boundary markers for the two max-scans: start index of each item's group
// and of its (group, chunk) run.
__global__ void k_marks(const uint64_t* keys, uint32_t A, uint32_t chunk_bits, uint32_t* gmark,
                        uint32_t* rmark) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x) {
    const bool gb = i == 0 || (keys[i] >> chunk_bits) != (keys[i - 1] >> chunk_bits);
    const bool rb = i == 0 || keys[i] != keys[i - 1];
    gmark[i] = gb ? i : 0;
    rmark[i] = rb ? i : 0;
  }
}

__global__ void k_resolve(const uint64_t* keys, const uint32_t* items, const uint32_t* gstart,
                          const uint32_t* rstart, uint32_t A, uint32_t k, RefineKey K,
                          uint32_t* out_pos, uint8_t* keep, uint32_t* next_grp) {
  const uint64_t cmask = K.chunk_bits >= 64 ? ~0ull : ((1ull << K.chunk_bits) - 1);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x) {
    const uint32_t item = items[i];
    const uint32_t g = uint32_t(keys[i] >> K.chunk_bits);
    const uint32_t pos = g + (i - gstart[i]);
    const bool run_head = rstart[i] == i;
    const bool next_head = i + 1 >= A || rstart[i + 1] == i + 1;
    const bool term = K.kind == 2 ? row_terminal(K, item, k) : string_terminal(K, keys[i] & cmask);
    if ((run_head && next_head) || term) {
      out_pos[item] = pos;
      keep[i] = 0;
    } else {
      keep[i] = 1;
    }
    next_grp[i] = g + (rstart[i] - gstart[i]);
  }
}

__global__ void k_iota(uint32_t* a, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[i] = i;
}

bool g_esc_table_ready = false;

void ensure_esc_table() {
  if (g_esc_table_ready) return;
  // Symbol value of each byte in escaped text (scoring.hpp:33-57): plain
  // bytes keep their value; escapes start with '\' (0x5C) then the escape
  // letter; \u00XX escapes append the byte itself (hex digits sort like the
  // byte). The fragment terminator '"' closes every value.
  std::vector<std::pair<uint32_t, int>> sym;
  for (int b = 0; b < 256; ++b) {
    uint32_t v;
    switch (b) {
      case '"': v = (0x5Cu << 16) | (0x22u << 8); break;
      case '\\': v = (0x5Cu << 16) | (0x5Cu << 8); break;
      case '\b': v = (0x5Cu << 16) | (uint32_t('b') << 8); break;
      case '\f': v = (0x5Cu << 16) | (uint32_t('f') << 8); break;
      case '\n': v = (0x5Cu << 16) | (uint32_t('n') << 8); break;
      case '\r': v = (0x5Cu << 16) | (uint32_t('r') << 8); break;
      case '\t': v = (0x5Cu << 16) | (uint32_t('t') << 8); break;
      default:
        v = b < 0x20 ? ((0x5Cu << 16) | (uint32_t('u') << 8) | uint32_t(b)) : (uint32_t(b) << 16);
    }
    sym.push_back({v, b});
  }
  sym.push_back({0x22u << 16, 256});
  std::sort(sym.begin(), sym.end());
  uint16_t code[257];
  for (size_t r = 0; r < sym.size(); ++r) code[sym[r].second] = uint16_t(r + 1);
  PO_CUDA(cudaMemcpyToSymbol(c_esc_code, code, sizeof(code)));
  g_esc_table_ready = true;
}

}  // namespace

uint32_t refine_chunk_bits(uint32_t grp_max) { return 64u - uint32_t(bits_for(grp_max)); }

void refine_sort(uint32_t n_items, const uint32_t* d_grp_init, uint32_t grp_max,
                 const RefineKey& key_in, uint32_t* d_out_pos, cudaStream_t s,
                 uint32_t* rounds_out) {
  if (rounds_out) *rounds_out = 0;
  if (n_items == 0) return;
  RefineKey key = key_in;
  key.chunk_bits = refine_chunk_bits(grp_max);
  if (key.kind != 2 && key.chunk_bits < 9) fail(PO_ERR_SIZE, "too many distinct values to rank");
  if (key.kind == 1) ensure_esc_table();

  DevBuf<uint32_t> items(n_items, s), items2(n_items, s);
  DevBuf<uint32_t> grp(n_items, s), grp2(n_items, s);
  DevBuf<uint64_t> keys(n_items, s), keys2(n_items, s);
  DevBuf<uint32_t> gstart(n_items, s), rstart(n_items, s);
  DevBuf<uint32_t> gmark(n_items, s), rmark(n_items, s);
  DevBuf<uint8_t> keep(n_items, s);
  DevBuf<int> nsel(1, s);

  PO_LAUNCH(k_iota, grid_for(n_items, 256), 256, 0, s, items.get(), n_items);
  PO_CUDA(cudaMemcpyAsync(grp.get(), d_grp_init, n_items * sizeof(uint32_t),
                          cudaMemcpyDeviceToDevice, s));

  // temp storage sized for the largest round
  size_t sort_bytes = 0, scan_bytes = 0, sel_bytes = 0;
  PO_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys.get(), keys2.get(),
                                          items.get(), items2.get(), n_items, 0, 64, s));
  PO_CUDA(cub::DeviceScan::InclusiveScan(nullptr, scan_bytes, gmark.get(), gstart.get(),
                                         cub::Max(), n_items, s));
  PO_CUDA(cub::DeviceSelect::Flagged(nullptr, sel_bytes, items2.get(), keep.get(), items.get(),
                                     nsel.get(), n_items, s));
  const size_t tb = std::max(sort_bytes, std::max(scan_bytes, sel_bytes));
  DevBuf<uint8_t> tmp(tb, s);
  const int end_bit = int(key.chunk_bits) + bits_for(grp_max);

  uint32_t A = n_items;
  for (uint32_t k = 0; A > 0; ++k) {
    PO_LAUNCH(k_build_keys, grid_for(A, 256), 256, 0, s, items.get(), grp.get(), A, k, key,
              keys.get());
    size_t b = tb;
    {
      ProfScope ps("cub_radix_sort", s);
      PO_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), b, keys.get(), keys2.get(), items.get(),
                                              items2.get(), A, 0, end_bit, s));
    }
    PO_LAUNCH(k_marks, grid_for(A, 256), 256, 0, s, keys2.get(), A, key.chunk_bits, gmark.get(),
              rmark.get());
    {
      ProfScope ps("cub_scan", s);
      b = tb;
      PO_CUDA(cub::DeviceScan::InclusiveScan(tmp.get(), b, gmark.get(), gstart.get(), cub::Max(),
                                             A, s));
      b = tb;
      PO_CUDA(cub::DeviceScan::InclusiveScan(tmp.get(), b, rmark.get(), rstart.get(), cub::Max(),
                                             A, s));
    }
    PO_LAUNCH(k_resolve, grid_for(A, 256), 256, 0, s, keys2.get(), items2.get(), gstart.get(),
              rstart.get(), A, k, key, d_out_pos, keep.get(), grp2.get());
    {
      ProfScope ps("cub_select", s);
      b = tb;
      PO_CUDA(cub::DeviceSelect::Flagged(tmp.get(), b, items2.get(), keep.get(), items.get(),
                                         nsel.get(), A, s));
      b = tb;
      PO_CUDA(cub::DeviceSelect::Flagged(tmp.get(), b, grp2.get(), keep.get(), grp.get(),
                                         nsel.get(), A, s));
    }
    int na = 0;
    PO_CUDA(cudaMemcpyAsync(&na, nsel.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    sync(s);
    A = uint32_t(na);
    if (rounds_out) ++*rounds_out;
  }
}

}  // namespace po
