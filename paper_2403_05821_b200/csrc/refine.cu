// Segmented refinement sort: the engine behind K3 rank_sort (distinct values
// in raw-byte and escaped-fragment order) and K8 multikey_sort (leaf row
// sorts of the statistics fallback, objective.hpp:154-171 / ggr.hpp:340-350,
// and the raw single-column base case, ggr.hpp:221-231).
//
// MSD by 63-bit chunks: each round stable-radix-sorts the still-unresolved
// items on (group, chunk) — group ids are final start positions, so every
// group keeps a contiguous range of output slots — then splits groups where
// the chunk changes. Most items resolve after one or two rounds, so later
// rounds touch only the long shared prefixes.

#include <cub/cub.cuh>
#include <cuda/std/tuple>

#include "internal.cuh"

namespace po {

namespace {

__constant__ uint16_t c_esc_code[257];  // byte -> code in escaped order; [256] = end

struct RKey {
  uint64_t chunk;
  uint32_t grp;
  uint32_t pad;
};

struct RKeyDecomposer {
  __host__ __device__ ::cuda::std::tuple<uint32_t&, uint64_t&> operator()(RKey& k) const {
    return {k.grp, k.chunk};
  }
};

constexpr uint16_t kRawEnd = 1;  // raw codes: end = 1, byte b = b + 2

// Chunk k of a string: 7 symbols of 9 bits (bytes 7k..7k+6, the end marker
// at position len, zero padding after). Raw order: end < every byte (a prefix
// sorts first). Escaped order: the code of each byte is the rank of its
// json_escape expansion, the end marker is the closing '"' (0x22) of the
// fragment, so comparing code strings == comparing escaped fragment keys.
__device__ __forceinline__ uint64_t string_chunk(const RefineKey& K, uint32_t item, uint32_t k,
                                                 bool& terminal) {
  const uint64_t i = uint64_t(K.item_cell_row[item]) * K.m + K.item_col[item];
  const uint64_t o0 = K.offsets[i];
  const uint64_t len = K.offsets[i + 1] - o0;
  const uint8_t* p = K.arena + o0;
  uint64_t chunk = 0;
  terminal = false;
  const uint64_t base = uint64_t(k) * 7;
  for (int j = 0; j < 7; ++j) {
    uint64_t pos = base + j;
    uint32_t code;
    if (pos < len) {
      uint8_t b = p[pos];
      code = K.kind == 0 ? uint32_t(b) + 2 : c_esc_code[b];
    } else if (pos == len) {
      code = K.kind == 0 ? kRawEnd : c_esc_code[256];
      terminal = true;
    } else {
      code = 0;
    }
    chunk = (chunk << 9) | code;
  }
  return chunk;
}

// Chunk k of a row: the packed ranks of the leaf's k-th key group.
__device__ __forceinline__ uint64_t row_chunk(const RefineKey& K, uint32_t row, uint32_t k,
                                              bool& terminal) {
  const uint32_t leaf = K.row_leaf[row];
  const uint32_t nch = K.leaf_nchunks[leaf];
  if (nch == 0) {
    terminal = true;
    return 0;
  }
  terminal = k + 1 >= nch;
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

__device__ __forceinline__ uint64_t key_chunk(const RefineKey& K, uint32_t item, uint32_t k,
                                              bool& terminal) {
  return K.kind == 2 ? row_chunk(K, item, k, terminal) : string_chunk(K, item, k, terminal);
}

__global__ void k_build_keys(const uint32_t* items, const uint32_t* grp, uint32_t A, uint32_t k,
                             RefineKey K, RKey* keys) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x) {
    bool term;
    RKey rk;
    rk.chunk = key_chunk(K, items[i], k, term);
    rk.grp = grp[i];
    rk.pad = term ? 1u : 0u;  // not part of the sort key
    keys[i] = rk;
  }
}

// Boundary markers for the two max-scans: start index of each item's group
// and of its (group, chunk) run.
__global__ void k_marks(const RKey* keys, uint32_t A, uint32_t* gstart, uint32_t* rstart) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x) {
    bool gb = i == 0 || keys[i].grp != keys[i - 1].grp;
    bool rb = gb || keys[i].chunk != keys[i - 1].chunk;
    gstart[i] = gb ? i : 0;
    rstart[i] = rb ? i : 0;
  }
}

__global__ void k_resolve(const RKey* keys, const uint32_t* items, const uint32_t* gstart,
                          const uint32_t* rstart, uint32_t A, uint32_t* out_pos, uint8_t* keep, uint32_t* next_grp) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < A; i += gridDim.x * blockDim.x) {
    const uint32_t item = items[i];
    const uint32_t g = keys[i].grp;
    const uint32_t pos = g + (i - gstart[i]);
    const bool run_head = rstart[i] == i;
    const bool next_head = i + 1 >= A || rstart[i + 1] == i + 1;
    if ((run_head && next_head) || keys[i].pad) {
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

void refine_sort(uint32_t n_items, const uint32_t* d_grp_init, uint32_t grp_max,
                 const RefineKey& key, uint32_t* d_out_pos, cudaStream_t s, uint32_t* rounds_out) {
  if (rounds_out) *rounds_out = 0;
  if (n_items == 0) return;
  if (key.kind == 1) ensure_esc_table();
  const int end_bit = 64 + bits_for(grp_max);

  DevBuf<uint32_t> items(n_items, s), items2(n_items, s);
  DevBuf<uint32_t> grp(n_items, s), grp2(n_items, s);
  DevBuf<RKey> keys(n_items, s), keys2(n_items, s);
  DevBuf<uint32_t> gstart(n_items, s), rstart(n_items, s);
  DevBuf<uint8_t> keep(n_items, s);
  DevBuf<int> nsel(1, s);

  PO_LAUNCH(k_iota, grid_for(n_items, 256), 256, 0, s, items.get(), n_items);
  PO_CUDA(cudaMemcpyAsync(grp.get(), d_grp_init, n_items * sizeof(uint32_t),
                          cudaMemcpyDeviceToDevice, s));

  // temp storage sized for the largest round
  size_t sort_bytes = 0, scan_bytes = 0, sel_bytes = 0;
  PO_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, keys.get(), keys2.get(),
                                          items.get(), items2.get(), n_items, RKeyDecomposer{}, 0,
                                          end_bit, s));
  PO_CUDA(cub::DeviceScan::InclusiveScan(nullptr, scan_bytes, gstart.get(), gstart.get(),
                                         cub::Max(), n_items, s));
  PO_CUDA(cub::DeviceSelect::Flagged(nullptr, sel_bytes, items2.get(), keep.get(), items.get(),
                                     nsel.get(), n_items, s));
  size_t tb = std::max(sort_bytes, std::max(scan_bytes, sel_bytes));
  DevBuf<uint8_t> tmp(tb, s);

  uint32_t A = n_items;
  for (uint32_t k = 0; A > 0; ++k) {
    PO_LAUNCH(k_build_keys, grid_for(A, 256), 256, 0, s, items.get(), grp.get(), A, k, key,
              keys.get());
    size_t b = tb;
    PO_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), b, keys.get(), keys2.get(), items.get(),
                                            items2.get(), A, RKeyDecomposer{}, 0, end_bit, s));
    PO_LAUNCH(k_marks, grid_for(A, 256), 256, 0, s, keys2.get(), A, gstart.get(), rstart.get());
    b = tb;
    PO_CUDA(cub::DeviceScan::InclusiveScan(tmp.get(), b, gstart.get(), gstart.get(), cub::Max(),
                                           A, s));
    b = tb;
    PO_CUDA(cub::DeviceScan::InclusiveScan(tmp.get(), b, rstart.get(), rstart.get(), cub::Max(),
                                           A, s));
    PO_LAUNCH(k_resolve, grid_for(A, 256), 256, 0, s, keys2.get(), items2.get(), gstart.get(),
              rstart.get(), A, d_out_pos, keep.get(), grp2.get());
    b = tb;
    PO_CUDA(cub::DeviceSelect::Flagged(tmp.get(), b, items2.get(), keep.get(), items.get(),
                                       nsel.get(), A, s));
    b = tb;
    PO_CUDA(cub::DeviceSelect::Flagged(tmp.get(), b, grp2.get(), keep.get(), grp.get(),
                                       nsel.get(), A, s));
    int na = 0;
    PO_CUDA(cudaMemcpyAsync(&na, nsel.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    sync(s);
    A = uint32_t(na);
    if (rounds_out) ++*rounds_out;
  }
}

}  // namespace po
