// Prompt rendering and byte-exact dedup: the step
// after the path in cmd_solve (run.hpp:457-466).
//
// render_prompt (objective.hpp:118-131): [system_prompt '\n'] [question '\n']
// then render_body (objective.hpp:102-115): '{' then, per field of the
// entry's order, [", "] '"' esc(name) '": "' esc(value) '"', then '}'.
// Escaping is json_escape (scoring.hpp:33-57). One warp per request: pass 1
// sums the escaped lengths (lanes stride over each cell's bytes, warp sum),
// an exclusive scan gives every prompt's offset, pass 2 writes the bytes —
// 32 input bytes per step, each lane's expansion (1, 2 or 6 bytes) placed
// by a warp prefix sum, so the output is written in order without gaps.
//
// dedup (cost.hpp:171-186): uniques in first-occurrence order + expansion
// map, from the exact dictionary of the prompts (encode() on a one-column
// table: equal ids <=> equal bytes) and the first index of every id.

#include <cub/cub.cuh>

#include "internal.cuh"

namespace po {

namespace {

__device__ __forceinline__ uint32_t esc_len_b(uint8_t c) {
  if (c == '"' || c == '\\' || c == '\b' || c == '\f' || c == '\n' || c == '\r' || c == '\t')
    return 2;
  return c < 0x20 ? 6 : 1;
}

__device__ __forceinline__ void esc_write(uint8_t c, uint8_t* o) {
  const char* hex = "0123456789abcdef";
  switch (c) {
    case '"': o[0] = '\\'; o[1] = '"'; return;
    case '\\': o[0] = '\\'; o[1] = '\\'; return;
    case '\b': o[0] = '\\'; o[1] = 'b'; return;
    case '\f': o[0] = '\\'; o[1] = 'f'; return;
    case '\n': o[0] = '\\'; o[1] = 'n'; return;
    case '\r': o[0] = '\\'; o[1] = 'r'; return;
    case '\t': o[0] = '\\'; o[1] = 't'; return;
    default:
      if (c < 0x20) {
        o[0] = '\\'; o[1] = 'u'; o[2] = '0'; o[3] = '0';
        o[4] = uint8_t(hex[c >> 4]); o[5] = uint8_t(hex[c & 15]);
      } else {
        o[0] = c;
      }
  }
}

struct Sched {
  const uint64_t* rows;
  const uint64_t* offs;
  const int32_t* fields;
};

__global__ void k_prompt_len(const uint8_t* __restrict__ arena, const uint8_t* arena_end,
                             const uint64_t* __restrict__ offsets,
                             uint64_t n_rows, uint32_t m, Sched sc, uint64_t n_entries,
                             const uint64_t* __restrict__ name_esc_len, uint64_t prefix_len,
                             uint64_t* out_len, int* err) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; i < n_entries;
       i += warps) {
    const uint64_t r = sc.rows[i];
    const uint64_t a = sc.offs[i], b = sc.offs[i + 1];
    uint64_t tot = 0;
    for (uint64_t p = a; p < b; ++p) {
      const int32_t f = sc.fields[p];
      if (r >= n_rows || f < 0 || uint32_t(f) >= m) {
        if (lane == 0) atomicExch(err, 1);
        break;
      }
      const uint64_t c = r * m + f;
      const uint8_t* v = arena + offsets[c];
      const uint64_t len = offsets[c + 1] - offsets[c];
      for (uint64_t j = 8 * lane; j < len; j += 256) {  // 8 bytes per lane per step
        const uint64_t w = load8_unaligned(v + j, arena_end);
        const uint32_t nb = len - j >= 8 ? 8u : uint32_t(len - j);
        for (uint32_t k = 0; k < nb; ++k) tot += esc_len_b(uint8_t(w >> (8 * k)));
      }
      if (lane == 0) tot += (p > a ? 2 : 0) + 1 + name_esc_len[f] + 4 + 1;
    }
    for (int d = 16; d > 0; d >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, d);
    if (lane == 0) out_len[i] = prefix_len + 2 + tot;
  }
}

// warp-cooperative escaped copy of `len` bytes to dst; returns bytes
// written. Each lane takes 8 bytes per step (256 per warp step): their
// escaped sizes are summed, one warp prefix sum places every lane's output.
__device__ __forceinline__ uint64_t warp_esc_copy(const uint8_t* src, uint64_t len, uint8_t* dst,
                                                  const uint8_t* src_end, uint32_t lane) {
  uint64_t pos = 0;
  for (uint64_t base = 0; base < len; base += 256) {
    const uint64_t j = base + 8 * lane;
    const uint32_t nb = j < len ? (len - j >= 8 ? 8u : uint32_t(len - j)) : 0u;
    const uint64_t w = nb ? load8_unaligned(src + j, src_end) : 0;
    uint32_t el = 0;
    for (uint32_t k = 0; k < nb; ++k) el += esc_len_b(uint8_t(w >> (8 * k)));
    uint32_t incl = el;
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (int(lane) >= d) incl += y;
    }
    uint8_t* o = dst + pos + (incl - el);
    if (el == nb) {  // nothing to escape: plain bytes
      for (uint32_t k = 0; k < nb; ++k) o[k] = uint8_t(w >> (8 * k));
    } else {
      for (uint32_t k = 0; k < nb; ++k) {
        const uint8_t c = uint8_t(w >> (8 * k));
        esc_write(c, o);
        o += esc_len_b(c);
      }
    }
    pos += __shfl_sync(0xffffffffu, incl, 31);
  }
  return pos;
}

__device__ __forceinline__ void warp_copy(const uint8_t* src, uint64_t len, uint8_t* dst,
                                          uint32_t lane) {
  for (uint64_t j = lane; j < len; j += 32) dst[j] = src[j];
}

__global__ void k_prompt_write(const uint8_t* __restrict__ arena, const uint8_t* arena_end,
                               const uint64_t* __restrict__ offsets,
                               uint32_t m, Sched sc, uint64_t n_entries,
                               const uint8_t* __restrict__ names_esc,
                               const uint64_t* __restrict__ name_off, const uint8_t* prefix,
                               uint64_t prefix_len, const uint64_t* __restrict__ out_off,
                               uint8_t* out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5; i < n_entries;
       i += warps) {
    uint8_t* o = out + out_off[i];
    warp_copy(prefix, prefix_len, o, lane);
    uint64_t w = prefix_len;
    if (lane == 0) o[w] = '{';
    ++w;
    const uint64_t r = sc.rows[i];
    const uint64_t a = sc.offs[i], b = sc.offs[i + 1];
    for (uint64_t p = a; p < b; ++p) {
      const int32_t f = sc.fields[p];
      const uint64_t nl = name_off[f + 1] - name_off[f];
      if (lane == 0) {
        if (p > a) {
          o[w] = ','; o[w + 1] = ' ';
        }
        o[w + (p > a ? 2 : 0)] = '"';
      }
      w += (p > a ? 2 : 0) + 1;
      warp_copy(names_esc + name_off[f], nl, o + w, lane);
      w += nl;
      if (lane == 0) {
        o[w] = '"'; o[w + 1] = ':'; o[w + 2] = ' '; o[w + 3] = '"';
      }
      w += 4;
      const uint64_t c = r * m + f;
      w += warp_esc_copy(arena + offsets[c], offsets[c + 1] - offsets[c], o + w, arena_end, lane);
      if (lane == 0) o[w] = '"';
      ++w;
    }
    if (lane == 0) o[w] = '}';
  }
}

__global__ void k_first_index(const uint32_t* vid, uint64_t n, uint32_t* first) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    atomicMin(&first[vid[i]], uint32_t(i));
}

__global__ void k_is_first(const uint32_t* vid, uint64_t n, const uint32_t* first, uint32_t* flag) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    flag[i] = first[vid[i]] == uint32_t(i) ? 1u : 0u;
}

__global__ void k_expand(const uint32_t* vid, uint64_t n, const uint32_t* first,
                         const uint32_t* uidx_excl, uint64_t* expansion, uint64_t* unique_first) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t f = first[vid[i]];
    expansion[i] = uidx_excl[f];
    if (f == uint32_t(i)) unique_first[uidx_excl[i]] = i;
  }
}

}  // namespace

std::string json_escape_bytes(const std::string& s) {
  static const char hexd[] = "0123456789abcdef";
  std::string o;
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          o += "\\u00";
          o += hexd[c >> 4];
          o += hexd[c & 15];
        } else {
          o += char(c);
        }
    }
  }
  return o;
}

void render_prompts_device(const DeviceTable& t, uint64_t n_entries, const uint64_t* rows,
                           const uint64_t* order_offsets, const int32_t* fields,
                           const std::string& system_prompt, const std::string& question,
                           DevBuf<uint64_t>& out_off, DevBuf<uint8_t>& out_bytes,
                           uint64_t& total, cudaStream_t s) {
  const uint32_t m = t.m;
  std::string prefix;
  if (!system_prompt.empty()) prefix += system_prompt + "\n";
  if (!question.empty()) prefix += question + "\n";
  std::vector<uint64_t> name_off(m + 1, 0), name_len(std::max<uint32_t>(m, 1), 0);
  std::string names;
  for (uint32_t f = 0; f < m; ++f) {
    const std::string e = json_escape_bytes(t.names[f]);
    names += e;
    name_len[f] = e.size();
    name_off[f + 1] = names.size();
  }
  auto d_name_off = to_device(name_off, s), d_name_len = to_device(name_len, s);
  std::vector<uint8_t> nb(names.begin(), names.end()), pb(prefix.begin(), prefix.end());
  if (nb.empty()) nb.push_back(0);
  if (pb.empty()) pb.push_back(0);
  auto d_names = to_device(nb, s), d_prefix = to_device(pb, s);
  out_off.alloc(n_entries + 1, s);
  total = 0;
  if (n_entries == 0) {
    out_off.zero();
    out_bytes.alloc(1, s);
    return;
  }
  Sched sc{rows, order_offsets, fields};
  DevBuf<uint64_t> lens(n_entries + 1, s);
  lens.zero();
  DevBuf<int> err(1, s);
  err.zero();
  PO_LAUNCH(k_prompt_len, grid_for(n_entries * 32, 256), 256, 0, s, t.arena,
            t.arena + t.arena_bytes, t.offsets, t.n, m, sc,
            n_entries, d_name_len.get(), uint64_t(prefix.size()), lens.get(), err.get());
  size_t tb = 0;
  PO_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, lens.get(), out_off.get(), int64_t(n_entries + 1), s));
  DevBuf<uint8_t> tmp(tb, s);
  PO_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, lens.get(), out_off.get(), int64_t(n_entries + 1), s));
  int herr = 0;
  err.download(&herr, 1);
  PO_CUDA(cudaMemcpyAsync(&total, out_off.get() + n_entries, 8, cudaMemcpyDeviceToHost, s));
  sync(s);
  if (herr) fail(PO_ERR_OUT_OF_RANGE, "schedule references a row or field outside the table");
  out_bytes.alloc(std::max<uint64_t>(total, 1), s);
  PO_LAUNCH(k_prompt_write, grid_for(n_entries * 32, 256), 256, 0, s, t.arena,
            t.arena + t.arena_bytes, t.offsets, m, sc,
            n_entries, d_names.get(), d_name_off.get(), d_prefix.get(), uint64_t(prefix.size()),
            out_off.get(), out_bytes.get());
}

void dedup_device(const DeviceTable& t, uint64_t* d_expansion, uint64_t* d_unique_first,
                  uint64_t& n_unique, cudaStream_t s) {
  const uint64_t n = t.n;
  n_unique = 0;
  if (n == 0) return;
  Encoded e;
  encode(t, PO_TOK_CHAR, PO_SCORE_VALUE, s, e, debug_hash_bits(), /*ordered=*/false);
  DevBuf<uint32_t> first(e.D, s), flag(n + 1, s), uex(n + 1, s);
  first.fill_bytes(0xFF);
  PO_LAUNCH(k_first_index, grid_for(n, 256), 256, 0, s, e.vid.get(), n, first.get());
  flag.zero();
  PO_LAUNCH(k_is_first, grid_for(n, 256), 256, 0, s, e.vid.get(), n, first.get(), flag.get());
  size_t tb = 0;
  PO_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.get(), uex.get(), int64_t(n + 1), s));
  DevBuf<uint8_t> tmp(tb, s);
  PO_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, flag.get(), uex.get(), int64_t(n + 1), s));
  PO_LAUNCH(k_expand, grid_for(n, 256), 256, 0, s, e.vid.get(), n, first.get(), uex.get(),
            d_expansion, d_unique_first);
  n_unique = e.D;
}

}  // namespace po
