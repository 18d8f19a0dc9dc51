// CSV ingest: prefixopt::load_csv (table.hpp:114-215,
// RFC 4180 reader detail::read_csv_record) on the GPU.
//
// The reader is a 6-state automaton over bytes:
//   R record start | C cell start after ',' | U unquoted content (or after a
//   closing quote) | Q inside quotes | P inside quotes, just saw '"' (a second
//   '"' is a literal quote, anything else closes) | A record start right
//   after '\r' (a following '\n' is swallowed).
// A '"' opens quoting only at R/C/A (empty cell, no content yet); in U it is
// content. Line numbers follow the reference: '\n' inside quotes, and each
// record end ('\r', '\r\n' once, or '\n'), advance the line.
// Parallel form (simultaneous automaton): every 4 KB chunk computes its
// transition function for all 6 start states; an exclusive scan composing
// the functions gives each chunk's true start state; a counting pass and an
// emitting pass then re-run the chunks from those states, writing content
// bytes, cell ends and record ends at scanned positions. The host applies the
// reference's checks in its order (missing header, duplicate header field,
// per-record cell counts / unterminated quote, empty field names) and drops a
// trailing blank line.

#include <cub/cub.cuh>

#include "internal.cuh"

namespace po {

namespace {

enum : uint8_t { kR = 0, kC, kU, kQ, kP, kA };
enum : uint8_t { kEmit = 8, kCell = 16, kRec = 32, kBlank = 64, kLine = 128 };

// [state][class]: class 0 '"', 1 ',', 2 '\n', 3 '\r', 4 other
__constant__ uint8_t c_csv[6][5] = {
    /* R */ {kQ, kC | kCell, kR | kCell | kRec | kBlank | kLine, kA | kCell | kRec | kBlank | kLine, kU | kEmit},
    /* C */ {kQ, kC | kCell, kR | kCell | kRec | kLine, kA | kCell | kRec | kLine, kU | kEmit},
    /* U */ {kU | kEmit, kC | kCell, kR | kCell | kRec | kLine, kA | kCell | kRec | kLine, kU | kEmit},
    /* Q */ {kP, kQ | kEmit, kQ | kEmit | kLine, kQ | kEmit, kQ | kEmit},
    /* P */ {kQ | kEmit, kC | kCell, kR | kCell | kRec | kLine, kA | kCell | kRec | kLine, kU | kEmit},
    /* A */ {kQ, kC | kCell, kR, kA | kCell | kRec | kBlank | kLine, kU | kEmit},
};

constexpr uint64_t kChunk = 4096;

__device__ __forceinline__ uint32_t cls(uint8_t c) {
  return c == '"' ? 0u : c == ',' ? 1u : c == '\n' ? 2u : c == '\r' ? 3u : 4u;
}

// Calls f on bytes d[a..b) in order, reading 16 bytes per load (a is
// kChunk-aligned; the arena base is at least 16-byte aligned: cudaMalloc /
// torch allocations), so a thread issues a sixteenth of the load
// instructions and keeps 16 bytes in registers.
template <class F>
__device__ __forceinline__ void for_bytes(const uint8_t* __restrict__ d, uint64_t a, uint64_t b,
                                          F&& f) {
  const bool aligned = (reinterpret_cast<uintptr_t>(d) & 15) == 0;
  uint64_t i = a;
  if (aligned)
    for (; i + 16 <= b; i += 16) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(d + i));
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k) f(uint8_t(ws[q] >> (8 * k)));
    }
  for (; i < b; ++i) f(d[i]);
}

struct Fn {  // transition function of a chunk: 6 x 3-bit end states
  uint32_t v;
};
struct Compose {  // a then b
  __device__ __forceinline__ Fn operator()(const Fn& a, const Fn& b) const {
    uint32_t r = 0;
    for (uint32_t s = 0; s < 6; ++s) r |= ((b.v >> (3 * ((a.v >> (3 * s)) & 7))) & 7u) << (3 * s);
    return Fn{r};
  }
};
__host__ __device__ constexpr uint32_t fn_identity() {
  return 0u | (1u << 3) | (2u << 6) | (3u << 9) | (4u << 12) | (5u << 15);
}

__global__ void k_csv_trans(const uint8_t* __restrict__ d, uint64_t len, uint64_t nch, Fn* out) {
  for (uint64_t ch = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; ch < nch;
       ch += uint64_t(gridDim.x) * blockDim.x) {
    uint8_t st[6] = {0, 1, 2, 3, 4, 5};
    const uint64_t a = ch * kChunk, b = a + kChunk < len ? a + kChunk : len;
    for_bytes(d, a, b, [&](uint8_t byte) {
      const uint32_t c = cls(byte);
#pragma unroll
      for (int s = 0; s < 6; ++s) st[s] = c_csv[st[s]][c] & 7;
    });
    uint32_t v = 0;
    for (int s = 0; s < 6; ++s) v |= uint32_t(st[s]) << (3 * s);
    out[ch] = Fn{v};
  }
}

// counts per chunk from its true start state: content bytes, cells, records, lines
__global__ void k_csv_count(const uint8_t* __restrict__ d, uint64_t len, uint64_t nch,
                            const Fn* __restrict__ pre, ulonglong4* cnt) {
  for (uint64_t ch = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; ch < nch;
       ch += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t st = pre[ch].v & 7;  // state at the chunk start (file starts in R)
    unsigned long long e = 0, cells = 0, recs = 0, lines = 0;
    const uint64_t a = ch * kChunk, b = a + kChunk < len ? a + kChunk : len;
    for_bytes(d, a, b, [&](uint8_t byte) {
      const uint8_t t = c_csv[st][cls(byte)];
      st = t & 7;
      e += (t & kEmit) != 0;
      cells += (t & kCell) != 0;
      recs += (t & kRec) != 0;
      lines += (t & kLine) != 0;
    });
    cnt[ch] = make_ulonglong4(e, cells, recs, lines);
  }
}

__global__ void k_csv_emit(const uint8_t* __restrict__ d, uint64_t len, uint64_t nch,
                           const Fn* __restrict__ pre, const ulonglong4* __restrict__ base,
                           uint8_t* arena, uint64_t* cell_end, uint64_t* rec_end_cell,
                           uint64_t* rec_next_line, uint8_t* rec_blank) {
  for (uint64_t ch = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; ch < nch;
       ch += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t st = pre[ch].v & 7;
    ulonglong4 p = base[ch];  // running: content byte, cell, record, line increments
    const uint64_t a = ch * kChunk, b = a + kChunk < len ? a + kChunk : len;
    // a chunk's content bytes form one contiguous run of the arena: bytes up
    // to the first 16-byte boundary are stored one by one, then gathered in
    // registers and stored 16 at a time (a sixteenth of the byte stores)
    uint32_t acc[4] = {0u, 0u, 0u, 0u};
    for_bytes(d, a, b, [&](uint8_t c) {
      const uint8_t t = c_csv[st][cls(c)];
      st = t & 7;
      if (t & kEmit) {
        const uint32_t k = uint32_t(p.x & 15);
        if (p.x - k < base[ch].x) {  // before the chunk's first full 16-byte slot
          arena[p.x] = c;
        } else {
          const uint32_t v = uint32_t(c) << (8 * (k & 3));
          switch (k >> 2) {
            case 0: acc[0] |= v; break;
            case 1: acc[1] |= v; break;
            case 2: acc[2] |= v; break;
            default: acc[3] |= v; break;
          }
          if (k == 15) {
            *reinterpret_cast<uint4*>(arena + (p.x - 15)) = make_uint4(acc[0], acc[1], acc[2], acc[3]);
            acc[0] = acc[1] = acc[2] = acc[3] = 0u;
          }
        }
        ++p.x;
      }
      if (t & kLine) ++p.w;
      if (t & kCell) cell_end[p.y++] = p.x;
      if (t & kRec) {
        rec_end_cell[p.z] = p.y;
        rec_next_line[p.z] = 1 + p.w;  // start line of the record that follows
        rec_blank[p.z] = (t & kBlank) ? 1 : 0;
        ++p.z;
      }
    });
    // the partial last slot
    const uint32_t k = uint32_t(p.x & 15);
    if (k && p.x - k >= base[ch].x)
      for (uint32_t q = 0; q < k; ++q) arena[p.x - k + q] = uint8_t(acc[q >> 2] >> (8 * (q & 3)));
  }
}

struct AddU4 {
  __device__ __forceinline__ ulonglong4 operator()(const ulonglong4& a, const ulonglong4& b) const {
    return make_ulonglong4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  }
};

}  // namespace

void load_csv_device(const uint8_t* d, uint64_t len, CsvParsed& out, cudaStream_t s) {
  out = CsvParsed{};
  const uint64_t nch = (len + kChunk - 1) / kChunk;
  uint32_t end_state = kR;
  ulonglong4 tot = make_ulonglong4(0, 0, 0, 0);
  DevBuf<Fn> fn(std::max<uint64_t>(nch, 1), s), pre(std::max<uint64_t>(nch + 1, 1), s);
  DevBuf<ulonglong4> cnt(std::max<uint64_t>(nch, 1), s), base(std::max<uint64_t>(nch + 1, 1), s);
  if (nch) {
    PO_LAUNCH(k_csv_trans, grid_for(nch, 128), 128, 0, s, d, len, nch, fn.get());
    size_t tb = 0;
    PO_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, tb, fn.get(), pre.get(), Compose{},
                                           Fn{fn_identity()}, int64_t(nch), s));
    DevBuf<uint8_t> tmp(tb, s);
    PO_CUDA(cub::DeviceScan::ExclusiveScan(tmp.get(), tb, fn.get(), pre.get(), Compose{},
                                           Fn{fn_identity()}, int64_t(nch), s));
    PO_LAUNCH(k_csv_count, grid_for(nch, 128), 128, 0, s, d, len, nch, pre.get(), cnt.get());
    size_t tb2 = 0;
    PO_CUDA(cub::DeviceScan::ExclusiveScan(nullptr, tb2, cnt.get(), base.get(), AddU4{},
                                           make_ulonglong4(0, 0, 0, 0), int64_t(nch), s));
    DevBuf<uint8_t> tmp2(tb2, s);
    PO_CUDA(cub::DeviceScan::ExclusiveScan(tmp2.get(), tb2, cnt.get(), base.get(), AddU4{},
                                           make_ulonglong4(0, 0, 0, 0), int64_t(nch), s));
    Fn last_pre, last_fn;
    ulonglong4 last_base, last_cnt;
    PO_CUDA(cudaMemcpyAsync(&last_pre, pre.get() + nch - 1, sizeof(Fn), cudaMemcpyDeviceToHost, s));
    PO_CUDA(cudaMemcpyAsync(&last_fn, fn.get() + nch - 1, sizeof(Fn), cudaMemcpyDeviceToHost, s));
    PO_CUDA(cudaMemcpyAsync(&last_base, base.get() + nch - 1, sizeof(ulonglong4),
                            cudaMemcpyDeviceToHost, s));
    PO_CUDA(cudaMemcpyAsync(&last_cnt, cnt.get() + nch - 1, sizeof(ulonglong4),
                            cudaMemcpyDeviceToHost, s));
    sync(s);
    const uint32_t s_last = last_pre.v & 7;
    end_state = (last_fn.v >> (3 * s_last)) & 7;
    tot = make_ulonglong4(last_base.x + last_cnt.x, last_base.y + last_cnt.y,
                          last_base.z + last_cnt.z, last_base.w + last_cnt.w);
  }
  // EOF closes a pending record (read_csv_record's end_record at EOF)
  const bool pending = end_state == kC || end_state == kU || end_state == kP || end_state == kQ;
  out.unterminated = end_state == kQ;
  out.content_bytes = tot.x;
  out.n_cells = tot.y + (pending ? 1 : 0);
  out.n_records = tot.z + (pending ? 1 : 0);
  out.arena.alloc(std::max<uint64_t>(tot.x, 1), s);
  out.cell_end.alloc(std::max<uint64_t>(out.n_cells, 1), s);
  DevBuf<uint64_t> rec_end(std::max<uint64_t>(out.n_records, 1), s),
      rec_line(std::max<uint64_t>(out.n_records, 1), s);
  DevBuf<uint8_t> rec_blank(std::max<uint64_t>(out.n_records, 1), s);
  if (nch)
    PO_LAUNCH(k_csv_emit, grid_for(nch, 128), 128, 0, s, d, len, nch, pre.get(), base.get(),
              out.arena.get(), out.cell_end.get(), rec_end.get(), rec_line.get(), rec_blank.get());
  out.rec_end_cell.assign(out.n_records, 0);
  out.rec_start_line.assign(out.n_records, 1);
  out.rec_blank.assign(out.n_records, 0);
  std::vector<uint64_t> nl(out.n_records);
  if (tot.z) {
    rec_end.download(out.rec_end_cell.data(), tot.z);
    rec_line.download(nl.data(), tot.z);
    rec_blank.download(out.rec_blank.data(), tot.z);
  }
  if (pending) {
    const uint64_t ce = tot.x;
    h2d_async(out.cell_end.get() + tot.y, &ce, 8, s);
  }
  sync(s);
  if (pending) out.rec_end_cell[out.n_records - 1] = out.n_cells;
  for (uint64_t r = 1; r < out.n_records; ++r) out.rec_start_line[r] = nl[r - 1];
}

}  // namespace po
