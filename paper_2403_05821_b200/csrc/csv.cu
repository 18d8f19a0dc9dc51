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
constexpr uint8_t kCsv[6][5] = {
    /* R */ {kQ, kC | kCell, kR | kCell | kRec | kBlank | kLine, kA | kCell | kRec | kBlank | kLine, kU | kEmit},
    /* C */ {kQ, kC | kCell, kR | kCell | kRec | kLine, kA | kCell | kRec | kLine, kU | kEmit},
    /* U */ {kU | kEmit, kC | kCell, kR | kCell | kRec | kLine, kA | kCell | kRec | kLine, kU | kEmit},
    /* Q */ {kP, kQ | kEmit, kQ | kEmit | kLine, kQ | kEmit, kQ | kEmit},
    /* P */ {kQ | kEmit, kC | kCell, kR | kCell | kRec | kLine, kA | kCell | kRec | kLine, kU | kEmit},
    /* A */ {kQ, kC | kCell, kR, kA | kCell | kRec | kBlank | kLine, kU | kEmit},
};

// The table held in registers (a per-lane __constant__ lookup with divergent
// indices is serialised): per class, byte s of kT8 is the transition from
// state s; nibble s of kT4 is its next state.
__host__ __device__ constexpr uint64_t t8_of(int c) {
  uint64_t v = 0;
  for (int s = 0; s < 6; ++s) v |= uint64_t(kCsv[s][c]) << (8 * s);
  return v;
}
__host__ __device__ constexpr uint32_t t4_of(int c) {
  uint32_t v = 0;
  for (int s = 0; s < 6; ++s) v |= uint32_t(kCsv[s][c] & 7) << (4 * s);
  return v;
}
__device__ __forceinline__ uint64_t t8(uint8_t b) {
  return b == '"' ? t8_of(0) : b == ',' ? t8_of(1) : b == '\n' ? t8_of(2) : b == '\r' ? t8_of(3) : t8_of(4);
}
__device__ __forceinline__ uint32_t t4(uint8_t b) {
  return b == '"' ? t4_of(0) : b == ',' ? t4_of(1) : b == '\n' ? t4_of(2) : b == '\r' ? t4_of(3) : t4_of(4);
}

constexpr uint64_t kChunk = 4096;

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

// Per 16-byte block, high-bit byte masks (two words) of quotes or CRs, commas
// and newlines (exact per byte).
struct BlockMasks {
  uint64_t qr[2], sep[2], nl[2];
};
__device__ __forceinline__ uint64_t eq_mask(uint64_t x, uint64_t c8) {
  const uint64_t y = x ^ c8;
  return ~(((y & 0x7F7F7F7F7F7F7F7Full) + 0x7F7F7F7F7F7F7F7Full) | y) & 0x8080808080808080ull;
}
__device__ __forceinline__ BlockMasks block_masks(const uint4& w) {
  BlockMasks m;
  const uint64_t x[2] = {uint64_t(w.x) | (uint64_t(w.y) << 32), uint64_t(w.z) | (uint64_t(w.w) << 32)};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    m.qr[h] = eq_mask(x[h], 0x2222222222222222ull) | eq_mask(x[h], 0x0D0D0D0D0D0D0D0Dull);
    m.sep[h] = eq_mask(x[h], 0x2C2C2C2C2C2C2C2Cull);
    m.nl[h] = eq_mask(x[h], 0x0A0A0A0A0A0A0A0Aull);
  }
  return m;
}

// Like for_bytes, but a whole aligned 16-byte block is first offered to
// fast(w, masks), which returns false to have its bytes walked one by one.
template <class Fast, class F>
__device__ __forceinline__ void for_blocks(const uint8_t* __restrict__ d, uint64_t a, uint64_t b,
                                           Fast&& fast, F&& f) {
  const bool aligned = (reinterpret_cast<uintptr_t>(d) & 15) == 0;
  uint64_t i = a;
  if (aligned && i + 16 <= b) {
    // the next block's load is issued before this one is processed
    uint4 nx = __ldg(reinterpret_cast<const uint4*>(d + i));
    for (; i + 16 <= b; i += 16) {
      const uint4 w = nx;
      if (i + 32 <= b) nx = __ldg(reinterpret_cast<const uint4*>(d + i + 16));
      if (fast(w, block_masks(w))) continue;
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k) f(uint8_t(ws[q] >> (8 * k)));
    }
  }
  for (; i < b; ++i) f(d[i]);
}

// state after a block without quotes or CRs from any state but Q: its last
// byte decides (',' -> C, '\n' -> R, anything else -> U)
__device__ __forceinline__ uint32_t plain_block_end(const uint4& w) {
  const uint8_t last = uint8_t(w.w >> 24);
  return last == ',' ? uint32_t(kC) : last == '\n' ? uint32_t(kR) : uint32_t(kU);
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
    uint32_t st4[6] = {0, 4, 8, 12, 16, 20};  // 4 x the state of each run
    const uint64_t a = ch * kChunk, b = a + kChunk < len ? a + kChunk : len;
    for_blocks(
        d, a, b,
        [&](const uint4& w, const BlockMasks& mk) {
          if (mk.qr[0] | mk.qr[1]) return false;
          const uint32_t g = plain_block_end(w) << 2;
#pragma unroll
          for (int s = 0; s < 6; ++s) st4[s] = st4[s] == 4u * kQ ? st4[s] : g;
          return true;
        },
        [&](uint8_t byte) {
          const uint32_t tb = t4(byte);
#pragma unroll
          for (int s = 0; s < 6; ++s) st4[s] = ((tb >> st4[s]) & 7u) << 2;
        });
    uint32_t v = 0;
    for (int s = 0; s < 6; ++s) v |= (st4[s] >> 2) << (3 * s);
    out[ch] = Fn{v};
  }
}

// counts per chunk from its true start state: content bytes, cells, records, lines
__global__ void k_csv_count(const uint8_t* __restrict__ d, uint64_t len, uint64_t nch,
                            const Fn* __restrict__ pre, ulonglong4* cnt) {
  for (uint64_t ch = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; ch < nch;
       ch += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t st8 = (pre[ch].v & 7) << 3;  // 8 x the state at the chunk start (file starts in R)
    uint32_t e = 0, cells = 0, recs = 0, lines = 0;
    const uint64_t a = ch * kChunk, b = a + kChunk < len ? a + kChunk : len;
    for_blocks(
        d, a, b,
        [&](const uint4& w, const BlockMasks& mk) {
          // outside quotes and not right after a CR: ',' and '\n' end a cell
          // ('\n' also a record and a line), every other byte is content
          if ((mk.qr[0] | mk.qr[1]) || st8 == 8u * kQ || st8 == 8u * kA) return false;
          const uint32_t nn = __popcll(mk.nl[0]) + __popcll(mk.nl[1]);
          const uint32_t ns = __popcll(mk.sep[0]) + __popcll(mk.sep[1]) + nn;
          e += 16 - ns;
          cells += ns;
          recs += nn;
          lines += nn;
          st8 = plain_block_end(w) << 3;
          return true;
        },
        [&](uint8_t byte) {
          const uint32_t t = uint32_t(t8(byte) >> st8) & 0xFFu;
          st8 = (t & 7u) << 3;
          e += (t >> 3) & 1u;  // kEmit
          cells += (t >> 4) & 1u;
          recs += (t >> 5) & 1u;
          lines += t >> 7;
        });
    cnt[ch] = make_ulonglong4(e, cells, recs, lines);
  }
}

__device__ __forceinline__ void shl128(uint64_t& lo, uint64_t& hi, uint32_t s) {  // s < 128
  if (s == 0) return;
  if (s < 64) {
    hi = (hi << s) | (lo >> (64 - s));
    lo <<= s;
  } else {
    hi = lo << (s - 64);
    lo = 0;
  }
}
__device__ __forceinline__ void shr128(uint64_t& lo, uint64_t& hi, uint32_t s) {  // s < 128
  if (s == 0) return;
  if (s < 64) {
    lo = (lo >> s) | (hi << (64 - s));
    hi >>= s;
  } else {
    lo = hi >> (s - 64);
    hi = 0;
  }
}
__device__ __forceinline__ void keep_low_bytes128(uint64_t& lo, uint64_t& hi, uint32_t n) {  // n <= 16
  if (n < 8) {
    lo &= n ? (~0ull >> (64 - 8 * n)) : 0ull;
    hi = 0;
  } else if (n < 16) {
    hi &= n > 8 ? (~0ull >> (64 - 8 * (n - 8))) : 0ull;
  }
}

// Writes a chunk's content bytes: one contiguous run of the arena starting at
// x0. Bytes up to the first 16-byte boundary at or after x0 are stored one by
// one; after that they gather in a 16-byte register slot (lo, hi) stored
// whole when full.
struct EmitRun {
  uint8_t* arena;
  uint64_t x0;
  uint64_t x;  // next content byte
  uint64_t lo = 0, hi = 0;
  // the low n (<= 16) bytes of (a, b)
  __device__ __forceinline__ void append(uint64_t a, uint64_t b, uint32_t n) {
    while (n && (x & ~uint64_t(15)) < x0) {  // the slot is shared with the previous chunk
      arena[x++] = uint8_t(a);
      shr128(a, b, 8);
      --n;
    }
    if (!n) return;
    keep_low_bytes128(a, b, n);
    const uint32_t k = uint32_t(x & 15);
    uint64_t sa = a, sb = b;
    shl128(sa, sb, 8 * k);
    lo |= sa;
    hi |= sb;
    if (k + n >= 16) {
      *reinterpret_cast<uint4*>(arena + (x - k)) =
          make_uint4(uint32_t(lo), uint32_t(lo >> 32), uint32_t(hi), uint32_t(hi >> 32));
      // what did not fit starts the next slot (nothing when k == 0: n == 16)
      lo = hi = 0;
      if (k) {
        lo = a;
        hi = b;
        shr128(lo, hi, 8 * (16 - k));
      }
    }
    x += n;
  }
  __device__ __forceinline__ void put(uint8_t c) { append(c, 0, 1); }
  // the partial last slot
  __device__ __forceinline__ void finish() {
    const uint32_t k = uint32_t(x & 15);
    if (k && x - k >= x0)
      for (uint32_t q = 0; q < k; ++q) arena[x - k + q] = uint8_t((q < 8 ? lo : hi) >> (8 * (q & 7)));
  }
};

__global__ void k_csv_emit(const uint8_t* __restrict__ d, uint64_t len, uint64_t nch,
                           const Fn* __restrict__ pre, const ulonglong4* __restrict__ base,
                           uint8_t* arena, uint64_t* cell_end, uint64_t* rec_end_cell,
                           uint64_t* rec_next_line, uint8_t* rec_blank) {
  for (uint64_t ch = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; ch < nch;
       ch += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t st8 = (pre[ch].v & 7) << 3;
    ulonglong4 p = base[ch];  // running: content byte, cell, record, line increments
    EmitRun run{arena, p.x, p.x};
    const uint64_t a = ch * kChunk, b = a + kChunk < len ? a + kChunk : len;
    auto end_cell = [&]() { cell_end[p.y++] = run.x; };
    auto end_record = [&](bool blank) {
      rec_end_cell[p.z] = p.y;
      rec_next_line[p.z] = 1 + p.w;  // start line of the record that follows
      rec_blank[p.z] = blank ? 1 : 0;
      ++p.z;
    };
    for_blocks(
        d, a, b,
        [&](const uint4& w, const BlockMasks& mk) {
          // a block without quotes or CRs, outside quotes and not right after
          // a CR: ',' ends a cell, '\n' a cell, a record and a line, every
          // other byte is content; the runs between separators are appended
          // 16 bytes at a time
          if ((mk.qr[0] | mk.qr[1]) || st8 == 8u * kQ || st8 == 8u * kA) return false;
          const uint64_t X0 = uint64_t(w.x) | (uint64_t(w.y) << 32), X1 = uint64_t(w.z) | (uint64_t(w.w) << 32);
          bool rec_start = st8 == 8u * kR;  // no content since the record began
          uint32_t used = 0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint64_t sm = mk.sep[h] | mk.nl[h];
            while (sm) {
              const uint32_t bit = uint32_t(__ffsll((long long)sm) - 1);
              sm &= sm - 1;
              const uint32_t j = 8 * h + (bit >> 3);
              if (j > used) {
                uint64_t s0 = X0, s1 = X1;
                shr128(s0, s1, 8 * used);
                run.append(s0, s1, j - used);
                rec_start = false;
              }
              const bool nl = (mk.nl[h] >> bit) & 1;
              end_cell();
              if (nl) {
                ++p.w;
                end_record(rec_start);
              }
              rec_start = nl;
              used = j + 1;
            }
          }
          if (used < 16) {
            uint64_t s0 = X0, s1 = X1;
            shr128(s0, s1, 8 * used);
            run.append(s0, s1, 16 - used);
          }
          st8 = plain_block_end(w) << 3;
          return true;
        },
        [&](uint8_t c) {
          const uint32_t t = uint32_t(t8(c) >> st8) & 0xFFu;
          st8 = (t & 7u) << 3;
          if (t & kEmit) run.put(c);
          if (t & kLine) ++p.w;
          if (t & kCell) end_cell();
          if (t & kRec) end_record((t & kBlank) != 0);
        });
    run.finish();
  }
}

// first record r in [1, hi) whose cell count (rec_end[r] - rec_end[r - 1])
// is not h
__global__ void k_csv_widths(const uint64_t* __restrict__ rec_end, uint64_t hi, uint64_t h,
                             unsigned long long* first) {
  for (uint64_t r = 1 + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < hi;
       r += uint64_t(gridDim.x) * blockDim.x)
    if (rec_end[r] - rec_end[r - 1] != h) atomicMin(first, (unsigned long long)r);
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
  out.n_closed = tot.z;
  out.rec_end = std::move(rec_end);
  out.rec_line = std::move(rec_line);
  out.rec_blank = std::move(rec_blank);
  if (pending) {
    const uint64_t ce = tot.x;
    h2d_async(out.cell_end.get() + tot.y, &ce, 8, s);
  }
  sync(s);
}

uint64_t CsvParsed::end_cell(uint64_t r, cudaStream_t s) const {
  if (r >= n_closed) return n_cells;  // the record pending at EOF
  uint64_t v = 0;
  PO_CUDA(cudaMemcpyAsync(&v, rec_end.get() + r, 8, cudaMemcpyDeviceToHost, s));
  sync(s);
  return v;
}

uint64_t CsvParsed::start_line(uint64_t r, cudaStream_t s) const {
  if (r == 0) return 1;
  uint64_t v = 1;
  PO_CUDA(cudaMemcpyAsync(&v, rec_line.get() + (r - 1), 8, cudaMemcpyDeviceToHost, s));
  sync(s);
  return v;
}

bool CsvParsed::blank(uint64_t r, cudaStream_t s) const {
  if (r >= n_closed) return false;
  uint8_t v = 0;
  PO_CUDA(cudaMemcpyAsync(&v, rec_blank.get() + r, 1, cudaMemcpyDeviceToHost, s));
  sync(s);
  return v != 0;
}

uint64_t CsvParsed::first_wrong_width(uint64_t h, cudaStream_t s) const {
  if (n_records < 3) return n_records;
  DevBuf<unsigned long long> first(1, s);
  first.fill_bytes(0xFF);
  // records [1, n_records - 1) all closed inside the text (r < n_closed)
  const uint64_t hi = n_records - 1;
  PO_LAUNCH(k_csv_widths, grid_for(hi, 256), 256, 0, s, rec_end.get(), hi, h, first.get());
  unsigned long long v = 0;
  first.download(&v, 1);
  sync(s);
  return v == ~0ull ? n_records : uint64_t(v);
}

}  // namespace po
