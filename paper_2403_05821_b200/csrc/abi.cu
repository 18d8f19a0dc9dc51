// extern "C" entry points of libprefixopt_cuda.so (include/prefixopt_cuda.h).
// Each call runs synchronously on the caller's stream; exceptions become
// PO_ERR_* codes with a thread-local message.

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <unordered_set>

#include "comm.cuh"
#include "internal.cuh"

namespace po {

std::atomic<uint64_t> g_launches{0};
thread_local uint64_t g_syncs = 0;
std::atomic<int> g_profile{0};

namespace {

struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof_pending;
std::vector<cudaEvent_t> g_prof_free;
std::map<std::string, std::pair<uint64_t, double>> g_prof_acc;  // name -> (count, ms)

cudaEvent_t prof_event() {
  if (!g_prof_free.empty()) {
    cudaEvent_t e = g_prof_free.back();
    g_prof_free.pop_back();
    return e;
  }
  cudaEvent_t e;
  PO_CUDA(cudaEventCreate(&e));
  return e;
}

void prof_drain() {  // caller holds g_prof_mu
  // device idle time between the recorded launches (sweep over the scopes'
  // [start, end) intervals in start order), charged to the launch that ends
  // the gap as "gap:<name>": the host work between two launches
  struct Iv {
    float a, b;
    const char* name;
  };
  std::vector<Iv> iv;
  iv.reserve(g_prof_pending.size());
  for (auto& r : g_prof_pending) {
    float ms = 0, a = 0;
    PO_CUDA(cudaEventSynchronize(r.b));
    PO_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    PO_CUDA(cudaEventElapsedTime(&a, g_prof_pending.front().a, r.a));
    iv.push_back({a, a + ms, r.name});
  }
  std::stable_sort(iv.begin(), iv.end(), [](const Iv& x, const Iv& y) { return x.a < y.a; });
  // a scope whose interval holds the next launch wraps other launches (a
  // library call or a multi-kernel sort): reported as "scope:<name>" so that
  // sums over kernels do not count its children twice
  for (size_t i = 0; i < iv.size(); ++i) {
    const bool outer = i + 1 < iv.size() && iv[i + 1].a < iv[i].b - 0.0005f;
    auto& acc = g_prof_acc[outer ? std::string("scope:") + iv[i].name : std::string(iv[i].name)];
    acc.first += 1;
    acc.second += iv[i].b - iv[i].a;
  }
  float covered = iv.empty() ? 0.f : iv.front().a, busy = 0.f;
  for (const Iv& x : iv) {
    if (x.a > covered + 0.002f) {
      auto& acc = g_prof_acc[std::string("gap:") + x.name];
      acc.first += 1;
      acc.second += x.a - covered;
    }
    if (x.b > covered) busy += x.b - std::max(x.a, covered);
    covered = std::max(covered, x.b);
  }
  if (!iv.empty()) {  // device time under any recorded launch (union of the intervals)
    auto& acc = g_prof_acc["busy:"];
    acc.first += 1;
    acc.second += busy;
  }
  for (auto& r : g_prof_pending) {
    g_prof_free.push_back(r.a);
    g_prof_free.push_back(r.b);
  }
  g_prof_pending.clear();
}

}  // namespace

void profile_begin(const char* name, cudaStream_t s, void** token) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (g_prof_pending.size() > 4096) prof_drain();
  ProfRec r{name, prof_event(), prof_event()};
  PO_CUDA(cudaEventRecord(r.a, s));
  g_prof_pending.push_back(r);
  *token = reinterpret_cast<void*>(g_prof_pending.size());
}

void profile_host(const char* name, double ms) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  auto& acc = g_prof_acc[std::string("host:") + name];
  acc.first += 1;
  acc.second += ms;
}

void profile_end(void* token, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  size_t i = reinterpret_cast<size_t>(token) - 1;
  if (i < g_prof_pending.size()) PO_CUDA(cudaEventRecord(g_prof_pending[i].b, s));
}

namespace {
thread_local std::vector<std::pair<std::string, double>> g_marks;
thread_local std::chrono::steady_clock::time_point g_mark_t0;
}  // namespace

// PO_DEBUG_TIMING=1: phase times with a stream sync at every mark (GPU time
// per phase); PO_DEBUG_TIMING=host: host timestamps only, no syncs (where the
// host thread itself waits).
int timing_mode() {
  static const int mode = [] {
    const char* v = std::getenv("PO_DEBUG_TIMING");
    if (!v || !*v || *v == '0') return 0;
    return std::string(v) == "host" ? 2 : 1;
  }();
  return mode;
}
bool debug_timing() { return timing_mode() != 0; }

void timing_mark(const char* phase, cudaStream_t s) {
  if (!debug_timing()) return;
  if (timing_mode() == 1) sync(s);
  auto now = std::chrono::steady_clock::now();
  if (!g_marks.empty() || phase[0] == '<')
    g_marks.push_back({phase, std::chrono::duration<double, std::milli>(now - g_mark_t0).count()});
  g_mark_t0 = now;
}

void timing_report(const char* call) {
  if (!debug_timing()) return;
  std::map<std::string, double> agg;
  std::vector<std::string> order;
  double tot = 0;
  for (auto& [k, v] : g_marks) {
    if (!agg.count(k)) order.push_back(k);
    agg[k] += v;
    tot += v;
  }
  std::string line = "[po timing] " + std::string(call) + " total " + std::to_string(tot) +
                     " ms, " + std::to_string(g_syncs) + " stream syncs:";
  g_syncs = 0;
  for (auto& k : order)
    if (k != "<start") line += " " + k + "=" + std::to_string(agg[k]);
  line += "\n";
  fputs(line.c_str(), stderr);  // one write: lines of concurrent ranks stay whole
  g_marks.clear();
}

namespace {
// Pinned staging memory is recycled across threads (a thread's arena goes
// back to a free list when the thread exits): callers that run each call on
// a fresh host thread must not pay cudaMallocHost / cudaFreeHost (which
// synchronises the device) per call.
std::mutex g_pin_mu;
std::vector<std::pair<uint8_t*, size_t>> g_pin_free;

struct PinnedArena {
  uint8_t* base = nullptr;
  size_t cap = 0, used = 0;
  // the last staged copy: its stream (compared only, never synchronised: the
  // caller may destroy it) and an event recorded after it, which orders
  // every earlier copy on that stream
  cudaStream_t last = nullptr;
  cudaEvent_t done = nullptr;
  int done_dev = -1;
  bool pending = false;
  void wait_copies() {
    if (pending) cudaEventSynchronize(done);
    pending = false;
  }
  ~PinnedArena() {
    if (!base) return;
    wait_copies();  // copies out of the arena are done
    if (done) cudaEventDestroy(done);
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_free.push_back({base, cap});
  }
  void acquire() {
    {
      std::lock_guard<std::mutex> lk(g_pin_mu);
      if (!g_pin_free.empty()) {
        base = g_pin_free.back().first;
        cap = g_pin_free.back().second;
        g_pin_free.pop_back();
        return;
      }
    }
    cap = 32u << 20;
    if (cudaMallocHost(reinterpret_cast<void**>(&base), cap) != cudaSuccess) {
      (void)cudaGetLastError();
      base = nullptr;
      cap = 0;
    }
  }
};
thread_local PinnedArena g_pin;
}  // namespace

namespace {
struct CachedBlock {
  void* p = nullptr;
  size_t bytes = 0;
  int device = 0;
  bool busy = false;
  cudaEvent_t released = nullptr;  // recorded on the releasing stream
};
std::mutex g_blocks_mu;
std::vector<CachedBlock> g_blocks;
}  // namespace

void* cached_block_acquire(size_t bytes, cudaStream_t s) {
  int dev = 0;
  PO_CUDA(cudaGetDevice(&dev));
  bytes = (bytes + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
  std::lock_guard<std::mutex> lk(g_blocks_mu);
  CachedBlock* best = nullptr;
  for (auto& b : g_blocks)  // best fit among free blocks of at most twice the size
    if (!b.busy && b.device == dev && b.bytes >= bytes && b.bytes <= 2 * bytes &&
        (!best || b.bytes < best->bytes))
      best = &b;
  if (best) {
    // always ordered on the release event: stream handles are not unique
    // identities (cudaStreamPerThread, reused handles); the wait is a no-op
    // once the event has completed
    PO_CUDA(cudaStreamWaitEvent(s, best->released, 0));
    best->busy = true;
    return best->p;
  }
  CachedBlock b;
  b.bytes = bytes;
  b.device = dev;
  b.busy = true;
  if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
    (void)cudaGetLastError();
    // free the idle cached blocks of this device and the stream-ordered
    // pool's unused reservation, then retry once
    PO_CUDA(cudaDeviceSynchronize());
    for (auto it = g_blocks.begin(); it != g_blocks.end();)
      if (!it->busy && it->device == dev) {
        cudaFree(it->p);
        cudaEventDestroy(it->released);
        it = g_blocks.erase(it);
      } else {
        ++it;
      }
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    PO_CUDA(cudaMalloc(&b.p, bytes));
  }
  PO_CUDA(cudaEventCreateWithFlags(&b.released, cudaEventDisableTiming));
  g_blocks.push_back(b);
  return b.p;
}

uint64_t trim_cached_blocks() {
  std::lock_guard<std::mutex> lk(g_blocks_mu);
  uint64_t freed = 0;
  for (auto it = g_blocks.begin(); it != g_blocks.end();)
    if (!it->busy) {
      int prev = 0;
      cudaGetDevice(&prev);
      cudaSetDevice(it->device);
      cudaEventSynchronize(it->released);  // its last user is done
      cudaFree(it->p);
      cudaEventDestroy(it->released);
      cudaSetDevice(prev);
      freed += it->bytes;
      it = g_blocks.erase(it);
    } else {
      ++it;
    }
  return freed;
}

void cached_block_release(void* p, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_blocks_mu);
  for (auto& b : g_blocks)
    if (b.p == p) {
      cudaEventRecord(b.released, s);
      b.busy = false;
      return;
    }
}

// Side streams are per thread and device, taken from a process-wide pool and
// returned when the thread exits: callers that run every call on a fresh
// host thread (pipelined e2e, thread ranks) neither create nor destroy
// streams per call.
namespace {
std::mutex g_stream_mu;
std::map<std::pair<int, int>, std::vector<cudaStream_t>> g_stream_free;  // (kind, device)

cudaStream_t pooled_stream(int kind) {
  struct Held {
    std::vector<std::pair<std::pair<int, int>, cudaStream_t>> s;
    ~Held() {
      std::lock_guard<std::mutex> lk(g_stream_mu);
      for (auto& [key, st] : s) g_stream_free[key].push_back(st);
    }
  };
  static thread_local Held held;
  int dev = 0;
  PO_CUDA(cudaGetDevice(&dev));
  const std::pair<int, int> key{kind, dev};
  for (auto& [k, st] : held.s)
    if (k == key) return st;
  cudaStream_t st = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_stream_mu);
    auto& f = g_stream_free[key];
    if (!f.empty()) {
      st = f.back();
      f.pop_back();
    }
  }
  if (!st) PO_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  held.s.push_back({key, st});
  return st;
}
}  // namespace

cudaStream_t copy_stream() { return pooled_stream(0); }
cudaStream_t aux_stream() { return pooled_stream(1); }

// Small device -> host reads that the host waits for (level results): through
// a per-thread pinned buffer, which completes sooner than a pageable copy.
bool debug_syncs() {
  static const bool on = [] {
    const char* v = std::getenv("PO_DEBUG_SYNCS");
    return v && *v && *v != '0';
  }();
  return on;
}

void d2h_sync(void* dst, const void* src, size_t bytes, cudaStream_t s, const char* file, int line) {
  // per-thread bounce buffer from a process-wide list (returned at thread
  // exit, never freed: cudaFreeHost synchronises the device)
  static std::mutex mu;
  static std::vector<std::pair<uint8_t*, size_t>> free_bufs;
  struct Pinned {
    uint8_t* p = nullptr;
    size_t cap = 0;
    ~Pinned() {
      if (p) {
        std::lock_guard<std::mutex> lk(mu);
        free_bufs.push_back({p, cap});
      }
    }
  };
  static thread_local Pinned buf;
  constexpr size_t kMax = 4u << 20;
  if (bytes > kMax) {
    PO_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    sync(s, file, line);
    return;
  }
  if (buf.cap < bytes) {
    std::lock_guard<std::mutex> lk(mu);
    if (buf.p) free_bufs.push_back({buf.p, buf.cap});
    buf.p = nullptr;
    buf.cap = 0;
    for (size_t i = 0; i < free_bufs.size(); ++i)
      if (free_bufs[i].second >= bytes) {
        buf.p = free_bufs[i].first;
        buf.cap = free_bufs[i].second;
        free_bufs.erase(free_bufs.begin() + i);
        break;
      }
    if (!buf.p) {
      const size_t cap = std::max<size_t>(bytes, 64u << 10);
      PO_CUDA(cudaMallocHost(reinterpret_cast<void**>(&buf.p), cap));
      buf.cap = cap;
    }
  }
  if (bytes) PO_CUDA(cudaMemcpyAsync(buf.p, src, bytes, cudaMemcpyDeviceToHost, s));
  sync(s, file, line);
  if (bytes) std::memcpy(dst, buf.p, bytes);
}

void h2d_async(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (!bytes) return;
  PinnedArena& a = g_pin;
  if (bytes > kPinnedSmallCopy) {
    PO_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  if (!a.base) {
    a.acquire();
    if (!a.base) {
      PO_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
      return;
    }
  }
  const size_t need = (bytes + 15) & ~size_t(15);
  int dev = 0;
  PO_CUDA(cudaGetDevice(&dev));
  if (a.used + need > a.cap || (a.pending && (a.last != s || a.done_dev != dev))) {
    // recycle: every earlier copy out of the arena must have completed
    a.wait_copies();
    a.used = 0;
  }
  if (a.done_dev != dev) {  // events record only on streams of their device
    if (a.done) cudaEventDestroy(a.done);
    PO_CUDA(cudaEventCreateWithFlags(&a.done, cudaEventDisableTiming));
    a.done_dev = dev;
  }
  uint8_t* p = a.base + a.used;
  a.used += need;
  a.last = s;
  std::memcpy(p, src, bytes);
  PO_CUDA(cudaMemcpyAsync(dst, p, bytes, cudaMemcpyHostToDevice, s));
  PO_CUDA(cudaEventRecord(a.done, s));
  a.pending = true;
}

namespace {

// Keep freed stream-ordered allocations cached in the device pool between
// calls instead of returning them to the driver at every synchronisation.
void init_pool_once() {
  static thread_local int done_dev = -1;
  int dev = 0;
  PO_CUDA(cudaGetDevice(&dev));
  if (done_dev == dev) return;
  cudaMemPool_t pool;
  PO_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = ~uint64_t(0);
  PO_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  done_dev = dev;
}

thread_local std::string g_err;

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return PO_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return PO_ERR_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PO_ERR_ERROR;
  }
}

void check_modes(int tok, int scoring) {
  if (tok < PO_TOK_CHAR || tok > PO_TOK_CUSTOM) fail(PO_ERR_INVALID_ARG, "unknown tokenizer kind");
  if (scoring != PO_SCORE_VALUE && scoring != PO_SCORE_FRAGMENT)
    fail(PO_ERR_INVALID_ARG, "unknown scoring mode");
}

}  // namespace

// PO_DEBUG_HASH_BITS=k keeps k bits of every cell hash (forces collisions:
// tests of the exact dictionary), 64 otherwise.
uint32_t debug_hash_bits() {
  const char* v = std::getenv("PO_DEBUG_HASH_BITS");
  if (!v || !*v) return 64;
  int b = std::atoi(v);
  return (b <= 0 || b > 64) ? 64u : uint32_t(b);
}

namespace {

struct Prepared {
  DeviceTable t;
  Encoded e;
};

// ordered = false for callers that only need value identity (phc, hit,
// compute_stats): the escaped-order rank job is not started.
// Unique columns stay unranked (Encoded::unranked) unless PO_RANK_UNIQUE=1.
bool rank_unique_columns() {
  const char* v = std::getenv("PO_RANK_UNIQUE");
  return v && *v == '1';
}

void prepare(const po_table* tv, int tok, int scoring, cudaStream_t s, Prepared& p,
             bool ordered = true) {
  check_modes(tok, scoring);
  init_pool_once();
  // host tables stream through the dictionary pass (row chunks copied while
  // the previous chunk is encoded); nothing after encode() reads the table
  make_device_table(tv, tok, s, p.t, /*stream_host=*/true);
  timing_mark("table_h2d", s);
  encode(p.t, tok, scoring, s, p.e, debug_hash_bits(), ordered, rank_unique_columns());
}

// offsets of the data cells of a parsed CSV (po_csv_copy)
__global__ void k_csv_offsets(const uint64_t* cell_end, uint64_t first, uint64_t count,
                              uint64_t base, uint64_t* out) {
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k <= count;
       k += uint64_t(gridDim.x) * blockDim.x)
    out[k] = (first + k == 0 ? 0 : cell_end[first + k - 1]) - base;
}

__global__ void k_u32_to_u64(const uint32_t* a, uint64_t n, uint64_t* b) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    b[i] = a[i];
}

// Copies a device u32 row array to the caller's u64 buffer (host or device).
void deliver_rows(const uint32_t* d_rows32, uint64_t n, uint32_t loc, uint64_t* out,
                  cudaStream_t s) {
  if (n == 0) return;
  if (loc == PO_LOC_DEVICE) {
    PO_LAUNCH(k_u32_to_u64, grid_for(n, 256), 256, 0, s, d_rows32, n, out);
  } else {
    DevBuf<uint64_t> tmp(n, s);
    PO_LAUNCH(k_u32_to_u64, grid_for(n, 256), 256, 0, s, d_rows32, n, tmp.get());
    tmp.download(out, n);
  }
}

template <class T>
const T* stage(const T* p, uint64_t count, uint32_t loc, DevBuf<T>& own, cudaStream_t s) {
  if (loc == PO_LOC_DEVICE || count == 0) return p;
  own.alloc(count, s);
  own.upload(p, count);
  return own.get();
}

uint64_t phc_call(const po_table* tv, int tok, int scoring, uint64_t n_entries,
                  const uint64_t* rows, const uint64_t* offs, const int32_t* fields, uint32_t loc,
                  cudaStream_t s, uint64_t first, uint64_t last_plus_one) {
  if (loc != PO_LOC_HOST && loc != PO_LOC_DEVICE) fail(PO_ERR_INVALID_ARG, "bad schedule location");
  if (n_entries && (!rows || !offs)) fail(PO_ERR_INVALID_ARG, "null schedule arrays");
  Prepared p;
  prepare(tv, tok, scoring, s, p, /*ordered=*/false);  // PHC needs identity only
  uint64_t nfields = 0;
  if (n_entries) {
    if (loc == PO_LOC_HOST) nfields = offs[n_entries];
    else {
      PO_CUDA(cudaMemcpyAsync(&nfields, offs + n_entries, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      sync(s);
    }
  }
  DevBuf<uint64_t> own_rows, own_offs;
  DevBuf<int32_t> own_fields;
  const uint64_t* d_rows = stage(rows, n_entries, loc, own_rows, s);
  const uint64_t* d_offs = stage(offs, n_entries + 1, loc, own_offs, s);
  const int32_t* d_fields = stage(fields, nfields, loc, own_fields, s);
  return phc_device(p.e, last_plus_one, d_rows, nullptr, d_offs, d_fields, s, first);
}

}  // namespace

}  // namespace po

using namespace po;

struct po_comm {
  std::unique_ptr<po::Comm> c;
};

struct po_csv {
  uint64_t rows = 0;
  uint32_t fields = 0;
  uint64_t first_cell = 0;   // first data cell
  uint64_t base = 0;         // arena offset of the first data byte
  uint64_t data_bytes = 0;
  std::string names;
  std::vector<uint64_t> name_off;
  po::CsvParsed parsed;
};

struct po_schedule {
  uint64_t n = 0, m = 0, total = 0;
  po::DevBuf<uint32_t> rows;
  po::DevBuf<uint64_t> offsets;  // empty: uniform (entry i at i*m)
  po::DevBuf<int32_t> fields;
};

struct po_slice {
  uint64_t offset = 0, count = 0;
  uint32_t m = 0;
  int device = 0;
  po::DevBuf<uint64_t> rows;
  po::DevBuf<int32_t> orders;  // (count + 1) * m, entry i at (i + 1) * m
};

extern "C" {

int po_ggr(const po_table* t, const po_fd_groups* fds, const po_ggr_config* cfg, int32_t tok,
           int32_t scoring, uint32_t out_location, uint64_t* out_row_ids,
           int32_t* out_field_orders, uint64_t* out_phc, po_solve_stats* out_stats,
           void* stream) {
  return guarded([&] {
    auto t0 = std::chrono::steady_clock::now();
    if (!cfg || !out_phc) fail(PO_ERR_INVALID_ARG, "null config or output");
    if (out_location != PO_LOC_HOST && out_location != PO_LOC_DEVICE)
      fail(PO_ERR_INVALID_ARG, "bad output location");
    if (cfg->stats_variant < 0 || cfg->stats_variant > 2)
      fail(PO_ERR_INVALID_ARG, "unknown stats variant");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    timing_mark("<start", s);
    std::vector<std::vector<int>> groups;
    if (fds && cfg->use_fds)
      for (uint32_t g = 0; g < fds->n_groups; ++g)
        groups.emplace_back(fds->members + fds->group_offsets[g],
                            fds->members + fds->group_offsets[g + 1]);
    Prepared p;
    prepare(t, tok, scoring, s, p);
    const uint64_t n = p.e.n, m = p.e.m;
    DevBuf<uint32_t> rows(n, s);
    int32_t* d_orders = nullptr;
    DevBuf<int32_t> own_orders;
    if (out_location == PO_LOC_DEVICE) d_orders = out_field_orders;
    else {
      own_orders.alloc(n * m, s);
      d_orders = own_orders.get();
    }
    GgrOutput go;
    ggr_device(p.e, groups, *cfg, rows.get(), d_orders, go, s);
    if (go.csr)
      fail(PO_ERR_SIZE,
           "FD groups repeat a field pair: some field orders are longer than n_fields; "
           "use po_ggr_schedule");
    deliver_rows(rows.get(), n, out_location, out_row_ids, s);
    if (out_location == PO_LOC_HOST) own_orders.download(out_field_orders, n * m);
    sync(s);
    timing_mark("deliver", s);
    timing_report("po_ggr");
    *out_phc = go.phc;
    if (out_stats) {
      *out_stats = go.stats;
      out_stats->wall_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

int po_ggr_schedule(const po_table* t, const po_fd_groups* fds, const po_ggr_config* cfg,
                    int32_t tok, int32_t scoring, po_schedule** out_schedule, uint64_t* out_phc,
                    po_solve_stats* out_stats, void* stream) {
  return guarded([&] {
    auto t0 = std::chrono::steady_clock::now();
    if (!cfg || !out_phc || !out_schedule) fail(PO_ERR_INVALID_ARG, "null config or output");
    if (cfg->stats_variant < 0 || cfg->stats_variant > 2)
      fail(PO_ERR_INVALID_ARG, "unknown stats variant");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::vector<std::vector<int>> groups;
    if (fds && cfg->use_fds)
      for (uint32_t g = 0; g < fds->n_groups; ++g)
        groups.emplace_back(fds->members + fds->group_offsets[g],
                            fds->members + fds->group_offsets[g + 1]);
    Prepared p;
    prepare(t, tok, scoring, s, p);
    const uint64_t n = p.e.n, m = p.e.m;
    auto sc = std::make_unique<po_schedule>();
    sc->n = n;
    sc->m = m;
    sc->rows.alloc(n, s);
    DevBuf<int32_t> orders(n * m, s);
    GgrOutput go;
    ggr_device(p.e, groups, *cfg, sc->rows.get(), orders.get(), go, s);
    if (go.csr) {
      sc->offsets = std::move(go.csr_offsets);
      sc->fields = std::move(go.csr_fields);
      sc->total = go.csr_total;
    } else {
      sc->fields = std::move(orders);
      sc->total = n * m;
    }
    sync(s);
    *out_phc = go.phc;
    if (out_stats) {
      *out_stats = go.stats;
      out_stats->wall_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    *out_schedule = sc.release();
  });
}

int po_schedule_info(const po_schedule* sc, uint64_t* out_entries, uint64_t* out_fields_total) {
  return guarded([&] {
    if (!sc) fail(PO_ERR_INVALID_ARG, "null schedule");
    if (out_entries) *out_entries = sc->n;
    if (out_fields_total) *out_fields_total = sc->total;
  });
}

int po_schedule_copy(const po_schedule* sc, uint32_t out_location, uint64_t* out_row_ids,
                     uint64_t* out_order_offsets, int32_t* out_order_fields, void* stream) {
  return guarded([&] {
    if (!sc) fail(PO_ERR_INVALID_ARG, "null schedule");
    if (out_location != PO_LOC_HOST && out_location != PO_LOC_DEVICE)
      fail(PO_ERR_INVALID_ARG, "bad output location");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t n = sc->n;
    if (n && (!out_row_ids || !out_order_offsets || (sc->total && !out_order_fields)))
      fail(PO_ERR_INVALID_ARG, "null output");
    deliver_rows(sc->rows.get(), n, out_location, out_row_ids, s);
    const cudaMemcpyKind k = out_location == PO_LOC_HOST ? cudaMemcpyDeviceToHost
                                                         : cudaMemcpyDeviceToDevice;
    if (sc->offsets.get()) {
      PO_CUDA(cudaMemcpyAsync(out_order_offsets, sc->offsets.get(), (n + 1) * 8, k, s));
    } else if (out_order_offsets) {  // uniform: entry i at i*m
      std::vector<uint64_t> h(n + 1);
      for (uint64_t i = 0; i <= n; ++i) h[i] = i * sc->m;
      PO_CUDA(cudaMemcpyAsync(out_order_offsets, h.data(), (n + 1) * 8,
                              out_location == PO_LOC_HOST ? cudaMemcpyHostToHost
                                                          : cudaMemcpyHostToDevice, s));
      sync(s);
    }
    if (sc->total)
      PO_CUDA(cudaMemcpyAsync(out_order_fields, sc->fields.get(), sc->total * 4, k, s));
    sync(s);
  });
}

void po_schedule_free(po_schedule* sc) { delete sc; }

// Test hook: the K8 radix sort on host arrays (tests/test_gpu_radix.py).
int po_debug_radix_sort(const uint64_t* keys, const uint32_t* vals, uint64_t n, int32_t begin_bit,
                        int32_t end_bit, uint64_t* out_keys, uint32_t* out_vals) {
  return guarded([&] {
    if (n >= (uint64_t(1) << 32)) fail(PO_ERR_SIZE, "too many items");
    if (begin_bit < 0 || end_bit > 64 || begin_bit > end_bit) fail(PO_ERR_INVALID_ARG, "bad bit range");
    cudaStream_t s = nullptr;
    DevBuf<uint64_t> k(n, s), k2(n, s);
    DevBuf<uint32_t> v(n, s), v2(n, s);
    if (n) {
      PO_CUDA(cudaMemcpyAsync(k.get(), keys, n * 8, cudaMemcpyHostToDevice, s));
      PO_CUDA(cudaMemcpyAsync(v.get(), vals, n * 4, cudaMemcpyHostToDevice, s));
    }
    radix_sort_pairs(k.get(), k2.get(), v.get(), v2.get(), uint32_t(n), begin_bit, end_bit, s);
    if (n) {
      PO_CUDA(cudaMemcpyAsync(out_keys, k2.get(), n * 8, cudaMemcpyDeviceToHost, s));
      PO_CUDA(cudaMemcpyAsync(out_vals, v2.get(), n * 4, cudaMemcpyDeviceToHost, s));
    }
    sync(s);
  });
}

int po_debug_merge_sort(const uint64_t* a, const uint64_t* b, const uint32_t* vals, uint64_t n,
                        uint64_t* out_a, uint64_t* out_b, uint32_t* out_vals) {
  return guarded([&] {
    if (n >= (uint64_t(1) << 32)) fail(PO_ERR_SIZE, "too many items");
    if (n && (!a || !b || !vals || !out_a || !out_b || !out_vals)) fail(PO_ERR_INVALID_ARG, "null argument");
    debug_merge_sort(a, b, vals, uint32_t(n), out_a, out_b, out_vals, nullptr);
  });
}

int po_phc(const po_table* t, int32_t tok, int32_t scoring, uint64_t n_entries,
           const uint64_t* row_ids, const uint64_t* order_offsets, const int32_t* order_fields,
           uint32_t sched_location, uint64_t* out_phc, void* stream) {
  return guarded([&] {
    if (!out_phc) fail(PO_ERR_INVALID_ARG, "null output");
    *out_phc = phc_call(t, tok, scoring, n_entries, row_ids, order_offsets, order_fields,
                        sched_location, static_cast<cudaStream_t>(stream), 1, n_entries);
  });
}

int po_hit(const po_table* t, int32_t tok, int32_t scoring, uint64_t n_entries,
           const uint64_t* row_ids, const uint64_t* order_offsets, const int32_t* order_fields,
           uint32_t sched_location, uint64_t r, uint64_t* out_hit, void* stream) {
  return guarded([&] {
    if (!out_hit) fail(PO_ERR_INVALID_ARG, "null output");
    if (r >= n_entries)  // objective.hpp:73-75
      fail(PO_ERR_DOMAIN, "hit: request index " + std::to_string(r) +
                              " out of range for schedule of " + std::to_string(n_entries));
    *out_hit = r == 0 ? 0
                      : phc_call(t, tok, scoring, n_entries, row_ids, order_offsets, order_fields,
                                 sched_location, static_cast<cudaStream_t>(stream), r, r + 1);
  });
}

int po_sort_rows_fixed_order(const po_table* t, const int32_t* field_order, uint32_t out_location,
                             uint64_t* out_row_ids, void* stream) {
  return guarded([&] {
    if (!t) fail(PO_ERR_INVALID_ARG, "null table");
    const uint32_t m = t->n_fields;
    // validate_field_permutation (objective.hpp:140-149)
    std::vector<char> seen(m, 0);
    std::vector<int> order(m);
    for (uint32_t i = 0; i < m; ++i) {
      int f = field_order[i];
      if (f < 0 || uint32_t(f) >= m || seen[f])
        fail(PO_ERR_SCHEMA, "field order is not a permutation of the schema");
      seen[f] = 1;
      order[i] = f;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Prepared p;
    prepare(t, PO_TOK_CHAR, PO_SCORE_VALUE, s, p);
    const uint64_t n = p.e.n;
    DevBuf<uint32_t> perm(n, s);
    if (m == 0) {
      std::vector<uint32_t> id(n);
      std::iota(id.begin(), id.end(), 0u);
      perm.upload(id.data(), n);
    } else {
      sort_all_rows(p.e, order, perm.get(), s);
    }
    deliver_rows(perm.get(), n, out_location, out_row_ids, s);
    sync(s);
  });
}

int po_compute_stats(const po_table* t, int32_t tok, int32_t scoring, uint64_t* out_card,
                     uint64_t* out_total, void* stream) {
  return guarded([&] {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Prepared p;
    prepare(t, tok, scoring, s, p, /*ordered=*/false);  // cardinality + lengths only
    for (uint32_t f = 0; f < p.e.m; ++f) {
      out_card[f] = p.e.card[f];
      out_total[f] = p.e.total_len[f];
    }
  });
}

int po_fixed_order_by_hitcount_stats(uint32_t m, uint64_t total_rows, const uint64_t* card,
                                     const double* avg, int32_t variant, int32_t* out) {
  return guarded([&] {
    if (variant < 0 || variant > 2) fail(PO_ERR_INVALID_ARG, "unknown stats variant");
    std::vector<uint64_t> c(card, card + m);
    std::vector<double> a(avg, avg + m);
    std::vector<int> o = hitcount_order(total_rows, c, a, variant);
    std::copy(o.begin(), o.end(), out);
  });
}

int po_fixed_order_by_stats(uint32_t m, uint64_t total_rows, const uint64_t* card,
                            const double* avg, int32_t* out) {
  return guarded([&] {
    std::vector<uint64_t> c(card, card + m);
    std::vector<double> a(avg, avg + m);
    std::vector<int> o = stats_order(total_rows, c, a);
    std::copy(o.begin(), o.end(), out);
  });
}

int po_fd_compare(const po_table* t, uint32_t n_pairs, const int32_t* pair_a,
                  const int32_t* pair_b, uint64_t* out_first_diff, uint64_t* out_sig_a,
                  uint64_t* out_sig_b, void* stream) {
  return guarded([&] {
    if (n_pairs && (!pair_a || !pair_b || !out_first_diff))
      fail(PO_ERR_INVALID_ARG, "null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Prepared p;
    init_pool_once();
    make_device_table(t, PO_TOK_CHAR, s, p.t);
    encode(p.t, PO_TOK_CHAR, PO_SCORE_VALUE, s, p.e, debug_hash_bits(), /*ordered=*/false);
    std::vector<int32_t> pa(pair_a, pair_a + n_pairs), pb(pair_b, pair_b + n_pairs);
    std::vector<uint64_t> fd, sa, sb;
    fd_compare_device(p.e, pa, pb, fd, sa, sb, s);
    for (uint32_t k = 0; k < n_pairs; ++k) {
      out_first_diff[k] = fd[k];
      if (out_sig_a) out_sig_a[k] = sa[k];
      if (out_sig_b) out_sig_b[k] = sb[k];
    }
  });
}

int po_render_prompts(const po_table* t, uint64_t n_entries, const uint64_t* rows,
                      const uint64_t* offs, const int32_t* fields, uint32_t sched_loc,
                      const uint8_t* sp, uint64_t sp_len, const uint8_t* q, uint64_t q_len,
                      uint32_t out_loc, uint64_t* out_offsets, uint8_t* out_bytes,
                      uint64_t out_capacity, uint64_t* out_total, void* stream) {
  return guarded([&] {
    if (sched_loc != PO_LOC_HOST && sched_loc != PO_LOC_DEVICE)
      fail(PO_ERR_INVALID_ARG, "bad schedule location");
    if (out_loc != PO_LOC_HOST && out_loc != PO_LOC_DEVICE)
      fail(PO_ERR_INVALID_ARG, "bad output location");
    if (!out_offsets || !out_total || (n_entries && (!rows || !offs)))
      fail(PO_ERR_INVALID_ARG, "null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    init_pool_once();
    DeviceTable dt;
    make_device_table(t, PO_TOK_CHAR, s, dt);
    uint64_t nfields = 0;
    if (n_entries) {
      if (sched_loc == PO_LOC_HOST) nfields = offs[n_entries];
      else {
        PO_CUDA(cudaMemcpyAsync(&nfields, offs + n_entries, 8, cudaMemcpyDeviceToHost, s));
        sync(s);
      }
    }
    DevBuf<uint64_t> own_rows, own_offs;
    DevBuf<int32_t> own_fields;
    const uint64_t* d_rows = stage(rows, n_entries, sched_loc, own_rows, s);
    const uint64_t* d_offs = stage(offs, n_entries + 1, sched_loc, own_offs, s);
    const int32_t* d_fields = stage(fields, nfields, sched_loc, own_fields, s);
    DevBuf<uint64_t> o;
    DevBuf<uint8_t> b;
    uint64_t total = 0;
    // the bytes go straight into a device destination; a host destination
    // gets them through a device buffer
    auto dst_for = [&](uint64_t tot) -> uint8_t* {
      if (!out_bytes) return nullptr;
      if (out_capacity < tot) fail(PO_ERR_SIZE, "render: output buffer too small");
      if (out_loc == PO_LOC_DEVICE) return out_bytes;
      b.alloc(std::max<uint64_t>(tot, 1), s);
      return b.get();
    };
    render_prompts_device(dt, n_entries, d_rows, d_offs, d_fields, nfields,
                          std::string(reinterpret_cast<const char*>(sp), sp ? sp_len : 0),
                          std::string(reinterpret_cast<const char*>(q), q ? q_len : 0), o, total,
                          dst_for, s);
    const cudaMemcpyKind k = out_loc == PO_LOC_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    PO_CUDA(cudaMemcpyAsync(out_offsets, o.get(), (n_entries + 1) * 8, k, s));
    *out_total = total;
    if (out_bytes && out_loc == PO_LOC_HOST && total)
      PO_CUDA(cudaMemcpyAsync(out_bytes, b.get(), total, k, s));
    sync(s);
  });
}

int po_dedup(uint64_t n, const uint8_t* arena, const uint64_t* offsets, uint32_t loc,
             uint64_t* out_expansion, uint64_t* out_unique_first, uint64_t* out_n_unique,
             void* stream) {
  return guarded([&] {
    if (!out_expansion || !out_unique_first || !out_n_unique || (n && (!arena || !offsets)))
      fail(PO_ERR_INVALID_ARG, "null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    init_pool_once();
    const char* name = "prompt";
    const uint64_t name_len = 6;
    po_table tv{n, 1u, loc, &name, &name_len, arena, offsets, nullptr};
    DeviceTable dt;
    make_device_table(&tv, PO_TOK_CHAR, s, dt);
    DevBuf<uint64_t> ex(std::max<uint64_t>(n, 1), s), uf(std::max<uint64_t>(n, 1), s);
    uint64_t nu = 0;
    dedup_device(dt, ex.get(), uf.get(), nu, s);
    ex.download(out_expansion, n);
    uf.download(out_unique_first, nu);
    sync(s);
    *out_n_unique = nu;
  });
}

int po_replay_unbounded(uint64_t n, const uint8_t* arena, const uint64_t* offsets, uint32_t loc,
                        int32_t tok, uint64_t min_cacheable, uint64_t* out_input,
                        uint64_t* out_hit, uint64_t* out_miss, uint64_t* out_written,
                        uint64_t* out_totals, void* stream) {
  return guarded([&] {
    if (n == 0) fail(PO_ERR_DOMAIN, "simulate: prompt list is empty");
    if (tok != PO_TOK_CHAR && tok != PO_TOK_WORD)
      fail(PO_ERR_INVALID_ARG, "replay: char or word tokenizer");
    if (!arena || !offsets) fail(PO_ERR_INVALID_ARG, "null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    init_pool_once();
    const char* name = "prompt";
    const uint64_t name_len = 6;
    po_table tv{n, 1u, loc, &name, &name_len, arena, offsets, nullptr};
    DeviceTable dt;
    make_device_table(&tv, PO_TOK_CHAR, s, dt);
    DevBuf<uint64_t> in(n, s), raw(n, s), hit(n, s), miss(n, s);
    DevBuf<unsigned long long> tot(3, s);
    replay_unbounded_device(dt, tok, in.get(), raw.get(), s);
    // the report on the device (cache_sim.hpp:266-279): raw becomes written
    replay_report_device(in.get(), raw.get(), n, min_cacheable, hit.get(), miss.get(), tot.get(), s);
    if (out_input) in.download(out_input, n);
    if (out_hit) hit.download(out_hit, n);
    if (out_miss) miss.download(out_miss, n);
    if (out_written) raw.download(out_written, n);
    unsigned long long ht[3];
    d2h_sync(ht, tot.get(), sizeof(ht), s);
    if (out_totals) {
      out_totals[0] = ht[0];
      out_totals[1] = ht[1];
      out_totals[2] = ht[2];
    }
  });
}

int po_load_csv(const uint8_t* data, uint64_t len, uint32_t loc, po_csv** out, void* stream) {
  return guarded([&] {
    if (!out || (len && !data)) fail(PO_ERR_INVALID_ARG, "null argument");
    if (loc != PO_LOC_HOST && loc != PO_LOC_DEVICE) fail(PO_ERR_INVALID_ARG, "bad location");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    init_pool_once();
    DevBuf<uint8_t> own;
    const uint8_t* d = data;
    if (loc == PO_LOC_HOST && len) {
      own.alloc(len, s);
      own.upload(data, len);
      d = own.get();
    }
    auto c = std::make_unique<po_csv>();
    CsvParsed& P = c->parsed;
    load_csv_device(d, len, P, s);
    const uint64_t R = P.n_records;
    auto unterminated = [&](uint64_t r) {
      fail(PO_ERR_STRUCTURAL, "csv: unterminated quoted field starting near line " +
                                  std::to_string(P.start_line(r, s)));
    };
    auto wrong_width = [&](uint64_t r, uint64_t cells, uint64_t h) {
      fail(PO_ERR_STRUCTURAL, "csv: line " + std::to_string(P.start_line(r, s)) + " has " +
                                  std::to_string(cells) + " cells, expected " + std::to_string(h));
    };
    // load_csv's order of checks (table.hpp:190-214)
    if (R == 0) fail(PO_ERR_STRUCTURAL, "csv: missing header row");
    if (R == 1 && P.unterminated) unterminated(0);
    const uint64_t H = P.end_cell(0, s);
    std::vector<uint64_t> hend(H);
    P.cell_end.download(hend.data(), H);
    uint64_t hbytes = H ? hend[H - 1] : 0;
    std::string hb(hbytes, '\0');
    if (hbytes) PO_CUDA(cudaMemcpyAsync(hb.data(), P.arena.get(), hbytes, cudaMemcpyDeviceToHost, s));
    sync(s);
    std::vector<std::string> names;
    for (uint64_t i = 0; i < H; ++i) names.push_back(hb.substr(i ? hend[i - 1] : 0, hend[i] - (i ? hend[i - 1] : 0)));
    {
      std::unordered_set<std::string> seen;
      for (const auto& nm : names)
        if (!seen.insert(nm).second) fail(PO_ERR_SCHEMA, "csv: duplicate header field: " + nm);
    }
    uint64_t rows_end = R;  // records [1, rows_end) are data rows
    if (R >= 2) {
      // records before the last: widths checked on the device, the first
      // wrong one reported
      const uint64_t bad = P.first_wrong_width(H, s);
      if (bad < R - 1) {
        const uint64_t cells = P.end_cell(bad, s) - P.end_cell(bad - 1, s);
        wrong_width(bad, cells, H);
      }
      const uint64_t r = R - 1;  // the last record
      if (P.unterminated) unterminated(r);
      if (P.blank(r, s)) {  // trailing blank line
        rows_end = r;
      } else {
        const uint64_t cells = P.end_cell(r, s) - P.end_cell(r - 1, s);
        if (cells != H) wrong_width(r, cells, H);
      }
    }
    for (uint64_t i = 0; i < H; ++i)  // Table's constructor (table.hpp:28-33)
      if (names[i].empty())
        fail(PO_ERR_SCHEMA, "field " + std::to_string(i) + " has an empty name");
    if (H >= (uint64_t(1) << 31)) fail(PO_ERR_SIZE, "csv: too many fields");
    c->fields = uint32_t(H);
    c->rows = rows_end - 1;
    c->first_cell = H;
    c->base = hbytes;
    uint64_t data_end = hbytes;
    if (c->rows && H) {
      const uint64_t last_cell = H + c->rows * H - 1;
      PO_CUDA(cudaMemcpyAsync(&data_end, P.cell_end.get() + last_cell, 8, cudaMemcpyDeviceToHost, s));
      sync(s);
    }
    c->data_bytes = data_end - hbytes;
    c->name_off.assign(1, 0);
    for (const auto& nm : names) {
      c->names += nm;
      c->name_off.push_back(c->names.size());
    }
    *out = c.release();
  });
}

int po_csv_info(const po_csv* c, uint64_t* rows, uint32_t* fields, uint64_t* arena_bytes,
                uint64_t* names_bytes) {
  return guarded([&] {
    if (!c) fail(PO_ERR_INVALID_ARG, "null csv");
    if (rows) *rows = c->rows;
    if (fields) *fields = c->fields;
    if (arena_bytes) *arena_bytes = c->data_bytes;
    if (names_bytes) *names_bytes = c->names.size();
  });
}

int po_csv_copy(const po_csv* c, uint32_t loc, uint8_t* arena, uint64_t* offsets, uint8_t* names,
                uint64_t* name_offsets, void* stream) {
  return guarded([&] {
    if (!c) fail(PO_ERR_INVALID_ARG, "null csv");
    if (loc != PO_LOC_HOST && loc != PO_LOC_DEVICE) fail(PO_ERR_INVALID_ARG, "bad location");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const cudaMemcpyKind k = loc == PO_LOC_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    const uint64_t cells = c->rows * c->fields;
    if (arena && c->data_bytes)
      PO_CUDA(cudaMemcpyAsync(arena, c->parsed.arena.get() + c->base, c->data_bytes, k, s));
    if (offsets) {
      DevBuf<uint64_t> tmp;
      uint64_t* dst = offsets;
      if (loc == PO_LOC_HOST) {
        tmp.alloc(cells + 1, s);
        dst = tmp.get();
      }
      PO_LAUNCH(k_csv_offsets, grid_for(cells + 1, 256), 256, 0, s, c->parsed.cell_end.get(),
                c->first_cell, cells, c->base, dst);
      if (loc == PO_LOC_HOST) tmp.download(offsets, cells + 1);
    }
    if (names && !c->names.empty()) std::memcpy(names, c->names.data(), c->names.size());
    if (name_offsets)
      std::memcpy(name_offsets, c->name_off.data(), c->name_off.size() * sizeof(uint64_t));
    sync(s);
  });
}

void po_csv_free(po_csv* c) { delete c; }

int po_comm_unique_id(uint8_t* out_id128) {
  return guarded([&] {
    if (!out_id128) fail(PO_ERR_INVALID_ARG, "null id buffer");
    nccl_unique_id(out_id128);
  });
}

int po_comm_init_nccl(const uint8_t* id128, int32_t nranks, int32_t rank, po_comm** out) {
  return guarded([&] {
    if (!id128 || !out) fail(PO_ERR_INVALID_ARG, "null argument");
    auto h = std::make_unique<po_comm>();
    h->c.reset(make_nccl_comm(id128, nranks, rank));
    *out = h.release();
  });
}

int po_comm_init_local(int32_t nranks, po_comm** out_array) {
  return guarded([&] {
    if (!out_array) fail(PO_ERR_INVALID_ARG, "null output array");
    std::vector<Comm*> cs = make_local_group(nranks);
    for (int32_t r = 0; r < nranks; ++r) {
      out_array[r] = new po_comm;
      out_array[r]->c.reset(cs[r]);
    }
  });
}

int po_comm_init_host(const po_host_collectives* ops, int32_t nranks, int32_t rank, po_comm** out) {
  return guarded([&] {
    if (!ops || !out) fail(PO_ERR_INVALID_ARG, "null argument");
    auto h = std::make_unique<po_comm>();
    h->c.reset(make_host_comm(*ops, nranks, rank));
    *out = h.release();
  });
}

int po_comm_destroy(po_comm* comm) {
  return guarded([&] { delete comm; });
}

int po_ggr_sharded(po_comm* comm, const po_table* t, const po_fd_groups* fds,
                   const po_ggr_config* cfg, int32_t tok, int32_t scoring, po_slice** out_slice,
                   uint64_t* out_phc, po_solve_stats* out_stats, void* stream) {
  return guarded([&] {
    auto t0 = std::chrono::steady_clock::now();
    if (!comm || !cfg || !out_slice || !out_phc) fail(PO_ERR_INVALID_ARG, "null argument");
    if (cfg->stats_variant < 0 || cfg->stats_variant > 2)
      fail(PO_ERR_INVALID_ARG, "unknown stats variant");
    check_modes(tok, scoring);
    init_pool_once();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    timing_mark("<start", s);
    std::vector<std::vector<int>> groups;
    if (fds && cfg->use_fds)
      for (uint32_t g = 0; g < fds->n_groups; ++g)
        groups.emplace_back(fds->members + fds->group_offsets[g],
                            fds->members + fds->group_offsets[g + 1]);
    DeviceTable dt;
    make_device_table(t, tok, s, dt);
    DistCtx dc;
    GgrOutput go;
    ggr_sharded(*comm->c, dt, tok, scoring, groups, *cfg, dc, go, s);
    auto sl = std::make_unique<po_slice>();
    sl->offset = dc.slice_offset;
    sl->count = dc.slice_count;
    sl->m = dt.m;
    PO_CUDA(cudaGetDevice(&sl->device));
    sl->rows = std::move(dc.rows);
    sl->orders = std::move(dc.orders);
    sync(s);
    timing_report("po_ggr_sharded");
    *out_phc = go.phc;
    if (out_stats) {
      *out_stats = go.stats;
      out_stats->wall_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    *out_slice = sl.release();
  });
}

int po_slice_info(const po_slice* slice, uint64_t* out_offset, uint64_t* out_count) {
  return guarded([&] {
    if (!slice) fail(PO_ERR_INVALID_ARG, "null slice");
    if (out_offset) *out_offset = slice->offset;
    if (out_count) *out_count = slice->count;
  });
}

int po_slice_copy(const po_slice* slice, uint32_t loc, uint64_t* out_rows, int32_t* out_orders,
                  void* stream) {
  return guarded([&] {
    if (!slice) fail(PO_ERR_INVALID_ARG, "null slice");
    if (loc != PO_LOC_HOST && loc != PO_LOC_DEVICE) fail(PO_ERR_INVALID_ARG, "bad location");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const cudaMemcpyKind k = loc == PO_LOC_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (slice->count && out_rows)
      PO_CUDA(cudaMemcpyAsync(out_rows, slice->rows.get(), slice->count * 8, k, s));
    if (slice->count && slice->m && out_orders)
      PO_CUDA(cudaMemcpyAsync(out_orders, slice->orders.get() + slice->m,
                              slice->count * slice->m * sizeof(int32_t), k, s));
    sync(s);
  });
}

void po_slice_free(po_slice* slice) { delete slice; }

const char* po_last_error(void) { return g_err.c_str(); }

}  // extern "C"

namespace po {
// for entry points defined in other translation units (jsonl.cpp)
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace po

extern "C" {

const char* po_build_info(void) { return "prefixopt-b200 sm_100a"; }

uint64_t po_trim_device_cache(void) { return po::trim_cached_blocks(); }

uint64_t po_kernel_launch_count(void) { return g_launches.load(); }

void po_profile_enable(int enable) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!enable) {
    try {
      prof_drain();
    } catch (...) {
    }
  }
  g_profile.store(enable ? 1 : 0);
}

uint64_t po_profile_report(char* buf, uint64_t cap) {
  std::string out;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    try {
      prof_drain();
    } catch (...) {
    }
    for (auto& [name, v] : g_prof_acc)
      out += name + " " + std::to_string(v.first) + " " + std::to_string(v.second) + "\n";
    g_prof_acc.clear();
  }
  if (buf && cap) {
    size_t k = std::min<size_t>(cap - 1, out.size());
    std::memcpy(buf, out.data(), k);
    buf[k] = 0;
  }
  return out.size() + 1;
}

}  // extern "C"
