// Transports for the row-sharded solver: NCCL (one process per GPU) and an
// in-process thread group (see comm.cuh).

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <memory>
#include <mutex>

#include "comm.cuh"

namespace po {

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
std::vector<uint64_t> Comm::allgather_host(const std::vector<uint64_t>& mine, cudaStream_t s) {
  const size_t k = mine.size();
  std::vector<uint64_t> all(k * size_);
  if (k == 0) return all;
  DevBuf<uint64_t> d_send(k, s), d_recv(k * size_, s);
  d_send.upload(mine.data(), k);
  allgather(d_send.get(), d_recv.get(), k * 8, s);
  d_recv.download(all.data(), k * size_);
  sync(s);
  return all;
}

std::vector<uint64_t> Comm::exchange_counts(const std::vector<uint64_t>& send, cudaStream_t s) {
  const std::vector<uint64_t> all = allgather_host(send, s);  // [src][dst]
  std::vector<uint64_t> recv(size_);
  for (int r = 0; r < size_; ++r) recv[r] = all[size_t(r) * size_ + rank_];
  return recv;
}

std::vector<uint64_t> Comm::allreduce_host(const std::vector<uint64_t>& v, COp op, cudaStream_t s) {
  std::vector<uint64_t> out(v);
  if (v.empty()) return out;
  DevBuf<uint64_t> d(v.size(), s);
  d.upload(v.data(), v.size());
  allreduce(d.get(), v.size(), CDtype::U64, op, s);
  d.download(out.data(), v.size());
  sync(s);
  return out;
}

namespace {

// ---------------------------------------------------------------------------
// NCCL (dlopen'd: the library has no link-time dependency on it)
// ---------------------------------------------------------------------------
struct NcclApi {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    // prefer the NCCL already loaded into the process (torch's), then the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = dlerror() ? dlerror() : "libnccl.so.2 not found";
      return;
    }
#define PO_SYM(f, name) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, name))
    PO_SYM(getUniqueId, "ncclGetUniqueId");
    PO_SYM(commInitRank, "ncclCommInitRank");
    PO_SYM(commDestroy, "ncclCommDestroy");
    PO_SYM(allReduce, "ncclAllReduce");
    PO_SYM(allGather, "ncclAllGather");
    PO_SYM(send, "ncclSend");
    PO_SYM(recv, "ncclRecv");
    PO_SYM(groupStart, "ncclGroupStart");
    PO_SYM(groupEnd, "ncclGroupEnd");
    PO_SYM(errStr, "ncclGetErrorString");
#undef PO_SYM
  });
  if (!api.commInitRank || !api.allReduce || !api.send)
    fail(PO_ERR_ERROR, "NCCL unavailable: " + (err.empty() ? std::string("missing symbols") : err));
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(PO_ERR_ERROR, std::string("NCCL error in ") + what + ": " +
                           (nccl().errStr ? nccl().errStr(r) : "?"));
}

class NcclComm final : public Comm {
 public:
  NcclComm(const uint8_t id[128], int nranks, int rank) {
    rank_ = rank;
    size_ = nranks;
    ncclUniqueId uid;
    static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(&uid, id, 128);
    nccl_check(nccl().commInitRank(&c_, nranks, uid, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (c_) nccl().commDestroy(c_);
  }
  void allreduce(void* d, size_t n, CDtype t, COp op, cudaStream_t s) override {
    if (!n || size_ == 1) return;
    nccl_check(nccl().allReduce(d, d, n, t == CDtype::U32 ? ncclUint32 : ncclUint64,
                                op == COp::Sum ? ncclSum : ncclMax, c_, s),
               "ncclAllReduce");
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    if (!bytes) return;
    nccl_check(nccl().allGather(send, recv, bytes, ncclUint8, c_, s), "ncclAllGather");
  }
  void allgatherv(const void* send, void* recv, const std::vector<uint64_t>& rb,
                  cudaStream_t s) override {
    nccl_check(nccl().groupStart(), "ncclGroupStart");
    uint64_t off = 0;
    for (int r = 0; r < size_; ++r) {
      if (rb[rank_]) nccl_check(nccl().send(send, rb[rank_], ncclUint8, r, c_, s), "ncclSend");
      if (rb[r])
        nccl_check(nccl().recv(static_cast<uint8_t*>(recv) + off, rb[r], ncclUint8, r, c_, s),
                   "ncclRecv");
      off += rb[r];
    }
    nccl_check(nccl().groupEnd(), "ncclGroupEnd");
  }
  void alltoallv(const void* send, const std::vector<uint64_t>& sb, void* recv,
                 const std::vector<uint64_t>& rb, cudaStream_t s) override {
    nccl_check(nccl().groupStart(), "ncclGroupStart");
    uint64_t so = 0, ro = 0;
    for (int r = 0; r < size_; ++r) {
      if (sb[r])
        nccl_check(nccl().send(static_cast<const uint8_t*>(send) + so, sb[r], ncclUint8, r, c_, s),
                   "ncclSend");
      if (rb[r])
        nccl_check(nccl().recv(static_cast<uint8_t*>(recv) + ro, rb[r], ncclUint8, r, c_, s),
                   "ncclRecv");
      so += sb[r];
      ro += rb[r];
    }
    nccl_check(nccl().groupEnd(), "ncclGroupEnd");
  }

 private:
  ncclComm_t c_ = nullptr;
};

// ---------------------------------------------------------------------------
// in-process thread group
// ---------------------------------------------------------------------------
struct LocalGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;
  std::vector<std::vector<uint64_t>> counts;  // [src] -> per-destination bytes
  int refs = 0;

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

template <class T>
__global__ void k_reduce_ranks(const T* all, size_t n, int nr, int is_max, T* out) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    T a = all[i];
    for (int r = 1; r < nr; ++r) {
      const T b = all[size_t(r) * n + i];
      a = is_max ? (b > a ? b : a) : T(a + b);
    }
    out[i] = a;
  }
}

class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalGroup> g, int rank) : g_(std::move(g)) {
    rank_ = rank;
    size_ = g_->n;
  }
  void allreduce(void* d, size_t n, CDtype t, COp op, cudaStream_t s) override {
    if (!n || size_ == 1) return;
    const size_t es = t == CDtype::U32 ? 4 : 8;
    DevBuf<uint8_t> all(n * es * size_, s);
    publish(d, {}, s);
    for (int r = 0; r < size_; ++r)
      PO_CUDA(cudaMemcpyAsync(all.get() + size_t(r) * n * es, g_->ptr[r], n * es,
                              cudaMemcpyDefault, s));
    sync(s);
    g_->barrier();  // every rank holds its copies: buffers may change now
    if (t == CDtype::U32)
      PO_LAUNCH(k_reduce_ranks<uint32_t>, grid_for(n, 256), 256, 0, s,
                reinterpret_cast<const uint32_t*>(all.get()), n, size_, op == COp::Max ? 1 : 0,
                static_cast<uint32_t*>(d));
    else
      PO_LAUNCH(k_reduce_ranks<unsigned long long>, grid_for(n, 256), 256, 0, s,
                reinterpret_cast<const unsigned long long*>(all.get()), n, size_,
                op == COp::Max ? 1 : 0, static_cast<unsigned long long*>(d));
    sync(s);
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    if (!bytes) return;
    publish(send, {}, s);
    for (int r = 0; r < size_; ++r)
      PO_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv) + size_t(r) * bytes, g_->ptr[r], bytes,
                              cudaMemcpyDefault, s));
    finish(s);
  }
  void allgatherv(const void* send, void* recv, const std::vector<uint64_t>& rb,
                  cudaStream_t s) override {
    publish(send, {}, s);
    uint64_t off = 0;
    for (int r = 0; r < size_; ++r) {
      if (rb[r])
        PO_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv) + off, g_->ptr[r], rb[r],
                                cudaMemcpyDefault, s));
      off += rb[r];
    }
    finish(s);
  }
  void alltoallv(const void* send, const std::vector<uint64_t>& sb, void* recv,
                 const std::vector<uint64_t>& rb, cudaStream_t s) override {
    publish(send, sb, s);
    uint64_t ro = 0;
    for (int r = 0; r < size_; ++r) {
      const std::vector<uint64_t>& c = g_->counts[r];
      uint64_t so = 0;
      for (int q = 0; q < rank_; ++q) so += c[q];
      if (c[rank_] != rb[r]) fail(PO_ERR_ERROR, "local alltoallv: size mismatch");
      if (rb[r])
        PO_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv) + ro,
                                static_cast<const uint8_t*>(g_->ptr[r]) + so, rb[r],
                                cudaMemcpyDefault, s));
      ro += rb[r];
    }
    finish(s);
  }

 private:
  // send buffers complete, then visible to every rank
  void publish(const void* p, const std::vector<uint64_t>& counts, cudaStream_t s) {
    sync(s);
    {
      std::lock_guard<std::mutex> lk(g_->mu);
      g_->ptr[rank_] = p;
      g_->counts[rank_] = counts;
    }
    g_->barrier();
  }
  void finish(cudaStream_t s) {
    sync(s);
    g_->barrier();  // nobody reuses a send buffer before every reader is done
  }
  std::shared_ptr<LocalGroup> g_;
};

// ---------------------------------------------------------------------------
// host-staged transport over caller-provided host collectives
// ---------------------------------------------------------------------------
class HostComm final : public Comm {
 public:
  HostComm(const po_host_collectives& ops, int nranks, int rank) : ops_(ops) {
    rank_ = rank;
    size_ = nranks;
  }
  void allreduce(void* d, size_t n, CDtype t, COp op, cudaStream_t s) override {
    if (!n || size_ == 1) return;
    const size_t es = t == CDtype::U32 ? 4 : 8;
    std::vector<uint8_t> mine(n * es), all(n * es * size_);
    down(d, mine.data(), n * es, s);
    call(ops_.allgather(ops_.ctx, mine.data(), all.data(), n * es), "allgather");
    DevBuf<uint8_t> d_all(all.size(), s);
    d_all.upload(all.data(), all.size());
    if (t == CDtype::U32)
      PO_LAUNCH(k_reduce_ranks<uint32_t>, grid_for(n, 256), 256, 0, s,
                reinterpret_cast<const uint32_t*>(d_all.get()), n, size_, op == COp::Max ? 1 : 0,
                static_cast<uint32_t*>(d));
    else
      PO_LAUNCH(k_reduce_ranks<unsigned long long>, grid_for(n, 256), 256, 0, s,
                reinterpret_cast<const unsigned long long*>(d_all.get()), n, size_,
                op == COp::Max ? 1 : 0, static_cast<unsigned long long*>(d));
    sync(s);
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    if (!bytes) return;
    std::vector<uint8_t> mine(bytes), all(bytes * size_);
    down(send, mine.data(), bytes, s);
    call(ops_.allgather(ops_.ctx, mine.data(), all.data(), bytes), "allgather");
    up(all.data(), recv, all.size(), s);
  }
  void allgatherv(const void* send, void* recv, const std::vector<uint64_t>& rb,
                  cudaStream_t s) override {
    uint64_t tot = 0;
    for (uint64_t b : rb) tot += b;
    std::vector<uint8_t> mine(rb[rank_] ? rb[rank_] : 1), all(tot ? tot : 1);
    down(send, mine.data(), rb[rank_], s);
    call(ops_.allgatherv(ops_.ctx, mine.data(), all.data(), rb.data()), "allgatherv");
    up(all.data(), recv, tot, s);
  }
  void alltoallv(const void* send, const std::vector<uint64_t>& sb, void* recv,
                 const std::vector<uint64_t>& rb, cudaStream_t s) override {
    uint64_t st = 0, rt = 0;
    for (int r = 0; r < size_; ++r) {
      st += sb[r];
      rt += rb[r];
    }
    std::vector<uint8_t> hs(st ? st : 1), hr(rt ? rt : 1);
    down(send, hs.data(), st, s);
    call(ops_.alltoallv(ops_.ctx, hs.data(), sb.data(), hr.data(), rb.data()), "alltoallv");
    up(hr.data(), recv, rt, s);
  }

 private:
  static void call(int rc, const char* what) {
    if (rc != 0) fail(PO_ERR_ERROR, std::string("host collective ") + what + " failed");
  }
  static void down(const void* d, void* h, size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    PO_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
    sync(s);
  }
  static void up(const void* h, void* d, size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    PO_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
    sync(s);  // the host staging buffer is freed on return
  }
  po_host_collectives ops_;
};

}  // namespace

Comm* make_host_comm(const po_host_collectives& ops, int nranks, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(PO_ERR_INVALID_ARG, "bad rank/world size");
  if (!ops.allgather || !ops.allgatherv || !ops.alltoallv)
    fail(PO_ERR_INVALID_ARG, "null host collective");
  return new HostComm(ops, nranks, rank);
}

void nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId uid;
  nccl_check(nccl().getUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out, &uid, 128);
}

Comm* make_nccl_comm(const uint8_t id[128], int nranks, int rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(PO_ERR_INVALID_ARG, "bad rank/world size");
  return new NcclComm(id, nranks, rank);
}

std::vector<Comm*> make_local_group(int nranks) {
  if (nranks < 1) fail(PO_ERR_INVALID_ARG, "bad world size");
  auto g = std::make_shared<LocalGroup>();
  g->n = nranks;
  g->ptr.assign(nranks, nullptr);
  g->counts.assign(nranks, {});
  std::vector<Comm*> out;
  for (int r = 0; r < nranks; ++r) out.push_back(new LocalComm(g, r));
  return out;
}

}  // namespace po
