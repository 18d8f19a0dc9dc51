// Collectives of the row-sharded solver.
//
// One rank per GPU. Three transports behind one interface:
//   * NcclComm  — production: NCCL over NVLink/NVSwitch, one process per GPU
//                 (libnccl.so.2 is opened lazily, so single-GPU users of the
//                 library never need it);
//   * HostComm  — caller-provided collectives on host buffers (MPI, gloo):
//                 device buffers staged through host memory; any process
//                 layout, several ranks per GPU included (tests);
//   * LocalComm — N ranks as host threads of ONE process (any devices,
//                 including N ranks on one GPU): collectives are peer
//                 cudaMemcpyAsync between the ranks' buffers behind a host
//                 barrier. This is what lets the sharded path be checked
//                 bit-exactly against the single-GPU solver on a 1-GPU box.
// Every collective is called by all ranks in the same order and returns with
// the result complete on the caller's stream.
#pragma once

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace po {

enum class CDtype { U32, U64 };
enum class COp { Sum, Max };

class Comm {
 public:
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int size() const { return size_; }

  // In-place element-wise reduction of n elements on the device.
  virtual void allreduce(void* d, size_t n, CDtype t, COp op, cudaStream_t s) = 0;
  // recv[r*bytes .. (r+1)*bytes) = rank r's send (device buffers).
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  // Variable-size allgather: rank r contributes recv_bytes[r] bytes; they are
  // laid out back to back in rank order.
  virtual void allgatherv(const void* send, void* recv, const std::vector<uint64_t>& recv_bytes,
                          cudaStream_t s) = 0;
  // send_bytes[r] bytes go to rank r (contiguous in rank order in `send`);
  // recv_bytes[r] bytes arrive from rank r (contiguous in rank order).
  virtual void alltoallv(const void* send, const std::vector<uint64_t>& send_bytes, void* recv,
                         const std::vector<uint64_t>& recv_bytes, cudaStream_t s) = 0;

  // ---- host helpers built on the device collectives (small vectors) ----
  // every rank's vector (same length k on all ranks), concatenated
  std::vector<uint64_t> allgather_host(const std::vector<uint64_t>& mine, cudaStream_t s);
  // recv[r] = what rank r sends to me (send[r] = what I send to rank r)
  std::vector<uint64_t> exchange_counts(const std::vector<uint64_t>& send, cudaStream_t s);
  std::vector<uint64_t> allreduce_host(const std::vector<uint64_t>& v, COp op, cudaStream_t s);

 protected:
  int rank_ = 0, size_ = 1;
};

// 128-byte NCCL unique id (ncclGetUniqueId) for rank 0 to broadcast.
void nccl_unique_id(uint8_t out[128]);
Comm* make_nccl_comm(const uint8_t id[128], int nranks, int rank);
// nranks communicators sharing one in-process group (rank i = out[i]).
std::vector<Comm*> make_local_group(int nranks);
// host-staged collectives provided by the caller (po_host_collectives)
Comm* make_host_comm(const po_host_collectives& ops, int nranks, int rank);

}  // namespace po
