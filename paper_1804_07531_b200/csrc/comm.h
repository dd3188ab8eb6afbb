// Collectives of the row-sharded path, behind one interface with two back ends:
//
//   NcclComm  one process (or thread) per GPU, NCCL loaded at run time (libnccl.so.2); calls are
//             captured in the algorithm's CUDA graph; completion is awaited by polling the stream
//             and ncclCommGetAsyncError with a timeout (a dead peer aborts the communicator
//             instead of hanging the call).
//   LoopComm  N virtual row shards of one A on ONE GPU (rsvd_loop_create / rsvd_comm_init_loopback):
//             every virtual rank is a ctx driven by its own host thread on its own stream; a
//             collective is a host barrier, cross-stream event waits and an ordered local sum
//             (ranks 0..N-1, the same order on every rank, so results are bitwise identical on
//             all ranks).  No kernel ever waits on another kernel: only streams wait on events.
//             Not graph-capturable (host barriers), so loopback calls enqueue directly.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace rsvd {

struct Comm {
  int nranks = 1, rank = 0;
  virtual ~Comm() {}
  // in place: p[0..count) <- sum over ranks
  virtual int allreduce(double* p, size_t count, cudaStream_t st, std::string* err) = 0;
  // recv[0..count) <- sum over ranks of send[rank*count .. (rank+1)*count); send != recv
  virtual int reduce_scatter(const double* send, double* recv, size_t count, cudaStream_t st, std::string* err) = 0;
  // recv[q*count .. (q+1)*count) <- rank q's send[0..count); send must not overlap recv
  virtual int allgather(const double* send, double* recv, size_t count, cudaStream_t st, std::string* err) = 0;
  virtual bool graph_ok() const = 0;
  // wait for the stream's work; polls the communicator's error state (timeout in seconds)
  virtual int wait(cudaStream_t st, double timeout_s, std::string* err) = 0;
  // a rank's call failed: release peers blocked in a collective of this group
  virtual void abort() {}
};

// NCCL back end (dlopen).  Returns nullptr with *err set on failure.
bool nccl_available();
int nccl_unique_id(void* id128);
Comm* nccl_comm_create(int nranks, int rank, const void* id128, std::string* err);

// loopback back end
struct LoopGroup;
LoopGroup* loop_group_create(int nranks, double timeout_s);
void loop_group_release(LoopGroup* g);   // refcounted: the creator and every LoopComm hold one
Comm* loop_comm_create(LoopGroup* g, int rank, int device, std::string* err);

}  // namespace rsvd
