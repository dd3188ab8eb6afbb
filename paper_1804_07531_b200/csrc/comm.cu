// Collectives of the row-sharded path: NCCL (dlopen) and the single-GPU loopback (comm.h).
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "comm.h"
#include "../../include/rsvd.h"

namespace rsvd {

// ================================================================ NCCL
namespace {
typedef int nccl_res_t;
typedef void* nccl_comm_t;
struct nccl_uid_t { char internal[128]; };
constexpr int kNcclFloat64 = 8, kNcclSum = 0, kNcclInProgress = 7;

struct NcclApi {
  void* h = nullptr;
  nccl_res_t (*get_uid)(nccl_uid_t*) = nullptr;
  nccl_res_t (*init_rank)(nccl_comm_t*, int, nccl_uid_t, int) = nullptr;
  nccl_res_t (*allreduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  nccl_res_t (*reduce_scatter)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  nccl_res_t (*allgather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
  nccl_res_t (*destroy)(nccl_comm_t) = nullptr;
  nccl_res_t (*abort)(nccl_comm_t) = nullptr;
  nccl_res_t (*async_error)(nccl_comm_t, nccl_res_t*) = nullptr;
  const char* (*errstr)(nccl_res_t) = nullptr;
  std::mutex mu;
  bool load() {
    std::lock_guard<std::mutex> lk(mu);
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    get_uid = (decltype(get_uid))dlsym(h, "ncclGetUniqueId");
    init_rank = (decltype(init_rank))dlsym(h, "ncclCommInitRank");
    allreduce = (decltype(allreduce))dlsym(h, "ncclAllReduce");
    reduce_scatter = (decltype(reduce_scatter))dlsym(h, "ncclReduceScatter");
    allgather = (decltype(allgather))dlsym(h, "ncclAllGather");
    destroy = (decltype(destroy))dlsym(h, "ncclCommDestroy");
    abort = (decltype(abort))dlsym(h, "ncclCommAbort");
    async_error = (decltype(async_error))dlsym(h, "ncclCommGetAsyncError");
    errstr = (decltype(errstr))dlsym(h, "ncclGetErrorString");
    return get_uid && init_rank && allreduce && reduce_scatter && allgather && destroy && abort && async_error;
  }
  std::string msg(nccl_res_t r) const { return errstr ? errstr(r) : std::to_string(r); }
};
NcclApi g_nccl;

struct NcclComm : Comm {
  nccl_comm_t c = nullptr;
  bool aborted = false;
  ~NcclComm() override {
    if (c && !aborted) g_nccl.destroy(c);
  }
  int fail(nccl_res_t r, const char* what, std::string* err) {
    if (err) *err = std::string(what) + " failed: " + g_nccl.msg(r);
    return RSVD_E_NCCL;
  }
  int allreduce(double* p, size_t count, cudaStream_t st, std::string* err) override {
    nccl_res_t r = g_nccl.allreduce(p, p, count, kNcclFloat64, kNcclSum, c, st);
    return r ? fail(r, "ncclAllReduce", err) : RSVD_OK;
  }
  int reduce_scatter(const double* s, double* d, size_t count, cudaStream_t st, std::string* err) override {
    nccl_res_t r = g_nccl.reduce_scatter(s, d, count, kNcclFloat64, kNcclSum, c, st);
    return r ? fail(r, "ncclReduceScatter", err) : RSVD_OK;
  }
  int allgather(const double* s, double* d, size_t count, cudaStream_t st, std::string* err) override {
    nccl_res_t r = g_nccl.allgather(s, d, count, kNcclFloat64, c, st);
    return r ? fail(r, "ncclAllGather", err) : RSVD_OK;
  }
  bool graph_ok() const override { return true; }
  int wait(cudaStream_t st, double timeout_s, std::string* err) override {
    // poll instead of blocking in cudaStreamSynchronize: a peer that died mid-collective leaves
    // this rank's kernel spinning forever; the async error (or the timeout) aborts the comm
    const auto t0 = std::chrono::steady_clock::now();
    int sleep_us = 5;
    for (;;) {
      cudaError_t q = cudaStreamQuery(st);
      if (q == cudaSuccess) return RSVD_OK;
      if (q != cudaErrorNotReady) {
        if (err) *err = std::string("CUDA error: ") + cudaGetErrorString(q);
        return RSVD_E_CUDA;
      }
      nccl_res_t ae = 0;
      if (g_nccl.async_error(c, &ae) == 0 && ae != 0 && ae != kNcclInProgress) {
        g_nccl.abort(c);
        aborted = true;
        if (err) *err = "NCCL asynchronous error: " + g_nccl.msg(ae);
        return RSVD_E_NCCL;
      }
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (timeout_s > 0 && el > timeout_s) {
        g_nccl.abort(c);
        aborted = true;
        char b[160];
        snprintf(b, sizeof b, "collective call did not complete within %.0f s (RSVD_COMM_TIMEOUT_S); "
                              "communicator aborted", timeout_s);
        if (err) *err = b;
        return RSVD_E_NCCL;
      }
      std::this_thread::sleep_for(std::chrono::microseconds(sleep_us));
      sleep_us = std::min(sleep_us * 2, 2000);
    }
  }
  void abort() override {
    if (c && !aborted) {
      g_nccl.abort(c);
      aborted = true;
    }
  }
};
}  // namespace

bool nccl_available() { return g_nccl.load(); }

int nccl_unique_id(void* id128) {
  if (!g_nccl.load()) return RSVD_E_NCCL;
  nccl_uid_t uid;
  if (g_nccl.get_uid(&uid) != 0) return RSVD_E_NCCL;
  memcpy(id128, &uid, 128);
  return RSVD_OK;
}

Comm* nccl_comm_create(int nranks, int rank, const void* id128, std::string* err) {
  if (!g_nccl.load()) {
    if (err) *err = "libnccl.so.2 not loadable (or lacks ncclCommGetAsyncError / ncclReduceScatter)";
    return nullptr;
  }
  nccl_uid_t uid;
  memcpy(&uid, id128, 128);
  nccl_comm_t c = nullptr;
  nccl_res_t r = g_nccl.init_rank(&c, nranks, uid, rank);
  if (r != 0) {
    if (err) *err = "ncclCommInitRank failed: " + g_nccl.msg(r);
    return nullptr;
  }
  NcclComm* nc = new NcclComm();
  nc->c = c;
  nc->nranks = nranks;
  nc->rank = rank;
  return nc;
}

// ================================================================ loopback (N virtual shards, one GPU)
constexpr int kLoopMaxRanks = 16;

struct LoopPtrs {
  const double* p[kLoopMaxRanks];
};

// out[i] = sum_{q < n} src_q[off + i], accumulated in rank order q = 0, 1, ..., n-1
__global__ void k_loop_sum(LoopPtrs src, int n, size_t off, size_t count, double* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double s = src.p[0][off + i];
    for (int q = 1; q < n; ++q) s += src.p[q][off + i];
    out[i] = s;
  }
}

static int loop_sum(const LoopPtrs& src, int n, size_t off, size_t count, double* out, cudaStream_t st) {
  if (count == 0) return RSVD_OK;
  const int threads = 256;
  const int blocks = (int)std::min<size_t>((count + threads - 1) / threads, 148 * 8);
  k_loop_sum<<<blocks, threads, 0, st>>>(src, n, off, count, out);
  return cudaGetLastError() == cudaSuccess ? RSVD_OK : RSVD_E_CUDA;
}

struct LoopGroup {
  int n = 0;
  double timeout_s = 120.0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  bool aborted = false;
  std::atomic<int> refs{1};
  const double* ptr[kLoopMaxRanks] = {};
  cudaEvent_t ev_in[kLoopMaxRanks] = {};
  cudaEvent_t ev_done[kLoopMaxRanks] = {};

  // generation barrier with timeout; RSVD_E_NCCL when a peer aborted or never arrived
  int barrier(std::string* err) {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) {
      if (err) *err = "loopback group aborted by a failing rank";
      return RSVD_E_NCCL;
    }
    const long gen = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return RSVD_OK;
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                [&] { return generation != gen || aborted; });
    if (!ok || aborted) {
      aborted = true;
      cv.notify_all();
      if (err) *err = ok ? "loopback group aborted by a failing rank"
                         : "loopback collective: a peer rank did not arrive within the timeout";
      return RSVD_E_NCCL;
    }
    return RSVD_OK;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

LoopGroup* loop_group_create(int nranks, double timeout_s) {
  if (nranks < 1 || nranks > kLoopMaxRanks) return nullptr;
  LoopGroup* g = new LoopGroup();
  g->n = nranks;
  if (timeout_s > 0) g->timeout_s = timeout_s;
  for (int q = 0; q < nranks; ++q) {
    if (cudaEventCreateWithFlags(&g->ev_in[q], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_done[q], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      delete g;
      return nullptr;
    }
  }
  return g;
}

void loop_group_release(LoopGroup* g) {
  if (!g) return;
  if (--g->refs == 0) {
    for (int q = 0; q < g->n; ++q) {
      if (g->ev_in[q]) cudaEventDestroy(g->ev_in[q]);
      if (g->ev_done[q]) cudaEventDestroy(g->ev_done[q]);
    }
    delete g;
  }
}

namespace {
struct LoopComm : Comm {
  LoopGroup* g = nullptr;
  double* scratch = nullptr;
  size_t scratch_n = 0;
  ~LoopComm() override {
    if (scratch) cudaFree(scratch);
    loop_group_release(g);
  }
  bool graph_ok() const override { return false; }
  void abort() override { g->abort(); }
  int wait(cudaStream_t st, double, std::string* err) override {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      if (err) *err = std::string("CUDA error: ") + cudaGetErrorString(e);
      return RSVD_E_CUDA;
    }
    return RSVD_OK;
  }
  int ensure_scratch(size_t count, std::string* err) {
    if (count <= scratch_n) return RSVD_OK;
    if (scratch) cudaFree(scratch);   // synchronous: no work of this rank still uses it
    scratch = nullptr;
    scratch_n = 0;
    if (cudaMalloc(&scratch, std::max<size_t>(count, 1) * 8) != cudaSuccess) {
      cudaGetLastError();
      if (err) *err = "loopback scratch allocation failed";
      return RSVD_E_NOMEM;
    }
    scratch_n = count;
    return RSVD_OK;
  }
  // phase 1: publish this rank's buffer (ready on st), wait until every rank's is ready
  int publish(const double* p, cudaStream_t st, std::string* err, LoopPtrs* all) {
    g->ptr[rank] = p;
    if (cudaEventRecord(g->ev_in[rank], st) != cudaSuccess) return RSVD_E_CUDA;
    int r = g->barrier(err);
    if (r) return r;
    for (int q = 0; q < nranks; ++q) {
      all->p[q] = g->ptr[q];
      if (q != rank && cudaStreamWaitEvent(st, g->ev_in[q], 0) != cudaSuccess) return RSVD_E_CUDA;
    }
    return RSVD_OK;
  }
  // phase 2: every rank has finished reading the published buffers before any rank writes them
  int retire(cudaStream_t st, std::string* err) {
    if (cudaEventRecord(g->ev_done[rank], st) != cudaSuccess) return RSVD_E_CUDA;
    int r = g->barrier(err);
    if (r) return r;
    for (int q = 0; q < nranks; ++q)
      if (q != rank && cudaStreamWaitEvent(st, g->ev_done[q], 0) != cudaSuccess) return RSVD_E_CUDA;
    return RSVD_OK;
  }
  int allreduce(double* p, size_t count, cudaStream_t st, std::string* err) override {
    int r = ensure_scratch(count, err);
    LoopPtrs all;
    if (!r) r = publish(p, st, err, &all);
    if (!r) r = loop_sum(all, nranks, 0, count, scratch, st);
    if (!r) r = retire(st, err);
    if (!r && count && cudaMemcpyAsync(p, scratch, count * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      r = RSVD_E_CUDA;
    return r;
  }
  int reduce_scatter(const double* s, double* d, size_t count, cudaStream_t st, std::string* err) override {
    LoopPtrs all;
    int r = publish(s, st, err, &all);
    if (!r) r = loop_sum(all, nranks, (size_t)rank * count, count, d, st);
    if (!r) r = retire(st, err);
    return r;
  }
  int allgather(const double* s, double* d, size_t count, cudaStream_t st, std::string* err) override {
    LoopPtrs all;
    int r = publish(s, st, err, &all);
    for (int q = 0; q < nranks && !r && count; ++q)
      if (cudaMemcpyAsync(d + (size_t)q * count, all.p[q], count * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        r = RSVD_E_CUDA;
    if (!r) r = retire(st, err);
    return r;
  }
};
}  // namespace

Comm* loop_comm_create(LoopGroup* g, int rank, int device, std::string* err) {
  (void)device;
  if (!g || rank < 0 || rank >= g->n) {
    if (err) *err = "bad loopback rank";
    return nullptr;
  }
  LoopComm* c = new LoopComm();
  ++g->refs;
  c->g = g;
  c->nranks = g->n;
  c->rank = rank;
  return c;
}

}  // namespace rsvd
