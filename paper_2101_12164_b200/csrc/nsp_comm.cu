// Collectives of the sharded path: in-place sum-allreduce of fp64 buffers on the
// context stream.  Two implementations behind one call:
//  - NCCL (production, one process per GPU): libnccl.so.2 resolved at run time with dlopen (the
//    process's already-loaded NCCL when torch.distributed is up), communicator created in
//    nsp_setup from the caller's ncclUniqueId, ncclAllReduce on the context stream (NVLink /
//    NVSwitch; NVLS when NCCL selects it).
//  - local group (testing the sharded path on ONE GPU): G host threads each drive one rank's
//    context on its own stream; the allreduce is two host barriers around a kernel in which
//    every rank sums all G buffers in rank order.  No kernel ever waits on another rank's kernel
//    (dependencies are host barriers + cudaStreamWaitEvent), so this is safe on one device.
// Both give every rank the bitwise-identical sum (a reduced chunk is computed once and
// distributed by NCCL's ring / tree / NVLS algorithms; in rank order locally), which keeps the
// replicated shared rows identical on all ranks.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "nsp_comm.h"

namespace {

struct NcclApi {
  bool loaded = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return;
    }
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.loaded = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy && api.GetErrorString;
    if (!api.loaded) api.err = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

constexpr int MAXR = 16;
struct PtrPack {
  const double* p[MAXR];
};

__global__ void k_sum_ranks(PtrPack src, int nr, size_t count, double* __restrict__ out) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = src.p[0][i];
  for (int q = 1; q < nr; ++q) s += src.p[q][i];
  out[i] = s;
}

}  // namespace

struct LocalGroup {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const double*> bufs;
  std::vector<cudaEvent_t> ev1, ev2;
  bool broken = false;
  // false if another rank never arrived within 120 s (a rank that failed and left the collective
  // sequence): the group is marked broken so every rank errors out instead of deadlocking
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (broken) return false;
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

struct NspComm {
  int kind = 0;  // 1 NCCL, 2 local group
  int nranks = 1, rank = 0;
  ncclComm_t nc = nullptr;
  LocalGroup* lg = nullptr;
  double* tmp = nullptr;
  size_t tmp_cap = 0;
};

extern "C" nsp_status nsp_nccl_unique_id(void* out128) {
  if (!out128) return NSP_ERR_ARG;
  NcclApi& a = nccl();
  if (!a.loaded) return NSP_ERR_NCCL;
  ncclUniqueId id;
  if (a.GetUniqueId(&id) != ncclSuccess) return NSP_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, 128);
  return NSP_OK;
}

// The production collective's exact call sequence (dlopen, ncclGetUniqueId, ncclCommInitRank, in-place
// ncclAllReduce(ncclDouble, ncclSum) on a stream, ncclCommDestroy) on a ONE-rank communicator: the sum over
// one rank is the identity, so the buffer must come back bitwise unchanged.  The pool has a single GPU, so
// this is how the NCCL branch of comm_init / comm_allreduce is exercised on hardware.
extern "C" nsp_status nsp_nccl_selftest(int device, size_t count, double* max_abs_err) {
  if (count == 0 || !max_abs_err) return NSP_ERR_ARG;
  *max_abs_err = -1.0;
  NcclApi& a = nccl();
  if (!a.loaded) return NSP_ERR_NCCL;
  if (cudaSetDevice(device) != cudaSuccess) return NSP_ERR_CUDA;
  std::vector<double> h(count), g(count);
  for (size_t i = 0; i < count; ++i) h[i] = 1.0 / (double)(i + 3) - 0.25 * (double)(i % 7);
  double* d = nullptr;
  cudaStream_t st = nullptr;
  ncclComm_t nc = nullptr;
  nsp_status ret = NSP_OK;
  ncclUniqueId id;
  if (cudaMalloc(&d, count * 8) != cudaSuccess || cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
    ret = NSP_ERR_CUDA;
  } else if (a.GetUniqueId(&id) != ncclSuccess || a.CommInitRank(&nc, 1, id, 0) != ncclSuccess) {
    ret = NSP_ERR_NCCL;
  } else {
    cudaMemcpyAsync(d, h.data(), count * 8, cudaMemcpyHostToDevice, st);
    if (a.AllReduce(d, d, count, ncclDouble, ncclSum, nc, st) != ncclSuccess) ret = NSP_ERR_NCCL;
    cudaMemcpyAsync(g.data(), d, count * 8, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) ret = NSP_ERR_CUDA;
    if (ret == NSP_OK) {
      double m = 0.0;
      for (size_t i = 0; i < count; ++i) m = std::max(m, std::fabs(g[i] - h[i]));
      *max_abs_err = m;
    }
  }
  if (nc) a.CommDestroy(nc);
  if (st) cudaStreamDestroy(st);
  if (d) cudaFree(d);
  return ret;
}

extern "C" void* nsp_local_group_create(int nranks) {
  if (nranks < 1 || nranks > MAXR) return nullptr;
  LocalGroup* g = new LocalGroup();
  g->n = nranks;
  g->bufs.assign(nranks, nullptr);
  g->ev1.assign(nranks, nullptr);
  g->ev2.assign(nranks, nullptr);
  return g;
}

extern "C" void nsp_local_group_destroy(void* grp) { delete (LocalGroup*)grp; }

namespace nspi {

nsp_status comm_init(nsp_ctx* c) {
  if (c->nranks <= 1) return NSP_OK;
  NspComm* cm = new NspComm();
  cm->nranks = c->nranks;
  cm->rank = c->rank;
  c->comm = cm;
  if (c->opts.local_group) {
    LocalGroup* g = (LocalGroup*)c->opts.local_group;
    if (g->n != c->nranks) {
      c->err = "nsp_setup: local group size != nranks";
      return NSP_ERR_ARG;
    }
    cm->kind = 2;
    cm->lg = g;
    NSP_CUDA_TRY(c, cudaEventCreateWithFlags(&g->ev1[c->rank], cudaEventDisableTiming));
    NSP_CUDA_TRY(c, cudaEventCreateWithFlags(&g->ev2[c->rank], cudaEventDisableTiming));
    if (!g->barrier()) {   // every rank's events exist before the first allreduce
      c->err = "nsp_setup: local group barrier timed out (another rank failed)";
      return NSP_ERR_STATE;
    }
    return NSP_OK;
  }
  if (!c->opts.nccl_id) {
    c->err = "nsp_setup: nranks > 1 needs opts.nccl_id (nsp_nccl_unique_id on rank 0, broadcast) or a local group";
    return NSP_ERR_ARG;
  }
  NcclApi& a = nccl();
  if (!a.loaded) {
    c->err = "nsp_setup: " + a.err;
    return NSP_ERR_NCCL;
  }
  ncclUniqueId id;
  std::memcpy(&id, c->opts.nccl_id, sizeof(id));
  const ncclResult_t r = a.CommInitRank(&cm->nc, c->nranks, id, c->rank);
  if (r != ncclSuccess) {
    c->err = std::string("ncclCommInitRank: ") + a.GetErrorString(r);
    return NSP_ERR_NCCL;
  }
  cm->kind = 1;
  return NSP_OK;
}

nsp_status comm_allreduce(nsp_ctx* c, double* buf, size_t count) {
  NspComm* cm = c->comm;
  if (!cm || cm->nranks <= 1 || count == 0) return NSP_OK;
  if (cm->kind == 1) {
    NcclApi& a = nccl();
    const ncclResult_t r = a.AllReduce(buf, buf, count, ncclDouble, ncclSum, cm->nc, c->stream);
    if (r != ncclSuccess) {
      c->err = std::string("ncclAllReduce: ") + a.GetErrorString(r);
      return NSP_ERR_NCCL;
    }
    return NSP_OK;
  }
  LocalGroup* g = cm->lg;
  const int me = cm->rank;
  if (cm->tmp_cap < count) {
    if (cm->tmp) cudaFree(cm->tmp);
    cm->tmp = nullptr;
    cm->tmp_cap = 0;
    NSP_CUDA_TRY(c, cudaMalloc(&cm->tmp, count * 8));
    cm->tmp_cap = count;
  }
  g->bufs[me] = buf;
  NSP_CUDA_TRY(c, cudaEventRecord(g->ev1[me], c->stream));
  if (!g->barrier()) {
    c->err = "local-group allreduce: barrier timed out (another rank failed)";
    return NSP_ERR_STATE;
  }
  PtrPack pk{};
  for (int q = 0; q < g->n; ++q) {
    NSP_CUDA_TRY(c, cudaStreamWaitEvent(c->stream, g->ev1[q], 0));
    pk.p[q] = g->bufs[q];
  }
  nsp_count_launch();
  k_sum_ranks<<<(unsigned)((count + 255) / 256), 256, 0, c->stream>>>(pk, g->n, count, cm->tmp);
  NSP_CUDA_TRY(c, cudaEventRecord(g->ev2[me], c->stream));
  if (!g->barrier()) {
    c->err = "local-group allreduce: barrier timed out (another rank failed)";
    return NSP_ERR_STATE;
  }
  for (int q = 0; q < g->n; ++q) NSP_CUDA_TRY(c, cudaStreamWaitEvent(c->stream, g->ev2[q], 0));
  NSP_CUDA_TRY(c, cudaMemcpyAsync(buf, cm->tmp, count * 8, cudaMemcpyDeviceToDevice, c->stream));
  return NSP_OK;
}

void comm_free(nsp_ctx* c) {
  NspComm* cm = c->comm;
  if (!cm) return;
  if (cm->kind == 1 && cm->nc) nccl().CommDestroy(cm->nc);
  if (cm->kind == 2 && cm->lg) {
    if (cm->lg->ev1[cm->rank]) cudaEventDestroy(cm->lg->ev1[cm->rank]);
    if (cm->lg->ev2[cm->rank]) cudaEventDestroy(cm->lg->ev2[cm->rank]);
    cm->lg->ev1[cm->rank] = nullptr;
    cm->lg->ev2[cm->rank] = nullptr;
  }
  if (cm->tmp) cudaFree(cm->tmp);
  delete cm;
  c->comm = nullptr;
}

}  // namespace nspi
