// gss_comm.cu — patient sharding (config C5) across GPUs: the communicator
// behind the cycle kernel's in-kernel cross-shard exchange (gss_cycle.cu
// cross_shard) and its C ABI (include/gss.h, "Patient sharding").
//
// A communicator gives every shard engine (one per rank) peer-visible
// pointers to all ranks' exchange buffers [2][nranks][kXrStride] doubles and
// arrival counters.  Two ways to build one:
//   * gss_comm_init  — one process per GPU: NCCL bootstraps the ranks (the
//     unique id travels over the caller's own channel, e.g. torch.distributed),
//     each rank exports its buffers with CUDA IPC and all-gathers the handles;
//     peers open them (NVLink peer access).  NCCL is loaded with dlopen, so
//     libgss has no link-time NCCL dependency.
//   * gss_comm_local — every shard in this process (same device: the shards
//     run in one batched launch; or one device each with peer access).
// Attaching a communicator makes the shards' fixed terms global (sums over
// shards in rank order); the shards then fit with gss_engine_fit (one process
// per GPU) or gss_sharded_fit_local (all shards of this process together).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gss.h"
#include "gss_kernels.cuh"

namespace gss {
int set_last_error(int code, const std::string& msg);                       // gss_capi.cu
int engine_attach_comm(gss_engine* e, int nranks, int rank, double* const* pay_ptrs,
                       unsigned int* const* bar_ptrs, int sys_scope);       // gss_capi.cu
int engine_fixed_terms(gss_engine* e, double** dev_fixed, int64_t* p, int* device,
                       cudaStream_t* stream);                               // gss_capi.cu
}  // namespace gss

using gss::set_last_error;

struct gss_comm {
  int nranks = 1, rank = 0, device = 0;
  double* pay = nullptr;             // this rank's buffer (owned)
  unsigned int* bar = nullptr;       // this rank's counter (owned)
  double** d_pay = nullptr;          // device array [nranks] of peer-mapped buffers
  unsigned int** d_bar = nullptr;    // device array [nranks] of peer-mapped counters
  std::vector<void*> opened;         // IPC-opened peer allocations
  void* nccl = nullptr;              // ncclComm_t (multi-process)
  bool sys_scope = true;             // ranks on several devices (false: one device)
};

namespace {

// ---- NCCL through dlopen (nccl.h ABI: ncclUniqueId is 128 bytes) ---------
struct NcclApi {
  void* h = nullptr;
  int (*get_id)(void*) = nullptr;
  int (*allgather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*destroy)(void*) = nullptr;
};

struct Uid {
  char internal[128];
};
using InitFn = int (*)(void**, int, Uid, int);

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (api.h) {
      api.get_id = reinterpret_cast<int (*)(void*)>(dlsym(api.h, "ncclGetUniqueId"));
      api.allgather = reinterpret_cast<int (*)(const void*, void*, size_t, int, void*, cudaStream_t)>(
          dlsym(api.h, "ncclAllGather"));
      api.destroy = reinterpret_cast<int (*)(void*)>(dlsym(api.h, "ncclCommDestroy"));
    }
  }
  return api;
}

InitFn nccl_init_fn() {
  NcclApi& a = nccl();
  return a.h ? reinterpret_cast<InitFn>(dlsym(a.h, "ncclCommInitRank")) : nullptr;
}

constexpr int kNcclUint8 = 1;  // ncclDataType_t ncclUint8 (nccl.h)

int alloc_rank_buffers(gss_comm* c) {
  const size_t doubles = 2 * size_t(c->nranks) * gss::kXrStride;
  if (cudaMalloc(reinterpret_cast<void**>(&c->pay), doubles * sizeof(double)) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&c->bar), 256) != cudaSuccess)
    return set_last_error(GSS_ERR_OOM, "gss_comm: exchange buffer allocation failed");
  cudaMemset(c->pay, 0, doubles * sizeof(double));
  cudaMemset(c->bar, 0, 256);
  return GSS_OK;
}

int upload_ptrs(gss_comm* c, const std::vector<double*>& pay, const std::vector<unsigned int*>& bar) {
  if (cudaMalloc(reinterpret_cast<void**>(&c->d_pay), pay.size() * sizeof(double*)) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&c->d_bar), bar.size() * sizeof(unsigned int*)) != cudaSuccess)
    return set_last_error(GSS_ERR_OOM, "gss_comm: pointer table allocation failed");
  cudaMemcpy(c->d_pay, pay.data(), pay.size() * sizeof(double*), cudaMemcpyHostToDevice);
  cudaMemcpy(c->d_bar, bar.data(), bar.size() * sizeof(unsigned int*), cudaMemcpyHostToDevice);
  return cudaDeviceSynchronize() == cudaSuccess
             ? GSS_OK
             : set_last_error(GSS_ERR_CUDA, "gss_comm: pointer table upload failed");
}

}  // namespace

extern "C" {

int gss_comm_local_finalize(gss_engine* const* shards, int count);
void gss_comm_destroy(gss_comm* c);
int gss_engine_get_colmax(gss_engine* e, double* out, int64_t p);
int gss_engine_set_colmax(gss_engine* e, const double* in, int64_t p);

int gss_comm_unique_id(unsigned char* out128) {
  if (!out128) return set_last_error(GSS_ERR_DOMAIN, "null argument");
  NcclApi& a = nccl();
  if (!a.get_id) return set_last_error(GSS_ERR_CUDA, "gss_comm_unique_id: libnccl not found");
  const int r = a.get_id(out128);
  return r == 0 ? GSS_OK : set_last_error(GSS_ERR_CUDA, "ncclGetUniqueId failed");
}

// ---- NCCL-free bootstrap: the caller all-gathers the 128-byte handles ------
struct Handles {
  cudaIpcMemHandle_t pay, bar;
};
static_assert(sizeof(Handles) == 128, "two CUDA IPC handles");

int gss_comm_create(int nranks, int rank, int device, gss_comm** out) {
  if (!out) return set_last_error(GSS_ERR_DOMAIN, "null argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return set_last_error(GSS_ERR_DOMAIN, "gss_comm_create: rank outside [0, nranks)");
  if (cudaSetDevice(device) != cudaSuccess)
    return set_last_error(GSS_ERR_NO_DEVICE, "gss_comm_create: no such CUDA device");
  auto* c = new gss_comm;
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  if (int rc = alloc_rank_buffers(c)) {
    gss_comm_destroy(c);
    return rc;
  }
  *out = c;
  return GSS_OK;
}

int gss_comm_ipc_handle(gss_comm* c, unsigned char* out128) {
  if (!c || !out128) return set_last_error(GSS_ERR_DOMAIN, "null argument");
  cudaSetDevice(c->device);
  Handles h{};
  if (cudaIpcGetMemHandle(&h.pay, c->pay) != cudaSuccess ||
      cudaIpcGetMemHandle(&h.bar, c->bar) != cudaSuccess)
    return set_last_error(GSS_ERR_CUDA, "cudaIpcGetMemHandle failed");
  std::memcpy(out128, &h, sizeof(h));
  return GSS_OK;
}

int gss_comm_connect(gss_comm* c, const unsigned char* all128) {
  if (!c || !all128) return set_last_error(GSS_ERR_DOMAIN, "null argument");
  cudaSetDevice(c->device);
  const int R = c->nranks;
  std::vector<double*> pay(static_cast<size_t>(R));
  std::vector<unsigned int*> bar(static_cast<size_t>(R));
  for (int q = 0; q < R; ++q) {
    if (q == c->rank) {
      pay[q] = c->pay;
      bar[q] = c->bar;
      continue;
    }
    Handles h;
    std::memcpy(&h, all128 + size_t(q) * sizeof(Handles), sizeof(Handles));
    void *pp = nullptr, *pb = nullptr;
    if (cudaIpcOpenMemHandle(&pp, h.pay, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&pb, h.bar, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
      return set_last_error(GSS_ERR_CUDA, "cudaIpcOpenMemHandle failed (no peer access?)");
    c->opened.push_back(pp);
    c->opened.push_back(pb);
    pay[q] = static_cast<double*>(pp);
    bar[q] = static_cast<unsigned int*>(pb);
  }
  return upload_ptrs(c, pay, bar);
}

int gss_comm_init(int nranks, int rank, const unsigned char* uid128, int device, gss_comm** out) {
  if (!out || !uid128) return set_last_error(GSS_ERR_DOMAIN, "null argument");
  *out = nullptr;
  NcclApi& a = nccl();
  InitFn init = nccl_init_fn();
  if (!init || !a.allgather) return set_last_error(GSS_ERR_CUDA, "gss_comm_init: libnccl not found");
  gss_comm* c = nullptr;
  if (int rc = gss_comm_create(nranks, rank, device, &c)) return rc;
  auto bail = [&](int rc) {
    gss_comm_destroy(c);
    return rc;
  };
  Uid uid;
  std::memcpy(uid.internal, uid128, sizeof(uid.internal));
  if (init(&c->nccl, nranks, uid, rank) != 0)
    return bail(set_last_error(GSS_ERR_CUDA, "ncclCommInitRank failed"));
  unsigned char mine[sizeof(Handles)];
  if (int rc = gss_comm_ipc_handle(c, mine)) return bail(rc);
  void *d_mine = nullptr, *d_all = nullptr;
  cudaMalloc(&d_mine, sizeof(Handles));
  cudaMalloc(&d_all, sizeof(Handles) * nranks);
  cudaMemcpy(d_mine, mine, sizeof(Handles), cudaMemcpyHostToDevice);
  const int rc = a.allgather(d_mine, d_all, sizeof(Handles), kNcclUint8, c->nccl, nullptr);
  std::vector<unsigned char> all(sizeof(Handles) * nranks);
  cudaMemcpy(all.data(), d_all, all.size(), cudaMemcpyDeviceToHost);
  cudaFree(d_mine);
  cudaFree(d_all);
  if (rc != 0) return bail(set_last_error(GSS_ERR_CUDA, "ncclAllGather (IPC handles) failed"));
  if (int rc2 = gss_comm_connect(c, all.data())) return bail(rc2);
  *out = c;
  return GSS_OK;
}

int gss_comm_local(gss_engine* const* shards, int count, gss_comm** comms_out) {
  if (!shards || !comms_out || count < 1) return set_last_error(GSS_ERR_DOMAIN, "null argument");
  std::vector<gss_comm*> cs(static_cast<size_t>(count), nullptr);
  std::vector<double*> pay(static_cast<size_t>(count));
  std::vector<unsigned int*> bar(static_cast<size_t>(count));
  auto bail = [&](int rc) {
    for (gss_comm* c : cs) gss_comm_destroy(c);
    return rc;
  };
  std::vector<int> devs(static_cast<size_t>(count));
  for (int r = 0; r < count; ++r) {
    double* fx = nullptr;
    int64_t p = 0;
    cudaStream_t st = nullptr;
    if (int rc = gss::engine_fixed_terms(shards[r], &fx, &p, &devs[r], &st)) return bail(rc);
    cudaSetDevice(devs[r]);
    cs[r] = new gss_comm;
    cs[r]->nranks = count;
    cs[r]->rank = r;
    cs[r]->device = devs[r];
    if (int rc = alloc_rank_buffers(cs[r])) return bail(rc);
    pay[r] = cs[r]->pay;
    bar[r] = cs[r]->bar;
  }
  for (int r = 0; r < count; ++r)
    for (int q = 0; q < count; ++q)
      if (devs[q] != devs[r]) {
        cudaSetDevice(devs[r]);
        const cudaError_t e = cudaDeviceEnablePeerAccess(devs[q], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return bail(set_last_error(GSS_ERR_CUDA, "gss_comm_local: no peer access between devices"));
        cudaGetLastError();
      }
  bool one_device = true;
  for (int r = 1; r < count; ++r) one_device &= devs[r] == devs[0];
  for (int r = 0; r < count; ++r) {
    cudaSetDevice(devs[r]);
    cs[r]->sys_scope = !one_device;
    if (int rc = upload_ptrs(cs[r], pay, bar)) return bail(rc);
  }
  for (int r = 0; r < count; ++r)
    if (int rc = gss_engine_attach_comm(shards[r], cs[r])) return bail(rc);
  if (int rc = gss_comm_local_finalize(shards, count)) return bail(rc);
  for (int r = 0; r < count; ++r) comms_out[r] = cs[r];
  return GSS_OK;
}

void gss_comm_destroy(gss_comm* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (void* q : c->opened) cudaIpcCloseMemHandle(q);
  for (void* q : {(void*)c->pay, (void*)c->bar, (void*)c->d_pay, (void*)c->d_bar})
    if (q) cudaFree(q);
  if (c->nccl && nccl().destroy) nccl().destroy(c->nccl);
  delete c;
}

int gss_comm_rank(const gss_comm* c, int* nranks, int* rank) {
  if (!c) return set_last_error(GSS_ERR_DOMAIN, "null argument");
  if (nranks) *nranks = c->nranks;
  if (rank) *rank = c->rank;
  return GSS_OK;
}

// Attach: the engine becomes shard `rank` of the communicator's fit.  The
// fixed terms delta' X_j become the sums over all shards in rank order
// (all-gathered over NCCL for gss_comm_init communicators; for local groups
// the caller attaches every shard, then calls gss_comm_local_finalize).
int gss_engine_attach_comm(gss_engine* e, gss_comm* c) {
  if (!e || !c) return set_last_error(GSS_ERR_DOMAIN, "null argument");
  double* fx = nullptr;
  int64_t p = 0;
  int dev = 0;
  cudaStream_t st = nullptr;
  if (int rc = gss::engine_fixed_terms(e, &fx, &p, &dev, &st)) return rc;
  if (dev != c->device)
    return set_last_error(GSS_ERR_DOMAIN, "gss_engine_attach_comm: engine and comm on different devices");
  if (c->nccl && c->nranks > 1) {  // global fixed terms: all-gather, sum in rank order
    cudaSetDevice(dev);
    double* all = nullptr;
    if (cudaMalloc(reinterpret_cast<void**>(&all), sizeof(double) * size_t(p) * c->nranks) != cudaSuccess)
      return set_last_error(GSS_ERR_OOM, "gss_engine_attach_comm: allocation failed");
    const int rc = nccl().allgather(fx, all, sizeof(double) * size_t(p), kNcclUint8, c->nccl, st);
    std::vector<double> h(size_t(p) * c->nranks), sum(size_t(p), 0.0);
    cudaMemcpyAsync(h.data(), all, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(all);
    if (rc != 0) return set_last_error(GSS_ERR_CUDA, "ncclAllGather (fixed terms) failed");
    for (int q = 0; q < c->nranks; ++q)
      for (int64_t j = 0; j < p; ++j) sum[j] += h[size_t(q) * p + j];
    cudaMemcpy(fx, sum.data(), sum.size() * sizeof(double), cudaMemcpyHostToDevice);
    // the fast overflow bound: max over ranks
    std::vector<double> cm(static_cast<size_t>(p));
    if (int rc2 = gss_engine_get_colmax(e, cm.data(), p)) return rc2;
    double* dcm = nullptr;
    cudaMalloc(reinterpret_cast<void**>(&dcm), sizeof(double) * size_t(p) * (c->nranks + 1));
    cudaMemcpy(dcm, cm.data(), sizeof(double) * size_t(p), cudaMemcpyHostToDevice);
    const int rc3 = nccl().allgather(dcm, dcm + p, sizeof(double) * size_t(p), kNcclUint8, c->nccl, st);
    cudaMemcpyAsync(h.data(), dcm + p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(dcm);
    if (rc3 != 0) return set_last_error(GSS_ERR_CUDA, "ncclAllGather (colmax) failed");
    for (int q = 0; q < c->nranks; ++q)
      for (int64_t j = 0; j < p; ++j) cm[j] = std::max(cm[j], h[size_t(q) * p + j]);
    if (int rc4 = gss_engine_set_colmax(e, cm.data(), p)) return rc4;
  }
  // GSS_XR_SCOPE=gpu: every rank is known to share one device (e.g. several
  // shard processes on one GPU under MPS): gpu-scope flags are sufficient
  const char* sc = std::getenv("GSS_XR_SCOPE");
  const bool sys = c->sys_scope && !(sc && std::strcmp(sc, "gpu") == 0);
  return gss::engine_attach_comm(e, c->nranks, c->rank, c->d_pay, c->d_bar, sys ? 1 : 0);
}

int gss_comm_local_finalize(gss_engine* const* shards, int count) {
  if (!shards || count < 1) return set_last_error(GSS_ERR_DOMAIN, "null argument");
  std::vector<std::vector<double>> fx(static_cast<size_t>(count));
  int64_t p0 = -1;
  for (int r = 0; r < count; ++r) {
    double* d = nullptr;
    int64_t p = 0;
    int dev = 0;
    cudaStream_t st = nullptr;
    if (int rc = gss::engine_fixed_terms(shards[r], &d, &p, &dev, &st)) return rc;
    if (p0 >= 0 && p != p0) return set_last_error(GSS_ERR_DOMAIN, "shards differ in p");
    p0 = p;
    cudaSetDevice(dev);
    fx[r].resize(size_t(p));
    cudaMemcpy(fx[r].data(), d, size_t(p) * sizeof(double), cudaMemcpyDeviceToHost);
  }
  std::vector<double> sum(size_t(p0), 0.0);
  for (int r = 0; r < count; ++r)
    for (int64_t j = 0; j < p0; ++j) sum[j] += fx[r][j];
  // the fast overflow bound: the max over shards, on every shard
  std::vector<double> cm(static_cast<size_t>(p0), 0.0), tmp(static_cast<size_t>(p0));
  for (int r = 0; r < count; ++r) {
    if (int rc = gss_engine_get_colmax(shards[r], tmp.data(), p0)) return rc;
    for (int64_t j = 0; j < p0; ++j) cm[j] = std::max(cm[j], tmp[j]);
  }
  for (int r = 0; r < count; ++r)
    if (int rc = gss_engine_set_colmax(shards[r], cm.data(), p0)) return rc;
  for (int r = 0; r < count; ++r) {
    double* d = nullptr;
    int64_t p = 0;
    int dev = 0;
    cudaStream_t st = nullptr;
    gss::engine_fixed_terms(shards[r], &d, &p, &dev, &st);
    cudaSetDevice(dev);
    cudaMemcpy(d, sum.data(), sum.size() * sizeof(double), cudaMemcpyHostToDevice);
  }
  return GSS_OK;
}

}  // extern "C"
