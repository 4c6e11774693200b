// The collectives of the sharded run (sgx_run_sharded): an NCCL exchange for
// one process per GPU, and an in-process exchange for one host thread per
// rank.  See include/satgrad_b200.h.
//
// NCCL is resolved at run time (dlopen/dlsym): a process that already loaded
// a libnccl.so.2 (e.g. torch's) gets that copy, so communicators and streams
// come from one NCCL; otherwise the system libnccl.so.2.  The library itself
// never links NCCL, and single-GPU use never touches it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/satgrad_b200.h"

namespace sgx {
void set_last_error(const std::string& msg);
}

namespace {

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string err;
};

NcclApi& nccl() {
  static NcclApi A = [] {
    NcclApi a;
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy this process already uses
    if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!a.h) {
      a.err = std::string("libnccl.so.2 not found: ") + dlerror();
      return a;
    }
    auto sym = [&](const char* s) {
      void* p = dlsym(a.h, s);
      if (!p && a.err.empty()) a.err = std::string("libnccl.so.2 lacks ") + s;
      return p;
    };
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(sym("ncclAllGather"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
    return a;
  }();
  if (!A.err.empty()) throw std::runtime_error(A.err);
  return A;
}

struct NcclEx {
  ncclComm_t comm = nullptr;
  int device = 0, nranks = 1;
  cudaStream_t hs = nullptr;  // host all-gathers
  int64_t* dbuf = nullptr;    // staging for them
  size_t dcap = 0;
};

int nccl_allgather_device(void* user, const void* send, void* recv, int64_t bytes, void* stream) {
  auto* e = static_cast<NcclEx*>(user);
  NcclApi& A = nccl();
  const ncclResult_t r = A.all_gather(send, recv, static_cast<size_t>(bytes), ncclUint8, e->comm,
                                      static_cast<cudaStream_t>(stream));
  return r == ncclSuccess ? 0 : -static_cast<int>(r) - 100;
}

int nccl_allgather_host(void* user, const int64_t* send, int64_t* recv, int32_t n) {
  auto* e = static_cast<NcclEx*>(user);
  NcclApi& A = nccl();
  const size_t need = static_cast<size_t>(n) * (1 + e->nranks);
  if (cudaSetDevice(e->device) != cudaSuccess) return -2;
  if (need > e->dcap) {
    if (e->dbuf) cudaFree(e->dbuf);
    if (cudaMalloc(&e->dbuf, need * sizeof(int64_t)) != cudaSuccess) return -3;
    e->dcap = need;
  }
  int64_t* dsend = e->dbuf;
  int64_t* drecv = e->dbuf + n;
  if (cudaMemcpyAsync(dsend, send, n * sizeof(int64_t), cudaMemcpyHostToDevice, e->hs) != cudaSuccess) return -2;
  const ncclResult_t r = A.all_gather(dsend, drecv, static_cast<size_t>(n), ncclInt64, e->comm, e->hs);
  if (r != ncclSuccess) return -static_cast<int>(r) - 100;
  if (cudaMemcpyAsync(recv, drecv, static_cast<size_t>(n) * e->nranks * sizeof(int64_t), cudaMemcpyDeviceToHost,
                      e->hs) != cudaSuccess)
    return -2;
  return cudaStreamSynchronize(e->hs) == cudaSuccess ? 0 : -2;
}

// ---------------------------------------------------------- in-process
struct LocalGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const void*> dsend;
  std::vector<const int64_t*> hsend;
  std::vector<struct LocalRank*> ranks;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LocalRank {
  LocalGroup* g = nullptr;
  int rank = 0;
};

// Every rank publishes its (ready) send buffer, then copies every rank's
// buffer into its own recv on its stream (device-to-device, peer or not),
// and waits for the copies before anyone may reuse a send buffer.
int local_allgather_device(void* user, const void* send, void* recv, int64_t bytes, void* stream) {
  auto* me = static_cast<LocalRank*>(user);
  LocalGroup* g = me->g;
  auto st = static_cast<cudaStream_t>(stream);
  if (cudaStreamSynchronize(st) != cudaSuccess) return -2;
  g->dsend[me->rank] = send;
  g->barrier();
  int rc = 0;
  for (int q = 0; q < g->n && rc == 0; ++q)
    if (cudaMemcpyAsync(static_cast<char*>(recv) + static_cast<size_t>(q) * bytes, g->dsend[q],
                        static_cast<size_t>(bytes), cudaMemcpyDefault, st) != cudaSuccess)
      rc = -2;
  if (rc == 0 && cudaStreamSynchronize(st) != cudaSuccess) rc = -2;
  g->barrier();
  return rc;
}

int local_allgather_host(void* user, const int64_t* send, int64_t* recv, int32_t n) {
  auto* me = static_cast<LocalRank*>(user);
  LocalGroup* g = me->g;
  g->hsend[me->rank] = send;
  g->barrier();
  for (int q = 0; q < g->n; ++q) std::memcpy(recv + static_cast<size_t>(q) * n, g->hsend[q], n * sizeof(int64_t));
  g->barrier();
  return 0;
}

template <typename F>
int wrap(F&& f) {
  try {
    f();
    return SGX_OK;
  } catch (const std::invalid_argument& e) {
    sgx::set_last_error(e.what());
    return SGX_E_INVALID;
  } catch (const std::exception& e) {
    sgx::set_last_error(e.what());
    return SGX_E_CUDA;
  }
}

}  // namespace

extern "C" {

int sgx_nccl_unique_id(uint8_t id[128]) {
  return wrap([&] {
    if (!id) throw std::invalid_argument("id is null");
    ncclUniqueId u;
    const ncclResult_t r = nccl().get_unique_id(&u);
    if (r != ncclSuccess) throw std::runtime_error(std::string("ncclGetUniqueId: ") + nccl().error_string(r));
    static_assert(sizeof(u.internal) == 128, "ncclUniqueId size");
    std::memcpy(id, u.internal, 128);
  });
}

int sgx_exchange_nccl_create(int32_t nranks, const uint8_t id[128], int32_t rank, int32_t device,
                             sgx_exchange* out) {
  return wrap([&] {
    if (!id || !out) throw std::invalid_argument("id / out is null");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("bad rank / nranks");
    NcclApi& A = nccl();
    if (cudaSetDevice(device) != cudaSuccess) throw std::runtime_error("cudaSetDevice failed");
    auto* e = new NcclEx;
    e->device = device;
    e->nranks = nranks;
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    const ncclResult_t r = A.comm_init_rank(&e->comm, nranks, u, rank);
    if (r != ncclSuccess) {
      delete e;
      throw std::runtime_error(std::string("ncclCommInitRank: ") + A.error_string(r));
    }
    cudaStreamCreateWithFlags(&e->hs, cudaStreamNonBlocking);
    out->user = e;
    out->rank = rank;
    out->nranks = nranks;
    out->allgather_device = nccl_allgather_device;
    out->allgather_host = nccl_allgather_host;
  });
}

int sgx_exchange_nccl_destroy(sgx_exchange* ex) {
  return wrap([&] {
    if (!ex || !ex->user) return;
    auto* e = static_cast<NcclEx*>(ex->user);
    cudaSetDevice(e->device);
    if (e->hs) cudaStreamSynchronize(e->hs);
    nccl().comm_destroy(e->comm);
    if (e->dbuf) cudaFree(e->dbuf);
    if (e->hs) cudaStreamDestroy(e->hs);
    delete e;
    ex->user = nullptr;
  });
}

int sgx_exchange_local_create(int32_t nranks, sgx_exchange* out) {
  return wrap([&] {
    if (!out) throw std::invalid_argument("out is null");
    if (nranks < 1) throw std::invalid_argument("nranks must be positive");
    auto* g = new LocalGroup;
    g->n = nranks;
    g->dsend.assign(nranks, nullptr);
    g->hsend.assign(nranks, nullptr);
    for (int r = 0; r < nranks; ++r) {
      auto* lr = new LocalRank{g, r};
      g->ranks.push_back(lr);
      out[r].user = lr;
      out[r].rank = r;
      out[r].nranks = nranks;
      out[r].allgather_device = local_allgather_device;
      out[r].allgather_host = local_allgather_host;
    }
  });
}

int sgx_exchange_local_destroy(sgx_exchange* ex) {
  return wrap([&] {
    if (!ex || !ex->user) return;
    LocalGroup* g = static_cast<LocalRank*>(ex->user)->g;
    for (LocalRank* r : g->ranks) delete r;
    delete g;
    ex->user = nullptr;
  });
}

}  // extern "C"
