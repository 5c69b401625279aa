// Inter-rank communication for the z-slab decomposition.
//
// Each rank's context holds its owned planes [kw_lo, kw_hi) plus one ghost
// plane on each side that has a neighbouring rank. Only two things cross
// ranks: the one-plane halo of a vector before every operator that reads
// neighbours (state before assembly; p-hat / s-hat / x before each SpMV),
// and the Krylov scalars (dot products) and Newton norms.
//
// Two transports behind one interface:
//   * NCCL (one process per GPU, NVLink/NVSwitch): grouped ncclSend/ncclRecv
//     of packed boundary planes, ncclAllReduce of the packed scalar slots on
//     the context's stream. libnccl is resolved at run time (dlopen) from the
//     process — torch has already loaded its NCCL — so the library still
//     loads on machines without NCCL.
//   * Hub (several contexts in one process, one host thread each): device
//     copies between the contexts' buffers and host barriers. Used to run the
//     multi-rank algorithm on a single GPU in tests; kernels never wait on
//     each other (only host threads do), so there is no cross-kernel spin.
#pragma once
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace isc {

// --- minimal NCCL ABI (types/values from nccl.h, resolved with dlsym) -------
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
enum { ncclSuccess_ = 0 };
enum { ncclFloat64_ = 8 };
enum { ncclSum_ = 0, ncclMax_ = 2 };

struct NcclApi {
  bool ok = false;
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

inline NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.CommInitRank = (int (*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(h, "ncclCommInitRank");
  api.CommDestroy = (int (*)(ncclComm_t))dlsym(h, "ncclCommDestroy");
  api.Send = (int (*)(const void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclSend");
  api.Recv = (int (*)(void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(h, "ncclRecv");
  api.AllReduce = (int (*)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t))dlsym(
      h, "ncclAllReduce");
  api.GroupStart = (int (*)())dlsym(h, "ncclGroupStart");
  api.GroupEnd = (int (*)())dlsym(h, "ncclGroupEnd");
  api.GetErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
  api.ok = api.CommInitRank && api.Send && api.Recv && api.AllReduce && api.GroupStart &&
           api.GroupEnd;
  return api;
}

// --- in-process hub ----------------------------------------------------------
struct Hub {
  int nranks = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  // per rank: device send buffers (lo, hi) and the event marking them ready
  std::vector<double*> send_lo, send_hi;
  std::vector<cudaEvent_t> ready;
  // host scalar exchange
  std::vector<double> red;   // nranks * 64
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct Comm {
  int rank = 0, nranks = 1;
  bool has_lo = false, has_hi = false;
  ncclComm_t nccl = nullptr;
  Hub* hub = nullptr;
  bool single = false;   // one-rank NCCL communicator driven through the slab path (tests)
  bool active() const { return nranks > 1 || single; }
};

// pack / unpack the `rows` x plane-k values of a storage-order vector. The
// buffer is in natural cell order within the plane, so ranks whose local
// colourings of the shared plane differ (odd plane offsets) still agree.
__global__ void k_pack_plane(Dims g, int rows, int k, const double* __restrict__ v,
                             double* __restrict__ buf) {
  const int64_t m = g.nxny;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * rows) return;
  const int r = (int)(t / m);
  const int64_t q = t - (int64_t)r * m;
  buf[t] = v[(int64_t)r * g.n + pos_of(g, (int64_t)k * m + q)];
}

__global__ void k_unpack_plane(Dims g, int rows, int k, const double* __restrict__ buf,
                               double* __restrict__ v) {
  const int64_t m = g.nxny;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * rows) return;
  const int r = (int)(t / m);
  const int64_t q = t - (int64_t)r * m;
  v[(int64_t)r * g.n + pos_of(g, (int64_t)k * m + q)] = buf[t];
}

}  // namespace isc
