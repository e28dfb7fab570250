// Multi-GPU step statistics. Environments are independent
// worlds (shell.hpp:392-397): one process per GPU, each owning a
// contiguous env range, no halo and no particle migration. The only exchange
// is the per-env-step statistics vector. It is reduced over the context's envs
// on the device and all-reduced with NCCL on the context's own stream, so the
// exchange is stream-ordered after the env step, capturable in a CUDA graph,
// and reaches the host only when the caller reads it.
//
// NCCL is resolved at run time from the process (RTLD_NOLOAD first: the
// libnccl torch already loaded, so communicators live in one library), else
// libnccl.so.2; the library itself does not link it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "msim_internal.h"

namespace msim_impl {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("NCCL not available: ") + dlerror();
      return a;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.all_reduce && a.comm_destroy && a.error_string;
    if (!a.ok) a.why = "NCCL symbols missing";
    return a;
  }();
  return api;
}

// sums[0..3] = particle-substeps, env-steps, CFL cycles, lost particles (summed
// over envs); maxs[4..5] = max penetration, max force-balance error.
__global__ void k_step_stats(const long long* env_off, const EnvRun* run, const unsigned* max_pen,
                             const double* balance, const long long* lost, int n_env, int substeps, double* out) {
  __shared__ double s[4], m[2];
  if (threadIdx.x < 4) s[threadIdx.x] = 0.0;
  if (threadIdx.x < 2) m[threadIdx.x] = 0.0;
  __syncthreads();
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0, p = 0, b = 0;
  for (int e = threadIdx.x; e < n_env; e += blockDim.x) {
    a0 += (double)(env_off[e + 1] - env_off[e]) * substeps;
    a1 += 1.0;
    a2 += run[e].cyc_sum;
    a3 += (double)lost[e];
    p = fmax(p, (double)__uint_as_float(max_pen[e]));
    b = fmax(b, balance[e]);
  }
  atomicAdd(&s[0], a0);
  atomicAdd(&s[1], a1);
  atomicAdd(&s[2], a2);
  atomicAdd(&s[3], a3);
  // non-negative doubles order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(&m[0]), (unsigned long long)__double_as_longlong(p));
  atomicMax(reinterpret_cast<unsigned long long*>(&m[1]), (unsigned long long)__double_as_longlong(b));
  __syncthreads();
  if (threadIdx.x < 4) out[threadIdx.x] = s[threadIdx.x];
  if (threadIdx.x < 2) out[4 + threadIdx.x] = m[threadIdx.x];
}

}  // namespace

const char* nccl_unique_id(unsigned char* id128) {
  const NcclApi& a = nccl();
  if (!a.ok) return a.why.c_str();
  ncclUniqueId u;
  const ncclResult_t r = a.get_unique_id(&u);
  if (r != ncclSuccess) return a.error_string(r);
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(id128, &u, sizeof u);
  return nullptr;
}

const char* nccl_comm_init(void** comm, int rank, int world, const unsigned char* id128) {
  const NcclApi& a = nccl();
  if (!a.ok) return a.why.c_str();
  ncclUniqueId u;
  std::memcpy(&u, id128, sizeof u);
  ncclComm_t c = nullptr;
  const ncclResult_t r = a.comm_init_rank(&c, world, u, rank);
  if (r != ncclSuccess) return a.error_string(r);
  *comm = c;
  return nullptr;
}

void nccl_comm_destroy(void* comm) {
  if (comm && nccl().ok) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}

const char* launch_step_stats(const SimParams& P, int substeps, double* stats_d, void* comm, cudaStream_t s) {
  k_step_stats<<<1, 256, 0, s>>>(P.env_off, P.run, P.max_pen_bits, P.balance_max, P.lost_count, P.n_env, substeps,
                                 stats_d);
  if (cudaGetLastError() != cudaSuccess) return "step statistics kernel failed to launch";
  if (!comm) return nullptr;
  const NcclApi& a = nccl();
  ncclResult_t r = a.all_reduce(stats_d, stats_d, 4, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm), s);
  if (r == ncclSuccess)
    r = a.all_reduce(stats_d + 4, stats_d + 4, 2, ncclFloat64, ncclMax, static_cast<ncclComm_t>(comm), s);
  return r == ncclSuccess ? nullptr : a.error_string(r);
}

}  // namespace msim_impl
