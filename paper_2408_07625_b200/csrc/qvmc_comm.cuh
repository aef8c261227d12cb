// Collectives of the sharded surrogate-E_loc path: the
// sample-set shards are all-gathered and the per-rank energy moments are
// gathered and summed in rank order. Two backends behind one interface:
//  * NCCL over NVLink/NVSwitch (device buffers, the handle's stream).
//    libnccl.so.2 is opened at run time (dlopen), so libqvmc_cuda.so has no
//    link dependency on it and a process that already loaded torch's NCCL
//    reuses that copy (same soname).
//  * a host all-gather callback (MPI, gloo, tests): the library stages the
//    device buffer through pinned host memory around the call.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>

namespace qvmc_b200 {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  const char* error = nullptr;  // why loading failed (null: loaded)
};

inline const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.error = "libnccl.so.2 not found";
      return a;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!a.GetUniqueId || !a.CommInitRank || !a.CommDestroy || !a.AllGather || !a.AllReduce || !a.GetErrorString)
      a.error = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

// rows [begin, end) of rank r in the contiguous balanced split of n rows
// (the first n % world ranks hold one extra row)
__host__ __device__ inline void shard_range(int64_t n, int world, int r, int64_t& begin, int64_t& end) {
  const int64_t base = n / world, rem = n % world;
  begin = r * base + (r < rem ? r : rem);
  end = begin + base + (r < rem ? 1 : 0);
}

// shard -> one padded record block [max_rows][W + 3] words (key words, then
// log|psi|, phase, log p bit patterns): one all-gather moves the whole shard
template <int W>
__global__ void k_pack_shard(const uint64_t* __restrict__ keys, const double* __restrict__ la,
                             const double* __restrict__ ph, const double* __restrict__ lp, int64_t rows,
                             uint64_t* __restrict__ out) {
  constexpr int R = W + 3;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t* o = out + i * R;
#pragma unroll
    for (int w = 0; w < W; ++w) o[w] = keys[i * W + w];
    o[W] = __double_as_longlong(la[i]);
    o[W + 1] = __double_as_longlong(ph[i]);
    o[W + 2] = lp ? __double_as_longlong(lp[i]) : 0ull;
  }
}

// gathered blocks [world][max_rows][W + 3] -> the whole sample set in rank order
template <int W>
__global__ void k_unpack_shards(const uint64_t* __restrict__ in, int world, int64_t max_rows, int64_t n,
                                uint64_t* __restrict__ keys, double* __restrict__ la, double* __restrict__ ph,
                                double* __restrict__ lp) {
  constexpr int R = W + 3;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    // rank of global row j in the balanced split
    const int64_t base = n / world, rem = n % world;
    const int64_t big = rem * (base + 1);
    const int64_t r = j < big ? j / (base + 1) : rem + (j - big) / (base > 0 ? base : 1);
    int64_t b, e;
    shard_range(n, world, static_cast<int>(r), b, e);
    const uint64_t* s = in + (r * max_rows + (j - b)) * R;
#pragma unroll
    for (int w = 0; w < W; ++w) keys[j * W + w] = s[w];
    la[j] = __longlong_as_double(s[W]);
    ph[j] = __longlong_as_double(s[W + 1]);
    lp[j] = __longlong_as_double(s[W + 2]);
  }
}

// [world][n] uint64 -> sum (integer: exact in any order); the host backend's all-reduce
__global__ void k_sum_ranks_u64(const unsigned long long* __restrict__ in, int world, int64_t n,
                                unsigned long long* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    unsigned long long s = 0;
    for (int r = 0; r < world; ++r) s += in[static_cast<int64_t>(r) * n + i];
    out[i] = s;
  }
}

// per-rank moments [world][8] -> sum in rank order (deterministic for a given world size)
__global__ void k_sum_rank_moments(const double* __restrict__ in, int world, double* __restrict__ out) {
  const int k = threadIdx.x;
  if (k < 5) {
    double s = 0.0;
    for (int r = 0; r < world; ++r) s += in[r * 8 + k];
    out[k] = s;
  }
}

}  // namespace qvmc_b200
