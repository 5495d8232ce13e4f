// nvlink_probe.cu — NVLink 5 peer-access microbenchmarks (tools only, not the
// product): how fast can one rank pull its 1/p slice of a buffer out of every
// peer, or push its slice into every peer, with
//   pull_ldg<U>   U x 16 B vector loads per peer in flight per thread
//   pull_tma      cp.async.bulk (TMA) peer -> shared memory, S-stage ring
//   push_st<U>    16 B stores into every peer
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared
//        -Xcompiler -fPIC tools/nvlink_probe.cu -o tools/_probe/libnvprobe.so
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

template <int U>
__global__ void __launch_bounds__(256) pull_ldg(const uint64_t* __restrict__ peers, int p, int rank,
                                                int64_t slice16, uint4* __restrict__ out) {
  uint32_t acc = 0;
  const int64_t base = rank * slice16;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x * U + threadIdx.x; i < slice16; i += stride) {
    uint4 v[U][8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q >= p) break;
      const uint4* src = reinterpret_cast<const uint4*>(peers[q]) + base;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * blockDim.x < slice16) v[u][q] = __ldcv(src + i + u * blockDim.x);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q >= p) break;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * blockDim.x < slice16) acc ^= v[u][q].x ^ v[u][q].y ^ v[u][q].z ^ v[u][q].w;
    }
  }
  if (acc == 0x12345678u) out[0] = make_uint4(acc, 0, 0, 0);
}

template <int U>
__global__ void __launch_bounds__(256) push_st(const uint64_t* __restrict__ peers, int p, int rank,
                                               int64_t slice16, const uint4* __restrict__ src) {
  const int64_t base = rank * slice16;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x * U + threadIdx.x; i < slice16; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * blockDim.x < slice16) v[u] = src[base + i + u * blockDim.x];
    for (int q = 0; q < p; ++q) {
      uint4* dst = reinterpret_cast<uint4*>(peers[q]) + base;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * blockDim.x < slice16) dst[i + u * blockDim.x] = v[u];
    }
  }
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// each CTA walks blocks of `blk` bytes: block j of the rank's slice from peer
// j % p; thread 0 keeps S-1 bulk copies in flight; every thread folds the
// landed stage (xor) before it is refilled
template <int S>
__global__ void __launch_bounds__(256) pull_tma(const uint64_t* __restrict__ peers, int p, int rank,
                                                int64_t slice_bytes, int blk, uint4* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[S];
  const int64_t nblk_peer = slice_bytes / blk;
  const int64_t nblk = nblk_peer * p;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int64_t j, int s) {
    const int q = (int)(j % p);
    const int64_t k = j / p;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(peers[q]) + rank * slice_bytes + k * blk;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar[s])),
                 "r"(blk));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(smem + (size_t)s * blk)),
        "l"(src), "r"(blk), "r"(smem_addr(&bar[s]))
        : "memory");
  };
  int64_t first = blockIdx.x, step = gridDim.x;
  int it = 0;
  if (threadIdx.x == 0)
    for (int s = 0; s < S - 1; ++s)
      if (first + s * step < nblk) issue(first + s * step, s);
  uint32_t acc = 0;
  for (int64_t j = first; j < nblk; j += step, ++it) {
    const int s = it % S;
    const uint32_t par = (it / S) & 1;
    if (threadIdx.x == 0) {
      const int64_t jn = j + (int64_t)(S - 1) * step;
      if (jn < nblk) issue(jn, (it + S - 1) % S);
    }
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
          : "=r"(done)
          : "r"(smem_addr(&bar[s])), "r"(par));
    const uint4* st = reinterpret_cast<const uint4*>(smem + (size_t)s * blk);
    for (int i = threadIdx.x; i < blk / 16; i += blockDim.x) {
      const uint4 v = st[i];
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    __syncthreads();  // stage s is consumed before thread 0 refills it
  }
  if (acc == 0x12345678u) out[0] = make_uint4(acc, 0, 0, 0);
}

}  // namespace

extern "C" {

// mode 0: pull_ldg<U>, 1: push_st<U>, 2: pull_tma<S = U>
int probe_run(int mode, int U, const uint64_t* peers, int p, int rank, int64_t slice_bytes,
              void* scratch, int grid, int blk, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t s16 = slice_bytes / 16;
  uint4* out = static_cast<uint4*>(scratch);
  if (mode == 0) {
    if (U == 1) pull_ldg<1><<<grid, 256, 0, s>>>(peers, p, rank, s16, out);
    else if (U == 2) pull_ldg<2><<<grid, 256, 0, s>>>(peers, p, rank, s16, out);
    else pull_ldg<4><<<grid, 256, 0, s>>>(peers, p, rank, s16, out);
  } else if (mode == 1) {
    if (U == 1) push_st<1><<<grid, 256, 0, s>>>(peers, p, rank, s16, out);
    else if (U == 2) push_st<2><<<grid, 256, 0, s>>>(peers, p, rank, s16, out);
    else push_st<4><<<grid, 256, 0, s>>>(peers, p, rank, s16, out);
  } else {
    const size_t sm = (size_t)U * blk;
    if (U == 2) {
      cudaFuncSetAttribute(pull_tma<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      pull_tma<2><<<grid, 256, sm, s>>>(peers, p, rank, slice_bytes, blk, out);
    } else if (U == 4) {
      cudaFuncSetAttribute(pull_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      pull_tma<4><<<grid, 256, sm, s>>>(peers, p, rank, slice_bytes, blk, out);
    } else {
      cudaFuncSetAttribute(pull_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      pull_tma<8><<<grid, 256, sm, s>>>(peers, p, rank, slice_bytes, blk, out);
    }
  }
  return (int)cudaGetLastError();
}
}
