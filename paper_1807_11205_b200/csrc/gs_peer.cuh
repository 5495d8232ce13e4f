// gs_peer.cuh — cross-GPU synchronisation over NVLink peer memory and the
// reference's pairwise binary16 tree, shared by the collective kernels
// (gs_collective.cu) and the fused collective + LARS kernels (gs_fused.cu).
#pragma once

#include "gs_common.cuh"

namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr uint64_t kPeerTimeoutNs = 120ull * 1000000000ull;

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// block-level cross-rank barrier on signal slot `phase`.
// RELEASE = true: the signal is a release store, cumulative over the block's
// writes ordered before it by the bar.sync (needed when THIS kernel wrote
// data a peer reads after the barrier, or stored into peer memory).
// RELEASE = false: a relaxed signal, for data written by EARLIER kernels into
// this GPU's own memory.  Not used: the signal slots are shared by kernels of
// different grid sizes, and a relaxed signal overtaken by a later kernel's
// signal to the same slot can move the slot's epoch backwards (a 4-GPU
// single-bucket run trapped on exactly such a lost wait); every barrier uses
// release signals.
template <bool RELEASE = true>
__device__ __forceinline__ void peer_barrier(const uint64_t* __restrict__ sig, int rank, int p,
                                             int phase, uint32_t epoch) {
  __syncthreads();
  if (threadIdx.x < p) {
    const int q = threadIdx.x;
    uint32_t* remote = reinterpret_cast<uint32_t*>(sig[q]) +
                       ((size_t)phase * gridDim.x + blockIdx.x) * p + rank;
    if (RELEASE)
      st_release_sys(remote, epoch);
    else
      st_relaxed_sys(remote, epoch);
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(sig[rank]) +
                           ((size_t)phase * gridDim.x + blockIdx.x) * p + q;
    // bounded by time, not spins: ranks can legitimately be seconds apart
    // (first-use setup on one host thread); a peer that never arrives traps
    // after kPeerTimeoutNs instead of hanging the GPU
    // epochs only grow: a peer that already moved on to a later call has
    // passed this barrier too (it only starts a call after finishing the
    // previous one on its stream), so "at least epoch" is the condition
    if ((int32_t)(ld_acquire_sys(mine) - epoch) < 0) {
      // poll with relaxed loads, then one acquire load once the value is in
      const uint64_t t0 = globaltimer_ns();
      while ((int32_t)(ld_relaxed_sys(mine) - epoch) < 0) {
        if (globaltimer_ns() - t0 > kPeerTimeoutNs) __trap();
      }
      (void)ld_acquire_sys(mine);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ float add_narrow(float a, float b) {
  return gs::widen(gs::narrow(__fadd_rn(a, b)));
}

template <int P>
__device__ __forceinline__ float tree(float (&v)[P]) {
#pragma unroll
  for (int s = 1; s < P; s *= 2) {
#pragma unroll
    for (int i = 0; i + s < P; i += 2 * s) v[i] = add_narrow(v[i], v[i + s]);
  }
  return v[0];
}

}  // namespace
