// gs_peer.cuh — cross-rank synchronisation over peer memory (NVLink on a
// real box, local memory when p ranks are emulated on one device) and the
// reference's pairwise binary16 tree, shared by the collective kernels
// (gs_collective.cu) and the fused collective + LARS kernels (gs_fused.cu).
//
// Every peer kernel is launched over a table of gs_rank_ctx: one entry on a
// multi-GPU box (this GPU's rank), p entries when the p ranks of a job are
// emulated on one device (gs_rank_ctx.rank = 0..p-1).  CTA b of a launch
// serves rank slot b / nb as that rank's local CTA b % nb, so one launch
// carries every emulated rank and all of them are co-resident by
// construction — the waits below then need no help from the scheduler (and
// survive ncu's kernel serialisation).
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

// The launch geometry of a peer kernel as seen by one CTA.
struct PeerCta {
  const gs_rank_ctx* R;  // this CTA's rank
  int lb, nb;            // local CTA index / local grid size
};

__device__ __forceinline__ PeerCta peer_cta(const gs_rank_ctx* __restrict__ ranks, int nb) {
  PeerCta c;
  c.R = ranks + blockIdx.x / nb;
  c.lb = blockIdx.x % nb;
  c.nb = nb;
  return c;
}

// Block-level cross-rank barrier on signal slot `phase`: thread q < p stores
// this CTA's arrival into peer q's slot (a release store, cumulative over
// the block's writes ordered before it by bar.sync — peer stores included),
// then waits for peer q's arrival in our slot.  Epochs only grow: a peer that
// already moved on to a later call has passed this barrier too.
//
// Bounded by time (gs_rank_ctx.timeout_ns, default 120 s), never by spins:
// ranks can legitimately be seconds apart.  A wait that times out records
// 0x80000000 | site << 20 | phase << 16 | peer << 8 | rank in *R.status
// (sticky) and gives up instead of trapping, so the context survives and the
// host reads the diagnosis (GradientPipeline.finish raises it); every later
// barrier of this rank sees the status and drains without waiting, so the
// stream empties in bounded time.
__device__ __forceinline__ void peer_barrier(const uint64_t* __restrict__ sig, const PeerCta& c,
                                             int p, int phase, uint32_t epoch, uint32_t site) {
  __syncthreads();
  GS_DCHECK(c.R->rank >= 0 && c.R->rank < p && c.lb < c.nb && phase < 3, "peer barrier geometry");
  if (threadIdx.x < p) {
    const int q = threadIdx.x;
    const int rank = c.R->rank;
    const size_t slot = ((size_t)phase * c.nb + c.lb) * p;
    st_release_sys(reinterpret_cast<uint32_t*>(sig[q]) + slot + rank, epoch);
    const uint32_t* mine = reinterpret_cast<const uint32_t*>(sig[rank]) + slot + q;
    if ((int32_t)(ld_acquire_sys(mine) - epoch) < 0) {
      uint32_t* status = c.R->status;
      const uint64_t limit = c.R->timeout_ns ? c.R->timeout_ns : kPeerTimeoutNs;
      const uint64_t t0 = globaltimer_ns();
      uint32_t spins = 0;
      while ((int32_t)(ld_relaxed_sys(mine) - epoch) < 0) {
        if ((++spins & 63u) == 0) {
          if (status != nullptr && *reinterpret_cast<volatile uint32_t*>(status) != 0u) break;
          if (globaltimer_ns() - t0 > limit) {
            if (status != nullptr)
              atomicOr(status, 0x80000000u | (site << 20) | ((uint32_t)phase << 16) |
                                   ((uint32_t)q << 8) | (uint32_t)rank);
            else
              __trap();  // no status word to report through
            break;
          }
        }
      }
      (void)ld_acquire_sys(mine);
    }
  }
  __syncthreads();
}

// the codes peer_barrier records in gs_rank_ctx.status (bits 20-27)
constexpr uint32_t kSiteOrderedAllreduce = 1;
constexpr uint32_t kSiteReduceScatter = 2;
constexpr uint32_t kSiteAllgather = 3;
constexpr uint32_t kSiteRsPass1 = 4;
constexpr uint32_t kSiteFence = 5;
constexpr uint32_t kSiteHierarchical = 6;

__device__ __forceinline__ float add_narrow(float a, float b) {
  return gs::widen(gs::narrow(__fadd_rn(a, b)));
}

// fold_f16_tree (collectives.py:273-283) over P widened values: level pairs
// (i, i + s), the odd tail carried to the next level
template <int P>
__device__ __forceinline__ float tree(float (&v)[P]) {
#pragma unroll
  for (int s = 1; s < P; s *= 2) {
#pragma unroll
    for (int i = 0; i + s < P; i += 2 * s) v[i] = add_narrow(v[i], v[i + s]);
  }
  return v[0];
}

// co-resident grid: every CTA of a peer launch may wait for its counterparts,
// so the whole launch (nranks x nb CTAs) must fit on the device at once.
// The clamp depends only on the kernel and the device, so every rank of a
// homogeneous box derives the same nb and the signal slots pair up.
inline int peer_grid(const void* kernel, int threads, size_t smem, int want, int nranks) {
  const int cap = gs_resident_ctas(kernel, threads, smem) / (nranks > 0 ? nranks : 1);
  int nb = want < cap ? want : cap;
  return nb < 1 ? 1 : nb;
}

}  // namespace
