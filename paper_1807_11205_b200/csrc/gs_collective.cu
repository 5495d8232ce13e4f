// gs_collective.cu — bit-exact (reference-ordered) all-reduce of binary16
// buckets over NVLink peer memory, one kernel per rank.
//
// Reference: allreduce_f16 / fold_f16_tree (collectives.py:273-283, 322-340):
// the sum is a pairwise tree over ranks 0..p-1 with widen-add-narrow
// combines.  NCCL sums in ring/NVLS order, which is not that tree; this
// kernel reproduces the tree exactly while moving the same bytes as a ring
// (2(p-1)/p * S inbound per GPU), like the reference's own TCP executor
// (tcp.py:122-130, 250-254: raw chunks go straight to their owner, the
// owner folds in rank order, folded chunks are gathered back).
//
//   A  entry barrier: every rank's bucket is packed (stream order on each
//      rank) -> block b signals block b of every peer and waits for them;
//   B  reduce-scatter: rank r folds its slice of the bucket, reading all p
//      peers' raw values over NVLink (pairwise tree, in registers) and
//      writes the folded slice in place into its own buffer;
//   C  barrier: the slices are complete (per block: block b of rank q only
//      reads the sub-ranges block b of every rank wrote);
//   D  all-gather: rank q copies every other rank's folded sub-range b from
//      that rank's buffer into its own.
// The caller double-buffers the wire across steps, so no exit barrier is
// needed: a rank can only overwrite a buffer after all peers passed the
// entry barrier of the following step, i.e. finished this kernel.
// Buffers come from a symmetric-memory window (torch's _symmetric_memory):
// peer pointers are plain device addresses mapped over NVLink; with p ranks
// emulated on one device they are plain local addresses and one launch
// carries every rank (gs_peer.cuh).  Every wait is time-bounded and reports
// a timeout through gs_rank_ctx.status instead of hanging the GPU.
#include "gs_peer.cuh"

namespace {

constexpr int kThreads = 512;

// [lo, hi) of sub-range `b` of slice `r` for an n-element bucket
__device__ __forceinline__ void subrange(int64_t n, int p, int r, int nb, int b, int64_t& lo,
                                         int64_t& hi) {
  const int64_t per = ((n + p - 1) / p + 7) / 8 * 8;
  const int64_t s0 = min(n, (int64_t)r * per), s1 = min(n, s0 + per);
  const int64_t sub = ((s1 - s0 + nb - 1) / nb + 7) / 8 * 8;
  lo = min(s1, s0 + (int64_t)b * sub);
  hi = min(s1, lo + sub);
  GS_DCHECK(0 <= lo && lo <= hi && hi <= n, "collective sub-range");
}

// fold [lo, hi) of every peer's buffer into mine (pairwise tree, P <= 8);
// PUSH: also store every folded vector into every peer's buffer at the same
// offset (only the slice's owner ever reads or writes those positions, and
// each thread reads its element from all peers before it overwrites it)
template <int P, int Q, bool PUSH>
__device__ __forceinline__ void fold_range_to(const uint16_t* const (&src)[P], uint16_t* const (&dst)[Q],
                                              uint16_t* mine, int64_t lo, int64_t hi, uint32_t& bad) {
  bool vec = gs::is_aligned16(mine + lo);
#pragma unroll
  for (int q = 0; q < P; ++q) vec = vec && gs::is_aligned16(src[q] + lo);
  const int64_t nv = vec ? (hi - lo) / 8 : 0;
  // kU vectors per thread in flight from every peer before any arithmetic
  // (NVLink latency is ~2 us; a ring's worth of bandwidth needs MBs in flight)
  constexpr int kU = P <= 4 ? 4 : 2;
  for (int64_t base = threadIdx.x; base < nv; base += kU * kThreads) {
    uint4 raw[kU][P];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = base + u * kThreads;
      if (i < nv) {
#pragma unroll
        for (int q = 0; q < P; ++q) raw[u][q] = __ldcv(reinterpret_cast<const uint4*>(src[q] + lo) + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = base + u * kThreads;
      if (i >= nv) break;
      uint32_t o[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        float a[P], b[P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
          const float2 f = gs::widen2((&raw[u][q].x)[h]);
          a[q] = f.x;
          b[q] = f.y;
        }
        o[h] = gs::narrow2(tree<P>(a), tree<P>(b));
        bad |= ((o[h] & 0x7C00u) == 0x7C00u) | ((o[h] & 0x7C000000u) == 0x7C000000u);
      }
      const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
      if (PUSH) {
#pragma unroll
        for (int q = 0; q < Q; ++q) reinterpret_cast<uint4*>(dst[q] + lo)[i] = ov;
      } else {
        reinterpret_cast<uint4*>(mine + lo)[i] = ov;
      }
    }
  }
  for (int64_t i = lo + nv * 8 + threadIdx.x; i < hi; i += kThreads) {
    float v[P];
#pragma unroll
    for (int q = 0; q < P; ++q) v[q] = gs::widen(__ldcv(src[q] + i));
    const uint16_t o = gs::narrow(tree<P>(v));
    bad |= (o & 0x7C00u) == 0x7C00u;
    if (PUSH) {
#pragma unroll
      for (int q = 0; q < Q; ++q) dst[q][i] = o;
    } else {
      mine[i] = o;
    }
  }
}

// the folded values stored into `mine` (pull) or into every source buffer
// (PUSH: the slice's final value lands in every peer as it is produced)
template <int P, bool PUSH = false>
__device__ __forceinline__ void fold_range(const uint16_t* const (&src)[P], uint16_t* mine, int64_t lo,
                                           int64_t hi, uint32_t& bad) {
  uint16_t* dst[P];
#pragma unroll
  for (int q = 0; q < P; ++q) dst[q] = const_cast<uint16_t*>(src[q]);
  fold_range_to<P, P, PUSH>(src, dst, mine, lo, hi, bad);
}

// fp32 form (fold_ascending, collectives.py:261-270): acc = b0; acc += b1;
// ... in rank order, each add rounded to fp32 (the mean's division by
// float32(p) is applied by the consumer, LARS pass 1, exactly as the
// reference divides the folded sum).  Same slice discipline as fold_range.
template <int P, bool PUSH = false>
__device__ __forceinline__ void fold_range_f32(const float* const (&src)[P], float* mine,
                                               int64_t lo, int64_t hi, uint32_t& bad) {
  bool vec = gs::is_aligned16(mine + lo);
#pragma unroll
  for (int q = 0; q < P; ++q) vec = vec && gs::is_aligned16(src[q] + lo);
  const int64_t nv = vec ? (hi - lo) / 4 : 0;
  constexpr int kU = P <= 4 ? 4 : 2;
  for (int64_t base = threadIdx.x; base < nv; base += kU * kThreads) {
    float4 raw[kU][P];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = base + u * kThreads;
      if (i < nv) {
#pragma unroll
        for (int q = 0; q < P; ++q) raw[u][q] = __ldcv(reinterpret_cast<const float4*>(src[q] + lo) + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = base + u * kThreads;
      if (i >= nv) break;
      float4 o = raw[u][0];
#pragma unroll
      for (int q = 1; q < P; ++q) {
        o.x = __fadd_rn(o.x, raw[u][q].x);
        o.y = __fadd_rn(o.y, raw[u][q].y);
        o.z = __fadd_rn(o.z, raw[u][q].z);
        o.w = __fadd_rn(o.w, raw[u][q].w);
      }
      bad |= !(gs::is_finite_f32(o.x) && gs::is_finite_f32(o.y) && gs::is_finite_f32(o.z) &&
               gs::is_finite_f32(o.w));
      if (PUSH) {
#pragma unroll
        for (int q = 0; q < P; ++q) reinterpret_cast<float4*>(const_cast<float*>(src[q]) + lo)[i] = o;
      } else {
        reinterpret_cast<float4*>(mine + lo)[i] = o;
      }
    }
  }
  for (int64_t i = lo + nv * 4 + threadIdx.x; i < hi; i += kThreads) {
    float o = __ldcv(src[0] + i);
#pragma unroll
    for (int q = 1; q < P; ++q) o = __fadd_rn(o, __ldcv(src[q] + i));
    bad |= !gs::is_finite_f32(o);
    if (PUSH) {
#pragma unroll
      for (int q = 0; q < P; ++q) const_cast<float*>(src[q])[i] = o;
    } else {
      mine[i] = o;
    }
  }
}

// copy bytes [lo, hi) of a peer buffer into mine
__device__ __forceinline__ void copy_range(const uint8_t* src, uint8_t* mine, int64_t lo, int64_t hi) {
  const bool v2 = ((reinterpret_cast<uintptr_t>(src + lo) | reinterpret_cast<uintptr_t>(mine + lo)) & 15) == 0;
  const int64_t m = v2 ? (hi - lo) / 16 : 0;
  const uint4* s4 = reinterpret_cast<const uint4*>(src + lo);
  uint4* d4 = reinterpret_cast<uint4*>(mine + lo);
  for (int64_t base = threadIdx.x; base < m; base += 8 * kThreads) {
    uint4 t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (base + u * kThreads < m) t[u] = __ldcv(s4 + base + u * kThreads);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (base + u * kThreads < m) d4[base + u * kThreads] = t[u];
  }
  for (int64_t i = lo + m * 16 + threadIdx.x; i < hi; i += kThreads) mine[i] = __ldcv(src + i);
}

// [lo, hi) of sub-range `b` of [s0, s1) split into nb pieces of whole 16 B
__device__ __forceinline__ void split_range(int64_t s0, int64_t s1, int nb, int b, int64_t grain,
                                            int64_t& lo, int64_t& hi) {
  const int64_t sub = ((s1 - s0 + nb - 1) / nb + grain - 1) / grain * grain;
  lo = min(s1, s0 + (int64_t)b * sub);
  hi = min(s1, lo + sub);
}

// A: entry barrier -> B: fold my slice -> C: barrier -> D: gather (pull
// form), or A -> fold my slice and store it into EVERY rank's buffer (push
// form: remote stores overlap the next loads) -> exit barrier.  Same bytes
// either way; push has one barrier and no gather phase.
template <int P, bool PUSH>
__global__ void __launch_bounds__(kThreads)
ordered_allreduce_kernel(const gs_rank_ctx* __restrict__ ranks, int nb,
                         const uint64_t* __restrict__ bufs, const uint64_t* __restrict__ sig,
                         int64_t offset, int64_t n, uint32_t epoch) {
  const PeerCta c = peer_cta(ranks, nb);
  const int rank = c.R->rank;
  if (c.R->epoch_base != nullptr) epoch += *c.R->epoch_base;  // graph-replayable epochs
  const uint16_t* src[P];
#pragma unroll
  for (int q = 0; q < P; ++q) src[q] = reinterpret_cast<const uint16_t*>(bufs[q]) + offset;
  uint16_t* mine = reinterpret_cast<uint16_t*>(bufs[rank]) + offset;

  peer_barrier(sig, c, P, 0, epoch, kSiteOrderedAllreduce);  // A: every bucket packed

  int64_t lo, hi;
  subrange(n, P, rank, nb, c.lb, lo, hi);
  uint32_t bad = 0;
  fold_range<P, PUSH>(src, mine, lo, hi, bad);
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (c.R->nonfinite != nullptr && bad && (threadIdx.x & 31) == 0) atomicOr(c.R->nonfinite, 1u);
  if (PUSH) {
    __threadfence_system();  // this thread's remote stores, before the release below
    peer_barrier(sig, c, P, 1, epoch, kSiteOrderedAllreduce);
    return;
  }
  peer_barrier(sig, c, P, 1, epoch, kSiteOrderedAllreduce);  // C: every slice folded
  // D: gather the other ranks' folded sub-ranges
#pragma unroll 1
  for (int d = 1; d < P; ++d) {
    const int r = (rank + d) % P;
    subrange(n, P, r, nb, c.lb, lo, hi);
    copy_range(reinterpret_cast<const uint8_t*>(src[r]), reinterpret_cast<uint8_t*>(mine), 2 * lo, 2 * hi);
  }
}

// The fp32-wire bucket all-reduce (the reference's own run_experiment path
// fuses fp32 gradients, experiment.py:282-301, 368-399): same structure as
// the binary16 kernel, ascending left fold per element.  For fp32 the
// reference's ring and hierarchical algorithms give the same left fold
// (test_collectives.py:168-173), which does not factor over groups, so this
// one kernel serves both.
template <int P, bool PUSH>
__global__ void __launch_bounds__(kThreads)
ordered_allreduce_f32_kernel(const gs_rank_ctx* __restrict__ ranks, int nb,
                             const uint64_t* __restrict__ bufs, const uint64_t* __restrict__ sig,
                             int64_t offset, int64_t n, uint32_t epoch) {
  const PeerCta c = peer_cta(ranks, nb);
  const int rank = c.R->rank;
  if (c.R->epoch_base != nullptr) epoch += *c.R->epoch_base;
  const float* src[P];
#pragma unroll
  for (int q = 0; q < P; ++q) src[q] = reinterpret_cast<const float*>(bufs[q]) + offset;
  float* mine = reinterpret_cast<float*>(bufs[rank]) + offset;
  peer_barrier(sig, c, P, 0, epoch, kSiteOrderedAllreduce);
  int64_t lo, hi;
  subrange(n, P, rank, nb, c.lb, lo, hi);
  uint32_t bad = 0;
  fold_range_f32<P, PUSH>(src, mine, lo, hi, bad);
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (c.R->nonfinite != nullptr && bad && (threadIdx.x & 31) == 0) atomicOr(c.R->nonfinite, 1u);
  if (PUSH) {
    __threadfence_system();
    peer_barrier(sig, c, P, 1, epoch, kSiteOrderedAllreduce);
    return;
  }
  peer_barrier(sig, c, P, 1, epoch, kSiteOrderedAllreduce);
#pragma unroll 1
  for (int d = 1; d < P; ++d) {
    const int r = (rank + d) % P;
    subrange(n, P, r, nb, c.lb, lo, hi);
    copy_range(reinterpret_cast<const uint8_t*>(src[r]), reinterpret_cast<uint8_t*>(mine), 4 * lo, 4 * hi);
  }
}

// Reduce-scatter with explicit slice bounds (elements, p + 1 entries):
// rank r folds [bounds[r], bounds[r+1]) of every peer's buffer into its own.
// One barrier: the raw values it reads are never written by their owners in
// this call, and the caller double-buffers the wire across steps.
template <int P>
__global__ void __launch_bounds__(kThreads)
ordered_reduce_scatter_kernel(const gs_rank_ctx* __restrict__ ranks, int nb,
                              const uint64_t* __restrict__ bufs, const uint64_t* __restrict__ sig,
                              const int64_t* __restrict__ bounds, uint32_t epoch) {
  const PeerCta c = peer_cta(ranks, nb);
  const int rank = c.R->rank;
  if (c.R->epoch_base != nullptr) epoch += *c.R->epoch_base;
  const uint16_t* src[P];
#pragma unroll
  for (int q = 0; q < P; ++q) src[q] = reinterpret_cast<const uint16_t*>(bufs[q]);
  uint16_t* mine = reinterpret_cast<uint16_t*>(bufs[rank]);
  peer_barrier(sig, c, P, 0, epoch, kSiteReduceScatter);  // every rank's bucket is packed
  int64_t lo, hi;
  split_range(bounds[rank], bounds[rank + 1], nb, c.lb, 8, lo, hi);
  uint32_t bad = 0;
  fold_range<P>(src, mine, lo, hi, bad);
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (c.R->nonfinite != nullptr && bad && (threadIdx.x & 31) == 0) atomicOr(c.R->nonfinite, 1u);
}

// All-gather of byte ranges: rank r owns [bounds[r], bounds[r+1]) of the
// buffer; every rank copies the others' ranges out of their buffers.  Entry
// barrier (the owners' ranges are final) and exit barrier (nobody reads a
// range its owner may overwrite next).
__global__ void __launch_bounds__(kThreads)
ordered_allgather_kernel(const gs_rank_ctx* __restrict__ ranks, int nb, int p,
                         const uint64_t* __restrict__ bufs, const uint64_t* __restrict__ sig,
                         const int64_t* __restrict__ bounds, uint32_t epoch) {
  const PeerCta c = peer_cta(ranks, nb);
  const int rank = c.R->rank;
  if (c.R->epoch_base != nullptr) epoch += *c.R->epoch_base;
  uint8_t* mine = reinterpret_cast<uint8_t*>(bufs[rank]);
  peer_barrier(sig, c, p, 0, epoch, kSiteAllgather);
#pragma unroll 1
  for (int d = 1; d < p; ++d) {
    const int r = (rank + d) % p;
    int64_t lo, hi;
    split_range(bounds[r], bounds[r + 1], nb, c.lb, 16, lo, hi);
    copy_range(reinterpret_cast<const uint8_t*>(bufs[r]), mine, lo, hi);
  }
  peer_barrier(sig, c, p, 1, epoch, kSiteAllgather);
}

// Hierarchical form for Topology(p = K*G, K) with K a power of two: the
// reference's pairwise tree over ranks 0..p-1 then factors into a tree over
// the K members of each group (its first log2(K) levels) followed by a tree
// over the G group partials (the remaining levels, odd tail carried the same
// way), so the paper's two-level exchange (collectives.py:
// 183-235) reproduces allreduce_f16 bit for bit.  The bucket is cut into p
// sub-slices u = j*G + g; rank (g, j) = g*K + j owns sub-slice j*G + g.
//   A  barrier (every rank's raw wire is packed)
//   B  intra-group reduce-scatter: rank (g, j) folds slice j (its group's
//      sub-slices j*G .. j*G+G-1) over the K members' raw values, in place
//   C  barrier; inter-group: rank (g, j) folds its own sub-slice over the G
//      same-offset ranks' group partials, in place
//   D  barrier; all-gather of the p final sub-slices by peer loads
// Every phase works on piece lb of each sub-slice, so CTA lb only ever reads
// what CTA lb of its peers wrote and the per-CTA barriers suffice.  Same
// inbound volume as the flat ring, 2(p-1)/p * S; no exit barrier (the wire
// is double-buffered across calls, as for the flat kernel).
template <int K, int G, bool PUSH>
__global__ void __launch_bounds__(kThreads)
hier_allreduce_kernel(const gs_rank_ctx* __restrict__ ranks, int nb,
                      const uint64_t* __restrict__ bufs, const uint64_t* __restrict__ sig,
                      int64_t offset, int64_t n, uint32_t epoch) {
  constexpr int P = K * G;
  const PeerCta c = peer_cta(ranks, nb);
  const int rank = c.R->rank;
  const int g = rank / K, j = rank % K;
  if (c.R->epoch_base != nullptr) epoch += *c.R->epoch_base;
  uint16_t* mine = reinterpret_cast<uint16_t*>(bufs[rank]) + offset;
  peer_barrier(sig, c, P, 0, epoch, kSiteHierarchical);  // A
  uint32_t bad = 0;
  {  // B: slice j over the group's members, member order
    const uint16_t* grp[K];
#pragma unroll
    for (int m = 0; m < K; ++m) grp[m] = reinterpret_cast<const uint16_t*>(bufs[g * K + m]) + offset;
#pragma unroll 1
    if (PUSH && G == 1) {
      // one group: the group fold is final -- store it into every member
      uint16_t* all[K];
#pragma unroll
      for (int m = 0; m < K; ++m) all[m] = const_cast<uint16_t*>(grp[m]);
      int64_t lo, hi;
      subrange(n, P, j, nb, c.lb, lo, hi);
      fold_range_to<K, K, true>(grp, all, mine, lo, hi, bad);
    } else {
#pragma unroll 1
      for (int gp = 0; gp < G; ++gp) {
        int64_t lo, hi;
        subrange(n, P, j * G + gp, nb, c.lb, lo, hi);
        fold_range<K>(grp, mine, lo, hi, bad);
      }
    }
  }
  if (G > 1) {
    peer_barrier(sig, c, P, 1, epoch, kSiteHierarchical);  // C
    bad = 0;
    const uint16_t* crs[G];
#pragma unroll
    for (int q = 0; q < G; ++q) crs[q] = reinterpret_cast<const uint16_t*>(bufs[q * K + j]) + offset;
    int64_t lo, hi;
    subrange(n, P, j * G + g, nb, c.lb, lo, hi);
    if (PUSH) {
      // the final sub-slice goes straight into every rank (no gather phase)
      uint16_t* all[P];
#pragma unroll
      for (int q = 0; q < P; ++q) all[q] = reinterpret_cast<uint16_t*>(bufs[q]) + offset;
      fold_range_to<G, P, true>(crs, all, mine, lo, hi, bad);
    } else {
      fold_range<G>(crs, mine, lo, hi, bad);
    }
  } else if (!PUSH) {
    // one group: the group partial of sub-slice j is the final value
    int64_t lo, hi;
    subrange(n, P, j, nb, c.lb, lo, hi);
    bad = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += kThreads) bad |= (mine[i] & 0x7C00u) == 0x7C00u;
  }
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (c.R->nonfinite != nullptr && bad && (threadIdx.x & 31) == 0) atomicOr(c.R->nonfinite, 1u);
  if (PUSH) {
    // every final sub-slice was stored into every rank: one exit barrier
    __threadfence_system();
    peer_barrier(sig, c, P, 2, epoch, kSiteHierarchical);
    return;
  }
  peer_barrier(sig, c, P, 2, epoch, kSiteHierarchical);  // D
#pragma unroll 1
  for (int d = 1; d < P; ++d) {
    const int r = (rank + d) % P;
    int64_t lo, hi;
    subrange(n, P, (r % K) * G + r / K, nb, c.lb, lo, hi);
    copy_range(reinterpret_cast<const uint8_t*>(bufs[r]) + 2 * offset,
               reinterpret_cast<uint8_t*>(mine), 2 * lo, 2 * hi);
  }
}

// One-shot form for small buckets (one barrier instead of two): every rank
// pushes its raw binary16 piece into slot [parity][rank] of every peer's
// inbox, fences and signals; after the barrier it folds the p slots of its
// OWN inbox (local memory) in the reference's tree order into its wire.
// (p-1) x S NVLink bytes out per rank instead of 2(p-1)/p x S, so it pays
// only while latency dominates.  CTA lb pushes and folds piece lb, so the
// per-CTA barrier suffices.  Slot reuse: consecutive one-shot calls
// alternate `parity`; a peer can push call c+2 only after this rank arrived
// at call c+1's barrier, i.e. after it folded call c.
template <int P>
__global__ void __launch_bounds__(kThreads)
oneshot_allreduce_kernel(const gs_rank_ctx* __restrict__ ranks, int nb,
                         const uint64_t* __restrict__ bufs, const uint64_t* __restrict__ inbox,
                         const uint64_t* __restrict__ sig, int64_t offset, int64_t n,
                         int64_t cap, uint32_t epoch, uint32_t parity) {
  const PeerCta c = peer_cta(ranks, nb);
  const int rank = c.R->rank;
  if (c.R->epoch_base != nullptr) epoch += *c.R->epoch_base;
  uint16_t* mine = reinterpret_cast<uint16_t*>(bufs[rank]) + offset;
  int64_t lo, hi;
  split_range(0, n, nb, c.lb, 8, lo, hi);
  const size_t slot = ((size_t)parity * P + rank) * (size_t)cap;
  {  // push my raw piece into every rank's inbox (own included)
    uint8_t* dst[P];
#pragma unroll
    for (int q = 0; q < P; ++q) dst[q] = reinterpret_cast<uint8_t*>(inbox[q]) + 2 * slot;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(mine);
    const int64_t b0 = 2 * lo, b1 = 2 * hi;
    const bool vec = gs::is_aligned16(src + b0) && gs::is_aligned16(dst[0] + b0);
    const int64_t nv = vec ? (b1 - b0) / 16 : 0;
    for (int64_t i = threadIdx.x; i < nv; i += kThreads) {
      const uint4 v = __ldcv(reinterpret_cast<const uint4*>(src + b0) + i);
#pragma unroll
      for (int q = 0; q < P; ++q) reinterpret_cast<uint4*>(dst[q] + b0)[i] = v;
    }
    for (int64_t i = b0 + 16 * nv + threadIdx.x; i < b1; i += kThreads) {
      const uint8_t v = src[i];
#pragma unroll
      for (int q = 0; q < P; ++q) dst[q][i] = v;
    }
  }
  __threadfence_system();
  peer_barrier(sig, c, P, 0, epoch, kSiteOrderedAllreduce);
  const uint16_t* src[P];
#pragma unroll
  for (int q = 0; q < P; ++q)
    src[q] = reinterpret_cast<const uint16_t*>(inbox[rank]) + ((size_t)parity * P + q) * cap;
  uint32_t bad = 0;
  fold_range<P>(src, mine, lo, hi, bad);
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (c.R->nonfinite != nullptr && bad && (threadIdx.x & 31) == 0) atomicOr(c.R->nonfinite, 1u);
}

// LL form (no barrier): every 4 bytes of payload (two binary16 values)
// travel as one 8-byte word {payload, epoch} into slot [parity][rank] of
// every rank's inbox (single 64-bit stores, two per 16-byte vector store);
// each rank polls ITS inbox -- all of a thread's words from all p slots are
// loaded at once and re-loaded until every flag carries this call's epoch --
// then folds in the reference's tree order into its wire.  The flag in the
// data is the synchronisation: no fence, no barrier.  Consecutive LL calls
// alternate parity (a peer can write call c+2 only after this rank's call
// c+1 words reached it, i.e. after this rank folded call c).
constexpr int kLLUnits = 4;  // 4-byte units per thread (8 halves, one uint4)

__device__ __forceinline__ void st_relaxed_sys_v2(uint64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_relaxed_sys_v2(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

template <int P>
__global__ void __launch_bounds__(kThreads)
ll_allreduce_kernel(const gs_rank_ctx* __restrict__ ranks, int nb,
                    const uint64_t* __restrict__ bufs, const uint64_t* __restrict__ inbox,
                    int64_t offset, int64_t n, int64_t cap, uint32_t epoch, uint32_t parity) {
  const PeerCta c = peer_cta(ranks, nb);
  const int rank = c.R->rank;
  if (c.R->epoch_base != nullptr) epoch += *c.R->epoch_base;
  uint16_t* mine = reinterpret_cast<uint16_t*>(bufs[rank]) + offset;
  // whole 8-half vectors (n % 8 == 0, 16-byte aligned: the host checks)
  const int64_t nv = n / 8;
  const uint64_t tag = (uint64_t)epoch << 32;
  const size_t slot_words = (size_t)cap / 2;
  uint64_t* dst[P];
#pragma unroll
  for (int q = 0; q < P; ++q)
    dst[q] = reinterpret_cast<uint64_t*>(inbox[q]) + ((size_t)parity * P + rank) * slot_words;
  const int64_t v = (int64_t)c.lb * kThreads + threadIdx.x;  // this thread's vector
  const int64_t stride = (int64_t)nb * kThreads;
  for (int64_t i = v; i < nv; i += stride) {
    const uint4 x = __ldcv(reinterpret_cast<const uint4*>(mine) + i);
    const uint64_t w0 = tag | x.x, w1 = tag | x.y, w2 = tag | x.z, w3 = tag | x.w;
#pragma unroll
    for (int q = 0; q < P; ++q) {
      st_relaxed_sys_v2(dst[q] + 4 * i, w0, w1);
      st_relaxed_sys_v2(dst[q] + 4 * i + 2, w2, w3);
    }
  }
  const uint64_t* src[P];
#pragma unroll
  for (int q = 0; q < P; ++q)
    src[q] = reinterpret_cast<const uint64_t*>(inbox[rank]) + ((size_t)parity * P + q) * slot_words;
  uint32_t bad = 0;
  for (int64_t i = v; i < nv; i += stride) {
    uint64_t w[P][4];
    const uint64_t t0 = globaltimer_ns();
    uint32_t spins = 0;
    for (;;) {
      int missing = -1;  // the first peer whose words are not in yet
#pragma unroll
      for (int q = 0; q < P; ++q) {
        ld_relaxed_sys_v2(src[q] + 4 * i, w[q][0], w[q][1]);
        ld_relaxed_sys_v2(src[q] + 4 * i + 2, w[q][2], w[q][3]);
      }
#pragma unroll
      for (int q = P - 1; q >= 0; --q)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if ((uint32_t)(w[q][k] >> 32) != epoch) missing = q;
      if (missing < 0) break;
      if ((++spins & 63u) == 0) {
        uint32_t* status = c.R->status;
        if (status != nullptr && *reinterpret_cast<volatile uint32_t*>(status) != 0u) break;
        const uint64_t limit = c.R->timeout_ns ? c.R->timeout_ns : kPeerTimeoutNs;
        if (globaltimer_ns() - t0 > limit) {
          if (status != nullptr)  // the first report wins (threads may miss different peers)
            atomicCAS(status, 0u, 0x80000000u | (kSiteOrderedAllreduce << 20) |
                                      ((uint32_t)missing << 8) | (uint32_t)rank);
          else
            __trap();
          break;
        }
      }
    }
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float a[P], b[P];
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const float2 f = gs::widen2((uint32_t)w[q][k]);
        a[q] = f.x;
        b[q] = f.y;
      }
      o[k] = gs::narrow2(tree<P>(a), tree<P>(b));
      bad |= ((o[k] & 0x7C00u) == 0x7C00u) | ((o[k] & 0x7C000000u) == 0x7C000000u);
    }
    reinterpret_cast<uint4*>(mine)[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (c.R->nonfinite != nullptr && bad && (threadIdx.x & 31) == 0) atomicOr(c.R->nonfinite, 1u);
}

__global__ void counter_add_kernel(uint32_t* counter, uint32_t inc) { *counter += inc; }

}  // namespace

// validation shared by the peer entry points
#define GS_PEER_ARGS(fn)                                                                       \
  GS_REQUIRE(p >= 1 && p <= 8, fn ": 1 <= p <= 8 (got %d)", p);                                \
  GS_REQUIRE(nranks >= 1 && nranks <= p, fn ": 1 <= nranks <= p (got %d)", nranks);            \
  GS_REQUIRE(nblocks >= 1 && nblocks <= 1024, fn ": bad block count %d", nblocks);              \
  GS_REQUIRE(epoch != 0, fn ": epoch 0 is the reset value")

extern "C" {

int gs_ordered_allreduce_f16(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* bufs,
                             const uint64_t* sig, int64_t offset, int64_t n, uint32_t epoch,
                             int nblocks, int push, void* stream) {
  GS_PEER_ARGS("gs_ordered_allreduce_f16");
  GS_REQUIRE(n >= 0 && offset >= 0, "gs_ordered_allreduce_f16: negative size/offset");
  if (p == 1 || n == 0) return GS_OK;
  GS_REQUIRE(ranks && bufs && sig, "gs_ordered_allreduce_f16: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
#define GS_OAR(P)                                                                                \
  case P: {                                                                                      \
    if (push) {                                                                                  \
      auto k = ordered_allreduce_kernel<P, true>;                                                \
      const int nb = peer_grid((const void*)k, kThreads, 0, nblocks, nranks);                    \
      k<<<nb * nranks, kThreads, 0, s>>>(ranks, nb, bufs, sig, offset, n, epoch);                \
    } else {                                                                                     \
      auto k = ordered_allreduce_kernel<P, false>;                                               \
      const int nb = peer_grid((const void*)k, kThreads, 0, nblocks, nranks);                    \
      k<<<nb * nranks, kThreads, 0, s>>>(ranks, nb, bufs, sig, offset, n, epoch);                \
    }                                                                                            \
    break;                                                                                       \
  }
  switch (p) {
    GS_OAR(2)
    GS_OAR(3)
    GS_OAR(4)
    GS_OAR(5)
    GS_OAR(6)
    GS_OAR(7)
    GS_OAR(8)
  }
#undef GS_OAR
  return gs_check_launch("gs_ordered_allreduce_f16");
}

int gs_ordered_reduce_scatter_f16(const gs_rank_ctx* ranks, int nranks, int p,
                                  const uint64_t* bufs, const uint64_t* sig, const int64_t* bounds,
                                  uint32_t epoch, int nblocks, void* stream) {
  GS_PEER_ARGS("gs_ordered_reduce_scatter_f16");
  if (p == 1) return GS_OK;
  GS_REQUIRE(ranks && bufs && sig && bounds, "gs_ordered_reduce_scatter_f16: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
#define GS_ORS(P)                                                                                \
  case P: {                                                                                      \
    auto k = ordered_reduce_scatter_kernel<P>;                                                   \
    const int nb = peer_grid((const void*)k, kThreads, 0, nblocks, nranks);                      \
    k<<<nb * nranks, kThreads, 0, s>>>(ranks, nb, bufs, sig, bounds, epoch);                     \
    break;                                                                                       \
  }
  switch (p) {
    GS_ORS(2)
    GS_ORS(3)
    GS_ORS(4)
    GS_ORS(5)
    GS_ORS(6)
    GS_ORS(7)
    GS_ORS(8)
  }
#undef GS_ORS
  return gs_check_launch("gs_ordered_reduce_scatter_f16");
}

int gs_ordered_allgather(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* bufs,
                         const uint64_t* sig, const int64_t* bounds, uint32_t epoch, int nblocks,
                         void* stream) {
  GS_PEER_ARGS("gs_ordered_allgather");
  if (p == 1) return GS_OK;
  GS_REQUIRE(ranks && bufs && sig && bounds, "gs_ordered_allgather: null pointer");
  const int nb = peer_grid((const void*)ordered_allgather_kernel, kThreads, 0, nblocks, nranks);
  ordered_allgather_kernel<<<nb * nranks, kThreads, 0, (cudaStream_t)stream>>>(ranks, nb, p, bufs,
                                                                               sig, bounds, epoch);
  return gs_check_launch("gs_ordered_allgather");
}

int gs_ordered_allreduce_f32(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* bufs,
                             const uint64_t* sig, int64_t offset, int64_t n, uint32_t epoch,
                             int nblocks, int push, void* stream) {
  GS_PEER_ARGS("gs_ordered_allreduce_f32");
  GS_REQUIRE(n >= 0 && offset >= 0, "gs_ordered_allreduce_f32: negative size/offset");
  if (p == 1 || n == 0) return GS_OK;
  GS_REQUIRE(ranks && bufs && sig, "gs_ordered_allreduce_f32: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
#define GS_OAR32(P)                                                                              \
  case P: {                                                                                      \
    if (push) {                                                                                  \
      auto k = ordered_allreduce_f32_kernel<P, true>;                                            \
      const int nb = peer_grid((const void*)k, kThreads, 0, nblocks, nranks);                    \
      k<<<nb * nranks, kThreads, 0, s>>>(ranks, nb, bufs, sig, offset, n, epoch);                \
    } else {                                                                                     \
      auto k = ordered_allreduce_f32_kernel<P, false>;                                           \
      const int nb = peer_grid((const void*)k, kThreads, 0, nblocks, nranks);                    \
      k<<<nb * nranks, kThreads, 0, s>>>(ranks, nb, bufs, sig, offset, n, epoch);                \
    }                                                                                            \
    break;                                                                                       \
  }
  switch (p) {
    GS_OAR32(2)
    GS_OAR32(3)
    GS_OAR32(4)
    GS_OAR32(5)
    GS_OAR32(6)
    GS_OAR32(7)
    GS_OAR32(8)
  }
#undef GS_OAR32
  return gs_check_launch("gs_ordered_allreduce_f32");
}

int gs_oneshot_allreduce_f16(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* bufs,
                             const uint64_t* inbox, const uint64_t* sig, int64_t offset, int64_t n,
                             int64_t cap, uint32_t epoch, int nblocks, uint32_t parity,
                             void* stream) {
  GS_PEER_ARGS("gs_oneshot_allreduce_f16");
  GS_REQUIRE(n >= 0 && offset >= 0 && n <= cap && parity <= 1,
             "gs_oneshot_allreduce_f16: need 0 <= n <= cap (n=%lld, cap=%lld) and parity 0/1",
             (long long)n, (long long)cap);
  if (p == 1 || n == 0) return GS_OK;
  GS_REQUIRE(ranks && bufs && inbox && sig, "gs_oneshot_allreduce_f16: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
#define GS_OS(P)                                                                                 \
  case P: {                                                                                      \
    auto k = oneshot_allreduce_kernel<P>;                                                        \
    const int nb = peer_grid((const void*)k, kThreads, 0, nblocks, nranks);                      \
    k<<<nb * nranks, kThreads, 0, s>>>(ranks, nb, bufs, inbox, sig, offset, n, cap, epoch,       \
                                       parity);                                                  \
    break;                                                                                       \
  }
  switch (p) {
    GS_OS(2)
    GS_OS(3)
    GS_OS(4)
    GS_OS(5)
    GS_OS(6)
    GS_OS(7)
    GS_OS(8)
  }
#undef GS_OS
  return gs_check_launch("gs_oneshot_allreduce_f16");
}

int gs_ll_allreduce_f16(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* bufs,
                        const uint64_t* inbox, int64_t offset, int64_t n, int64_t cap,
                        uint32_t epoch, int nblocks, uint32_t parity, void* stream) {
  GS_PEER_ARGS("gs_ll_allreduce_f16");
  GS_REQUIRE(n >= 0 && offset >= 0 && n <= cap && n % 8 == 0 && offset % 8 == 0 &&
                 parity <= 1 && cap % 8 == 0,
             "gs_ll_allreduce_f16: need whole 8-element vectors at an 8-element offset, "
             "n <= cap and parity 0/1");
  if (p == 1 || n == 0) return GS_OK;
  GS_REQUIRE(ranks && bufs && inbox, "gs_ll_allreduce_f16: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
#define GS_LL(P)                                                                                 \
  case P: {                                                                                      \
    auto k = ll_allreduce_kernel<P>;                                                             \
    const int nb = peer_grid((const void*)k, kThreads, 0, nblocks, nranks);                      \
    k<<<nb * nranks, kThreads, 0, s>>>(ranks, nb, bufs, inbox, offset, n, cap, epoch, parity);   \
    break;                                                                                       \
  }
  switch (p) {
    GS_LL(2)
    GS_LL(3)
    GS_LL(4)
    GS_LL(5)
    GS_LL(6)
    GS_LL(7)
    GS_LL(8)
  }
#undef GS_LL
  return gs_check_launch("gs_ll_allreduce_f16");
}

int gs_hier_allreduce_f16(const gs_rank_ctx* ranks, int nranks, int p, int k,
                          const uint64_t* bufs, const uint64_t* sig, int64_t offset, int64_t n,
                          uint32_t epoch, int nblocks, int push, void* stream) {
  GS_PEER_ARGS("gs_hier_allreduce_f16");
  GS_REQUIRE(k == 2 || k == 4 || k == 8, "gs_hier_allreduce_f16: group size k must be 2, 4 or 8 "
             "(the reference tree factors over groups only for power-of-two k; got %d)", k);
  GS_REQUIRE(p % k == 0, "gs_hier_allreduce_f16: k=%d does not divide p=%d", k, p);
  GS_REQUIRE(n >= 0 && offset >= 0, "gs_hier_allreduce_f16: negative size/offset");
  if (n == 0) return GS_OK;
  GS_REQUIRE(ranks && bufs && sig, "gs_hier_allreduce_f16: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  bool done = false;
#define GS_HAR(K, G)                                                                             \
  if (!done && k == K && p == K * G) {                                                           \
    auto kern = push ? hier_allreduce_kernel<K, G, true> : hier_allreduce_kernel<K, G, false>;    \
    const int nb = peer_grid((const void*)kern, kThreads, 0, nblocks, nranks);                   \
    kern<<<nb * nranks, kThreads, 0, s>>>(ranks, nb, bufs, sig, offset, n, epoch);               \
    done = true;                                                                                 \
  }
  GS_HAR(2, 1)
  GS_HAR(2, 2)
  GS_HAR(2, 3)
  GS_HAR(2, 4)
  GS_HAR(4, 1)
  GS_HAR(4, 2)
  GS_HAR(8, 1)
#undef GS_HAR
  return gs_check_launch("gs_hier_allreduce_f16");
}

int gs_counter_add(uint32_t* counter, uint32_t inc, void* stream) {
  GS_REQUIRE(counter != nullptr, "gs_counter_add: null pointer");
  counter_add_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(counter, inc);
  return gs_check_launch("gs_counter_add");
}

}  // extern "C"
