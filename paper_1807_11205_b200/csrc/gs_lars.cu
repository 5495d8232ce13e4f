// gs_lars.cu — the fused mixed-precision LARS update over a segment table.
//
// Reference semantics (pkg/src/gradsync):
//   experiment.py:401-412  merged mean grads -> LossScale.update (finite test
//                          on the still-scaled mean) -> unscale by the
//                          pre-update scale -> grad-norm metric -> lars_step
//   lars.py:158-181        global finite gate; per group eff = g (+ wd*w),
//                          local = eta*||w||/(||eff||+eps) (fp64) or 1,
//                          scale = f32(local*gamma), v = m*v + scale*eff,
//                          w -= v, w16 = f32_to_f16(w)
//
// Kernels (all HBM-bound; no tensor cores — nothing here is a contraction):
//   pass1        reads g (2 B fp16 or 4 B fp32) + w (4 B, LARS groups only),
//                optionally writes the raw g chunk into the fusion wire
//                (gs_segment.gcopy, the fused packer), emits per-chunk fp64
//                partials {sum w^2, sum eff^2, sum g^2} and the two
//                non-finite flag bits.                     6 (+2) B/elem
//   pass1_trust  pass1 + the trust ratio: the last CTA of every segment folds
//                the segment's partials in chunk order (no extra launch).
//   trust        the same fold as a separate single-CTA kernel.
//   pass2        early-exits on the flags, otherwise reads g, w, v and writes
//                v, w, w16.                                 20 B/elem
// Chunks never straddle a segment, so a CTA handles one (segment, range) pair
// with uniform control flow, and its partial sums land in a fixed slot: the
// reduction order depends only on the chunk table, never on timing.
//
// Specialisation (host hints, gradsync_b200.h GS_HINT_*): with power-of-two p
// and loss scale the mean and unscale are one exact multiplication by `mul`
// (one FMUL per element), and for fp16 input with mul <= 1 the finite tests reduce to
// an integer test of the binary16 exponent field; full 8192-element chunks
// issue all their loads before any arithmetic.
#include "gs_lars_device.cuh"

namespace {

// FUSE: the last CTA to finish a segment (per-segment arrival counter) folds
// that segment's partials in chunk order and writes its trust ratio; the last
// segment to finish writes the empty segments and the grad norm.  Which CTA
// arrives last is timing-dependent, the result is not: the fold always runs
// over the same chunk range in the same fixed tree.
template <bool F16, bool POW2, bool RAWFLAG, bool GNORM, bool FUSE>
__global__ void __launch_bounds__(kThreads, F16 ? GS_P1_MINB : 1)
lars_pass1_kernel(const gs_segment* __restrict__ segs, int nseg, int nseg_active,
                  const gs_chunk* __restrict__ chunks, int chunk0,
                  const gs_step_params* __restrict__ params, double* __restrict__ partials,
                  uint32_t* __restrict__ flags, uint32_t* __restrict__ counters,
                  float* __restrict__ seg_scale, double* __restrict__ seg_out,
                  double* __restrict__ grad_norm_out) {
  using T = typename G<F16>::T;
  const int c = chunk0 + blockIdx.x;
  const gs_chunk ch = chunks[c];
  const gs_segment* sgp = segs + ch.seg;
  const uint32_t sflags = sgp->flags;
  const T* g = static_cast<const T*>(sgp->g) + ch.start;
  const float* w = sgp->w + ch.start;
  uint16_t* gcopy = F16 && sgp->gcopy != nullptr ? static_cast<uint16_t*>(sgp->gcopy) + ch.start
                                                 : nullptr;
  Ctx cx;
  cx.u.load(params);
  cx.mul = params->mul;
  cx.wd = params->weight_decay;
  const bool lars = (sflags & GS_SEG_LARS_ENABLED) != 0;
  const bool decay = (cx.u.mode & GS_MODE_DECAY) && !(sflags & GS_SEG_DECAY_EXEMPT);
  Acc a;
  if (lars && decay)
    p1_chunk<F16, POW2, RAWFLAG, GNORM, true, true>(g, w, gcopy, ch.len, cx, a);
  else if (lars)
    p1_chunk<F16, POW2, RAWFLAG, GNORM, true, false>(g, w, gcopy, ch.len, cx, a);
  else
    p1_chunk<F16, POW2, RAWFLAG, GNORM, false, false>(g, w, gcopy, ch.len, cx, a);
  if (lars && !decay) {
    a.se = a.sg;  // eff == g exactly: same terms, same order
    if (!GNORM) a.sg = 0.0;
  }
  uint32_t fl = a.fl | ((a.raw & 0x80008000u) ? kBoth : 0u);
  fl = __reduce_or_sync(0xFFFFFFFFu, fl);
  if (fl != 0u && (threadIdx.x & 31) == 0) atomicOr(flags, fl);
  double sw = a.sw, se = a.se, sg = a.sg;
  gs::block_sum3<kThreads>(sw, se, sg);
  if (!FUSE) {
    if (threadIdx.x == 0) {
      partials[3 * (int64_t)c + 0] = sw;
      partials[3 * (int64_t)c + 1] = se;
      partials[3 * (int64_t)c + 2] = sg;
    }
    return;
  }
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    partials[3 * (int64_t)c + 0] = sw;
    partials[3 * (int64_t)c + 1] = se;
    partials[3 * (int64_t)c + 2] = sg;
    const uint32_t prev = arrive_release(&counters[ch.seg]);
    s_last = (prev + 1 == (uint32_t)sgp->chunk_count);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // fold this segment's chunk partials: fixed strided order + fixed tree
  const int cb = sgp->chunk_begin, cn = sgp->chunk_count;
  double x = 0.0, y = 0.0, z = 0.0;
  for (int i = threadIdx.x; i < cn; i += kThreads) {
    const double* pp = partials + 3 * (int64_t)(cb + i);
    x += __ldcg(pp + 0);
    y += __ldcg(pp + 1);
    z += __ldcg(pp + 2);
  }
  __syncthreads();  // block_sum3's shared scratch is reused
  gs::block_sum3<kThreads>(x, y, z);
  if (threadIdx.x == 0) {
    trust_eval(sflags, x, y, z, params, seg_scale + ch.seg, seg_out + 4 * (int64_t)ch.seg);
    const uint32_t prev = arrive_release(&counters[nseg]);
    if (prev + 1 == (uint32_t)nseg_active) {
      __threadfence();
      for (int s = 0; s < nseg; ++s)
        if (segs[s].chunk_count == 0)
          trust_eval(segs[s].flags, 0.0, 0.0, 0.0, params, seg_scale + s, seg_out + 4 * (int64_t)s);
      __threadfence();
      if (grad_norm_out != nullptr) *grad_norm_out = grad_norm_eval(seg_out, nseg);
    }
  }
}

// ------------------------------------------------ pass 1, TMA-pipelined
// Persistent, warp-specialised form of pass 1 for fp16 gradients (one CTA per
// SM).  Warp 8 is the producer: for every chunk of the CTA (chunks
// blockIdx.x, blockIdx.x + gridDim.x, ...) it waits for a free stage of a
// kStages-deep ring, arms the stage's `full` mbarrier with the byte count and
// streams the chunk's gradient (16 KB) and master (32 KB) into shared memory
// with bulk-async copies (the TMA engine: cp.async.bulk + complete_tx).
// Warps 0-7 are consumers: they wait on `full`, reduce the chunk from shared
// memory, hand their warp partial over through shared memory and release the
// stage on its `empty` mbarrier — no __syncthreads in the loop.  The last
// consumer warp of a chunk (shared-memory arrival counter) folds the 8 warp
// partials in warp order into the chunk partial and, for the fused trust,
// does the per-segment arrival; so the chunk partial and everything after it
// are identical to the register-staged kernel.  Chunks that are
// not 16-byte aligned (or not a multiple of 8 elements) are reduced from
// global memory directly by the consumers.
#ifndef GS_TMA_STAGES
#define GS_TMA_STAGES 2   // stages per CTA
#endif
#ifndef GS_TMA_CTAS
#define GS_TMA_CTAS 2     // CTAs per SM (consumer warps per SM = 8 x this)
#endif
constexpr int kStages = GS_TMA_STAGES;
constexpr int kStageG = kFullChunk * 2;      // 16 KB of binary16
constexpr int kStageW = kFullChunk * 4;      // 32 KB of fp32 master
constexpr int kStageBytes = kStageG + kStageW;
constexpr int kConsumerWarps = kThreads / 32;  // 8
constexpr int kProducerWarp = kConsumerWarps;  // warp 8
constexpr int kFinisherWarp = kConsumerWarps + 1;  // warp 9
constexpr int kTmaThreads = kThreads + 64;
constexpr int kRing = 64;                      // finisher queue entries

// Everything a consumer needs about the staged chunk (written by the
// producer before it arms the stage; the mbarrier orders it), so consumers
// never touch global metadata on the critical path.
struct StageMeta {
  const uint16_t* g;
  const float* w;
  uint16_t* gcopy;
  int32_t len, seg, chunk;
  uint32_t sflags;
  int32_t bulk;
  int32_t pad;
};

struct FinishItem {
  double sw, se, sg;
  int32_t chunk, seg;
};

struct TmaShared {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  StageMeta meta[kStages];
  double red[kStages][kConsumerWarps][3];
  uint32_t cnt[kStages];
  FinishItem ring[kRing];
  volatile uint32_t ring_tail;  // written by consumers (last warp of a chunk)
  volatile uint32_t ring_head;  // written by the finisher
};
constexpr int kTmaSmem = kStages * kStageBytes + (int)sizeof(TmaShared);

template <bool POW2, bool RAWFLAG, bool GNORM, bool LARS, bool DECAY>
__device__ __forceinline__ void p1_smem(const uint16_t* sg, const float* sw, uint16_t* gcopy,
                                        int len, const Ctx& cx, Acc& a) {
  const int nv = len / 8;
#pragma unroll 4
  for (int i = threadIdx.x; i < nv; i += kThreads) {
    const uint4 gv = reinterpret_cast<const uint4*>(sg)[i];
    // the fused packer: plain 128-bit stores of the staged gradient (a bulk
    // shared->global store would queue behind the next stages' loads in the
    // SM's TMA unit and hold the stage)
    if (gcopy != nullptr) reinterpret_cast<uint4*>(gcopy)[i] = gv;
    F8 wv{};
    if (LARS) {
      wv.a = reinterpret_cast<const float4*>(sw)[2 * i];
      wv.b = reinterpret_cast<const float4*>(sw)[2 * i + 1];
    }
    p1_vec<true, POW2, RAWFLAG, GNORM, LARS, DECAY>(gv, wv, cx, a);
  }
}

// chunk reduced straight from global memory (misaligned / odd-length chunks)
template <bool POW2, bool RAWFLAG, bool GNORM>
__device__ __noinline__ void p1_global_chunk(const StageMeta& m, const Ctx& cx, Acc& a) {
  const bool lars = (m.sflags & GS_SEG_LARS_ENABLED) != 0;
  const bool decay = (cx.u.mode & GS_MODE_DECAY) && !(m.sflags & GS_SEG_DECAY_EXEMPT);
  if (lars && decay)
    p1_chunk<true, POW2, RAWFLAG, GNORM, true, true>(m.g, m.w, m.gcopy, m.len, cx, a);
  else if (lars)
    p1_chunk<true, POW2, RAWFLAG, GNORM, true, false>(m.g, m.w, m.gcopy, m.len, cx, a);
  else
    p1_chunk<true, POW2, RAWFLAG, GNORM, false, false>(m.g, m.w, m.gcopy, m.len, cx, a);
}

// Chunk partial + (FUSE) segment arrival, trust fold, empty segments and
// grad norm for one finished chunk — executed by the finisher warp, so its
// global-memory latency never sits on the consumers' critical path.
template <bool FUSE>
__device__ __forceinline__ void finish_chunk_warp(const gs_segment* __restrict__ segs, int nseg,
                                                  int nseg_active, const FinishItem& it,
                                                  const gs_step_params* __restrict__ params,
                                                  double* __restrict__ partials,
                                                  uint32_t* __restrict__ counters,
                                                  float* __restrict__ seg_scale,
                                                  double* __restrict__ seg_out,
                                                  double* __restrict__ grad_norm_out) {
  const int lane = threadIdx.x & 31;
  const int c = it.chunk, seg = it.seg;
  uint32_t last = 0;
  if (lane == 0) {
    partials[3 * (int64_t)c + 0] = it.sw;
    partials[3 * (int64_t)c + 1] = it.se;
    partials[3 * (int64_t)c + 2] = it.sg;
    if (FUSE) last = (arrive_release(&counters[seg]) + 1 == (uint32_t)segs[seg].chunk_count);
  }
  if (!FUSE) return;
  last = __shfl_sync(0xFFFFFFFFu, last, 0);
  if (!last) return;
  __threadfence();
  // fold the segment's chunk partials in a fixed order: exactly the
  // block-wide fold of the register-staged kernel (256 lanes strided, then
  // warps in order), done by one warp, so both kernels produce the same bits
  const gs_segment* sp = segs + seg;
  const int cb = sp->chunk_begin, cn = sp->chunk_count;
  double x = 0.0, y = 0.0, z = 0.0;
  for (int w8 = 0; w8 < kConsumerWarps; ++w8) {
    double px = 0.0, py = 0.0, pz = 0.0;
    for (int i = w8 * 32 + lane; i < cn; i += kThreads) {
      const double* pp = partials + 3 * (int64_t)(cb + i);
      px += __ldcg(pp + 0);
      py += __ldcg(pp + 1);
      pz += __ldcg(pp + 2);
    }
    px = gs::warp_sum(px);
    py = gs::warp_sum(py);
    pz = gs::warp_sum(pz);
    if (w8 == 0) {
      x = px; y = py; z = pz;
    } else {
      x += px; y += py; z += pz;
    }
  }
  if (lane == 0) {
    trust_eval(sp->flags, x, y, z, params, seg_scale + seg, seg_out + 4 * (int64_t)seg);
    if (arrive_release(&counters[nseg]) + 1 == (uint32_t)nseg_active) {
      __threadfence();
      for (int s2 = 0; s2 < nseg; ++s2)
        if (segs[s2].chunk_count == 0)
          trust_eval(segs[s2].flags, 0.0, 0.0, 0.0, params, seg_scale + s2, seg_out + 4 * (int64_t)s2);
      __threadfence();
      if (grad_norm_out != nullptr) *grad_norm_out = grad_norm_eval(seg_out, nseg);
    }
  }
}

template <bool POW2, bool RAWFLAG, bool GNORM, bool FUSE>
__global__ void __launch_bounds__(kTmaThreads, GS_TMA_CTAS)
lars_pass1_tma_kernel(const gs_segment* __restrict__ segs, int nseg, int nseg_active,
                      const gs_chunk* __restrict__ chunks, int chunk0, int nchunk,
                      const gs_step_params* __restrict__ params, double* __restrict__ partials,
                      uint32_t* __restrict__ flags, uint32_t* __restrict__ counters,
                      float* __restrict__ seg_scale, double* __restrict__ seg_out,
                      double* __restrict__ grad_norm_out) {
  extern __shared__ __align__(128) uint8_t smem[];
  TmaShared& sh = *reinterpret_cast<TmaShared*>(smem + kStages * kStageBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nmine = blockIdx.x < nchunk ? (nchunk - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      gs::mbar_init(&sh.full[s], 1);
      gs::mbar_init(&sh.empty[s], kConsumerWarps);
      sh.cnt[s] = 0;
    }
    sh.ring_tail = 0;
    sh.ring_head = 0;
    gs::mbar_fence_init();
  }
  __syncthreads();

  if (warp == kProducerWarp) {
    // ------------------------------------------------------ producer warp
    // the 32 lanes fetch the metadata of 32 upcoming chunks at once, so the
    // dependent chunk -> segment loads cost one latency per 32 chunks
    StageMeta mine{};
    for (int base = 0; base < nmine; base += 32) {
      const int kk = base + lane;
      if (kk < nmine) {
        const int c = chunk0 + blockIdx.x + kk * gridDim.x;
        const gs_chunk ch = chunks[c];
        const gs_segment* sp = segs + ch.seg;
        const uint32_t fl = sp->flags;
        const uint16_t* g = static_cast<const uint16_t*>(sp->g) + ch.start;
        const float* w = sp->w + ch.start;
        uint16_t* gc = sp->gcopy != nullptr ? static_cast<uint16_t*>(sp->gcopy) + ch.start : nullptr;
        const bool lars = (fl & GS_SEG_LARS_ENABLED) != 0;
        // a stage holds kFullChunk elements: longer chunks take the global path
        const bool bulk = (ch.len & 7) == 0 && ch.len <= kFullChunk && gs::is_aligned16(g) &&
                          (!lars || gs::is_aligned16(w)) && (gc == nullptr || gs::is_aligned16(gc));
        mine = StageMeta{g, w, gc, ch.len, ch.seg, c, fl, bulk ? 1 : 0, 0};
      }
      const int cnt = min(32, nmine - base);
      for (int j = 0; j < cnt; ++j) {
        StageMeta m;
        m.g = reinterpret_cast<const uint16_t*>(__shfl_sync(0xFFFFFFFFu, (unsigned long long)mine.g, j));
        m.w = reinterpret_cast<const float*>(__shfl_sync(0xFFFFFFFFu, (unsigned long long)mine.w, j));
        m.gcopy = reinterpret_cast<uint16_t*>(__shfl_sync(0xFFFFFFFFu, (unsigned long long)mine.gcopy, j));
        m.len = __shfl_sync(0xFFFFFFFFu, mine.len, j);
        m.seg = __shfl_sync(0xFFFFFFFFu, mine.seg, j);
        m.chunk = __shfl_sync(0xFFFFFFFFu, mine.chunk, j);
        m.sflags = __shfl_sync(0xFFFFFFFFu, mine.sflags, j);
        m.bulk = __shfl_sync(0xFFFFFFFFu, mine.bulk, j);
        m.pad = 0;
        const int k = base + j;
        const int s = k % kStages;
        const uint32_t ph = (uint32_t)(k / kStages) & 1u;
        if (lane == 0) {
          gs::mbar_wait(&sh.empty[s], ph ^ 1u);  // fresh barrier: passes at once
          sh.meta[s] = m;
          if (m.bulk) {
            const uint32_t bg = 2u * m.len;
            const uint32_t bw = (m.sflags & GS_SEG_LARS_ENABLED) ? 4u * m.len : 0u;
            uint8_t* st = smem + s * kStageBytes;
            gs::mbar_arrive_expect_tx(&sh.full[s], bg + bw);
            gs::bulk_g2s(st, m.g, bg, &sh.full[s]);
            if (bw) gs::bulk_g2s(st + kStageG, m.w, bw, &sh.full[s]);
          } else {
            gs::mbar_arrive_expect_tx(&sh.full[s], 0);
          }
        }
        __syncwarp();
      }
    }
    return;
  }

  if (warp == kFinisherWarp) {
    // ------------------------------------------------------ finisher warp
    for (int k = 0; k < nmine; ++k) {
      uint32_t spins = 0;
      while (sh.ring_tail == (uint32_t)k) {
        __nanosleep(64);
        if (++spins > (1u << 26)) __trap();
      }
      __threadfence_block();
      const FinishItem it = sh.ring[k % kRing];
      finish_chunk_warp<FUSE>(segs, nseg, nseg_active, it, params, partials, counters, seg_scale,
                              seg_out, grad_norm_out);
      __syncwarp();
      if (lane == 0) sh.ring_head = (uint32_t)(k + 1);
    }
    return;
  }

  // ------------------------------------------------------ consumer warps
  Ctx cx;
  cx.u.load(params);
  cx.mul = params->mul;
  cx.wd = params->weight_decay;
  for (int k = 0; k < nmine; ++k) {
    const int s = k % kStages;
    const uint32_t ph = (uint32_t)(k / kStages) & 1u;
    gs::mbar_wait(&sh.full[s], ph);
    const StageMeta m = sh.meta[s];
    const bool lars = (m.sflags & GS_SEG_LARS_ENABLED) != 0;
    const bool decay = (cx.u.mode & GS_MODE_DECAY) && !(m.sflags & GS_SEG_DECAY_EXEMPT);
    Acc a;
    if (m.bulk) {
      const uint16_t* sgp = reinterpret_cast<const uint16_t*>(smem + s * kStageBytes);
      const float* swp = reinterpret_cast<const float*>(smem + s * kStageBytes + kStageG);
      if (lars && decay)
        p1_smem<POW2, RAWFLAG, GNORM, true, true>(sgp, swp, m.gcopy, m.len, cx, a);
      else if (lars)
        p1_smem<POW2, RAWFLAG, GNORM, true, false>(sgp, swp, m.gcopy, m.len, cx, a);
      else
        p1_smem<POW2, RAWFLAG, GNORM, false, false>(sgp, swp, m.gcopy, m.len, cx, a);
    } else {
      p1_global_chunk<POW2, RAWFLAG, GNORM>(m, cx, a);
    }
    if (lars && !decay) {
      a.se = a.sg;
      if (!GNORM) a.sg = 0.0;
    }
    uint32_t fl = a.fl | ((a.raw & 0x80008000u) ? kBoth : 0u);
    fl = __reduce_or_sync(0xFFFFFFFFu, fl);
    const double sw = gs::warp_sum(a.sw), se = gs::warp_sum(a.se), sg = gs::warp_sum(a.sg);
    uint32_t order = 0;
    if (lane == 0) {
      if (fl) atomicOr(flags, fl);
      sh.red[s][warp][0] = sw;
      sh.red[s][warp][1] = se;
      sh.red[s][warp][2] = sg;
      __threadfence_block();
      order = atomicAdd(&sh.cnt[s], 1u);
      if (order == kConsumerWarps - 1) {
        // last warp of this chunk: fold the warp partials in warp order and
        // queue the chunk for the finisher
        __threadfence_block();
        double tw = sh.red[s][0][0], te = sh.red[s][0][1], tg = sh.red[s][0][2];
#pragma unroll
        for (int i = 1; i < kConsumerWarps; ++i) {
          tw += sh.red[s][i][0];
          te += sh.red[s][i][1];
          tg += sh.red[s][i][2];
        }
        sh.cnt[s] = 0;
        uint32_t spins = 0;
        while ((uint32_t)k - sh.ring_head >= (uint32_t)kRing) {  // queue full (rare)
          __nanosleep(64);
          if (++spins > (1u << 26)) __trap();
        }
        sh.ring[k % kRing] = FinishItem{tw, te, tg, m.chunk, m.seg};
        __threadfence_block();
        sh.ring_tail = (uint32_t)(k + 1);
      }
    }
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(gs::smem_u32(&sh.empty[s]))
                   : "memory");
  }
}

// ----------------------------------------------------------------- trust
// One CTA per segment folds the segment's chunk partials (256-strided, then
// the fixed block tree: the same order as the fused and TMA paths), and the
// last CTA to finish (arrival counter, zeroed with the flags) writes the grad
// norm, summing the per-segment sums in segment order.
__global__ void __launch_bounds__(kThreads)
lars_trust_kernel(const gs_segment* __restrict__ segs, int nseg, const double* __restrict__ partials,
                  const gs_step_params* __restrict__ params, float* __restrict__ seg_scale,
                  double* __restrict__ seg_out, double* __restrict__ grad_norm_out,
                  uint32_t* __restrict__ counter, const uint64_t* __restrict__ peer_flags,
                  int npeers, uint32_t* __restrict__ flags) {
  gs::griddep_wait();                 // pass 1's partials are complete
  gs::griddep_launch_dependents();    // let pass 2 start issuing its loads now
  if (npeers > 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    // sharded update: the step is rejected if any rank saw a non-finite value
    uint32_t f = 0;
    for (int q = 0; q < npeers; ++q) f |= *reinterpret_cast<const volatile uint32_t*>(peer_flags[q]);
    if (f) atomicOr(flags, f);
  }
  const int s = blockIdx.x;
  const int cb = segs[s].chunk_begin, cn = segs[s].chunk_count;
  double x = 0.0, y = 0.0, z = 0.0;
  for (int i = threadIdx.x; i < cn; i += kThreads) {
    const double* pp = partials + 3 * (int64_t)(cb + i);
    x += pp[0];
    y += pp[1];
    z += pp[2];
  }
  gs::block_sum3<kThreads>(x, y, z);
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    trust_eval(segs[s].flags, x, y, z, params, seg_scale + s, seg_out + 4 * (int64_t)s);
    s_last = grad_norm_out != nullptr && arrive_release(counter) + 1 == (uint32_t)nseg;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  extern __shared__ double sq[];  // nseg doubles (dynamic)
  for (int i = threadIdx.x; i < nseg; i += kThreads) sq[i] = __ldcg(seg_out + 4 * (int64_t)i + 3);
  __syncthreads();
  if (threadIdx.x == 0) {
    // experiment.py:408-411: sqrt of the per-group dots summed in group order
    double acc = 0.0;
    for (int i = 0; i < nseg; ++i) acc = __dadd_rn(acc, sq[i]);
    *grad_norm_out = __dsqrt_rn(acc);
  }
}

// `scale_of()` yields the segment's fp32 trust scale; it is called by every
// thread after the first batch's loads are in flight, so a scale that has to
// be derived on the spot (TRUST) overlaps the loads' latency.
template <bool F16, bool POW2, bool DECAY, typename ScaleFn>
__device__ __forceinline__ void p2_chunk(const typename G<F16>::T* __restrict__ g,
                                         float* __restrict__ w, float* __restrict__ v,
                                         uint16_t* __restrict__ w16, int len, const Ctx& cx,
                                         ScaleFn scale_of) {
  using Gt = G<F16>;
  const bool vec = gs::is_aligned16(g) && gs::is_aligned16(w) && gs::is_aligned16(v) &&
                   gs::is_aligned16(w16);
  const int nv = vec ? len / 8 : 0;
  const int t = threadIdx.x;
  // batches of two vectors per thread: both vectors' loads are issued before
  // the arithmetic and stores (stores cannot alias the next batch's loads,
  // but the compiler cannot prove it through the casts)
  int done = 0;
  float s = 0.0f;
  bool have_s = false;
  for (; done + 2 * kThreads <= nv; done += 2 * kThreads) {
    const int i0 = done + t, i1 = i0 + kThreads;
    const typename Gt::V g0 = Gt::ld(g + 8 * i0), g1 = Gt::ld(g + 8 * i1);
    const F8 w0 = ld8(w, i0), w1 = ld8(w, i1), v0 = ld8(v, i0), v1 = ld8(v, i1);
    if (!have_s) {  // uniform: every thread runs the first batch
      if (!scale_of(s)) return;
      have_s = true;
    }
    p2_vec<F16, POW2, DECAY>(g0, w0, v0, w, v, w16, i0, cx, s);
    p2_vec<F16, POW2, DECAY>(g1, w1, v1, w, v, w16, i1, cx, s);
  }
  if (!have_s && !scale_of(s)) return;
  for (int i = done + t; i < nv; i += kThreads) {
    const typename Gt::V gv = Gt::ld(g + 8 * i);
    p2_vec<F16, POW2, DECAY>(gv, ld8(w, i), ld8(v, i), w, v, w16, i, cx, s);
  }
  for (int i = nv * 8 + t; i < len; i += kThreads) {
    float2 ww = make_float2(w[i], 0.0f), vv = make_float2(v[i], 0.0f);
    p2_pair<POW2, DECAY>(make_float2(Gt::one(g + i), 0.0f), ww, vv, cx, s);
    v[i] = vv.x;
    w[i] = ww.x;
    w16[i] = gs::narrow(ww.x);
  }
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// TRUST: the CTA derives its segment's trust ratio itself — the fold of
// gs_lars_trust (256-strided + fixed block tree, so the same bits in every
// CTA of the segment) — while its first batch of loads is in flight; the
// first CTA of a segment publishes seg_scale/seg_out and the last to do so
// (arrival counter) the empty segments and grad norm.  This removes the
// separate trust launch and its serial tail.
template <bool F16, bool POW2, bool TRUST>
__global__ void __launch_bounds__(kThreads, 4)
lars_pass2_kernel(const gs_segment* __restrict__ segs, int nseg, int nseg_active,
                  const gs_chunk* __restrict__ chunks,
                  int chunk0, const gs_step_params* __restrict__ params,
                  const double* __restrict__ partials, float* __restrict__ seg_scale,
                  double* __restrict__ seg_out, double* __restrict__ grad_norm_out,
                  uint32_t* __restrict__ counter, const uint32_t* __restrict__ flags,
                  uint32_t flag_mask) {
  using T = typename G<F16>::T;
  // lars.py:161-163 — a non-finite step mutates nothing (the non-TRUST form
  // checks after griddep_wait: it may run ahead of the trust kernel)
  if (TRUST && (*flags & flag_mask)) return;
  const int c = chunk0 + blockIdx.x;
  const gs_chunk ch = chunks[c];
  const gs_segment* sgp = segs + ch.seg;
  const uint32_t sflags = sgp->flags;
  const T* g = static_cast<const T*>(sgp->g) + ch.start;
  float* w = sgp->w + ch.start;
  float* v = sgp->v + ch.start;
  uint16_t* w16 = sgp->w16 + ch.start;
  Ctx cx;
  cx.u.load(params);
  cx.mul = params->mul;
  cx.wd = params->weight_decay;
  cx.m = params->momentum;
  // returns false when the step is rejected (nothing may be stored)
  auto scale_of = [&](float& out) -> bool {
    if (!TRUST) {
      // launched with PDL behind the trust kernel: everything above and the
      // first batch of loads overlapped it; scales and flags come after
      gs::griddep_wait();
      if (*flags & flag_mask) return false;
      out = seg_scale[ch.seg];
      return true;
    }
    __shared__ float s_scale;
    __shared__ int s_last;
    const int cb = sgp->chunk_begin, cn = sgp->chunk_count;
    double x = 0.0, y = 0.0, z = 0.0;
    for (int i = threadIdx.x; i < cn; i += kThreads) {
      const double* pp = partials + 3 * (int64_t)(cb + i);
      x += pp[0];
      y += pp[1];
      z += pp[2];
    }
    gs::block_sum3<kThreads>(x, y, z);
    if (threadIdx.x == 0) {
      double o[4];
      float sc;
      trust_eval(sflags, x, y, z, params, &sc, o);
      s_scale = sc;
      s_last = 0;
      if (c == cb) {  // the segment's first chunk publishes its statistics
        seg_scale[ch.seg] = sc;
        double* so = seg_out + 4 * (int64_t)ch.seg;
        so[0] = o[0];
        so[1] = o[1];
        so[2] = o[2];
        so[3] = o[3];
        if (grad_norm_out != nullptr && counter != nullptr &&
            arrive_release(counter) + 1 == (uint32_t)nseg_active) {
          __threadfence();
          for (int q = 0; q < nseg; ++q)
            if (segs[q].chunk_count == 0)
              trust_eval(segs[q].flags, 0.0, 0.0, 0.0, params, seg_scale + q, seg_out + 4 * (int64_t)q);
          *grad_norm_out = grad_norm_eval(seg_out, nseg);
        }
      }
    }
    __syncthreads();
    out = s_scale;
    return true;
  };
  const bool decay = (cx.u.mode & GS_MODE_DECAY) && !(sflags & GS_SEG_DECAY_EXEMPT);
  if (decay)
    p2_chunk<F16, POW2, true>(g, w, v, w16, ch.len, cx, scale_of);
  else
    p2_chunk<F16, POW2, false>(g, w, v, w16, ch.len, cx, scale_of);
}

// ------------------------------------------------------------ dispatch
int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <bool P, bool R, bool N, bool FUSE>
int launch_tma(const gs_segment* segs, int nseg, int nseg_active, const gs_chunk* chunks, int chunk0,
               int nchunk, const gs_step_params* params, double* partials, uint32_t* flags,
               uint32_t* counters, float* seg_scale, double* seg_out, double* gn, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(lars_pass1_tma_kernel<P, R, N, FUSE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem) != cudaSuccess)
      return gs_check_launch("gs_lars_pass1 (smem attribute)");
    attr = true;
  }
  int grid = GS_TMA_CTAS * sm_count();
  if (grid > nchunk) grid = nchunk;
  lars_pass1_tma_kernel<P, R, N, FUSE><<<grid, kTmaThreads, kTmaSmem, s>>>(
      segs, nseg, nseg_active, chunks, chunk0, nchunk, params, partials, flags, counters, seg_scale,
      seg_out, gn);
  return gs_check_launch(FUSE ? "gs_lars_pass1_trust" : "gs_lars_pass1");
}

template <bool FUSE>
int launch_pass1(const gs_segment* segs, int nseg, int nseg_active, const gs_chunk* chunks,
                 int chunk0, int nchunk, int f16, const gs_step_params* params, uint32_t hint,
                 double* partials, uint32_t* flags, uint32_t* counters, float* seg_scale,
                 double* seg_out, double* gn, cudaStream_t s) {
  const bool pow2 = hint & GS_HINT_POW2, raw = f16 && pow2 && (hint & GS_HINT_RAWFLAG),
             gnorm = hint & GS_HINT_GRADNORM;
  if (f16 && !(hint & GS_HINT_NO_BULK)) {
#define GS_T(P, R, N)                                                                              \
  return launch_tma<P, R, N, FUSE>(segs, nseg, nseg_active, chunks, chunk0, nchunk, params, partials, \
                                   flags, counters, seg_scale, seg_out, gn, s)
    if (raw) {
      if (gnorm) GS_T(true, true, true); else GS_T(true, true, false);
    } else if (pow2) {
      if (gnorm) GS_T(true, false, true); else GS_T(true, false, false);
    } else {
      if (gnorm) GS_T(false, false, true); else GS_T(false, false, false);
    }
#undef GS_T
  }
#define GS_P1(F, P, R, N)                                                                      \
  lars_pass1_kernel<F, P, R, N, FUSE><<<nchunk, kThreads, 0, s>>>(                             \
      segs, nseg, nseg_active, chunks, chunk0, params, partials, flags, counters, seg_scale,    \
      seg_out, gn)
  if (f16) {
    if (raw) {
      if (gnorm) GS_P1(true, true, true, true); else GS_P1(true, true, true, false);
    } else if (pow2) {
      if (gnorm) GS_P1(true, true, false, true); else GS_P1(true, true, false, false);
    } else {
      if (gnorm) GS_P1(true, false, false, true); else GS_P1(true, false, false, false);
    }
  } else {
    if (pow2) {
      if (gnorm) GS_P1(false, true, false, true); else GS_P1(false, true, false, false);
    } else {
      if (gnorm) GS_P1(false, false, false, true); else GS_P1(false, false, false, false);
    }
  }
#undef GS_P1
  return gs_check_launch(FUSE ? "gs_lars_pass1_trust" : "gs_lars_pass1");
}

}  // namespace

extern "C" {

int gs_lars_pass1(const gs_segment* segs, const gs_chunk* chunks, int chunk0, int nchunk,
                  int g_is_f16, const gs_step_params* params, uint32_t hint, double* partials,
                  uint32_t* flags, void* stream) {
  GS_REQUIRE(nchunk >= 0 && chunk0 >= 0, "gs_lars_pass1: bad chunk range");
  if (nchunk == 0) return GS_OK;
  GS_REQUIRE(segs && chunks && params && partials && flags, "gs_lars_pass1: null pointer");
  return launch_pass1<false>(segs, 0, 0, chunks, chunk0, nchunk, g_is_f16, params, hint, partials,
                             flags, nullptr, nullptr, nullptr, nullptr, (cudaStream_t)stream);
}

int gs_lars_pass1_trust(const gs_segment* segs, int nseg, int nseg_active, const gs_chunk* chunks,
                        int chunk0, int nchunk, int g_is_f16, const gs_step_params* params,
                        uint32_t hint, double* partials, uint32_t* flags, uint32_t* counters,
                        float* seg_scale, double* seg_out, double* grad_norm_out, void* stream) {
  GS_REQUIRE(nchunk >= 0 && chunk0 >= 0, "gs_lars_pass1_trust: bad chunk range");
  GS_REQUIRE(nseg_active >= 1 && nseg_active <= nseg,
             "gs_lars_pass1_trust: need 1 <= nseg_active <= nseg (use gs_lars_trust otherwise)");
  if (nchunk == 0) return GS_OK;
  GS_REQUIRE(segs && chunks && params && partials && flags && counters && seg_scale && seg_out,
             "gs_lars_pass1_trust: null pointer");
  return launch_pass1<true>(segs, nseg, nseg_active, chunks, chunk0, nchunk, g_is_f16, params, hint,
                            partials, flags, counters, seg_scale, seg_out, grad_norm_out,
                            (cudaStream_t)stream);
}

int gs_lars_trust(const gs_segment* segs, int nseg, const double* partials,
                  const gs_step_params* params, float* seg_scale, double* seg_out,
                  double* grad_norm_out, uint32_t* counter, const uint64_t* peer_flags,
                  int npeers, uint32_t* flags, void* stream) {
  GS_REQUIRE(nseg >= 0, "gs_lars_trust: negative segment count");
  if (nseg == 0) return GS_OK;
  GS_REQUIRE(segs && partials && params && seg_scale && seg_out, "gs_lars_trust: null pointer");
  GS_REQUIRE(grad_norm_out == nullptr || counter != nullptr,
             "gs_lars_trust: the grad norm needs a zeroed arrival counter");
  GS_REQUIRE(nseg <= 24 * 1024, "gs_lars_trust: at most 24576 segments");
  GS_REQUIRE(npeers == 0 || (peer_flags != nullptr && flags != nullptr),
             "gs_lars_trust: peer flags need both tables");
  const size_t dyn = grad_norm_out != nullptr ? sizeof(double) * (size_t)nseg : 0;
  if (dyn > 48 * 1024) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(lars_trust_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
      attr = true;
    }
  }
  const cudaError_t e = gs_launch_pdl(lars_trust_kernel, dim3(nseg), dim3(kThreads), dyn,
                                      (cudaStream_t)stream, segs, nseg, partials, params, seg_scale,
                                      seg_out, grad_norm_out, counter, peer_flags, npeers, flags);
  if (e != cudaSuccess) {
    gs_set_error("gs_lars_trust: %s", cudaGetErrorString(e));
    return GS_ECUDA;
  }
  return gs_check_launch("gs_lars_trust");
}

int gs_lars_pass2(const gs_segment* segs, const gs_chunk* chunks, int chunk0, int nchunk,
                  int g_is_f16, const gs_step_params* params, uint32_t hint,
                  const float* seg_scale, const uint32_t* flags, uint32_t flag_mask,
                  void* stream) {
  GS_REQUIRE(nchunk >= 0 && chunk0 >= 0, "gs_lars_pass2: bad chunk range");
  if (nchunk == 0) return GS_OK;
  GS_REQUIRE(segs && chunks && params && seg_scale && flags, "gs_lars_pass2: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const bool pow2 = hint & GS_HINT_POW2;
  float* sc = const_cast<float*>(seg_scale);
  cudaError_t err = cudaSuccess;
#define GS_P2(F, P)                                                                              \
  err = gs_launch_pdl(lars_pass2_kernel<F, P, false>, dim3(nchunk), dim3(kThreads), 0, s, segs, 0, \
                      0, chunks, chunk0, params, (const double*)nullptr, sc, (double*)nullptr,     \
                      (double*)nullptr, (uint32_t*)nullptr, flags, flag_mask)
  if (g_is_f16) {
    if (pow2) GS_P2(true, true); else GS_P2(true, false);
  } else {
    if (pow2) GS_P2(false, true); else GS_P2(false, false);
  }
#undef GS_P2
  if (err != cudaSuccess) {
    gs_set_error("gs_lars_pass2: %s", cudaGetErrorString(err));
    return GS_ECUDA;
  }
  return gs_check_launch("gs_lars_pass2");
}

int gs_lars_pass2_trust(const gs_segment* segs, int nseg, int nseg_active, const gs_chunk* chunks,
                        int chunk0, int nchunk, int g_is_f16, const gs_step_params* params, uint32_t hint,
                        const double* partials, float* seg_scale, double* seg_out,
                        double* grad_norm_out, uint32_t* counter, const uint32_t* flags,
                        uint32_t flag_mask, void* stream) {
  GS_REQUIRE(nchunk >= 0 && chunk0 >= 0 && nseg_active >= 1 && nseg_active <= nseg,
             "gs_lars_pass2_trust: bad range (1 <= nseg_active <= nseg)");
  if (nchunk == 0) return GS_OK;
  GS_REQUIRE(segs && chunks && params && partials && seg_scale && seg_out && flags,
             "gs_lars_pass2_trust: null pointer");
  GS_REQUIRE(grad_norm_out == nullptr || counter != nullptr,
             "gs_lars_pass2_trust: the grad norm needs a zeroed arrival counter");
  cudaStream_t s = (cudaStream_t)stream;
  const bool pow2 = hint & GS_HINT_POW2;
#define GS_P2T(F, P)                                                                             \
  lars_pass2_kernel<F, P, true><<<nchunk, kThreads, 0, s>>>(segs, nseg, nseg_active, chunks,     \
                                                            chunk0, params,                      \
                                                            partials, seg_scale, seg_out,        \
                                                            grad_norm_out, counter, flags,       \
                                                            flag_mask)
  if (g_is_f16) {
    if (pow2) GS_P2T(true, true); else GS_P2T(true, false);
  } else {
    if (pow2) GS_P2T(false, true); else GS_P2T(false, false);
  }
#undef GS_P2T
  return gs_check_launch("gs_lars_pass2_trust");
}

}  // extern "C"
