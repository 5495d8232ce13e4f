// gs_fused.cu — collective + LARS pass fused into single kernels over NVLink
// peer memory (the sharded, ZeRO-1 form of the step).
//
//   gs_rs_pass1   reduce-scatter fused with pass 1: the owner of a chunk reads
//                 every peer's raw binary16 values of that chunk over NVLink,
//                 folds them in the reference's pairwise-tree order
//                 (fold_f16_tree, collectives.py:273-283), stores the reduced
//                 chunk in its own wire and immediately runs pass 1 on the
//                 folded registers (no re-read), then PUSHES the chunk's fp64
//                 partials to every peer and ORs its flags into every peer's
//                 flag word (remote stores / atomics) — no gather kernel.
//   gs_pass2_push pass 2 over the owned chunks that also pushes each updated
//                 binary16 working-weight vector to every peer's working
//                 arena — no all-gather kernel.
//   gs_peer_fence one CTA per rank: every rank has finished the previous
//                 kernels' remote stores (system fence + release/acquire
//                 signals).
// Every kernel runs over a gs_rank_ctx table (gs_peer.cuh): one rank per
// launch on a multi-GPU box, all p ranks in one launch when they are
// emulated on a single device.
// The per-chunk arithmetic (p1_vec / p2_pair / block_sum3, thread-to-element
// mapping, fold order) is exactly the LARS kernels', so the partials, trust
// scales and updates are bit-identical to the replicated path.
#include "gs_lars_device.cuh"
#include "gs_peer.cuh"

namespace {

// vectors per thread in flight per batch (P raw loads each).  One vector
// keeps the kernel at <= 64 registers for P = 2 / 4 (4 co-resident CTAs per
// SM) and <= 80 for P = 8 (3 per SM): the reduce-scatter is bound by NVLink
// load latency per chunk, so more resident CTAs = more chunks in flight
// (two vectors took 124-206 registers, 1-2 CTAs per SM)
template <int P>
constexpr int kU = 1;

template <int P, bool POW2, bool RAWFLAG, bool GNORM, bool LARS, bool DECAY>
__device__ __forceinline__ void rs_p1_chunk(const uint16_t* const (&src)[P], uint16_t* mine,
                                            const float* __restrict__ w, int len, const Ctx& cx,
                                            Acc& a) {
  bool vec = gs::is_aligned16(mine) && (!LARS || gs::is_aligned16(w));
#pragma unroll
  for (int q = 0; q < P; ++q) vec = vec && gs::is_aligned16(src[q]);
  const int nv = vec ? len / 8 : 0;
  const int t = threadIdx.x;
  // vectors t, t+256, ... in increasing order: the summation order of pass 1
  for (int base = t; base < nv; base += kU<P> * kThreads) {
    uint4 raw[kU<P>][P];
    F8 wv[kU<P>];
#pragma unroll
    for (int u = 0; u < kU<P>; ++u) {
      const int i = base + u * kThreads;
      if (i < nv) {
#pragma unroll
        for (int q = 0; q < P; ++q) raw[u][q] = __ldcv(reinterpret_cast<const uint4*>(src[q]) + i);
        if (LARS) wv[u] = ldw(w + 8 * i);
      }
    }
#pragma unroll
    for (int u = 0; u < kU<P>; ++u) {
      const int i = base + u * kThreads;
      if (i >= nv) break;
      uint4 o;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        float x[P], y[P];
#pragma unroll
        for (int q = 0; q < P; ++q) {
          const float2 f = gs::widen2((&raw[u][q].x)[h]);
          x[q] = f.x;
          y[q] = f.y;
        }
        (&o.x)[h] = gs::narrow2(tree<P>(x), tree<P>(y));
      }
      reinterpret_cast<uint4*>(mine)[i] = o;
      p1_vec<true, POW2, RAWFLAG, GNORM, LARS, DECAY>(o, LARS ? wv[u] : F8{}, cx, a);
    }
  }
  for (int i = nv * 8 + t; i < len; i += kThreads) {
    float v[P];
#pragma unroll
    for (int q = 0; q < P; ++q) v[q] = gs::widen(__ldcv(src[q] + i));
    const uint16_t h = gs::narrow(tree<P>(v));
    mine[i] = h;
    if (RAWFLAG) a.raw |= raw_nonfinite_bits(h);
    Acc b;
    p1_pair<POW2, RAWFLAG, GNORM, LARS, DECAY>(make_float2(gs::widen(h), 0.0f),
                                               make_float2(LARS ? w[i] : 0.0f, 0.0f), cx, b);
    a.sw += b.sw;
    a.se += b.se;
    a.sg += b.sg;
    a.fl |= b.fl;
  }
}

// residency: every CTA waits for its peers at entry, so the whole launch
// must fit at once (peer_grid clamps nb with the occupancy calculator)
// (the power-of-two form with per-element finite tests needs more than 64
// registers at P = 4: 3 CTAs / SM so it does not spill)
template <int P, bool POW2, bool RAWFLAG>
constexpr int kRsMinBlocks = !POW2 ? 2 : (P <= 4 && RAWFLAG) ? 4 : 3;

// owned chunks [own_off[b0], own_off[b1]) of the rank's chunk list
__device__ __forceinline__ void own_range(const gs_rank_ctx& R, int b0, int b1, int& i0, int& i1) {
  i0 = R.own_off[b0];
  i1 = R.own_off[b1];
  GS_DCHECK(0 <= i0 && i0 <= i1, "owned chunk list range");
}

template <int P, bool POW2, bool RAWFLAG, bool GNORM>
__global__ void __launch_bounds__(kThreads, (kRsMinBlocks<P, POW2, RAWFLAG>))
rs_pass1_kernel(const gs_rank_ctx* __restrict__ ranks, int nb, const uint64_t* __restrict__ wires,
                const uint64_t* __restrict__ sig, const uint64_t* __restrict__ peer_partials,
                const uint64_t* __restrict__ peer_ctl, int b0, int b1, const gs_step_params params,
                uint32_t parity, uint32_t epoch) {
  const PeerCta pc = peer_cta(ranks, nb);
  const gs_rank_ctx& R = *pc.R;
  if (R.epoch_base != nullptr) epoch += *R.epoch_base;
  // every rank's raw gradients are in its wire -- a release signal,
  // cumulative over the stream-ordered stores that put them there
  peer_barrier(sig, pc, P, 0, epoch, kSiteRsPass1);
  Ctx cx;
  cx.u.load(&params);
  cx.mul = params.mul;
  cx.wd = params.weight_decay;
  // src[q] = wires[q] + (chunk's byte offset in my reduced wire): the raw
  // wires are only read, the folded chunk goes to my reduced wire
  const uint8_t* mybase = reinterpret_cast<const uint8_t*>(R.red);
  int i0, i1;
  own_range(R, b0, b1, i0, i1);
  uint32_t flag_acc = 0;
  for (int ci = i0 + pc.lb; ci < i1; ci += nb) {
    const int c = R.own_list[ci];
    const gs_chunk ch = R.chunks[c];
    const gs_segment* sp = R.segs + ch.seg;
    GS_DCHECK(c >= 0 && ch.len >= 0 && ch.start + ch.len <= sp->n, "rs_pass1: owned chunk");
    const uint32_t sflags = sp->flags;
    uint16_t* mine = const_cast<uint16_t*>(static_cast<const uint16_t*>(sp->g)) + ch.start;
    const size_t off = reinterpret_cast<const uint8_t*>(mine) - mybase;
    const uint16_t* src[P];
#pragma unroll
    for (int q = 0; q < P; ++q) src[q] = reinterpret_cast<const uint16_t*>(wires[q] + off);
    const float* w = sp->w + ch.start;
    const bool lars = (sflags & GS_SEG_LARS_ENABLED) != 0;
    const bool decay = (cx.u.mode & GS_MODE_DECAY) && !(sflags & GS_SEG_DECAY_EXEMPT);
    Acc a;
    if (lars && decay)
      rs_p1_chunk<P, POW2, RAWFLAG, GNORM, true, true>(src, mine, w, ch.len, cx, a);
    else if (lars)
      rs_p1_chunk<P, POW2, RAWFLAG, GNORM, true, false>(src, mine, w, ch.len, cx, a);
    else
      rs_p1_chunk<P, POW2, RAWFLAG, GNORM, false, false>(src, mine, w, ch.len, cx, a);
    if (lars && !decay) {
      a.se = a.sg;
      if (!GNORM) a.sg = 0.0;
    }
    flag_acc |= a.fl | ((a.raw & 0x80008000u) ? kBoth : 0u);
    double sw = a.sw, se = a.se, sg = a.sg;
    gs::block_sum3<kThreads>(sw, se, sg);
    // push the chunk partial into every rank's partials (own included)
    __shared__ double s_part[3];
    if (threadIdx.x == 0) {
      s_part[0] = sw;
      s_part[1] = se;
      s_part[2] = sg;
    }
    __syncthreads();
    if (threadIdx.x < P) {
      double* dst = reinterpret_cast<double*>(peer_partials[threadIdx.x]) + 3 * (int64_t)c;
      dst[0] = s_part[0];
      dst[1] = s_part[1];
      dst[2] = s_part[2];
    }
    __syncthreads();  // block_sum3 scratch and s_part are reused next chunk
  }
  flag_acc = __reduce_or_sync(0xFFFFFFFFu, flag_acc);
  if (flag_acc != 0u && (threadIdx.x & 31) == 0) {
    for (int q = 0; q < P; ++q)
      atomicOr_system(&reinterpret_cast<gs_ctl*>(peer_ctl[q])->flags[parity], flag_acc);
  }
}

// pass 2 over owned chunks, pushing the binary16 result into every peer's
// working arena (one 16-byte store per peer per vector)
template <bool POW2, bool DECAY>
__device__ __forceinline__ void p2_push_chunk(const uint16_t* __restrict__ g, float* __restrict__ w,
                                              float* __restrict__ v, uint16_t* __restrict__ w16,
                                              int len, const Ctx& cx, float s,
                                              const uint64_t* __restrict__ peer_working, int p,
                                              size_t woff) {
  using Gt = G<true>;
  const bool vec = gs::is_aligned16(g) && gs::is_aligned16(w) && gs::is_aligned16(v) &&
                   gs::is_aligned16(w16);
  const int nv = vec ? len / 8 : 0;
  const int t = threadIdx.x;
  // one 8-element vector: update in registers, local v/w streaming stores,
  // binary16 result stored into every rank's working arena (own included)
  auto one = [&](const uint4& gv, const F8& wv, const F8& vv, int i) {
    float2 ww[4] = {make_float2(wv.a.x, wv.a.y), make_float2(wv.a.z, wv.a.w),
                    make_float2(wv.b.x, wv.b.y), make_float2(wv.b.z, wv.b.w)};
    float2 xv[4] = {make_float2(vv.a.x, vv.a.y), make_float2(vv.a.z, vv.a.w),
                    make_float2(vv.b.x, vv.b.y), make_float2(vv.b.z, vv.b.w)};
#pragma unroll
    for (int q = 0; q < 4; ++q) p2_pair<POW2, DECAY>(Gt::pair(gv, q), ww[q], xv[q], cx, s);
    float4* vp = reinterpret_cast<float4*>(v) + 2 * i;
    float4* wp = reinterpret_cast<float4*>(w) + 2 * i;
    __stcs(vp, make_float4(xv[0].x, xv[0].y, xv[1].x, xv[1].y));
    __stcs(vp + 1, make_float4(xv[2].x, xv[2].y, xv[3].x, xv[3].y));
    __stcs(wp, make_float4(ww[0].x, ww[0].y, ww[1].x, ww[1].y));
    __stcs(wp + 1, make_float4(ww[2].x, ww[2].y, ww[3].x, ww[3].y));
    const uint4 h = make_uint4(pack_w16(ww[0]), pack_w16(ww[1]), pack_w16(ww[2]), pack_w16(ww[3]));
    for (int q = 0; q < p; ++q)
      reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(peer_working[q]) + woff)[i] = h;
  };
  // batches of two vectors per thread with every load issued first (the
  // stores cannot alias the next batch's loads, which the compiler cannot
  // prove through the casts) -- the same batching as lars_pass2
  int done = 0;
  for (; done + 2 * kThreads <= nv; done += 2 * kThreads) {
    const int i0 = done + t, i1 = i0 + kThreads;
    const uint4 g0 = Gt::ld(g + 8 * i0), g1 = Gt::ld(g + 8 * i1);
    const F8 w0 = ld8(w, i0), w1 = ld8(w, i1), v0 = ld8(v, i0), v1 = ld8(v, i1);
    one(g0, w0, v0, i0);
    one(g1, w1, v1, i1);
  }
  for (int i = done + t; i < nv; i += kThreads) one(Gt::ld(g + 8 * i), ld8(w, i), ld8(v, i), i);
  for (int i = nv * 8 + t; i < len; i += kThreads) {
    float2 ww = make_float2(w[i], 0.0f), vv = make_float2(v[i], 0.0f);
    p2_pair<POW2, DECAY>(make_float2(Gt::one(g + i), 0.0f), ww, vv, cx, s);
    v[i] = vv.x;
    w[i] = ww.x;
    const uint16_t h = gs::narrow(ww.x);
    for (int q = 0; q < p; ++q)
      reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(peer_working[q]) + woff)[i] = h;
  }
}

// wait (one thread) until *w == epoch: a gpu-scope acquire, bounded like
// every peer wait (gives up when the rank's status records a failure or
// after the rank's timeout)
__device__ __forceinline__ void wait_epoch(const uint32_t* w, uint32_t epoch, const gs_rank_ctx& R) {
  uint32_t v, spins = 0;
  const uint64_t t0 = globaltimer_ns();
  const uint64_t limit = R.timeout_ns ? R.timeout_ns : kPeerTimeoutNs;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(w) : "memory");
    if (v == epoch) break;
    if ((++spins & 63u) == 0) {
      if (R.status != nullptr && *reinterpret_cast<volatile uint32_t*>(R.status) != 0u) break;
      if (globaltimer_ns() - t0 > limit) break;
    }
  }
}

template <bool POW2>
__device__ __forceinline__ void pass2_push_cta(const PeerCta& pc, const uint64_t* __restrict__ peer_working,
                                               int p, int b0, int b1, const gs_step_params& params,
                                               uint32_t parity, uint32_t flag_mask,
                                               uint32_t ready_epoch);
__device__ __forceinline__ void trust_fence_cta(const gs_rank_ctx* __restrict__ ranks, int nranks,
                                                const uint64_t* __restrict__ sig, int p,
                                                uint32_t epoch, int nseg, int nchunk,
                                                const gs_step_params& params, uint32_t parity,
                                                int b, bool publish);

// one CTA per owned chunk (grid = nranks x max owned count; a rank's surplus
// CTAs exit), visited in reverse of rs_pass1's order: the chunks rs_pass1
// folded last are still in L2
template <bool POW2>
__global__ void __launch_bounds__(kThreads, POW2 ? 4 : 2)
pass2_push_kernel(const gs_rank_ctx* __restrict__ ranks, int nb, const uint64_t* __restrict__ peer_working,
                  int p, int b0, int b1, const gs_step_params params, uint32_t parity,
                  uint32_t flag_mask) {
  gs::griddep_wait();  // the trust kernel's scales (PDL launch)
  const PeerCta pc = peer_cta(ranks, nb);
  pass2_push_cta<POW2>(pc, peer_working, p, b0, b1, params, parity, flag_mask, 0u);
}

// the fence CTAs, the trust CTAs and the pass-2 CTAs of the sharded step in
// one grid (gs_zero_update); a pass-2 CTA waits for its segment's epoch in
// seg_ready, which its trust CTA publishes after the scale
template <bool POW2>
__global__ void __launch_bounds__(kThreads, POW2 ? 4 : 2)
zero_update_kernel(const gs_rank_ctx* __restrict__ ranks, int nranks, const uint64_t* __restrict__ sig,
                   const uint64_t* __restrict__ peer_working, int p, uint32_t epoch, int nseg,
                   int nchunk, int b0, int b1, int max_chunks, const gs_step_params params,
                   uint32_t parity, uint32_t flag_mask) {
  const int nfence = nranks, ntrust = nranks * (nseg + 1);
  const int b = blockIdx.x;
  if (b < nfence + ntrust) {
    trust_fence_cta(ranks, nranks, sig, p, epoch, nseg, nchunk, params, parity, b, true);
    return;
  }
  const int b2 = b - nfence - ntrust;
  PeerCta pc;
  pc.R = ranks + b2 / max_chunks;
  pc.lb = b2 % max_chunks;
  pc.nb = max_chunks;
  const uint32_t ep = epoch + (pc.R->epoch_base != nullptr ? *pc.R->epoch_base : 0u);
  pass2_push_cta<POW2>(pc, peer_working, p, b0, b1, params, parity, flag_mask, ep);
}

// the work of one pass2_push CTA; ready_epoch != 0: first wait until the
// chunk's segment has published its scale (gs_zero_update)
template <bool POW2>
__device__ __forceinline__ void pass2_push_cta(const PeerCta& pc, const uint64_t* __restrict__ peer_working,
                                               int p, int b0, int b1, const gs_step_params& params,
                                               uint32_t parity, uint32_t flag_mask,
                                               uint32_t ready_epoch) {
  const gs_rank_ctx& R = *pc.R;
  int i0, i1;
  own_range(R, b0, b1, i0, i1);
  if (pc.lb >= i1 - i0) return;
  const int c = R.own_list[i1 - 1 - pc.lb];
  const gs_chunk ch = R.chunks[c];
  if (ready_epoch != 0u) {
    if (threadIdx.x == 0) wait_epoch(&R.seg_ready[ch.seg], ready_epoch, R);
    __syncthreads();
  }
  if (R.ctl->flags[parity] & flag_mask) return;  // lars.py:161-163
  const gs_segment* sp = R.segs + ch.seg;
  const uint32_t sflags = sp->flags;
  Ctx cx;
  cx.u.load(&params);
  cx.mul = params.mul;
  cx.wd = params.weight_decay;
  cx.m = params.momentum;
  const float s = R.seg_scale[ch.seg];
  uint16_t* w16 = sp->w16 + ch.start;
  const size_t woff = reinterpret_cast<const uint8_t*>(w16) -
                      reinterpret_cast<const uint8_t*>(peer_working[R.rank]);
  const bool decay = (cx.u.mode & GS_MODE_DECAY) && !(sflags & GS_SEG_DECAY_EXEMPT);
  const uint16_t* g = static_cast<const uint16_t*>(sp->g) + ch.start;
  if (decay)
    p2_push_chunk<POW2, true>(g, sp->w + ch.start, sp->v + ch.start, w16, ch.len, cx, s,
                              peer_working, p, woff);
  else
    p2_push_chunk<POW2, false>(g, sp->w + ch.start, sp->v + ch.start, w16, ch.len, cx, s,
                               peer_working, p, woff);
}

// gs_peer_fence + gs_lars_trust in one launch.  Blocks [0, nranks): one
// fence CTA per rank (fence.sys, the peer barrier of gs_peer_fence, then
// `epoch` published in ctl->counter[0]); blocks nranks + r * (nseg + 1) + s:
// trust CTA s of rank r, which waits for its rank's word.  The fence CTAs
// come first in the grid, so they are dispatched before any waiting trust
// CTA and the launch cannot deadlock even when it does not fit at once.
__device__ __forceinline__ void trust_fence_cta(const gs_rank_ctx* __restrict__ ranks, int nranks,
                                                const uint64_t* __restrict__ sig, int p,
                                                uint32_t epoch, int nseg, int nchunk,
                                                const gs_step_params& params, uint32_t parity,
                                                int b, bool publish) {
  if (b < nranks) {
    PeerCta pc;
    pc.R = ranks + b;
    pc.lb = 0;
    pc.nb = 1;
    if (pc.R->epoch_base != nullptr) epoch += *pc.R->epoch_base;
    if (threadIdx.x < p) __threadfence_system();  // this GPU's earlier remote stores
    peer_barrier(sig, pc, p, 1, epoch, kSiteFence);
    if (threadIdx.x == 0)
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&pc.R->ctl->counter[0]), "r"(epoch)
                   : "memory");
    return;
  }
  b -= nranks;
  const gs_rank_ctx& R = ranks[b / (nseg + 1)];
  const int s = b % (nseg + 1);
  if (R.epoch_base != nullptr) epoch += *R.epoch_base;
  if (threadIdx.x == 0) wait_epoch(&R.ctl->counter[0], epoch, R);
  __syncthreads();
  trust_cta(R.segs, s, nseg, nchunk, R.partials, params, const_cast<float*>(R.seg_scale),
            R.seg_out, R.ctl, parity, nullptr, 0);
  if (publish && s < nseg && threadIdx.x == 0) {
    // thread 0 wrote the scale: publish the segment (release, gpu scope)
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&R.seg_ready[s]), "r"(epoch)
                 : "memory");
  }
}

__global__ void __launch_bounds__(kThreads)
trust_fence_kernel(const gs_rank_ctx* __restrict__ ranks, int nranks, const uint64_t* __restrict__ sig,
                   int p, uint32_t epoch, int nseg, int nchunk, const gs_step_params params,
                   uint32_t parity) {
  gs::griddep_launch_dependents();  // pass 2 (PDL) may start issuing its loads
  trust_fence_cta(ranks, nranks, sig, p, epoch, nseg, nchunk, params, parity, blockIdx.x, false);
}

__global__ void peer_fence_kernel(const gs_rank_ctx* __restrict__ ranks, const uint64_t* __restrict__ sig,
                                  int p, uint32_t epoch, uint32_t epoch_inc) {
  const PeerCta pc = peer_cta(ranks, 1);
  if (pc.R->epoch_base != nullptr) epoch += *pc.R->epoch_base;
  if (threadIdx.x < p) __threadfence_system();  // this GPU's earlier remote stores
  peer_barrier(sig, pc, p, 1, epoch, kSiteFence);
  // the step's last kernel: advance the rank's epoch base for the next step
  // (every kernel of this step read it at its start; saves a launch)
  if (epoch_inc != 0u && threadIdx.x == 0 && pc.R->epoch_base != nullptr)
    *const_cast<uint32_t*>(pc.R->epoch_base) += epoch_inc;
}

}  // namespace

extern "C" {

int gs_rs_pass1(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* wires,
                const uint64_t* sig, const uint64_t* peer_partials, const uint64_t* peer_ctl,
                int b0, int b1, gs_step_params params, uint32_t hint, uint32_t parity,
                uint32_t epoch, int nblocks, void* stream) {
  GS_REQUIRE(p == 2 || p == 4 || p == 8, "gs_rs_pass1: p must be 2, 4 or 8 (got %d)", p);
  GS_REQUIRE(nranks >= 1 && nranks <= p && b0 >= 0 && b1 >= b0 && nblocks >= 1 && parity <= 1,
             "gs_rs_pass1: bad arguments");
  GS_REQUIRE(epoch != 0, "gs_rs_pass1: epoch 0 is the reset value");
  GS_REQUIRE(ranks && wires && sig && peer_partials && peer_ctl, "gs_rs_pass1: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const bool pow2 = hint & GS_HINT_POW2, raw = pow2 && (hint & GS_HINT_RAWFLAG),
             gnorm = hint & GS_HINT_GRADNORM;
#define GS_RSP(P, PW, RW, GN)                                                                     \
  {                                                                                               \
    auto k = rs_pass1_kernel<P, PW, RW, GN>;                                                      \
    const int nb = peer_grid((const void*)k, kThreads, 0, nblocks, nranks);                       \
    k<<<nb * nranks, kThreads, 0, s>>>(ranks, nb, wires, sig, peer_partials, peer_ctl, b0, b1,    \
                                       params, parity, epoch);                                    \
  }
#define GS_RSP_P(P)                                      \
  if (raw) {                                             \
    if (gnorm) GS_RSP(P, true, true, true)               \
    else GS_RSP(P, true, true, false)                    \
  } else if (pow2) {                                     \
    if (gnorm) GS_RSP(P, true, false, true)              \
    else GS_RSP(P, true, false, false)                   \
  } else {                                               \
    if (gnorm) GS_RSP(P, false, false, true)             \
    else GS_RSP(P, false, false, false)                  \
  }
  if (p == 2) GS_RSP_P(2)
  else if (p == 4) GS_RSP_P(4)
  else GS_RSP_P(8)
#undef GS_RSP_P
#undef GS_RSP
  return gs_check_launch("gs_rs_pass1");
}

int gs_pass2_push(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* peer_working,
                  int b0, int b1, int max_chunks, gs_step_params params, uint32_t hint,
                  uint32_t parity, uint32_t flag_mask, void* stream) {
  GS_REQUIRE(nranks >= 1 && nranks <= p && p <= 32 && b0 >= 0 && b1 >= b0 && max_chunks >= 0 &&
                 parity <= 1,
             "gs_pass2_push: bad arguments");
  if (max_chunks == 0) return GS_OK;
  GS_REQUIRE(ranks && peer_working, "gs_pass2_push: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const dim3 grid(max_chunks * nranks);
  cudaError_t e;
  if (hint & GS_HINT_POW2)
    e = gs_launch_pdl(pass2_push_kernel<true>, grid, dim3(kThreads), 0, s, ranks, max_chunks,
                      peer_working, p, b0, b1, params, parity, flag_mask);
  else
    e = gs_launch_pdl(pass2_push_kernel<false>, grid, dim3(kThreads), 0, s, ranks, max_chunks,
                      peer_working, p, b0, b1, params, parity, flag_mask);
  if (e != cudaSuccess) {
    gs_set_error("gs_pass2_push: %s", cudaGetErrorString(e));
    return GS_ECUDA;
  }
  return gs_check_launch("gs_pass2_push");
}

int gs_trust_fence(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* sig,
                   uint32_t epoch, int nseg, int nchunk, gs_step_params params, uint32_t parity,
                   void* stream) {
  GS_REQUIRE(p >= 1 && p <= 32 && nranks >= 1 && nranks <= p && nseg >= 0 && nchunk >= 0 &&
                 parity <= 1,
             "gs_trust_fence: bad arguments");
  GS_REQUIRE(ranks && sig, "gs_trust_fence: null pointer");
  GS_REQUIRE(epoch != 0, "gs_trust_fence: epoch 0 is the reset value");
  trust_fence_kernel<<<nranks * (nseg + 2), kThreads, 0, (cudaStream_t)stream>>>(
      ranks, nranks, sig, p, epoch, nseg, nchunk, params, parity);
  return gs_check_launch("gs_trust_fence");
}

int gs_zero_update(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* sig,
                   const uint64_t* peer_working, uint32_t epoch, int nseg, int nchunk, int b0,
                   int b1, int max_chunks, gs_step_params params, uint32_t hint, uint32_t parity,
                   uint32_t flag_mask, void* stream) {
  GS_REQUIRE(p >= 1 && p <= 32 && nranks >= 1 && nranks <= p && nseg >= 0 && nchunk >= 0 &&
                 parity <= 1 && b0 >= 0 && b1 >= b0 && max_chunks >= 0,
             "gs_zero_update: bad arguments");
  GS_REQUIRE(ranks && sig && peer_working, "gs_zero_update: null pointer");
  GS_REQUIRE(epoch != 0, "gs_zero_update: epoch 0 is the reset value");
  const int mc = max_chunks > 0 ? max_chunks : 1;
  const dim3 grid(nranks * (nseg + 2) + nranks * mc);
  cudaStream_t s = (cudaStream_t)stream;
  if (hint & GS_HINT_POW2)
    zero_update_kernel<true><<<grid, kThreads, 0, s>>>(ranks, nranks, sig, peer_working, p, epoch,
                                                        nseg, nchunk, b0, b1, mc, params, parity,
                                                        flag_mask);
  else
    zero_update_kernel<false><<<grid, kThreads, 0, s>>>(ranks, nranks, sig, peer_working, p,
                                                         epoch, nseg, nchunk, b0, b1, mc, params,
                                                         parity, flag_mask);
  return gs_check_launch("gs_zero_update");
}

int gs_peer_fence(const gs_rank_ctx* ranks, int nranks, int p, const uint64_t* sig, uint32_t epoch,
                  uint32_t epoch_inc, void* stream) {
  GS_REQUIRE(p >= 1 && p <= 32 && nranks >= 1 && nranks <= p, "gs_peer_fence: bad arguments");
  if (p == 1) return GS_OK;
  GS_REQUIRE(ranks && sig, "gs_peer_fence: null pointer");
  GS_REQUIRE(epoch != 0, "gs_peer_fence: epoch 0 is the reset value");
  peer_fence_kernel<<<nranks, 32, 0, (cudaStream_t)stream>>>(ranks, sig, p, epoch, epoch_inc);
  return gs_check_launch("gs_peer_fence");
}

}  // extern "C"
