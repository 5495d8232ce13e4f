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
//   pass1   reads g (2 B fp16 or 4 B fp32) + w (4 B, LARS groups only),
//           emits per-chunk fp64 partials {sum w^2, sum eff^2, sum g^2} and
//           the two non-finite flag bits.                        6 B/elem
//   trust   one CTA per segment folds its chunk partials and derives the
//           fp32 trust scale; one more CTA folds the grad-norm metric.
//   pass2   early-exits on the flags, otherwise reads g, w, v and writes
//           v, w, w16, visiting the chunks in reverse of pass 1's order so
//           the chunks pass 1 read last are still in L2.       20 B/elem
// Chunks never straddle a segment, so a CTA handles one (segment, range) pair
// with uniform control flow, and its partial sums land in a fixed slot: the
// reduction order depends only on the chunk table, never on timing.
//
// Step scalars travel BY VALUE (gs_step_params kernel argument): a step needs
// no host->device copy.  The flag words are double-buffered by step parity in
// gs_ctl: step k ORs into flags[k & 1], and its trust kernel clears
// flags[(k + 1) & 1] for the next step (the host read it after step k - 1).
//
// Specialisation (host hints, gradsync_b200.h GS_HINT_*): with power-of-two p
// and loss scale the mean and unscale are one exact multiplication by `mul`
// (one FMUL per element), and for fp16 input with mul <= 1 the finite tests
// reduce to an integer test of the binary16 exponent field; full 8192-element
// chunks issue all their loads before any arithmetic.
#include "gs_lars_device.cuh"

namespace {

// ------------------------------------------------------------------ pass 1
// One CTA per chunk (one 8192-element batch: 4 vectors of g and of w per
// thread, every load issued before any arithmetic).  Per-thread vector order
// t, t+256, t+512, t+768, then the scalar tail: the summation order of every
// other pass-1 form (rs_pass1, p1_chunk), so the partials are bit-identical.
// Measured alternatives on ResNet-50 (profiles/r02_pass1_variants.md): a
// persistent software-pipelined form (3 CTAs/SM: 39.3 us), two chunks per
// CTA (2 CTAs/SM: 42.9 us), 3 CTAs/SM (37.4 us), a TMA bulk L2 prefetch of
// the chunk one wave ahead (35.8 us) and a persistent cp.async-staged 4-stage
// ring (45.6 us: latency hidden, but twice the instructions) all lost to 4
// CTAs/SM x one chunk (34.3 us).
struct P1Meta {
  const void* g;
  const float* w;
  double wc;  // sum w^2 left by the previous pass 2 (NaN: not available)
  int len, c;
  uint32_t sflags;
};

template <bool F16>
__device__ __forceinline__ P1Meta p1_meta(const gs_segment* __restrict__ segs,
                                          const gs_chunk* __restrict__ chunks, int c,
                                          const double* __restrict__ wsq) {
  using T = typename G<F16>::T;
  P1Meta m;
  m.c = c;
  m.wc = wsq != nullptr ? wsq[c] : __longlong_as_double(0x7FF8000000000000ll);
  const gs_chunk ch = chunks[c];
  GS_DCHECK(ch.seg >= 0 && ch.len >= 0 && ch.start >= 0, "pass 1: chunk table entry");
  GS_DCHECK(ch.start + ch.len <= segs[ch.seg].n, "pass 1: chunk inside its segment");
  const gs_segment* sp = segs + ch.seg;
  m.g = static_cast<const T*>(sp->g) + ch.start;
  m.w = sp->w + ch.start;
  m.len = ch.len;
  m.sflags = sp->flags;
  return m;
}

template <bool F16>
struct P1Batch {
  typename G<F16>::V gv[kP1Rounds];
  F8 wv[kP1Rounds];
};

// is the chunk on the 16-byte vector path (the summation order pass 2's
// carried sum w^2 was formed in)
__device__ __forceinline__ bool p1_vec_ok(const P1Meta& m) {
  const bool lars = (m.sflags & GS_SEG_LARS_ENABLED) != 0;
  return m.len <= kThreads * 8 * kP1Rounds &&
         (lars ? p1_vec_path<true>(m.g, m.w) : p1_vec_path<false>(m.g, m.w));
}

// does the chunk take the register-batched path (else p1_chunk).  fp32
// gradients (8 registers per vector) and the IEEE-division forms take
// p1_chunk with 2-vector batches, which keeps them at 3 CTAs/SM instead of
// 1-2 (same per-thread order, same bits)
template <bool F16, bool POW2>
__device__ __forceinline__ bool p1_batched(const P1Meta& m) {
  return F16 && POW2 && p1_vec_ok(m);
}

template <bool F16, bool POW2>
__device__ __forceinline__ void p1_issue(const P1Meta& m, P1Batch<F16>& bt) {
  using Gt = G<F16>;
  if (!p1_batched<F16, POW2>(m)) return;
  const int nv = m.len / 8, t = threadIdx.x;
  const bool lars = (m.sflags & GS_SEG_LARS_ENABLED) != 0;
  const typename Gt::T* g = static_cast<const typename Gt::T*>(m.g);
#pragma unroll
  for (int k = 0; k < kP1Rounds; ++k)
    if (t + k * kThreads < nv) bt.gv[k] = Gt::ld(g + 8 * (t + k * kThreads));
  if (lars) {
#pragma unroll
    for (int k = 0; k < kP1Rounds; ++k)
      if (t + k * kThreads < nv) bt.wv[k] = ldw(m.w + 8 * (t + k * kThreads));
  }
}

template <bool F16, bool POW2, bool RAWFLAG, bool GNORM, bool LARS, bool DECAY, bool W2>
__device__ __forceinline__ void p1_consume(const P1Meta& m, const P1Batch<F16>& bt, const Ctx& cx,
                                           Acc& a) {
  using Gt = G<F16>;
  if (!p1_batched<F16, POW2>(m)) {  // fp32 / IEEE division / misaligned: the generic loop
    p1_chunk<F16, POW2, RAWFLAG, GNORM, LARS, DECAY, W2, (F16 && POW2) ? kP1Rounds : 2>(
        static_cast<const typename Gt::T*>(m.g), m.w, m.len, cx, a);
    return;
  }
  const int nv = m.len / 8, t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < kP1Rounds; ++k)
    if (t + k * kThreads < nv)
      p1_vec<F16, POW2, RAWFLAG, GNORM, LARS, DECAY, W2>(bt.gv[k], LARS ? bt.wv[k] : F8{}, cx, a);
  // scalar tail, exactly as p1_chunk's
  const typename Gt::T* g = static_cast<const typename Gt::T*>(m.g);
  for (int i = nv * 8 + t; i < m.len; i += kThreads) {
    if (F16 && RAWFLAG) a.raw |= raw_nonfinite_bits(reinterpret_cast<const uint16_t*>(g)[i]);
    Acc b;
    p1_pair<POW2, RAWFLAG, GNORM, LARS, DECAY, W2>(make_float2(Gt::one(g + i), 0.0f),
                                                   make_float2(LARS ? m.w[i] : 0.0f, 0.0f), cx, b);
    a.sw += b.sw;
    a.se += b.se;
    a.sg += b.sg;
    a.fl |= b.fl;
  }
}

// 3 resident CTAs per SM for the power-of-two forms (80 registers: one batch
// in flight + the next chunk's table entries); the IEEE-division forms get
// 128 registers so nothing spills
#ifndef GS_P1_MINB
#define GS_P1_MINB 4
#endif
// (the power-of-two form with per-element finite tests, mul > 1, needs a few
// more registers than 64: 3 CTAs / SM so it does not spill)
template <bool F16, bool POW2, bool RAWFLAG>
constexpr int kP1MinBlocks = (F16 && POW2 && RAWFLAG) ? GS_P1_MINB : 3;

// one chunk's partials: the fixed block tree of gs::block_sum3 over
// double-buffered scratch (one barrier per chunk)
__device__ __forceinline__ void p1_finish(const P1Meta& m, bool cached, const Acc& a, int it,
                                          double (*red)[3][kThreads / 32],
                                          double* __restrict__ partials) {
  double x = gs::warp_sum(a.sw), y = gs::warp_sum(a.se), z = gs::warp_sum(a.sg);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double(*rb)[kThreads / 32] = red[it & 1];
  if (lane == 0) {
    rb[0][warp] = x;
    rb[1][warp] = y;
    rb[2][warp] = z;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w8 = 1; w8 < kThreads / 32; ++w8) {
      x += rb[0][w8];
      y += rb[1][w8];
      z += rb[2][w8];
    }
    partials[3 * (int64_t)m.c + 0] = cached ? m.wc : x;
    partials[3 * (int64_t)m.c + 1] = y;
    partials[3 * (int64_t)m.c + 2] = z;
  }
}

template <bool F16, bool POW2, bool RAWFLAG, bool GNORM>
__device__ __forceinline__ uint32_t p1_run(const P1Meta& cur, const P1Batch<F16>& bt,
                                           const Ctx& cx, bool& cached_out, Acc& a) {
  const bool lars = (cur.sflags & GS_SEG_LARS_ENABLED) != 0;
  const bool decay = (cx.u.mode & GS_MODE_DECAY) && !(cur.sflags & GS_SEG_DECAY_EXEMPT);
  // the previous pass 2's sum w^2 stands in for this chunk's when it was
  // formed in this very order (pass 2 stores NaN where it was not)
  const bool cached = lars && !isnan(cur.wc) && p1_vec_ok(cur);
  if (lars && decay) {
    if (cached)
      p1_consume<F16, POW2, RAWFLAG, GNORM, true, true, false>(cur, bt, cx, a);
    else
      p1_consume<F16, POW2, RAWFLAG, GNORM, true, true, true>(cur, bt, cx, a);
  } else if (lars) {
    if (cached)
      p1_consume<F16, POW2, RAWFLAG, GNORM, true, false, false>(cur, bt, cx, a);
    else
      p1_consume<F16, POW2, RAWFLAG, GNORM, true, false, true>(cur, bt, cx, a);
  } else {
    p1_consume<F16, POW2, RAWFLAG, GNORM, false, false, true>(cur, bt, cx, a);
  }
  if (lars && !decay) {
    a.se = a.sg;  // eff == g exactly: same terms, same order
    if (!GNORM) a.sg = 0.0;
  }
  cached_out = cached;
  return a.fl | ((a.raw & 0x80008000u) ? kBoth : 0u);
}

template <bool F16, bool POW2, bool RAWFLAG, bool GNORM>
__global__ void __launch_bounds__(kThreads, (kP1MinBlocks<F16, POW2, RAWFLAG>))
lars_pass1_kernel(const gs_segment* __restrict__ segs, const gs_chunk* __restrict__ chunks,
                  int chunk0, int nchunk, const gs_step_params params,
                  double* __restrict__ partials, gs_ctl* __restrict__ ctl, uint32_t parity,
                  const double* __restrict__ wsq) {
  Ctx cx;
  cx.u.load(&params);
  cx.mul = params.mul;
  cx.wd = params.weight_decay;
  __shared__ double red[2][3][kThreads / 32];
  uint32_t flag_acc = 0;
  const int i = blockIdx.x;
  const P1Meta m = p1_meta<F16>(segs, chunks, chunk0 + i, wsq);
  P1Batch<F16> bt;
  p1_issue<F16, POW2>(m, bt);
  Acc a;
  bool cached;
  flag_acc |= p1_run<F16, POW2, RAWFLAG, GNORM>(m, bt, cx, cached, a);
  p1_finish(m, cached, a, 0, red, partials);
  flag_acc = __reduce_or_sync(0xFFFFFFFFu, flag_acc);
  if (flag_acc != 0u && (threadIdx.x & 31) == 0) atomicOr(&ctl->flags[parity], flag_acc);
}

// ----------------------------------------------------------------- trust
// nseg + 1 independent CTAs, no arrival counters: CTA s < nseg folds segment
// s's chunk partials (256-strided in chunk order, then the fixed block tree,
// the same order on every path) and derives its trust scale; CTA nseg folds
// every chunk's sum g^2 for the grad-norm metric (experiment.py:408-411; a
// fixed tree over chunks instead of numpy's per-group dots summed in group
// order — the reference's own ddot order is unpinned).  The
// kernel's latency is one L2 round trip plus a block reduction; pass 2 (PDL)
// has issued its first loads meanwhile.
__global__ void __launch_bounds__(kThreads)
lars_trust_kernel(const gs_segment* __restrict__ segs, int nseg, int nchunk,
                  const double* __restrict__ partials, const gs_step_params params,
                  float* __restrict__ seg_scale, double* __restrict__ seg_out,
                  gs_ctl* __restrict__ ctl, uint32_t parity, const uint64_t* __restrict__ peer_ctl,
                  int npeers) {
  gs::griddep_wait();                 // pass 1's partials are complete
  gs::griddep_launch_dependents();    // let pass 2 start issuing its loads now
  trust_cta(segs, blockIdx.x, nseg, nchunk, partials, params, seg_scale, seg_out, ctl, parity,
            peer_ctl, npeers);
}

// W2: also sum the updated masters' squares in pass 1's order and store the
// chunk's sum in *wsq_out (NaN when this chunk cannot take the vector path,
// whose order pass 1 uses) for the next step's pass 1
template <bool F16, bool POW2, bool DECAY, bool W2>
__device__ __forceinline__ void p2_chunk(const typename G<F16>::T* __restrict__ g,
                                         float* __restrict__ w, float* __restrict__ v,
                                         uint16_t* __restrict__ w16, int len, const Ctx& cx,
                                         const float* __restrict__ seg_scale, int seg,
                                         const uint32_t* __restrict__ flag, uint32_t flag_mask,
                                         double* __restrict__ wsq_out) {
  using Gt = G<F16>;
  const bool vec = gs::is_aligned16(g) && gs::is_aligned16(w) && gs::is_aligned16(v) &&
                   gs::is_aligned16(w16);
  const int nv = vec ? len / 8 : 0;
  const int t = threadIdx.x;
  // launched with PDL behind the trust kernel: everything above and the
  // first batch of loads overlap it; the scale and the flags come after
  float s = 0.0f;
  double sw = 0.0;
  bool have_s = false;
  auto scale_of = [&]() -> bool {
    gs::griddep_wait();
    if (*flag & flag_mask) return false;  // lars.py:161-163: mutate nothing
    s = seg_scale[seg];
    return true;
  };
  // batches of two vectors per thread: both vectors' loads are issued before
  // the arithmetic and stores (stores cannot alias the next batch's loads,
  // but the compiler cannot prove it through the casts)
  int done = 0;
  for (; done + 2 * kThreads <= nv; done += 2 * kThreads) {
    const int i0 = done + t, i1 = i0 + kThreads;
    const typename Gt::V g0 = Gt::ld(g + 8 * i0), g1 = Gt::ld(g + 8 * i1);
    const F8 w0 = ld8(w, i0), w1 = ld8(w, i1), v0 = ld8(v, i0), v1 = ld8(v, i1);
    if (!have_s) {  // uniform: every thread runs the first batch
      if (!scale_of()) return;
      have_s = true;
    }
    p2_vec<F16, POW2, DECAY, W2>(g0, w0, v0, w, v, w16, i0, cx, s, &sw);
    p2_vec<F16, POW2, DECAY, W2>(g1, w1, v1, w, v, w16, i1, cx, s, &sw);
  }
  if (!have_s && !scale_of()) return;
  for (int i = done + t; i < nv; i += kThreads) {
    const typename Gt::V gv = Gt::ld(g + 8 * i);
    p2_vec<F16, POW2, DECAY, W2>(gv, ld8(w, i), ld8(v, i), w, v, w16, i, cx, s, &sw);
  }
  for (int i = nv * 8 + t; i < len; i += kThreads) {
    float2 ww = make_float2(w[i], 0.0f), vv = make_float2(v[i], 0.0f);
    p2_pair<POW2, DECAY>(make_float2(Gt::one(g + i), 0.0f), ww, vv, cx, s);
    v[i] = vv.x;
    w[i] = ww.x;
    w16[i] = gs::narrow(ww.x);
    if (W2) w2_tail(ww.x, sw);
  }
  if (W2) {
    double z1 = 0.0, z2 = 0.0;
    gs::block_sum3<kThreads>(sw, z1, z2);  // the fixed tree of pass 1's block_sum3
    if (threadIdx.x == 0) *wsq_out = vec ? sw : __longlong_as_double(0x7FF8000000000000ll);
  }
}

// one CTA per chunk, chunks visited in REVERSE order: pass 1 streamed them
// forward, so the first chunks pass 2 needs are the ones still in L2
// (ResNet-50: 84.0 -> 81.2 us, profiles/r02a)
template <bool F16, bool POW2>
__global__ void __launch_bounds__(kThreads, F16 && POW2 ? 4 : (F16 || POW2) ? 3 : 2)
lars_pass2_kernel(const gs_segment* __restrict__ segs, const gs_chunk* __restrict__ chunks,
                  int chunk0, const gs_step_params params, const float* __restrict__ seg_scale,
                  const gs_ctl* __restrict__ ctl, uint32_t parity, uint32_t flag_mask,
                  double* __restrict__ wsq) {
  using T = typename G<F16>::T;
  const int c = chunk0 + (int)(gridDim.x - 1 - blockIdx.x);
  const gs_chunk ch = chunks[c];
  GS_DCHECK(ch.seg >= 0 && ch.len >= 0 && ch.start >= 0, "pass 2: chunk table entry");
  const gs_segment* sgp = segs + ch.seg;
  GS_DCHECK(ch.start + ch.len <= sgp->n, "pass 2: chunk inside its segment");
  const uint32_t sflags = sgp->flags;
  const T* g = static_cast<const T*>(sgp->g) + ch.start;
  Ctx cx;
  cx.u.load(&params);
  cx.mul = params.mul;
  cx.wd = params.weight_decay;
  cx.m = params.momentum;
  const bool decay = (cx.u.mode & GS_MODE_DECAY) && !(sflags & GS_SEG_DECAY_EXEMPT);
  const bool w2 = wsq != nullptr && (sflags & GS_SEG_LARS_ENABLED);
  float* w = sgp->w + ch.start;
  float* v = sgp->v + ch.start;
  uint16_t* w16 = sgp->w16 + ch.start;
  const uint32_t* flag = &ctl->flags[parity];
  double* wo = wsq + c;
  if (decay) {
    if (w2)
      p2_chunk<F16, POW2, true, true>(g, w, v, w16, ch.len, cx, seg_scale, ch.seg, flag, flag_mask, wo);
    else
      p2_chunk<F16, POW2, true, false>(g, w, v, w16, ch.len, cx, seg_scale, ch.seg, flag, flag_mask, wo);
  } else {
    if (w2)
      p2_chunk<F16, POW2, false, true>(g, w, v, w16, ch.len, cx, seg_scale, ch.seg, flag, flag_mask, wo);
    else
      p2_chunk<F16, POW2, false, false>(g, w, v, w16, ch.len, cx, seg_scale, ch.seg, flag, flag_mask, wo);
  }
}

}  // namespace

extern "C" {

int gs_lars_pass1(const gs_segment* segs, const gs_chunk* chunks, int chunk0, int nchunk,
                  int g_is_f16, gs_step_params params, uint32_t hint, double* partials, gs_ctl* ctl,
                  uint32_t parity, const double* wsq, void* stream) {
  GS_REQUIRE(nchunk >= 0 && chunk0 >= 0 && parity <= 1, "gs_lars_pass1: bad chunk range / parity");
  if (nchunk == 0) return GS_OK;
  GS_REQUIRE(segs && chunks && partials && ctl, "gs_lars_pass1: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const bool pow2 = hint & GS_HINT_POW2, raw = g_is_f16 && pow2 && (hint & GS_HINT_RAWFLAG),
             gnorm = hint & GS_HINT_GRADNORM;
#define GS_P1(F, P, R, N)                                                                       \
  do {                                                                                          \
    lars_pass1_kernel<F, P, R, N><<<nchunk, kThreads, 0, s>>>(segs, chunks, chunk0, nchunk,     \
                                                               params, partials, ctl, parity,   \
                                                               wsq);                            \
  } while (0)
  if (g_is_f16) {
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
  return gs_check_launch("gs_lars_pass1");
}

int gs_lars_trust(const gs_segment* segs, int nseg, int nchunk, const double* partials,
                  gs_step_params params, float* seg_scale, double* seg_out, gs_ctl* ctl,
                  uint32_t parity, const uint64_t* peer_ctl, int npeers, void* stream) {
  GS_REQUIRE(nseg >= 0 && nchunk >= 0 && parity <= 1,
             "gs_lars_trust: negative segment / chunk count or bad parity");
  GS_REQUIRE(segs && partials && seg_scale && seg_out && ctl, "gs_lars_trust: null pointer");
  GS_REQUIRE(npeers == 0 || peer_ctl != nullptr, "gs_lars_trust: peer flags need the peer table");
  const cudaError_t e = gs_launch_pdl(lars_trust_kernel, dim3(nseg + 1), dim3(kThreads), 0,
                                      (cudaStream_t)stream, segs, nseg, nchunk, partials, params,
                                      seg_scale, seg_out, ctl, parity, peer_ctl, npeers);
  if (e != cudaSuccess) {
    gs_set_error("gs_lars_trust: %s", cudaGetErrorString(e));
    return GS_ECUDA;
  }
  return gs_check_launch("gs_lars_trust");
}

int gs_lars_pass2(const gs_segment* segs, const gs_chunk* chunks, int chunk0, int nchunk,
                  int g_is_f16, gs_step_params params, uint32_t hint, const float* seg_scale,
                  const gs_ctl* ctl, uint32_t parity, uint32_t flag_mask, double* wsq,
                  void* stream) {
  GS_REQUIRE(nchunk >= 0 && chunk0 >= 0 && parity <= 1, "gs_lars_pass2: bad chunk range / parity");
  if (nchunk == 0) return GS_OK;
  GS_REQUIRE(segs && chunks && seg_scale && ctl, "gs_lars_pass2: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const bool pow2 = hint & GS_HINT_POW2;
  cudaError_t err = cudaSuccess;
#define GS_P2(F, P)                                                                              \
  err = gs_launch_pdl(lars_pass2_kernel<F, P>, dim3(nchunk), dim3(kThreads), 0, s, segs, chunks, \
                      chunk0, params, seg_scale, ctl, parity, flag_mask, wsq)
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

}  // extern "C"
