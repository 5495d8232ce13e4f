// gs_lars_device.cuh — device-side building blocks of the LARS passes
// (element arithmetic, chunk reductions, trust evaluation), shared by the
// LARS kernels (gs_lars.cu) and the fused collective + LARS kernels
// (gs_fused.cu).  See gs_lars.cu for the semantics and reference lines.
#pragma once

#include "gs_common.cuh"

namespace {

constexpr int kThreads = 256;
#ifndef GS_P1_ROUNDS
#define GS_P1_ROUNDS 4   // pass-1 load batch (vectors per thread)
#endif
constexpr int kP1Rounds = GS_P1_ROUNDS;
constexpr int kTrustThreads = 1024;
constexpr uint32_t kBoth = GS_FLAG_SCALED_NONFINITE | GS_FLAG_GRAD_NONFINITE;

// Pairwise fp32 ops, each lane rounded separately.  NOT the packed
// __fmul2_rn/__fadd2_rn intrinsics: ptxas 12.9 contracts mul.rn.f32x2 feeding
// add.rn.f32x2 into FFMA2 even under -fmad=false (seen in SASS), which would
// break the separate roundings numpy performs; scalar mul.rn/add.rn are kept.
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  return make_float2(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y));
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  return make_float2(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y));
}

__device__ __forceinline__ void sq_acc(double& acc, float x) {
  const double d = (double)x;
  acc = fma(d, d, acc);
}

// release-ordered arrival: the values this thread stored become visible no
// later than the counter increment (the last arriver fences before reading
// everyone's data)
__device__ __forceinline__ uint32_t arrive_release(uint32_t* p) {
  uint32_t old;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

// raw binary16 non-finite detector for two halves in one word: adding 0x0400
// to an all-ones exponent field carries into the (masked-off) sign position
__device__ __forceinline__ uint32_t raw_nonfinite_bits(uint32_t w) {
  return (w & 0x7C007C00u) + 0x04000400u;
}

struct Ctx {
  gs::Unscale u;
  float mul, wd, m;
};

struct Acc {
  double sw = 0.0, se = 0.0, sg = 0.0;
  uint32_t fl = 0u, raw = 0u;
};

// ------------------------------------------------------------ pass 1 body
// One element pair (x = widened gradient, w = master).  Every square is
// widened by F2F.F64.F32 and accumulated with an fp64 fma (exact products,
// fixed order): the integer widening forms measured slower on B200 (the ALU
// pipe, not XU, became the limiter; profiles/r01u_pass1_widen_modes.log).
// W2 = false: sum w^2 is not accumulated (pass 2 of the previous step
// already produced it for this chunk, in this very order: w2_vec below).
template <bool POW2, bool RAWFLAG, bool GNORM, bool LARS, bool DECAY, bool W2 = true>
__device__ __forceinline__ void p1_pair(float2 x, float2 w, const Ctx& cx, Acc& a) {
  float2 gu;
  if (POW2) {
    gu = mul2(x, make_float2(cx.mul, cx.mul));
    if (!RAWFLAG) {
      // the mean x/p (p >= 1) is non-finite iff x is; the unscaled value
      // can additionally overflow when mul > 1
      a.fl |= (gs::is_finite_f32(x.x) && gs::is_finite_f32(x.y)) ? 0u : kBoth;
      a.fl |= (gs::is_finite_f32(gu.x) && gs::is_finite_f32(gu.y)) ? 0u : GS_FLAG_GRAD_NONFINITE;
    }
  } else {
    const float mx = cx.u.mean(x.x), my = cx.u.mean(x.y);
    a.fl |= (gs::is_finite_f32(mx) && gs::is_finite_f32(my)) ? 0u : GS_FLAG_SCALED_NONFINITE;
    gu = make_float2(cx.u.unscale(mx), cx.u.unscale(my));
    a.fl |= (gs::is_finite_f32(gu.x) && gs::is_finite_f32(gu.y)) ? 0u : GS_FLAG_GRAD_NONFINITE;
  }
  if (LARS) {
    if (W2) {
      sq_acc(a.sw, w.x);
      sq_acc(a.sw, w.y);
    }
    if (DECAY) {
      // eff = g + float32(wd) * w, two roundings (lars.py:172)
      const float2 eff = add2(gu, mul2(make_float2(cx.wd, cx.wd), w));
      sq_acc(a.se, eff.x);
      sq_acc(a.se, eff.y);
    }
  }
  if (GNORM || (LARS && !DECAY)) {
    sq_acc(a.sg, gu.x);
    sq_acc(a.sg, gu.y);
  }
}

template <bool F16>
struct G;
template <>
struct G<true> {
  using T = uint16_t;
  using V = uint4;  // 8 halves
  static __device__ __forceinline__ V ld(const T* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }
  static __device__ __forceinline__ float2 pair(const V& v, int q) {
    return gs::widen2((&v.x)[q]);
  }
  static __device__ __forceinline__ float one(const T* p) { return gs::widen(*p); }
};
struct F8 {
  float4 a, b;
};
template <>
struct G<false> {
  using T = float;
  using V = F8;
  static __device__ __forceinline__ V ld(const T* p) {
    return F8{__ldg(reinterpret_cast<const float4*>(p)), __ldg(reinterpret_cast<const float4*>(p) + 1)};
  }
  static __device__ __forceinline__ float2 pair(const V& v, int q) {
    return q == 0 ? make_float2(v.a.x, v.a.y) : q == 1 ? make_float2(v.a.z, v.a.w)
         : q == 2 ? make_float2(v.b.x, v.b.y) : make_float2(v.b.z, v.b.w);
  }
  static __device__ __forceinline__ float one(const T* p) { return *p; }
};

__device__ __forceinline__ F8 ldw(const float* p) {
  return F8{__ldg(reinterpret_cast<const float4*>(p)), __ldg(reinterpret_cast<const float4*>(p) + 1)};
}
__device__ __forceinline__ float2 wpair(const F8& v, int q) {
  return q == 0 ? make_float2(v.a.x, v.a.y) : q == 1 ? make_float2(v.a.z, v.a.w)
       : q == 2 ? make_float2(v.b.x, v.b.y) : make_float2(v.b.z, v.b.w);
}

template <bool F16, bool POW2, bool RAWFLAG, bool GNORM, bool LARS, bool DECAY, bool W2 = true>
__device__ __forceinline__ void p1_vec(const typename G<F16>::V& gv, const F8& wv, const Ctx& cx,
                                       Acc& a) {
  if (RAWFLAG) {
    const uint4& r = reinterpret_cast<const uint4&>(gv);
    a.raw |= raw_nonfinite_bits(r.x) | raw_nonfinite_bits(r.y) | raw_nonfinite_bits(r.z) |
             raw_nonfinite_bits(r.w);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    p1_pair<POW2, RAWFLAG, GNORM, LARS, DECAY, W2>(G<F16>::pair(gv, q),
                                                   LARS ? wpair(wv, q) : make_float2(0.f, 0.f), cx,
                                                   a);
}

// the vector path of pass 1 (the order its sums run in)
template <bool LARS>
__device__ __forceinline__ bool p1_vec_path(const void* g, const float* w) {
  return gs::is_aligned16(g) && (!LARS || gs::is_aligned16(w));
}

// R: vectors per thread per load batch (any R gives the same per-thread
// order, hence the same bits)
template <bool F16, bool POW2, bool RAWFLAG, bool GNORM, bool LARS, bool DECAY, bool W2 = true,
          int R = kP1Rounds>
__device__ __forceinline__ void p1_chunk(const typename G<F16>::T* __restrict__ g,
                                         const float* __restrict__ w, int len, const Ctx& cx,
                                         Acc& a) {
  using Gt = G<F16>;
  constexpr bool kW = LARS && (W2 || DECAY);  // does pass 1 read w at all
  const bool vec = p1_vec_path<LARS>(g, w);
  const int nv = vec ? len / 8 : 0;
  const int t = threadIdx.x;
  // full batches of kP1Rounds vectors per thread: issue every load of the
  // batch (4 x 16 B of g, 4 x 32 B of w) before any arithmetic; each thread
  // still visits its vectors t, t+256, t+512, ... in increasing order, so
  // the batching never changes the summation order
  constexpr int kBatch = R * kThreads;
  int done = 0;
  for (; done + kBatch <= nv; done += kBatch) {
    typename Gt::V gv[R];
    F8 wv[R];
#pragma unroll
    for (int k = 0; k < R; ++k) gv[k] = Gt::ld(g + 8 * (done + t + k * kThreads));
    if (kW) {
#pragma unroll
      for (int k = 0; k < R; ++k) wv[k] = ldw(w + 8 * (done + t + k * kThreads));
    }
#pragma unroll
    for (int k = 0; k < R; ++k)
      p1_vec<F16, POW2, RAWFLAG, GNORM, LARS, DECAY, W2>(gv[k], kW ? wv[k] : F8{}, cx, a);
  }
  for (int i = done + t; i < nv; i += kThreads) {
    const typename Gt::V gv = Gt::ld(g + 8 * i);
    F8 wv{};
    if (kW) wv = ldw(w + 8 * i);
    p1_vec<F16, POW2, RAWFLAG, GNORM, LARS, DECAY, W2>(gv, wv, cx, a);
  }
  // scalar tail (and misaligned segments): pair the element with a zero
  // partner that contributes nothing
  for (int i = nv * 8 + t; i < len; i += kThreads) {
    if (F16) {
      if (RAWFLAG) a.raw |= raw_nonfinite_bits(reinterpret_cast<const uint16_t*>(g)[i]);
    }
    const float x = Gt::one(g + i);
    const float wx = kW ? w[i] : 0.0f;
    Acc b;
    p1_pair<POW2, RAWFLAG, GNORM, LARS, DECAY, W2>(make_float2(x, 0.0f), make_float2(wx, 0.0f), cx,
                                                   b);
    a.sw += b.sw;
    a.se += b.se;
    a.sg += b.sg;
    a.fl |= b.fl;
  }
}

// lars_local_lr (lars.py:142-150) + lars.py:177 for one segment: norms are
// sqrt of the fp64 dots, local = (eta * w_norm) / (g_norm + eps) or 1.0 when
// degenerate / LARS disabled, scale = float32(local * gamma).
__device__ __forceinline__ void trust_eval(uint32_t sflags, double sw, double se, double sg,
                                           const gs_step_params& params, float* scale_out,
                                           double* o) {
  const double w_norm = __dsqrt_rn(sw);
  const double g_norm = __dsqrt_rn(se);
  double local = 1.0;
  if (sflags & GS_SEG_LARS_ENABLED) {
    const double denom = __dadd_rn(g_norm, params.epsilon);
    if (!(w_norm == 0.0 || denom == 0.0)) local = __ddiv_rn(__dmul_rn(params.eta, w_norm), denom);
  }
  *scale_out = __double2float_rn(__dmul_rn(local, params.gamma));
  o[0] = w_norm;
  o[1] = g_norm;
  o[2] = local;
  o[3] = sg;
}

// One CTA of the trust kernel (gs_lars.cu lars_trust_kernel, gs_fused.cu
// trust_fence_kernel): CTA s < nseg folds segment s's chunk partials
// (256-strided in chunk order, then the fixed block tree -- the same order on
// every path) and derives its trust scale; CTA nseg clears the next step's
// flag word, ORs the peers' flags in (sharded update with separate
// collectives) and folds every chunk's sum g^2 for the grad-norm metric
// (experiment.py:408-411).
__device__ __forceinline__ void trust_cta(const gs_segment* __restrict__ segs, int s, int nseg,
                                          int nchunk, const double* __restrict__ partials,
                                          const gs_step_params& params,
                                          float* __restrict__ seg_scale,
                                          double* __restrict__ seg_out, gs_ctl* __restrict__ ctl,
                                          uint32_t parity, const uint64_t* __restrict__ peer_ctl,
                                          int npeers) {
  if (s == nseg) {
    if (threadIdx.x == 0) {
      // the next step's flag word (the host read it after the previous step;
      // nobody touches it before this step ends)
      ctl->flags[parity ^ 1u] = 0u;
      if (npeers > 0) {
        // sharded update with separate collectives: the step is rejected if
        // any rank saw a non-finite value
        uint32_t f = 0;
        for (int q = 0; q < npeers; ++q)
          f |= *reinterpret_cast<const volatile uint32_t*>(
              &reinterpret_cast<const gs_ctl*>(peer_ctl[q])->flags[parity]);
        if (f) atomicOr(&ctl->flags[parity], f);
      }
    }
    if (!(params.mode & GS_MODE_GRADNORM)) return;
    double x = 0.0, y = 0.0, z = 0.0;
#pragma unroll 8
    for (int i = threadIdx.x; i < nchunk; i += kThreads) z += partials[3 * (int64_t)i + 2];
    gs::block_sum3<kThreads>(x, y, z);
    if (threadIdx.x == 0) ctl->grad_norm = __dsqrt_rn(z);
    return;
  }
  const int cb = segs[s].chunk_begin, cn = segs[s].chunk_count;
  GS_DCHECK(cb >= 0 && cn >= 0 && cb + cn <= nchunk, "trust: segment's chunk range");
  double x = 0.0, y = 0.0, z = 0.0;
#pragma unroll 2
  for (int i = threadIdx.x; i < cn; i += kThreads) {
    const double* pp = partials + 3 * (int64_t)(cb + i);
    x += pp[0];
    y += pp[1];
    z += pp[2];
  }
  gs::block_sum3<kThreads>(x, y, z);
  if (threadIdx.x == 0)
    trust_eval(segs[s].flags, x, y, z, params, seg_scale + s, seg_out + 4 * (int64_t)s);
}

// ----------------------------------------------------------------- pass 2
// v = m*v + s*eff (lars.py:178), w -= v (:179), w16 = f32_to_f16(w) (:180),
// eff = g or g + wd*w (:169-172); every product and sum rounded separately.
template <bool POW2, bool DECAY>
__device__ __forceinline__ void p2_pair(float2 x, float2& w, float2& v, const Ctx& cx, float s) {
  float2 gu;
  if (POW2) {
    gu = mul2(x, make_float2(cx.mul, cx.mul));
  } else {
    gu = make_float2(cx.u.unscale(cx.u.mean(x.x)), cx.u.unscale(cx.u.mean(x.y)));
  }
  const float2 eff = DECAY ? add2(gu, mul2(make_float2(cx.wd, cx.wd), w)) : gu;
  v = add2(mul2(make_float2(cx.m, cx.m), v), mul2(make_float2(s, s), eff));
  w = sub2(w, v);
}

// sum w^2 of the UPDATED masters in exactly pass 1's order (p1_vec: pairs
// q = 0..3, x then y; the scalar tail pairs an element with a zero partner
// and adds the pair sum), so the next step's pass 1 can take the chunk's sum
// instead of re-deriving it (one F2F + DFMA less per LARS element there)
__device__ __forceinline__ void w2_vec(const float2 (&ww)[4], double& s) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    sq_acc(s, ww[q].x);
    sq_acc(s, ww[q].y);
  }
}
__device__ __forceinline__ void w2_tail(float w, double& s) {
  double b = 0.0;
  sq_acc(b, w);
  sq_acc(b, 0.0f);
  s += b;
}

// binary16 pack with NaN canonicalisation for two lanes
__device__ __forceinline__ uint32_t pack_w16(float2 w) {
  __half2 h = __floats2half2_rn(w.x, w.y);
  uint32_t bits = *reinterpret_cast<uint32_t*>(&h);
  // any half with |h| > 0x7C00 is a NaN: force 0x7E00 (halfprec.py:76-77)
  const uint32_t nan = __vcmpgtu2(bits & 0x7FFF7FFFu, 0x7C007C00u);
  return (bits & ~nan) | (0x7E007E00u & nan);
}

template <bool F16, bool POW2, bool DECAY, bool W2 = false>
__device__ __forceinline__ void p2_vec(const typename G<F16>::V& gv, const F8& wv, const F8& vv,
                                       float* __restrict__ w, float* __restrict__ v,
                                       uint16_t* __restrict__ w16, int i, const Ctx& cx, float s,
                                       double* w2 = nullptr) {
  float2 ww[4] = {make_float2(wv.a.x, wv.a.y), make_float2(wv.a.z, wv.a.w),
                  make_float2(wv.b.x, wv.b.y), make_float2(wv.b.z, wv.b.w)};
  float2 xv[4] = {make_float2(vv.a.x, vv.a.y), make_float2(vv.a.z, vv.a.w),
                  make_float2(vv.b.x, vv.b.y), make_float2(vv.b.z, vv.b.w)};
#pragma unroll
  for (int q = 0; q < 4; ++q) p2_pair<POW2, DECAY>(G<F16>::pair(gv, q), ww[q], xv[q], cx, s);
  if (W2) w2_vec(ww, *w2);
  float4* vp = reinterpret_cast<float4*>(v) + 2 * i;
  float4* wp = reinterpret_cast<float4*>(w) + 2 * i;
  __stcs(vp, make_float4(xv[0].x, xv[0].y, xv[1].x, xv[1].y));
  __stcs(vp + 1, make_float4(xv[2].x, xv[2].y, xv[3].x, xv[3].y));
  __stcs(wp, make_float4(ww[0].x, ww[0].y, ww[1].x, ww[1].y));
  __stcs(wp + 1, make_float4(ww[2].x, ww[2].y, ww[3].x, ww[3].y));
  __stcs(reinterpret_cast<uint4*>(w16) + i,
         make_uint4(pack_w16(ww[0]), pack_w16(ww[1]), pack_w16(ww[2]), pack_w16(ww[3])));
}

__device__ __forceinline__ F8 ld8(const float* p, int i) {
  const float4* q = reinterpret_cast<const float4*>(p) + 2 * i;
  return F8{q[0], q[1]};
}

}  // namespace
