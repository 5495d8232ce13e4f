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
// Three kernels, all HBM-bound (no tensor cores: nothing is a contraction):
//   pass1  reads g (2 B fp16 or 4 B fp32) + w (4 B, LARS groups only) and
//          emits per-chunk fp64 partials {sum w^2, sum eff^2, sum g^2} and
//          the two non-finite flag bits;                       6 B/elem
//   trust  one CTA folds the partials per segment in fixed chunk order and
//          evaluates the trust ratio in fp64;                 O(#chunks)
//   pass2  early-exits on the flags, otherwise reads g, w, v and writes
//          v, w, w16;                                          20 B/elem
// Chunks never straddle a segment, so a CTA handles one (segment, range)
// pair with uniform control flow, and its partial sums land in a fixed slot:
// the reduction order depends only on the chunk table, never on timing.
#include "gs_common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kTrustThreads = 1024;

template <bool F16>
struct GradIO;

template <>
struct GradIO<true> {
  using T = uint16_t;
  static __device__ __forceinline__ void load8(const T* p, float (&g)[8]) {
    const uint4 r = *reinterpret_cast<const uint4*>(p);
    const float2 a = gs::widen2(r.x), b = gs::widen2(r.y), c = gs::widen2(r.z), d = gs::widen2(r.w);
    g[0] = a.x; g[1] = a.y; g[2] = b.x; g[3] = b.y;
    g[4] = c.x; g[5] = c.y; g[6] = d.x; g[7] = d.y;
  }
  static __device__ __forceinline__ float load1(const T* p) { return gs::widen(*p); }
};

template <>
struct GradIO<false> {
  using T = float;
  static __device__ __forceinline__ void load8(const T* p, float (&g)[8]) {
    const float4 a = reinterpret_cast<const float4*>(p)[0];
    const float4 b = reinterpret_cast<const float4*>(p)[1];
    g[0] = a.x; g[1] = a.y; g[2] = a.z; g[3] = a.w;
    g[4] = b.x; g[5] = b.y; g[6] = b.z; g[7] = b.w;
  }
  static __device__ __forceinline__ float load1(const T* p) { return *p; }
};

__device__ __forceinline__ void load8f(const float* p, float (&x)[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0];
  const float4 b = reinterpret_cast<const float4*>(p)[1];
  x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
  x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
}

__device__ __forceinline__ void store8f(float* p, const float (&x)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(x[0], x[1], x[2], x[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(x[4], x[5], x[6], x[7]);
}

__device__ __forceinline__ void sq_acc(double& acc, float x) {
  const double d = (double)x;
  acc = fma(d, d, acc);
}

// ----------------------------------------------------------------- pass 1
template <bool F16, bool LARS>
__device__ __forceinline__ void pass1_body(const typename GradIO<F16>::T* __restrict__ g,
                                           const float* __restrict__ w, int len, const gs::Unscale& u,
                                           bool decay, float wd, bool gnorm, double& sw, double& se,
                                           double& sg, uint32_t& fl) {
  auto elem = [&](float graw, float wv) {
    const float gm = u.mean(graw);
    fl |= gs::is_finite_f32(gm) ? 0u : GS_FLAG_SCALED_NONFINITE;
    const float gu = u.unscale(gm);
    fl |= gs::is_finite_f32(gu) ? 0u : GS_FLAG_GRAD_NONFINITE;
    if (LARS) {
      const float eff = decay ? __fadd_rn(gu, __fmul_rn(wd, wv)) : gu;
      sq_acc(sw, wv);
      sq_acc(se, eff);
    }
    if (gnorm) sq_acc(sg, gu);
  };
  const bool vec = gs::is_aligned16(g) && (!LARS || gs::is_aligned16(w));
  const int nv = vec ? len / 8 : 0;
#pragma unroll 4
  for (int i = threadIdx.x; i < nv; i += kThreads) {
    float gf[8], wf[8];
    GradIO<F16>::load8(g + 8 * i, gf);
    if (LARS) load8f(w + 8 * i, wf);
#pragma unroll
    for (int k = 0; k < 8; ++k) elem(gf[k], LARS ? wf[k] : 0.0f);
  }
  for (int i = nv * 8 + threadIdx.x; i < len; i += kThreads)
    elem(GradIO<F16>::load1(g + i), LARS ? w[i] : 0.0f);
}

// lars_local_lr (lars.py:142-150) + lars.py:177 for one segment: norms are
// sqrt of the fp64 dots, local = (eta * w_norm) / (g_norm + eps) or 1.0 when
// degenerate / LARS disabled, scale = float32(local * gamma).
__device__ __forceinline__ void trust_eval(uint32_t sflags, double sw, double se, double sg,
                                           const gs_step_params* __restrict__ params,
                                           float* scale_out, double* o) {
  const double w_norm = __dsqrt_rn(sw);
  const double g_norm = __dsqrt_rn(se);
  double local = 1.0;
  if (sflags & GS_SEG_LARS_ENABLED) {
    const double denom = __dadd_rn(g_norm, params->epsilon);
    if (!(w_norm == 0.0 || denom == 0.0)) local = __ddiv_rn(__dmul_rn(params->eta, w_norm), denom);
  }
  *scale_out = __double2float_rn(__dmul_rn(local, params->gamma));
  o[0] = w_norm;
  o[1] = g_norm;
  o[2] = local;
  o[3] = sg;
}

// experiment.py:408-411: sqrt(sum over groups of float(dot(g, g))), summed in
// group order starting from 0.
__device__ __forceinline__ double grad_norm_eval(const double* seg_out, int nseg) {
  double acc = 0.0;
  for (int s = 0; s < nseg; ++s) acc = __dadd_rn(acc, __ldcg(seg_out + 4 * (int64_t)s + 3));
  return __dsqrt_rn(acc);
}

// FUSE = false: plain pass 1 (partials + flags).
// FUSE = true : additionally the last CTA to finish a segment (per-segment
// arrival counter) folds that segment's partials in chunk order and writes its
// trust ratio, and the last segment to finish writes the grad norm and the
// empty segments — the trust step costs no extra launch and no tail.  Which
// CTA arrives last is timing-dependent; the result is not: the fold always
// runs over the same chunk range in the same fixed tree.
template <bool F16, bool FUSE>
__global__ void __launch_bounds__(kThreads)
lars_pass1_kernel(const gs_segment* __restrict__ segs, int nseg, int nseg_active,
                  const gs_chunk* __restrict__ chunks, int chunk0,
                  const gs_step_params* __restrict__ params, double* __restrict__ partials,
                  uint32_t* __restrict__ flags, uint32_t* __restrict__ counters,
                  float* __restrict__ seg_scale, double* __restrict__ seg_out,
                  double* __restrict__ grad_norm_out) {
  using T = typename GradIO<F16>::T;
  const int c = chunk0 + blockIdx.x;
  const gs_chunk ch = chunks[c];
  const gs_segment* sg = segs + ch.seg;
  const uint32_t sflags = sg->flags;
  const T* g = static_cast<const T*>(sg->g) + ch.start;
  const float* w = sg->w + ch.start;
  gs::Unscale u;
  u.load(params);
  const float wd = params->weight_decay;
  const bool decay = (u.mode & GS_MODE_DECAY) && !(sflags & GS_SEG_DECAY_EXEMPT);
  const bool gnorm = (u.mode & GS_MODE_GRADNORM) != 0;
  double sw = 0.0, se = 0.0, sgn = 0.0;
  uint32_t fl = 0;
  if (sflags & GS_SEG_LARS_ENABLED)
    pass1_body<F16, true>(g, w, ch.len, u, decay, wd, gnorm, sw, se, sgn, fl);
  else
    pass1_body<F16, false>(g, w, ch.len, u, decay, wd, gnorm, sw, se, sgn, fl);

  fl = __reduce_or_sync(0xFFFFFFFFu, fl);
  if (fl != 0u && (threadIdx.x & 31) == 0) atomicOr(flags, fl);
  gs::block_sum3<kThreads>(sw, se, sgn);
  if (!FUSE) {
    if (threadIdx.x == 0) {
      partials[3 * (int64_t)c + 0] = sw;
      partials[3 * (int64_t)c + 1] = se;
      partials[3 * (int64_t)c + 2] = sgn;
    }
    return;
  }
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    partials[3 * (int64_t)c + 0] = sw;
    partials[3 * (int64_t)c + 1] = se;
    partials[3 * (int64_t)c + 2] = sgn;
    __threadfence();
    const uint32_t prev = atomicAdd(&counters[ch.seg], 1u);
    s_last = (prev + 1 == (uint32_t)sg->chunk_count);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // fold this segment's chunk partials: fixed strided order + fixed tree
  const int cb = sg->chunk_begin, cn = sg->chunk_count;
  double a = 0.0, b = 0.0, d = 0.0;
  for (int i = threadIdx.x; i < cn; i += kThreads) {
    const double* pp = partials + 3 * (int64_t)(cb + i);
    a += __ldcg(pp + 0);
    b += __ldcg(pp + 1);
    d += __ldcg(pp + 2);
  }
  __syncthreads();  // block_sum3's shared scratch is reused
  gs::block_sum3<kThreads>(a, b, d);
  if (threadIdx.x == 0) {
    trust_eval(sflags, a, b, d, params, seg_scale + ch.seg, seg_out + 4 * (int64_t)ch.seg);
    __threadfence();
    const uint32_t prev = atomicAdd(&counters[nseg], 1u);
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

// ----------------------------------------------------------------- trust
__global__ void __launch_bounds__(kTrustThreads)
lars_trust_kernel(const gs_segment* __restrict__ segs, int nseg, const double* __restrict__ partials,
                  const gs_step_params* __restrict__ params, float* __restrict__ seg_scale,
                  double* __restrict__ seg_out, double* __restrict__ grad_norm_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int s = warp; s < nseg; s += kTrustThreads / 32) {
    const int cb = segs[s].chunk_begin, cn = segs[s].chunk_count;
    const uint32_t sflags = segs[s].flags;
    double sw = 0.0, se = 0.0, sg = 0.0;
    for (int i = lane; i < cn; i += 32) {
      const double* p = partials + 3 * (int64_t)(cb + i);
      sw += p[0];
      se += p[1];
      sg += p[2];
    }
    sw = gs::warp_sum(sw);
    se = gs::warp_sum(se);
    sg = gs::warp_sum(sg);
    if (lane == 0) trust_eval(sflags, sw, se, sg, params, seg_scale + s, seg_out + 4 * (int64_t)s);
  }
  __syncthreads();
  if (threadIdx.x == 0 && grad_norm_out != nullptr) *grad_norm_out = grad_norm_eval(seg_out, nseg);
}

// ----------------------------------------------------------------- pass 2
template <bool F16>
__global__ void __launch_bounds__(kThreads)
lars_pass2_kernel(const gs_segment* __restrict__ segs, const gs_chunk* __restrict__ chunks, int chunk0,
                  const gs_step_params* __restrict__ params, const float* __restrict__ seg_scale,
                  const uint32_t* __restrict__ flags, uint32_t flag_mask) {
  using T = typename GradIO<F16>::T;
  // lars.py:161-163 — a non-finite step mutates nothing
  if (*flags & flag_mask) return;
  const int c = chunk0 + blockIdx.x;
  const gs_chunk ch = chunks[c];
  const gs_segment* sg = segs + ch.seg;
  const uint32_t sflags = sg->flags;
  const T* __restrict__ g = static_cast<const T*>(sg->g) + ch.start;
  float* __restrict__ w = sg->w + ch.start;
  float* __restrict__ v = sg->v + ch.start;
  uint16_t* __restrict__ w16 = sg->w16 + ch.start;
  gs::Unscale u;
  u.load(params);
  const float wd = params->weight_decay;
  const float m = params->momentum;
  const float s = seg_scale[ch.seg];
  const bool decay = (u.mode & GS_MODE_DECAY) && !(sflags & GS_SEG_DECAY_EXEMPT);
  const int len = ch.len;

  auto upd = [&](float graw, float& wv, float& vv) {
    const float gu = u.unscale(u.mean(graw));
    const float eff = decay ? __fadd_rn(gu, __fmul_rn(wd, wv)) : gu;  // lars.py:172
    vv = __fadd_rn(__fmul_rn(m, vv), __fmul_rn(s, eff));               // lars.py:178
    wv = __fsub_rn(wv, vv);                                             // lars.py:179
  };

  const bool vec = gs::is_aligned16(g) && gs::is_aligned16(w) && gs::is_aligned16(v) &&
                   gs::is_aligned16(w16);
  const int nv = vec ? len / 8 : 0;
#pragma unroll 2
  for (int i = threadIdx.x; i < nv; i += kThreads) {
    float gf[8], wf[8], vf[8];
    GradIO<F16>::load8(g + 8 * i, gf);
    load8f(w + 8 * i, wf);
    load8f(v + 8 * i, vf);
#pragma unroll
    for (int k = 0; k < 8; ++k) upd(gf[k], wf[k], vf[k]);
    store8f(v + 8 * i, vf);
    store8f(w + 8 * i, wf);
    uint4 h;
    h.x = gs::narrow2(wf[0], wf[1]);
    h.y = gs::narrow2(wf[2], wf[3]);
    h.z = gs::narrow2(wf[4], wf[5]);
    h.w = gs::narrow2(wf[6], wf[7]);
    *reinterpret_cast<uint4*>(w16 + 8 * i) = h;  // lars.py:180
  }
  for (int i = nv * 8 + threadIdx.x; i < len; i += kThreads) {
    float wv = w[i], vv = v[i];
    upd(GradIO<F16>::load1(g + i), wv, vv);
    v[i] = vv;
    w[i] = wv;
    w16[i] = gs::narrow(wv);
  }
}

}  // namespace

extern "C" {

int gs_lars_pass1(const gs_segment* segs, const gs_chunk* chunks, int chunk0, int nchunk,
                  int g_is_f16, const gs_step_params* params, double* partials, uint32_t* flags,
                  void* stream) {
  GS_REQUIRE(nchunk >= 0 && chunk0 >= 0, "gs_lars_pass1: bad chunk range");
  if (nchunk == 0) return GS_OK;
  GS_REQUIRE(segs && chunks && params && partials && flags, "gs_lars_pass1: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  if (g_is_f16)
    lars_pass1_kernel<true, false><<<nchunk, kThreads, 0, s>>>(
        segs, 0, 0, chunks, chunk0, params, partials, flags, nullptr, nullptr, nullptr, nullptr);
  else
    lars_pass1_kernel<false, false><<<nchunk, kThreads, 0, s>>>(
        segs, 0, 0, chunks, chunk0, params, partials, flags, nullptr, nullptr, nullptr, nullptr);
  return gs_check_launch("gs_lars_pass1");
}

int gs_lars_pass1_trust(const gs_segment* segs, int nseg, int nseg_active, const gs_chunk* chunks,
                        int chunk0, int nchunk, int g_is_f16, const gs_step_params* params,
                        double* partials, uint32_t* flags, uint32_t* counters, float* seg_scale,
                        double* seg_out, double* grad_norm_out, void* stream) {
  GS_REQUIRE(nchunk >= 0 && chunk0 >= 0, "gs_lars_pass1_trust: bad chunk range");
  GS_REQUIRE(nseg_active >= 1 && nseg_active <= nseg,
             "gs_lars_pass1_trust: need 1 <= nseg_active <= nseg (use gs_lars_trust otherwise)");
  if (nchunk == 0) return GS_OK;
  GS_REQUIRE(segs && chunks && params && partials && flags && counters && seg_scale && seg_out,
             "gs_lars_pass1_trust: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  if (g_is_f16)
    lars_pass1_kernel<true, true><<<nchunk, kThreads, 0, s>>>(
        segs, nseg, nseg_active, chunks, chunk0, params, partials, flags, counters, seg_scale,
        seg_out, grad_norm_out);
  else
    lars_pass1_kernel<false, true><<<nchunk, kThreads, 0, s>>>(
        segs, nseg, nseg_active, chunks, chunk0, params, partials, flags, counters, seg_scale,
        seg_out, grad_norm_out);
  return gs_check_launch("gs_lars_pass1_trust");
}

int gs_lars_trust(const gs_segment* segs, int nseg, const double* partials,
                  const gs_step_params* params, float* seg_scale, double* seg_out,
                  double* grad_norm_out, void* stream) {
  GS_REQUIRE(nseg >= 0, "gs_lars_trust: negative segment count");
  if (nseg == 0) return GS_OK;
  GS_REQUIRE(segs && partials && params && seg_scale && seg_out, "gs_lars_trust: null pointer");
  lars_trust_kernel<<<1, kTrustThreads, 0, (cudaStream_t)stream>>>(segs, nseg, partials, params,
                                                                   seg_scale, seg_out, grad_norm_out);
  return gs_check_launch("gs_lars_trust");
}

int gs_lars_pass2(const gs_segment* segs, const gs_chunk* chunks, int chunk0, int nchunk,
                  int g_is_f16, const gs_step_params* params, const float* seg_scale,
                  const uint32_t* flags, uint32_t flag_mask, void* stream) {
  GS_REQUIRE(nchunk >= 0 && chunk0 >= 0, "gs_lars_pass2: bad chunk range");
  if (nchunk == 0) return GS_OK;
  GS_REQUIRE(segs && chunks && params && seg_scale && flags, "gs_lars_pass2: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  if (g_is_f16)
    lars_pass2_kernel<true><<<nchunk, kThreads, 0, s>>>(segs, chunks, chunk0, params, seg_scale, flags,
                                                        flag_mask);
  else
    lars_pass2_kernel<false><<<nchunk, kThreads, 0, s>>>(segs, chunks, chunk0, params, seg_scale,
                                                         flags, flag_mask);
  return gs_check_launch("gs_lars_pass2");
}

}  // extern "C"
