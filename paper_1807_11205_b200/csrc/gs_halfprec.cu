// gs_halfprec.cu — binary16 conversions, unscale and the finite test.
//
// Replaces the numpy bit manipulation of the reference
//   f32_to_f16 / _narrow_bits   halfprec.py:40-85, 108-121
//   f16_to_f32 / _widen_bits    halfprec.py:88-105, 124-132
//   quantize_tensor             halfprec.py:135-137
//   unscale_gradients           halfprec.py:230-234
//   LossScale.update isfinite   halfprec.py:209-210
// All kernels are grid-stride, 8 elements per thread per iteration with
// 128-bit accesses when every pointer is 16-byte aligned, scalar otherwise.
#include "gs_common.cuh"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ bool half2_nonfinite(uint32_t w) {
  return ((w & 0x7C00u) == 0x7C00u) | ((w & 0x7C000000u) == 0x7C000000u);
}

inline int grid_for(int64_t work_items) {
  int64_t b = (work_items + kThreads - 1) / kThreads;
  const int64_t cap = 148 * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

__global__ void __launch_bounds__(kThreads)
f32_to_f16_kernel(const float* __restrict__ x, uint16_t* __restrict__ h, int64_t n, float scale,
                  int apply_scale, uint32_t* __restrict__ nonfinite, int vec) {
  uint32_t bad = 0;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t tail_begin = 0;
  if (vec) {
    const int64_t nv = n / 8;
    for (int64_t i = tid; i < nv; i += stride) {
      const float4 a = reinterpret_cast<const float4*>(x)[2 * i];
      const float4 b = reinterpret_cast<const float4*>(x)[2 * i + 1];
      float f[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      if (apply_scale) {
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = __fmul_rn(f[k], scale);
      }
      uint4 o;
      o.x = gs::narrow2(f[0], f[1]);
      o.y = gs::narrow2(f[2], f[3]);
      o.z = gs::narrow2(f[4], f[5]);
      o.w = gs::narrow2(f[6], f[7]);
      // a half is non-finite iff its exponent field is all ones
      bad |= half2_nonfinite(o.x) | half2_nonfinite(o.y) | half2_nonfinite(o.z) |
             half2_nonfinite(o.w);
      reinterpret_cast<uint4*>(h)[i] = o;
    }
    tail_begin = nv * 8;
  }
  for (int64_t i = tail_begin + tid; i < n; i += stride) {
    float f = x[i];
    if (apply_scale) f = __fmul_rn(f, scale);
    const uint16_t o = gs::narrow(f);
    bad |= (o & 0x7C00u) == 0x7C00u;
    h[i] = o;
  }
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (nonfinite != nullptr && bad && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1u);
}

// f16_to_f32's NaN is numpy's float32 NaN, 0x7FC00000, whatever the binary16
// payload or sign (halfprec.py:103-104); cvt.f32.f16 would keep both
__device__ __forceinline__ float canon(float x) {
  return x != x ? __uint_as_float(0x7FC00000u) : x;
}

__global__ void __launch_bounds__(kThreads)
f16_to_f32_kernel(const uint16_t* __restrict__ h, float* __restrict__ x, int64_t n, int vec) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t tail_begin = 0;
  if (vec) {
    const int64_t nv = n / 8;
    for (int64_t i = tid; i < nv; i += stride) {
      const uint4 a = reinterpret_cast<const uint4*>(h)[i];
      const float2 p0 = gs::widen2(a.x), p1 = gs::widen2(a.y), p2 = gs::widen2(a.z),
                   p3 = gs::widen2(a.w);
      reinterpret_cast<float4*>(x)[2 * i] =
          make_float4(canon(p0.x), canon(p0.y), canon(p1.x), canon(p1.y));
      reinterpret_cast<float4*>(x)[2 * i + 1] =
          make_float4(canon(p2.x), canon(p2.y), canon(p3.x), canon(p3.y));
    }
    tail_begin = nv * 8;
  }
  for (int64_t i = tail_begin + tid; i < n; i += stride) x[i] = canon(gs::widen(h[i]));
}

__global__ void __launch_bounds__(kThreads)
quantize_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n, int vec) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t tail_begin = 0;
  if (vec) {
    const int64_t nv = n / 4;
    for (int64_t i = tid; i < nv; i += stride) {
      float4 a = reinterpret_cast<const float4*>(x)[i];
      a.x = gs::widen(gs::narrow(a.x));
      a.y = gs::widen(gs::narrow(a.y));
      a.z = gs::widen(gs::narrow(a.z));
      a.w = gs::widen(gs::narrow(a.w));
      reinterpret_cast<float4*>(y)[i] = a;
    }
    tail_begin = nv * 4;
  }
  for (int64_t i = tail_begin + tid; i < n; i += stride) y[i] = gs::widen(gs::narrow(x[i]));
}

__global__ void __launch_bounds__(kThreads)
unscale_kernel(const float* __restrict__ g, float* __restrict__ out, int64_t n, float scale,
               int vec) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t tail_begin = 0;
  if (vec) {
    const int64_t nv = n / 4;
    for (int64_t i = tid; i < nv; i += stride) {
      float4 a = reinterpret_cast<const float4*>(g)[i];
      a.x = __fdiv_rn(a.x, scale);
      a.y = __fdiv_rn(a.y, scale);
      a.z = __fdiv_rn(a.z, scale);
      a.w = __fdiv_rn(a.w, scale);
      reinterpret_cast<float4*>(out)[i] = a;
    }
    tail_begin = nv * 4;
  }
  for (int64_t i = tail_begin + tid; i < n; i += stride) out[i] = __fdiv_rn(g[i], scale);
}

// grid: (x = blocks over the longest tensor, y = tensor index)
__global__ void __launch_bounds__(kThreads)
nonfinite_kernel(const uint64_t* __restrict__ ptrs, const int64_t* __restrict__ lens, int is_f16,
                 uint32_t* __restrict__ flag, uint32_t bit) {
  const int t = blockIdx.y;
  const int64_t n = lens[t];
  const int64_t per_block = (int64_t)kThreads * 16;
  const int64_t begin = blockIdx.x * per_block;
  if (begin >= n) return;
  const int64_t end = begin + per_block < n ? begin + per_block : n;
  uint32_t bad = 0;
  if (is_f16) {
    const uint16_t* p = reinterpret_cast<const uint16_t*>(ptrs[t]);
    for (int64_t i = begin + threadIdx.x; i < end; i += kThreads) bad |= (p[i] & 0x7C00u) == 0x7C00u;
  } else {
    const float* p = reinterpret_cast<const float*>(ptrs[t]);
    for (int64_t i = begin + threadIdx.x; i < end; i += kThreads) bad |= !gs::is_finite_f32(p[i]);
  }
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (bad && (threadIdx.x & 31) == 0) atomicOr(flag, bit);
}

}  // namespace

extern "C" {

int gs_f32_to_f16(const float* x, uint16_t* h, int64_t n, float scale, uint32_t* nonfinite,
                  void* stream) {
  GS_REQUIRE(n >= 0, "gs_f32_to_f16: negative length");
  if (n == 0) return GS_OK;
  GS_REQUIRE(x && h, "gs_f32_to_f16: null pointer");
  const int vec = gs::is_aligned16(x) && gs::is_aligned16(h);
  const int apply = !(scale == 1.0f);
  f32_to_f16_kernel<<<grid_for(vec ? n / 8 + 1 : n), kThreads, 0, (cudaStream_t)stream>>>(
      x, h, n, scale, apply, nonfinite, vec);
  return gs_check_launch("gs_f32_to_f16");
}

int gs_f16_to_f32(const uint16_t* h, float* x, int64_t n, void* stream) {
  GS_REQUIRE(n >= 0, "gs_f16_to_f32: negative length");
  if (n == 0) return GS_OK;
  GS_REQUIRE(x && h, "gs_f16_to_f32: null pointer");
  const int vec = gs::is_aligned16(x) && gs::is_aligned16(h);
  f16_to_f32_kernel<<<grid_for(vec ? n / 8 + 1 : n), kThreads, 0, (cudaStream_t)stream>>>(h, x, n,
                                                                                          vec);
  return gs_check_launch("gs_f16_to_f32");
}

int gs_quantize_f32(const float* x, float* y, int64_t n, void* stream) {
  GS_REQUIRE(n >= 0, "gs_quantize_f32: negative length");
  if (n == 0) return GS_OK;
  GS_REQUIRE(x && y, "gs_quantize_f32: null pointer");
  const int vec = gs::is_aligned16(x) && gs::is_aligned16(y);
  quantize_kernel<<<grid_for(vec ? n / 4 + 1 : n), kThreads, 0, (cudaStream_t)stream>>>(x, y, n,
                                                                                        vec);
  return gs_check_launch("gs_quantize_f32");
}

int gs_unscale_f32(const float* g, float* out, int64_t n, float scale, void* stream) {
  GS_REQUIRE(n >= 0, "gs_unscale_f32: negative length");
  if (n == 0) return GS_OK;
  GS_REQUIRE(g && out, "gs_unscale_f32: null pointer");
  const int vec = gs::is_aligned16(g) && gs::is_aligned16(out);
  unscale_kernel<<<grid_for(vec ? n / 4 + 1 : n), kThreads, 0, (cudaStream_t)stream>>>(g, out, n,
                                                                                       scale, vec);
  return gs_check_launch("gs_unscale_f32");
}

int gs_nonfinite(const uint64_t* ptrs, const int64_t* lens, int ntensors, int64_t max_len,
                       int is_f16, uint32_t* flag, uint32_t bit, void* stream) {
  GS_REQUIRE(ntensors >= 0 && ntensors <= 65535, "gs_nonfinite: bad tensor count %d", ntensors);
  GS_REQUIRE(max_len >= 0, "gs_nonfinite: negative max_len");
  if (ntensors == 0 || max_len == 0) return GS_OK;
  GS_REQUIRE(ptrs && lens && flag, "gs_nonfinite: null pointer");
  const int64_t per_block = (int64_t)kThreads * 16;
  const int64_t bx = (max_len + per_block - 1) / per_block;
  GS_REQUIRE(bx < (1LL << 31), "gs_nonfinite: tensor too long");
  dim3 grid((unsigned)bx, (unsigned)ntensors);
  nonfinite_kernel<<<grid, kThreads, 0, (cudaStream_t)stream>>>(ptrs, lens, is_f16, flag, bit);
  return gs_check_launch("gs_nonfinite");
}

}  // extern "C"
