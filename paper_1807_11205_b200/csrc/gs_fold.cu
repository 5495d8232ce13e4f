// gs_fold.cu — the reference's fixed-order reductions, one pass over p slots.
//
//   fold_ascending  collectives.py:261-270  fp32 left fold b0+b1+...; mean
//                                           divides by float32(p) afterwards
//   fold_f16_tree   collectives.py:273-283  pairwise tree over binary16
//                                           patterns: level pairs (i, i+1),
//                                           each combine widen-add-narrow,
//                                           odd tail carried to the next level
//
// The slots are device pointers — local buffers for the single-process list
// API (ring_allreduce([...]) with p buffers), or peer-mapped NVLink pointers
// of a symmetric-memory window for the multi-GPU ordered all-reduce, where
// rank r folds chunk r straight out of every peer's HBM.
//
// The in-register tree below reproduces the reference level structure
// exactly: at level L (stride s = 2^(L-1)) item i (i a multiple of 2s)
// combines with item i+s when i+s < p, otherwise it is carried unchanged.
#include "gs_common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kMaxGenericP = 64;

inline int grid_for(int64_t items) {
  int64_t b = (items + kThreads - 1) / kThreads;
  if (b > 148 * 8) b = 148 * 8;
  if (b < 1) b = 1;
  return (int)b;
}

__device__ __forceinline__ float add_narrow(float a, float b) {
  // combine of fold_f16_tree: f32_to_f16(f16_to_f32(a) + f16_to_f32(b));
  // kept widened so the next level reads it back exactly
  return gs::widen(gs::narrow(__fadd_rn(a, b)));
}

template <int P>
__device__ __forceinline__ float tree_fixed(float (&v)[P]) {
#pragma unroll
  for (int s = 1; s < P; s *= 2) {
#pragma unroll
    for (int i = 0; i + s < P; i += 2 * s) v[i] = add_narrow(v[i], v[i + s]);
  }
  return v[0];
}

__device__ __forceinline__ float tree_generic(float* v, int p) {
  for (int s = 1; s < p; s *= 2)
    for (int i = 0; i + s < p; i += 2 * s) v[i] = add_narrow(v[i], v[i + s]);
  return v[0];
}

// ---- fp16 tree fold, compile-time p, 8 elements per thread (uint4) ----
template <int P>
__global__ void __launch_bounds__(kThreads)
fold_f16_fixed_kernel(const uint64_t* __restrict__ slots, int64_t offset, uint16_t* out, int64_t n,
                      uint32_t* __restrict__ nonfinite, int vec) {
  const uint16_t* src[P];
#pragma unroll
  for (int r = 0; r < P; ++r) {
    src[r] = reinterpret_cast<const uint16_t*>(slots[r]) + offset;
    vec = vec && gs::is_aligned16(src[r]);
  }
  uint32_t bad = 0;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t tail_begin = 0;
  if (vec) {
    const int64_t nv = n / 8;
    for (int64_t i = tid; i < nv; i += stride) {
      uint4 raw[P];
#pragma unroll
      for (int r = 0; r < P; ++r) raw[r] = reinterpret_cast<const uint4*>(src[r])[i];
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float lo[P], hi[P];
#pragma unroll
        for (int r = 0; r < P; ++r) {
          const uint32_t w = (&raw[r].x)[q];
          const float2 f = gs::widen2(w);
          lo[r] = f.x;
          hi[r] = f.y;
        }
        uint32_t bits;
        if (P == 1) {
          bits = (&raw[0].x)[q];
        } else {
          bits = gs::narrow2(tree_fixed<P>(lo), tree_fixed<P>(hi));
        }
        bad |= ((bits & 0x7C00u) == 0x7C00u) | ((bits & 0x7C000000u) == 0x7C000000u);
        o[q] = bits;
      }
      reinterpret_cast<uint4*>(out)[i] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    tail_begin = nv * 8;
  }
  for (int64_t i = tail_begin + tid; i < n; i += stride) {
    uint16_t bits;
    if (P == 1) {
      bits = src[0][i];
    } else {
      float v[P];
#pragma unroll
      for (int r = 0; r < P; ++r) v[r] = gs::widen(src[r][i]);
      bits = gs::narrow(tree_fixed<P>(v));
    }
    bad |= (bits & 0x7C00u) == 0x7C00u;
    out[i] = bits;
  }
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (nonfinite != nullptr && bad && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1u);
}

__global__ void __launch_bounds__(kThreads)
fold_f16_generic_kernel(const uint64_t* __restrict__ slots, int p, int64_t offset, uint16_t* out,
                        int64_t n, uint32_t* __restrict__ nonfinite) {
  uint32_t bad = 0;
  float v[kMaxGenericP];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int r = 0; r < p; ++r) v[r] = gs::widen(reinterpret_cast<const uint16_t*>(slots[r])[offset + i]);
    const uint16_t bits = p == 1 ? reinterpret_cast<const uint16_t*>(slots[0])[offset + i]
                                 : gs::narrow(tree_generic(v, p));
    bad |= (bits & 0x7C00u) == 0x7C00u;
    out[i] = bits;
  }
  bad = __reduce_or_sync(0xFFFFFFFFu, bad);
  if (nonfinite != nullptr && bad && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1u);
}

// ---- fp32 ascending left fold, 4 elements per thread (float4) ----
__global__ void __launch_bounds__(kThreads)
fold_f32_kernel(const uint64_t* __restrict__ slots, int p, int64_t offset, float* out, int64_t n,
                int mean, float divisor, int pow2, float rcp, int vec) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto finish = [&](float a) {
    if (mean) a = pow2 ? __fmul_rn(a, rcp) : __fdiv_rn(a, divisor);
    return a;
  };
  for (int r = 0; r < p && vec; ++r)
    vec = gs::is_aligned16(reinterpret_cast<const float*>(slots[r]) + offset);
  int64_t tail_begin = 0;
  if (vec) {
    const int64_t nv = n / 4;
    for (int64_t i = tid; i < nv; i += stride) {
      float4 acc = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(slots[0]) + offset)[i];
      for (int r = 1; r < p; ++r) {
        const float4 b =
            reinterpret_cast<const float4*>(reinterpret_cast<const float*>(slots[r]) + offset)[i];
        acc.x = __fadd_rn(acc.x, b.x);
        acc.y = __fadd_rn(acc.y, b.y);
        acc.z = __fadd_rn(acc.z, b.z);
        acc.w = __fadd_rn(acc.w, b.w);
      }
      acc.x = finish(acc.x);
      acc.y = finish(acc.y);
      acc.z = finish(acc.z);
      acc.w = finish(acc.w);
      reinterpret_cast<float4*>(out)[i] = acc;
    }
    tail_begin = nv * 4;
  }
  for (int64_t i = tail_begin + tid; i < n; i += stride) {
    float acc = reinterpret_cast<const float*>(slots[0])[offset + i];
    for (int r = 1; r < p; ++r) acc = __fadd_rn(acc, reinterpret_cast<const float*>(slots[r])[offset + i]);
    out[i] = finish(acc);
  }
}

bool is_pow2_float(int p) { return p > 0 && (p & (p - 1)) == 0; }

}  // namespace

extern "C" {

int gs_fold_f32(const uint64_t* slots, int p, int64_t offset, float* out, int64_t n, int mean,
                void* stream) {
  GS_REQUIRE(p >= 1, "gs_fold_f32: need at least one slot");
  GS_REQUIRE(n >= 0 && offset >= 0, "gs_fold_f32: negative size/offset");
  if (n == 0) return GS_OK;
  GS_REQUIRE(slots && out, "gs_fold_f32: null pointer");
  // the kernel additionally requires every slot + offset to be 16-byte aligned
  const int vec = gs::is_aligned16(out);
  const float divisor = (float)p;
  const int pow2 = is_pow2_float(p);
  fold_f32_kernel<<<grid_for(vec ? n / 4 + 1 : n), kThreads, 0, (cudaStream_t)stream>>>(
      slots, p, offset, out, n, mean, divisor, pow2, 1.0f / divisor, vec);
  return gs_check_launch("gs_fold_f32");
}

// Variant selector: compile-time p for the common world sizes, a generic
// single-pass kernel up to kMaxGenericP.  The kernels themselves drop to the
// scalar path when any slot + offset is not 16-byte aligned.
static int fold_f16_launch(const uint64_t* slots, int p, int64_t offset, uint16_t* out, int64_t n,
                           uint32_t* nonfinite, cudaStream_t s) {
  const int vec = gs::is_aligned16(out);
  const int grid = grid_for(vec ? n / 8 + 1 : n);
#define GS_FOLD_CASE(P)                                                                         \
  case P:                                                                                       \
    fold_f16_fixed_kernel<P><<<grid, kThreads, 0, s>>>(slots, offset, out, n, nonfinite, vec); \
    break;
  switch (p) {
    GS_FOLD_CASE(1)
    GS_FOLD_CASE(2)
    GS_FOLD_CASE(3)
    GS_FOLD_CASE(4)
    GS_FOLD_CASE(5)
    GS_FOLD_CASE(6)
    GS_FOLD_CASE(7)
    GS_FOLD_CASE(8)
    GS_FOLD_CASE(16)
    default:
      if (p > kMaxGenericP) {
        gs_set_error("gs_fold_f16_tree: p=%d exceeds the single-pass limit %d", p, kMaxGenericP);
        return GS_EINVAL;
      }
      fold_f16_generic_kernel<<<grid_for(n), kThreads, 0, s>>>(slots, p, offset, out, n, nonfinite);
  }
#undef GS_FOLD_CASE
  return gs_check_launch("gs_fold_f16_tree");
}

int gs_fold_f16_tree(const uint64_t* slots, int p, int64_t offset, uint16_t* out, int64_t n,
                     uint32_t* nonfinite, void* stream) {
  GS_REQUIRE(p >= 1, "gs_fold_f16_tree: need at least one slot");
  GS_REQUIRE(n >= 0 && offset >= 0, "gs_fold_f16_tree: negative size/offset");
  if (n == 0) return GS_OK;
  GS_REQUIRE(slots && out, "gs_fold_f16_tree: null pointer");
  return fold_f16_launch(slots, p, offset, out, n, nonfinite, (cudaStream_t)stream);
}

}  // extern "C"
