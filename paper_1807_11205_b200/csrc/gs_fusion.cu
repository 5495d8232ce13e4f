// gs_fusion.cu — the fusion-buffer packer (reference FusionBuffer._emit,
// fusion.py:83-94, which np.concatenate's the pending tensors in arrival
// order into one fresh payload).
//
// One CTA per gs_copy entry.  The host splits every tensor into pieces of at
// most kPieceBytes so the grid load-balances over the skewed tensor sizes of
// ResNet-50 / AlexNet (64 B ... 75 MB).  Body copies are 128-bit with 8
// independent loads in flight per thread before the stores; misaligned
// entries fall back to the widest element size both ends share.
#include "gs_common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 8;  // uint4 per thread per round -> 32 KiB per CTA round

template <typename T>
__device__ __forceinline__ void copy_elems(const T* __restrict__ s, T* __restrict__ d, int64_t n) {
  for (int64_t i = threadIdx.x; i < n; i += kThreads) d[i] = s[i];
}

__global__ void __launch_bounds__(kThreads)
batched_copy_kernel(const gs_copy* __restrict__ copies) {
  const gs_copy c = copies[blockIdx.x];
  const uint8_t* s = static_cast<const uint8_t*>(c.src);
  uint8_t* d = static_cast<uint8_t*>(c.dst);
  int64_t n = c.nbytes;
  const uintptr_t sa = reinterpret_cast<uintptr_t>(s), da = reinterpret_cast<uintptr_t>(d);
  if (((sa ^ da) & 15u) == 0) {
    // same phase mod 16: scalar head up to the 16-byte boundary, uint4 body
    int64_t head = (int64_t)((16 - (da & 15u)) & 15u);
    if (head > n) head = n;
    if (threadIdx.x < head) d[threadIdx.x] = s[threadIdx.x];
    s += head;
    d += head;
    n -= head;
    const int64_t nv = n / 16;
    const uint4* __restrict__ sv = reinterpret_cast<const uint4*>(s);
    uint4* __restrict__ dv = reinterpret_cast<uint4*>(d);
    int64_t base = 0;
    for (; base + (int64_t)kThreads * kUnroll <= nv; base += (int64_t)kThreads * kUnroll) {
      uint4 r[kUnroll];
#pragma unroll
      for (int k = 0; k < kUnroll; ++k) r[k] = __ldcs(sv + base + k * kThreads + threadIdx.x);
#pragma unroll
      for (int k = 0; k < kUnroll; ++k) dv[base + k * kThreads + threadIdx.x] = r[k];
    }
    for (int64_t i = base + threadIdx.x; i < nv; i += kThreads) dv[i] = __ldcs(sv + i);
    const int64_t tail = n - nv * 16;
    if (threadIdx.x < tail) d[nv * 16 + threadIdx.x] = s[nv * 16 + threadIdx.x];
  } else if (((sa | da | (uintptr_t)n) & 3u) == 0) {
    copy_elems(reinterpret_cast<const uint32_t*>(s), reinterpret_cast<uint32_t*>(d), n / 4);
  } else if (((sa | da | (uintptr_t)n) & 1u) == 0) {
    copy_elems(reinterpret_cast<const uint16_t*>(s), reinterpret_cast<uint16_t*>(d), n / 2);
  } else {
    copy_elems(s, d, n);
  }
}

}  // namespace

extern "C" {

int gs_batched_copy(const gs_copy* copies, int ncopies, void* stream) {
  GS_REQUIRE(ncopies >= 0, "gs_batched_copy: negative count");
  if (ncopies == 0) return GS_OK;
  GS_REQUIRE(copies != nullptr, "gs_batched_copy: null table");
  batched_copy_kernel<<<ncopies, kThreads, 0, (cudaStream_t)stream>>>(copies);
  return gs_check_launch("gs_batched_copy");
}

}  // extern "C"
