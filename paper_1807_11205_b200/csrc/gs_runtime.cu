// gs_runtime.cu — error reporting, version and device queries for the C ABI.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <mutex>

#include "gs_common.cuh"

// the Python mirrors (_native.py *_DTYPE) assert the same sizes
static_assert(sizeof(gs_segment) == 64, "gs_segment layout");
static_assert(sizeof(gs_chunk) == 16, "gs_chunk layout");
static_assert(sizeof(gs_copy) == 24, "gs_copy layout");
static_assert(sizeof(gs_step_params) == 56, "gs_step_params layout");
static_assert(sizeof(gs_ctl) == 48, "gs_ctl layout");
static_assert(sizeof(gs_rank_ctx) == 120, "gs_rank_ctx layout");
static_assert(sizeof(gs_step_rank) == 96, "gs_step_rank layout");

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

void gs_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int gs_check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    gs_set_error("%s: %s", what, cudaGetErrorString(e));
    return GS_ECUDA;
  }
  return GS_OK;
}

int gs_resident_ctas(const void* kernel, int threads, size_t smem) {
  struct Entry {
    const void* k;
    int threads, dev;
    size_t smem;
    int ctas;
  };
  static Entry cache[256];
  static int n = 0;
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < n; ++i)
      if (cache[i].k == kernel && cache[i].threads == threads && cache[i].smem == smem &&
          cache[i].dev == dev)
        return cache[i].ctas;
  }
  int per_sm = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  const int ctas = (per_sm > 0 ? per_sm : 1) * (sms > 0 ? sms : 148);
  std::lock_guard<std::mutex> lock(mu);
  if (n < 256) cache[n++] = Entry{kernel, threads, dev, smem, ctas};
  return ctas;
}

namespace {
__global__ void fill_zero_kernel(uint4* __restrict__ dst, int64_t n16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = make_uint4(0, 0, 0, 0);
}
__global__ void fill_zero_bytes_kernel(uint8_t* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = 0;
}
}  // namespace

extern "C" {

int gs_abi_version(void) { return GS_ABI_VERSION; }

const char* gs_last_error(void) { return g_err; }

int64_t gs_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int gs_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    gs_set_error("cudaDeviceGetAttribute failed for device %d", device);
    return GS_ECUDA;
  }
  return v;
}

int gs_fill_zero(void* dst, int64_t nbytes, void* stream) {
  GS_REQUIRE(nbytes >= 0, "gs_fill_zero: negative size");
  if (nbytes == 0) return GS_OK;
  GS_REQUIRE(dst != nullptr, "gs_fill_zero: null dst");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && (nbytes & 15) == 0) {
    const int64_t n16 = nbytes / 16;
    int64_t blocks = (n16 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    fill_zero_kernel<<<(int)blocks, 256, 0, s>>>(static_cast<uint4*>(dst), n16);
  } else {
    int64_t blocks = (nbytes + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    fill_zero_bytes_kernel<<<(int)blocks, 256, 0, s>>>(static_cast<uint8_t*>(dst), nbytes);
  }
  return gs_check_launch("gs_fill_zero");
}

}  // extern "C"
