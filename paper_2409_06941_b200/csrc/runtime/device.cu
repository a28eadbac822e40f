// Stream / device helpers of the C-ABI (freeride_gpu.h).
#include "freeride_gpu.h"
#include "kernels/common.cuh"

namespace {

// One warp spins for `cycles` SM clocks and records (clock64 delta,
// globaltimer delta): the SM frequency the GPU is running at right now.
__global__ void clock_probe_kernel(unsigned long long* out, long long cycles) {
  if (threadIdx.x != 0) return;
  const long long c0 = clock64();
  const unsigned long long t0 = frk::globaltimer_ns();
  long long c = c0;
  while (c - c0 < cycles) c = clock64();
  const unsigned long long t1 = frk::globaltimer_ns();
  out[0] = static_cast<unsigned long long>(c - c0);
  out[1] = t1 - t0;
}

// L2 bandwidth probe: every CTA streams its slice of an L2-resident buffer
// `passes` times with 16 B ld.global.cg (L2, not L1), so after the first pass
// the bytes come from L2 -- the bound of a kernel whose working set stays in
// L2 (PageRank at RMAT-20).  The xor into `sink` keeps the loads alive.
__global__ void l2_read_kernel(const int4* __restrict__ p, int64_t n, int passes, int4* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int q = 0; q < passes; ++q)
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
      const int4 v = __ldcg(p + i);
      acc.x ^= v.x;
      acc.y ^= v.y;
      acc.z ^= v.z;
      acc.w ^= v.w;
    }
  if ((acc.x & acc.y & acc.z & acc.w) == 0x7fffffff) sink[0] = acc;  // practically never
}

}  // namespace

extern "C" {

int fr_l2_read_probe(const void* buf, int64_t bytes, int32_t passes, void* sink16, void* stream) {
  if (!buf || !sink16 || bytes < 16 || passes < 1) return frcapi::fail(FR_ERR_ARGUMENT, "bad probe args");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  l2_read_kernel<<<sms * 4, 512, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const int4*>(buf), bytes / 16, passes, static_cast<int4*>(sink16));
  FR_CUDA_LAUNCHED("l2_read_probe");
  return FR_OK;
}

int fr_clock_probe(uint64_t* out_cycles_ns, int64_t cycles, void* stream) {
  if (!out_cycles_ns || cycles < 1) return frcapi::fail(FR_ERR_ARGUMENT, "bad probe args");
  clock_probe_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<unsigned long long*>(out_cycles_ns), cycles);
  FR_CUDA_LAUNCHED("clock_probe");
  return FR_OK;
}

int fr_memcpy(void* dst, const void* src, int64_t bytes) {
  if (bytes < 0) return frcapi::fail(FR_ERR_ARGUMENT, "negative size");
  if (bytes) FR_CUDA_TRY(cudaMemcpy(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault));
  return FR_OK;
}

int fr_stream_create(int32_t priority_class, void** stream) {
  if (!stream) return frcapi::fail(FR_ERR_ARGUMENT, "null stream out");
  int least = 0, greatest = 0;  // CUDA: numerically lower = higher priority
  FR_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  cudaStream_t s = nullptr;
  FR_CUDA_TRY(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking,
                                           priority_class == 0 ? least : greatest));
  *stream = s;
  return FR_OK;
}

int fr_stream_destroy(void* stream) {
  if (stream) FR_CUDA_TRY(cudaStreamDestroy(static_cast<cudaStream_t>(stream)));
  return FR_OK;
}

int fr_stream_synchronize(void* stream) {
  FR_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return FR_OK;
}

// The library links its own (static) CUDA runtime: make its current device
// explicit for the calling thread instead of relying on the driver context
// another runtime (torch's) left current.
int fr_set_device(int32_t device) {
  FR_CUDA_TRY(cudaSetDevice(device));
  return FR_OK;
}

int fr_get_device(int32_t* device) {
  if (!device) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  int d = 0;
  FR_CUDA_TRY(cudaGetDevice(&d));
  *device = d;
  return FR_OK;
}

int fr_device_sm_count(int32_t* sms) {
  int dev = 0, n = 0;
  FR_CUDA_TRY(cudaGetDevice(&dev));
  FR_CUDA_TRY(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  *sms = n;
  return FR_OK;
}

}  // extern "C"
