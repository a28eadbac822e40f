// Stream / device helpers of the C-ABI (freeride_gpu.h).
#include "freeride_gpu.h"
#include "kernels/common.cuh"

extern "C" {

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

int fr_device_sm_count(int32_t* sms) {
  int dev = 0, n = 0;
  FR_CUDA_TRY(cudaGetDevice(&dev));
  FR_CUDA_TRY(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  *sms = n;
  return FR_OK;
}

}  // extern "C"
