// Synthetic side task (reference SideTaskSpec,
// task.hpp:33-50): steps of a known GPU duration, a known memory demand and
// the two Fig. 9 misbehaviours (task.hpp:26-31), as real GPU work, so the
// framework-enforced limits can be exercised on the device.
//
// A step is a spin kernel with one CTA per SM that holds the SMs for step_ns
// (device %globaltimer).  In cooperative mode it also polls a host-mapped
// cancel word, so a kill ends it within a poll interval.  Memory comes from
// cudaMallocAsync -- i.e. from whatever pool the worker made current for
// this task -- and every allocation (including the "leaked" ones) is freed
// by StopSideTask.
#include <cuda_runtime.h>

#include <cstring>
#include <new>
#include <vector>

#include "capi_util.hpp"
#include "freeride_gpu.h"
#include "kernels/common.cuh"

namespace {

__global__ void spin_kernel(int64_t ns, const volatile uint32_t* cancel) {
  __shared__ uint64_t t0;
  if (threadIdx.x == 0) t0 = frk::globaltimer_ns();
  __syncthreads();
  if (threadIdx.x != 0) return;
  while (frk::globaltimer_ns() - t0 < static_cast<uint64_t>(ns)) {
    if (cancel && *cancel) return;
    __nanosleep(500);
  }
}

struct SynthTask {
  fr_synthetic_task_config cfg{};
  bool profiled = false;  // first Stop ends the profiling instance
  void* demand = nullptr;
  std::vector<void*> leaked;
  uint32_t* cancel = nullptr;      // host-mapped
  uint32_t* cancel_dev = nullptr;
  cudaStream_t last = nullptr;
  int sms = 148;
};

int cu(cudaError_t e, const char* what) {
  return e == cudaSuccess ? FR_OK
                          : frcapi::fail(FR_ERR_CUDA_BASE + static_cast<int>(e),
                                         std::string(what) + ": " + cudaGetErrorString(e));
}

size_t gib_bytes(double gib) { return static_cast<size_t>(gib * 1024.0 * 1024.0 * 1024.0); }

int syn_init(void* u, void* stream) {
  auto* t = static_cast<SynthTask*>(u);
  auto s = static_cast<cudaStream_t>(stream);
  t->last = s;
  *t->cancel = 0;
  if (t->cfg.memory_demand_gib > 0) {
    const int rc = cu(cudaMallocAsync(&t->demand, gib_bytes(t->cfg.memory_demand_gib), s), "demand");
    if (rc != FR_OK) return rc;
  }
  if (t->cfg.init_ns > 0) {
    spin_kernel<<<1, 32, 0, s>>>(t->cfg.init_ns, t->cfg.cooperative ? t->cancel_dev : nullptr);
    return cu(cudaGetLastError(), "init spin");
  }
  return FR_OK;
}

int syn_step(void* u, void* stream) {
  auto* t = static_cast<SynthTask*>(u);
  auto s = static_cast<cudaStream_t>(stream);
  t->last = s;
  if (t->cfg.leak_gib_per_step > 0) {  // MemoryLeak: never freed by the step
    void* p = nullptr;
    const int rc = cu(cudaMallocAsync(&p, gib_bytes(t->cfg.leak_gib_per_step), s), "leak");
    if (rc != FR_OK) return rc;
    t->leaked.push_back(p);
  }
  const int64_t ns = (!t->profiled && t->cfg.profile_step_ns > 0) ? t->cfg.profile_step_ns : t->cfg.step_ns;
  spin_kernel<<<t->sms, 32, 0, s>>>(ns, t->cfg.cooperative ? t->cancel_dev : nullptr);
  return cu(cudaGetLastError(), "spin");
}

int syn_stop(void* u) {
  auto* t = static_cast<SynthTask*>(u);
  int rc = FR_OK;
  if (t->demand) rc = cu(cudaFreeAsync(t->demand, t->last), "free demand");
  t->demand = nullptr;
  for (void* p : t->leaked)
    if (rc == FR_OK) rc = cu(cudaFreeAsync(p, t->last), "free leak");
  t->leaked.clear();
  t->profiled = true;
  return rc;
}

int syn_cancel(void* u) {
  auto* t = static_cast<SynthTask*>(u);
  *reinterpret_cast<volatile uint32_t*>(t->cancel) = 1;  // seen by the polling kernel
  return FR_OK;
}

int syn_finished(void* u, int64_t done, int32_t* out) {
  auto* t = static_cast<SynthTask*>(u);
  *out = t->cfg.total_steps > 0 && done >= t->cfg.total_steps;
  return FR_OK;
}

void syn_destroy(void* u) {
  auto* t = static_cast<SynthTask*>(u);
  if (t->last) cudaStreamSynchronize(t->last);
  syn_stop(t);
  if (t->last) cudaStreamSynchronize(t->last);
  if (t->cancel) cudaFreeHost(t->cancel);
  delete t;
}

}  // namespace

extern "C" int fr_synthetic_task_create(const fr_synthetic_task_config* c, fr_side_task_vtable* vt,
                                        void** user) {
  if (!c || !vt || !user) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (c->step_ns < 1) return frcapi::fail(FR_ERR_VALIDATION, "step_ns must be >= 1", "step_ns");
  if (c->init_ns < 0) return frcapi::fail(FR_ERR_VALIDATION, "init_ns must be >= 0", "init_ns");
  if (c->memory_demand_gib < 0 || c->leak_gib_per_step < 0)
    return frcapi::fail(FR_ERR_VALIDATION, "memory sizes must be >= 0", "memory_demand");
  auto* t = new (std::nothrow) SynthTask;
  if (!t) return frcapi::fail(FR_ERR_INVARIANT, "out of host memory");
  t->cfg = *c;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&t->sms, cudaDevAttrMultiProcessorCount, dev);
  int rc = cu(cudaHostAlloc(reinterpret_cast<void**>(&t->cancel), 64, cudaHostAllocMapped), "cancel word");
  if (rc == FR_OK) {
    *t->cancel = 0;
    rc = cu(cudaHostGetDevicePointer(reinterpret_cast<void**>(&t->cancel_dev), t->cancel, 0), "cancel word");
  }
  if (rc != FR_OK) {
    if (t->cancel) cudaFreeHost(t->cancel);
    delete t;
    return rc;
  }
  std::memset(vt, 0, sizeof(*vt));
  vt->carveout_hint = -1;
  vt->init = syn_init;
  vt->run_next_step = syn_step;
  vt->stop = syn_stop;
  vt->finished = syn_finished;
  vt->destroy = syn_destroy;
  vt->cancel = syn_cancel;
  vt->work_units_per_step = 1.0;  // steps
  *user = t;
  return FR_OK;
}
