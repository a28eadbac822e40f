// Built-in image side task: InitSideTask materialises a batch
// of 4K frames and the watermark on the GPU (or in pinned host memory for the
// end-to-end mode), every RunNextStep resizes + watermarks `images_per_step`
// frames with the K5 kernel, StopSideTask releases everything.  Device memory
// is stream-ordered (cudaMallocAsync / cudaFreeAsync) so no transition ever
// synchronises the device -- a cudaFree inside a bubble would stall the
// training stream's host thread.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "capi_util.hpp"
#include "freeride_gpu.h"

namespace {

struct ImageTask {
  fr_image_task_config cfg{};
  fr_img_plan* plan = nullptr;
  uint8_t* src = nullptr;  // device: batch (resident) or one step (host_io)
  uint8_t* dst = nullptr;
  uint8_t* wm = nullptr;
  void* wmp = nullptr;  // prepared watermark (fr_img_prepare_watermark)
  uint8_t* h_src = nullptr;  // pinned host batch (host_io)
  uint8_t* h_dst = nullptr;
  // host_io: a ring of `ring` step slots in device memory, fed like a data
  // loader.  The copy engines run ahead of the steps: slot j's H2D (stream
  // pf) waits only for the slot's previous D2H (stream dh), so while the
  // pipeline computes -- when no step may run -- PCIe keeps filling the ring,
  // and a bubble's steps find their frames resident.  A step is just the
  // K5 kernel behind its slot's `ready` event; its D2H leaves on dh.
  cudaStream_t pf = nullptr, dh = nullptr;
  std::vector<cudaEvent_t> e_ready, e_done, e_free;
  int ring = 0;
  int64_t issued = 0;   // steps whose frames were queued on pf
  bool primed = false;
  uint32_t* ctr = nullptr;   // imperative: preemptible row cursor + rows completed
  uint64_t rows_base = 0;    // rows completed by earlier Init..Stop lifetimes
  int64_t cursor = 0;
  int64_t steps = 0;
  cudaStream_t last = nullptr;
  int32_t max_sms = 0;  // set_sm_budget

  std::size_t src_img() const { return static_cast<std::size_t>(cfg.sw) * cfg.sh * 3; }
  std::size_t dst_img() const { return static_cast<std::size_t>(cfg.dw) * cfg.dh * 3; }
};

int cu(cudaError_t e, const char* what) {
  return e == cudaSuccess ? FR_OK : frcapi::fail(FR_ERR_CUDA_BASE + static_cast<int>(e), std::string(what) + ": " + cudaGetErrorString(e));
}

int release(ImageTask* t, cudaStream_t s) {
  int rc = FR_OK;
  if (t->primed) {  // the copy streams may still run ahead: join them before freeing
    for (cudaStream_t q : {t->pf, t->dh}) {
      cudaEvent_t e = t->e_free.empty() ? nullptr : t->e_free[0];
      if (e && cudaEventRecord(e, q) == cudaSuccess) cudaStreamWaitEvent(s, e, 0);
    }
    t->primed = false;
  }
  if (t->ctr) {  // keep the completed-row count across Stop/Init
    uint64_t done = 0;
    if (cudaMemcpyAsync(&done, t->ctr + 2, sizeof(done), cudaMemcpyDeviceToHost, s) == cudaSuccess &&
        cudaStreamSynchronize(s) == cudaSuccess)
      t->rows_base += done;
  }
  for (void** p : {reinterpret_cast<void**>(&t->src), reinterpret_cast<void**>(&t->dst),
                   reinterpret_cast<void**>(&t->wm), &t->wmp, reinterpret_cast<void**>(&t->ctr)})
    if (*p) {
      if (rc == FR_OK) rc = cu(cudaFreeAsync(*p, s), "cudaFreeAsync");
      *p = nullptr;
    }
  return rc;
}

int img_create(void* u) {
  auto* t = static_cast<ImageTask*>(u);
  if (t->plan) return FR_OK;
  int rc = fr_img_plan_create(t->cfg.sw, t->cfg.sh, t->cfg.dw, t->cfg.dh, &t->plan);
  if (rc == FR_OK) rc = fr_img_plan_set_max_sms(t->plan, t->max_sms);
  // resident frames are produced at Init, never by the kernel before a step
  if (rc == FR_OK && !t->cfg.host_io) rc = fr_img_plan_set_overlap(t->plan, 1);
  return rc;
}

int host_frames(ImageTask* t, cudaStream_t s);

int img_init(void* u, void* stream) {
  auto* t = static_cast<ImageTask*>(u);
  auto s = static_cast<cudaStream_t>(stream);
  t->last = s;
  const fr_image_task_config& c = t->cfg;
  const std::size_t resident = c.host_io ? static_cast<std::size_t>(t->ring) * c.images_per_step
                                         : static_cast<std::size_t>(c.batch);
  int rc = cu(cudaMallocAsync(reinterpret_cast<void**>(&t->src), resident * t->src_img(), s), "src");
  if (rc == FR_OK) rc = cu(cudaMallocAsync(reinterpret_cast<void**>(&t->dst), resident * t->dst_img(), s), "dst");
  if (rc == FR_OK && c.host_io) {
    if (!t->pf) {
      rc = cu(cudaStreamCreateWithFlags(&t->pf, cudaStreamNonBlocking), "prefetch stream");
      if (rc == FR_OK) rc = cu(cudaStreamCreateWithFlags(&t->dh, cudaStreamNonBlocking), "D2H stream");
      for (auto* v : {&t->e_ready, &t->e_done, &t->e_free}) {
        v->assign(t->ring, nullptr);
        for (cudaEvent_t& e : *v)
          if (rc == FR_OK) rc = cu(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "ring events");
      }
    }
    t->issued = 0;
    t->primed = false;
  }
  if (rc == FR_OK) rc = cu(cudaMallocAsync(reinterpret_cast<void**>(&t->wm), static_cast<std::size_t>(c.dw) * c.dh * 4, s), "wm");
  int64_t pbytes = 0;
  if (rc == FR_OK) rc = fr_img_prepared_bytes(t->plan, &pbytes);
  if (rc == FR_OK) rc = cu(cudaMallocAsync(&t->wmp, static_cast<std::size_t>(pbytes), s), "prepared wm");
  if (rc == FR_OK) rc = fr_img_generate_watermark(t->wm, c.dw, c.dh, c.seed ^ 0x77ull, s);
  if (rc == FR_OK) rc = fr_img_prepare_watermark(t->plan, t->wm, t->wmp, s);
  if (rc == FR_OK && c.interface_kind == FR_IMPERATIVE) {
    rc = cu(cudaMallocAsync(reinterpret_cast<void**>(&t->ctr), 8 * sizeof(uint32_t), s), "counters");
    if (rc == FR_OK) rc = cu(cudaMemsetAsync(t->ctr, 0, 8 * sizeof(uint32_t), s), "counters");
  }
  if (rc != FR_OK) return rc;
  if (!c.host_io) return fr_img_generate(t->src, c.batch, c.sw, c.sh, 3, c.seed, 0, s);
  rc = host_frames(t, s);
  // every slot starts free once Init's work on s is done (the first Init
  // uses the device ring as scratch to generate the host frames)
  for (int j = 0; rc == FR_OK && j < t->ring; ++j) rc = cu(cudaEventRecord(t->e_free[j], s), "ring events");
  return rc;
}

int host_frames(ImageTask* t, cudaStream_t s) {
  const fr_image_task_config& c = t->cfg;
  int rc = FR_OK;
  if (!t->h_src) {  // host frames: generated once, kept across Stop/Init cycles
    rc = cu(cudaMallocHost(reinterpret_cast<void**>(&t->h_src), static_cast<std::size_t>(c.batch) * t->src_img()), "pinned src");
    if (rc == FR_OK) rc = cu(cudaMallocHost(reinterpret_cast<void**>(&t->h_dst), static_cast<std::size_t>(c.batch) * t->dst_img()), "pinned dst");
    for (int i = 0; rc == FR_OK && i < c.batch; i += c.images_per_step) {
      const int n = std::min(c.images_per_step, c.batch - i);
      rc = fr_img_generate(t->src, n, c.sw, c.sh, 3, c.seed, i, s);
      if (rc == FR_OK) rc = cu(cudaMemcpyAsync(t->h_src + i * t->src_img(), t->src, n * t->src_img(), cudaMemcpyDeviceToHost, s), "D2H frames");
    }
  }
  return rc;
}

int img_step(void* u, void* stream) {
  auto* t = static_cast<ImageTask*>(u);
  auto s = static_cast<cudaStream_t>(stream);
  t->last = s;
  const fr_image_task_config& c = t->cfg;
  const int64_t i0 = t->cursor;
  const int n = c.images_per_step;
  int rc;
  if (c.host_io) {
    const std::size_t fb = static_cast<std::size_t>(n) * t->src_img(), ob = static_cast<std::size_t>(n) * t->dst_img();
    // queue H2D for the steps up to `ring` ahead of this one (each waits for
    // its slot's previous D2H; the first call after Init fills the ring)
    auto prefetch = [&](int64_t k) {  // step k = frames (i0 + (k - steps) n) % batch
      const int j = static_cast<int>(k % t->ring);
      const int64_t f = (i0 + (k - t->steps) * n) % c.batch;
      int r = cu(cudaStreamWaitEvent(t->pf, t->e_free[j], 0), "ring wait");
      if (r == FR_OK) r = cu(cudaMemcpyAsync(t->src + j * fb, t->h_src + f * t->src_img(), fb, cudaMemcpyHostToDevice, t->pf), "H2D ring");
      if (r == FR_OK) r = cu(cudaEventRecord(t->e_ready[j], t->pf), "ring ready");
      return r;
    };
    rc = FR_OK;
    if (!t->primed) {
      t->issued = t->steps;
      t->primed = true;
    }
    // copy-ahead depth: the whole ring, or under an SM budget 2 slots per
    // SM-equivalent -- PCIe DMA into HBM while the pipeline computes costs
    // the GEMMs clock like the SMs' work does (ring 8 / 24 /
    // 128 -> +0.0 / +0.9 / +1.1 % pipeline ΔT), so the ΔT controller's budget
    // rations the copies too
    const int64_t depth = t->max_sms > 0 ? std::clamp<int64_t>(2 * t->max_sms, 2, t->ring) : t->ring;
    while (rc == FR_OK && t->issued < t->steps + depth) rc = prefetch(t->issued++);
    const int j = static_cast<int>(t->steps % t->ring);
    if (rc == FR_OK) rc = cu(cudaStreamWaitEvent(s, t->e_ready[j], 0), "frames ready");
    if (rc == FR_OK) rc = fr_img_resize_watermark_prepared(t->plan, t->src + j * fb, t->dst + j * ob, t->wmp, n, s);
    if (rc == FR_OK) rc = cu(cudaEventRecord(t->e_done[j], s), "step done");
    if (rc == FR_OK) rc = cu(cudaStreamWaitEvent(t->dh, t->e_done[j], 0), "D2H wait");
    if (rc == FR_OK) rc = cu(cudaMemcpyAsync(t->h_dst + i0 * t->dst_img(), t->dst + j * ob, ob, cudaMemcpyDeviceToHost, t->dh), "D2H step");
    if (rc == FR_OK) rc = cu(cudaEventRecord(t->e_free[j], t->dh), "slot free");
  } else {
    rc = fr_img_resize_watermark_prepared(t->plan, t->src + i0 * t->src_img(), t->dst + i0 * t->dst_img(), t->wmp, n, s);
  }
  if (rc != FR_OK) return rc;
  t->cursor = (i0 + n) % c.batch;
  t->steps++;
  return FR_OK;
}

// Imperative: one preemptible launch of up to kWorkloadPasses passes over
// the batch; it resumes at the first row the previous launch did not take
// and stops taking rows when the stage's bubble-end word reaches the token.
constexpr int64_t kWorkloadPasses = 4;

int img_workload(void* u, void* stream, const fr_preempt* pre) {
  auto* t = static_cast<ImageTask*>(u);
  t->last = static_cast<cudaStream_t>(stream);
  const int64_t rows = static_cast<int64_t>(t->cfg.batch) * t->cfg.dh;
  return fr_img_resize_watermark_preemptible(t->plan, t->src, t->dst, t->wmp, t->cfg.batch, t->ctr,
                                             std::min<int64_t>(kWorkloadPasses * rows, (int64_t{1} << 31) - 1),
                                             pre, stream);
}

int img_work_done(void* u, void* stream, double* units) {
  auto* t = static_cast<ImageTask*>(u);
  uint64_t done = 0;
  if (t->ctr) {
    auto s = static_cast<cudaStream_t>(stream);
    int rc = cu(cudaMemcpyAsync(&done, t->ctr + 2, sizeof(done), cudaMemcpyDeviceToHost, s), "rows done");
    if (rc == FR_OK) rc = cu(cudaStreamSynchronize(s), "rows done");
    if (rc != FR_OK) return rc;
  }
  *units = static_cast<double>(t->rows_base + done) * t->cfg.dw;  // output pixels
  return FR_OK;
}

int img_stop(void* u) {
  auto* t = static_cast<ImageTask*>(u);
  return release(t, t->last);
}

int img_sm_budget(void* u, int32_t sms) {
  auto* t = static_cast<ImageTask*>(u);
  t->max_sms = sms;
  return t->plan ? fr_img_plan_set_max_sms(t->plan, sms) : FR_OK;
}

int img_finished(void* u, int64_t done, int32_t* out) {
  auto* t = static_cast<ImageTask*>(u);
  *out = t->cfg.total_steps > 0 && done >= t->cfg.total_steps;
  return FR_OK;
}

void img_destroy(void* u) {
  auto* t = static_cast<ImageTask*>(u);
  if (t->last) cudaStreamSynchronize(t->last);
  release(t, t->last);
  if (t->last) cudaStreamSynchronize(t->last);
  if (t->h_src) cudaFreeHost(t->h_src);
  if (t->h_dst) cudaFreeHost(t->h_dst);
  for (auto* v : {&t->e_ready, &t->e_done, &t->e_free})
    for (cudaEvent_t e : *v)
      if (e) cudaEventDestroy(e);
  for (cudaStream_t q : {t->pf, t->dh})
    if (q) cudaStreamDestroy(q);
  fr_img_plan_destroy(t->plan);
  delete t;
}

}  // namespace

extern "C" {

int fr_image_task_memory(const fr_image_task_config* c, double* gib) {
  if (!c || !gib) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  const double resident = c->host_io ? double(std::max(2, c->host_ring)) * c->images_per_step : c->batch;
  const double bytes = resident * (double(c->sw) * c->sh * 3 + double(c->dw) * c->dh * 3) +
                       double(c->dw) * c->dh * 12;
  *gib = bytes / (1024.0 * 1024.0 * 1024.0);
  return FR_OK;
}

int fr_image_task_create(const fr_image_task_config* c, fr_side_task_vtable* vt, void** user) {
  if (!c || !vt || !user) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (c->batch < 1 || c->images_per_step < 1 || c->batch % c->images_per_step != 0)
    return frcapi::fail(FR_ERR_VALIDATION, "batch must be a positive multiple of images_per_step", "images_per_step");
  if (c->interface_kind != FR_ITERATIVE && c->interface_kind != FR_IMPERATIVE)
    return frcapi::fail(FR_ERR_VALIDATION, "interface_kind must be FR_ITERATIVE or FR_IMPERATIVE", "interface_kind");
  if (c->interface_kind == FR_IMPERATIVE && c->host_io)
    return frcapi::fail(FR_ERR_UNSUPPORTED, "the imperative image task keeps its batch resident (host_io = 0)");
  if (c->host_ring < 0) return frcapi::fail(FR_ERR_VALIDATION, "host_ring must be >= 0", "host_ring");
  auto* t = new (std::nothrow) ImageTask;
  if (!t) return frcapi::fail(FR_ERR_INVARIANT, "out of host memory");
  t->cfg = *c;
  t->ring = std::max(2, c->host_ring);
  std::memset(vt, 0, sizeof(*vt));
  vt->carveout_hint = 100;
  vt->create = img_create;
  vt->init = img_init;
  vt->run_next_step = img_step;
  vt->stop = img_stop;
  vt->finished = img_finished;
  vt->destroy = img_destroy;
  vt->set_sm_budget = img_sm_budget;
  vt->work_units_per_step = double(c->images_per_step) * c->dw * c->dh;  // output pixels
  if (c->interface_kind == FR_IMPERATIVE) {
    vt->interface_kind = FR_IMPERATIVE;
    vt->run_gpu_workload = img_workload;
    vt->work_done = img_work_done;
  }
  *user = t;
  return FR_OK;
}

int fr_image_task_buffers(void* user, const uint8_t** src, uint8_t** dst, const uint8_t** wm, int64_t* steps) {
  auto* t = static_cast<ImageTask*>(user);
  if (!t) return frcapi::fail(FR_ERR_ARGUMENT, "null task");
  if (src) *src = t->src;
  if (dst) *dst = t->dst;
  if (wm) *wm = t->wm;
  if (steps) *steps = t->steps;
  return FR_OK;
}

int fr_image_task_host_output(void* user, const uint8_t** h_dst) {
  auto* t = static_cast<ImageTask*>(user);
  if (!t || !h_dst) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (t->dh) {  // readout point: the ring's D2H landed
    const int rc = cu(cudaStreamSynchronize(t->dh), "D2H ring");
    if (rc != FR_OK) return rc;
  }
  *h_dst = t->h_dst;
  return FR_OK;
}

}  // extern "C"
