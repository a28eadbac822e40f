/*
 * freeride_gpu.h -- C-ABI of the sm_100a side-task steps and the GPU
 * bubble-harvesting runtime (product library only).
 *
 * The reference has no GPU code: its side tasks are synthetic step durations
 * (proj/include/bubblesim/task.hpp:36-38) and the paper's workloads come from
 * unvendored sources.  What these entry points replace is the
 * *body* of RunNextStep() -- the per-step GPU work the reference's iterative
 * interface (task.hpp:87, iterative_run) only models as `actual_step_ticks`.
 * Each call is one bounded-duration step, asynchronous on the caller's
 * (low-priority) stream.  Device buffers are caller-owned unless a *_create
 * function says otherwise.  Status codes as in freeride.h.
 */
#ifndef FREERIDE_GPU_H_
#define FREERIDE_GPU_H_

#include "freeride.h"

#ifdef __cplusplus
extern "C" {
#endif

/* --------------------------------------------------------------- device */
/* cudaStream_t created with the lowest (numerically greatest) priority, the
 * class side-task steps run in so pipeline kernels always win the SMs. */
int fr_stream_create(int32_t priority_class /* 0 = lowest, 1 = highest */, void** stream);
int fr_stream_destroy(void* stream);
int fr_stream_synchronize(void* stream);
int fr_device_sm_count(int32_t* sms);

/* ------------------------------------------- K5: image resize + watermark */
/* Plan for one (src WxH -> dst WxH) shape.  Coefficients follow cv2's
 * INTER_LINEAR_EXACT (8-bit fixed point, half-pixel centres); the plan picks
 * the TMA-staged exact-2x kernel when the shape allows (sw == 2 dw,
 * sh == 2 dh, dw % 16 == 0) and the table-driven general kernel otherwise. */
typedef struct fr_img_plan fr_img_plan;
enum fr_img_path { FR_IMG_PATH_GENERAL = 0, FR_IMG_PATH_TMA_2X = 1 };
int fr_img_plan_create(int32_t sw, int32_t sh, int32_t dw, int32_t dh, fr_img_plan** out);
int fr_img_plan_destroy(fr_img_plan* plan);
int fr_img_plan_path(const fr_img_plan* plan, int32_t* path);
/* n images: src [n][sh][sw][3] u8, dst [n][dh][dw][3] u8, wm [dh][dw][4] u8
 * (RGBA, straight alpha): dst = (resize(src)*(255-a) + wm*a + 127) / 255 */
int fr_img_resize_watermark(const fr_img_plan* plan, const uint8_t* src, uint8_t* dst,
                            const uint8_t* wm_rgba, int32_t n, void* stream);
/* synthetic inputs (same counter-based arithmetic as oracle/sidetasks.c) */
int fr_img_generate(uint8_t* dst, int32_t n, int32_t w, int32_t h, int32_t channels,
                    uint64_t seed, int32_t first_index, void* stream);
int fr_img_generate_watermark(uint8_t* wm, int32_t w, int32_t h, uint64_t seed, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FREERIDE_GPU_H_ */
