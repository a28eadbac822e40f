/* ORACLE / TEST INFRASTRUCTURE ONLY -- CPU restatement of the side-task
 * arithmetic the north star dispatches into bubbles.  The reference ships no
 * side-task code (tasks are synthetic durations, task.hpp:36-38); the paper's
 * workloads come from unvendored third-party sources:
 *   - Gardenia PageRank / SGD (cite key xu_gardenia_2019, no version pinned)
 *   - NVIDIA image resize + watermark sample (nvidia_developers_image_2019)
 * so this file restates their published algorithms and is pinned instead
 * against independent libraries in this container (cv2 INTER_LINEAR_EXACT,
 * scipy.sparse power iteration, numpy SGD) via committed golden fixtures.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. */
#ifndef FR_ORACLE_SIDETASKS_H_
#define FR_ORACLE_SIDETASKS_H_
#include <stdint.h>

/* ---- shared deterministic generators (identical arithmetic on the GPU) -- */
uint64_t orc_splitmix64(uint64_t x);
/* synthetic RGB/RGBA images: gradient + splitmix64 noise */
void orc_img_generate(uint8_t* dst, int n, int w, int h, int channels, uint64_t seed,
                      int first_index, int nthreads);
void orc_img_generate_watermark(uint8_t* wm, int w, int h, uint64_t seed, int nthreads);

/* ---- K5: bilinear resize (cv2 INTER_LINEAR_EXACT, 8-bit fixed point) +
 *          integer alpha blend with an RGBA watermark at output size ------ */
void orc_img_coeffs(int src_n, int dst_n, int32_t* idx0, int32_t* idx1, int32_t* w1);
void orc_img_resize_watermark(const uint8_t* src, uint8_t* dst, const uint8_t* wm, int n,
                              int sw, int sh, int dw, int dh, int nthreads);

/* ---- K1/K2: PageRank pull over the incoming CSR ------------------------ */
/* RMAT edge list (Graph500 a,b,c; no noise), scale s, m edges, seed */
void orc_rmat_edges(int scale, int64_t m, uint64_t seed, int32_t* src, int32_t* dst,
                    int nthreads);
/* r' = (1-d)/V + d * sum_{u in in(v)} r[u]*inv_outdeg[u]; dangling mass
 * dropped.  Accumulates in double; `r` holds the start ranks and is
 * overwritten with the ranks after `iters` iterations. */
void orc_pr_run(int32_t V, const int32_t* offsets, const int32_t* col_idx,
                const int32_t* outdeg, double damping, int iters, double* r, int nthreads);

/* ---- K3/K4: Graph-SGD matrix factorisation (rank k) -------------------- */
void orc_sgd_edges(int32_t V, int64_t E, uint64_t seed, int32_t* u, int32_t* v, float* r,
                   int nthreads);
int32_t orc_sgd_item_blocks(int32_t V, int k);
void orc_sgd_group_by_user(int32_t V, int64_t E, int64_t window, int k, int32_t* u, int32_t* v, float* r);
void orc_sgd_init(int32_t V, int k, uint64_t seed, float* L, int nthreads);
/* one epoch over edges [0,E) in order; sequential when nthreads == 1,
 * Hogwild (racy by design) otherwise */
void orc_sgd_epoch(int64_t E, const int32_t* u, const int32_t* v, const float* r, float* L,
                   int k, float eta, float lambda, int nthreads);
double orc_sgd_rmse(int64_t E, const int32_t* u, const int32_t* v, const float* r,
                    const float* L, int k, int nthreads);

#endif
