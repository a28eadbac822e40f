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
/* the library's current device for the calling thread (it links its own
 * CUDA runtime; set it once per thread, e.g. after torch.cuda.set_device) */
int fr_set_device(int32_t device);
int fr_get_device(int32_t* device);
/* synchronous copy between any host/device buffers (unified addressing) */
int fr_memcpy(void* dst, const void* src, int64_t bytes);
/* diagnostics: spin `cycles` SM clocks on one warp, write {cycles, ns} */
int fr_clock_probe(uint64_t* out_cycles_ns, int64_t cycles, void* stream);
/* L2 read bandwidth probe: `passes` coalesced 16 B ld.global.cg sweeps of
 * `buf` (size it to fit in L2); time it with events on `stream`.  sink16:
 * 16 device bytes the kernel may write (keeps the loads alive). */
int fr_l2_read_probe(const void* buf, int64_t bytes, int32_t passes, void* sink16, void* stream);

/* Device-side preemption for the imperative interface: the workload stops
 * taking new work items once *stop_word >= token.  The harness's gap kernel
 * raises stop_word (device memory, gpu-scope) at the instant the next op's
 * dependency arrives, i.e. the bubble end, so the pause reaches the GPU
 * without a host round trip and lands within one work item. */
typedef struct fr_preempt {
  const uint32_t* stop_word; /* device pointer, read with ld.relaxed.gpu */
  uint32_t token;
  uint32_t reserved;
} fr_preempt;

/* ------------------------------------------- K5: image resize + watermark */
/* Plan for one (src WxH -> dst WxH) shape.  Coefficients follow cv2's
 * INTER_LINEAR_EXACT (8-bit fixed point, half-pixel centres); the plan picks
 * the TMA-staged exact-2x kernel when the shape allows (sw == 2 dw,
 * sh == 2 dh, dw % 16 == 0) and the table-driven general kernel otherwise. */
typedef struct fr_img_plan fr_img_plan;
enum fr_img_path { FR_IMG_PATH_GENERAL = 0, FR_IMG_PATH_TMA_2X = 1 };
int fr_img_plan_create(int32_t sw, int32_t sh, int32_t dw, int32_t dh, fr_img_plan** out);
/* Consecutive exact-2x launches on this plan may overlap (programmatic
 * dependent launch: a launch's CTAs start as soon as every CTA of the previous
 * one has taken its last row).  Only a launch that directly follows another
 * exact-2x step of this plan on the same stream is made a dependent; the
 * watermark preparation, a preemptible launch or a call of this function
 * restart the chain.  The caller promises not to enqueue a producer of a
 * step's frames between two such steps (the built-in image task: frames
 * materialised at InitSideTask, which also prepares the watermark). */
int fr_img_plan_set_overlap(fr_img_plan* plan, int32_t overlap);
/* launches of this plan occupy at most `sms` SMs (0 = all): the grid is
 * sized for that many SMs (rows are handed out dynamically, so any grid is
 * correct) */
int fr_img_plan_set_max_sms(fr_img_plan* plan, int32_t sms);
int fr_img_plan_destroy(fr_img_plan* plan);
int fr_img_plan_path(const fr_img_plan* plan, int32_t* path);
/* n images: src [n][sh][sw][3] u8, dst [n][dh][dw][3] u8, wm [dh][dw][4] u8
 * (RGBA, straight alpha): dst = (resize(src)*(255-a) + wm*a + 127) / 255 */
int fr_img_resize_watermark(const fr_img_plan* plan, const uint8_t* src, uint8_t* dst,
                            const uint8_t* wm_rgba, int32_t n, void* stream);
/* The watermark is a task constant: prepare it once (InitSideTask) into the
 * plan's layout and run the prepared variant per step (exact-2x path: per
 * pixel pair the premultiplied w*a+127 of the blend lanes [R0,B0] [G0,R1]
 * [B1,G1] and the two 255-a, group-transposed, 10 B/px; 8 B/px with the
 * round-1 math FR_IMG_MATH=0; general path: RGBA copy, 4 B/px -- always size
 * the buffer with fr_img_prepared_bytes of the plan that runs it).
 * fr_img_resize_watermark prepares into a plan-owned buffer on every call.
 * Exact-2x launches claim rows in units of the same output row in up to 16
 * consecutive frames (the consumers keep that row's watermark in registers);
 * the output is byte-identical for any unit size, grid or SM budget. */
int fr_img_prepared_bytes(const fr_img_plan* plan, int64_t* bytes);
int fr_img_prepare_watermark(const fr_img_plan* plan, const uint8_t* wm_rgba, void* prepared,
                             void* stream);
int fr_img_resize_watermark_prepared(const fr_img_plan* plan, const uint8_t* src, uint8_t* dst,
                                     const void* prepared, int32_t n, void* stream);
/* Preemptible K5 over a resident batch of n frames (fast 2x path only).
 * Work is claimed in units of U = fr_img_preemptible_unit_rows(plan, n) rows
 * (the same output row of U consecutive frames; U depends on n only): a
 * launch takes up to floor(max_rows / U) units, unit (base + t) mod
 * (n * dh / U) for the t-th unit taken, base = counters[0] -- so a launch may
 * loop over the batch and the next launch resumes at the first unit this one
 * did not take.  counters: 8 x uint32 of zeroed device memory owned by the
 * caller (the unit cursor, scheduler state, and counters[2..3] = rows
 * completed, uint64).  Stops taking units once *preempt->stop_word >=
 * preempt->token (preempt may be null); every unit taken is completed
 * before the launch ends. */
int fr_img_resize_watermark_preemptible(const fr_img_plan* plan, const uint8_t* src, uint8_t* dst,
                                        const void* prepared, int32_t n, uint32_t* counters,
                                        int64_t max_rows, const fr_preempt* preempt, void* stream);
int fr_img_preemptible_unit_rows(const fr_img_plan* plan, int32_t n, int32_t* rows);
/* synthetic inputs (same counter-based arithmetic as oracle/sidetasks.c) */
int fr_img_generate(uint8_t* dst, int32_t n, int32_t w, int32_t h, int32_t channels,
                    uint64_t seed, int32_t first_index, void* stream);
int fr_img_generate_watermark(uint8_t* wm, int32_t w, int32_t h, uint64_t seed, void* stream);

/* ------------------------------------------------ K1/K2: PageRank (pull) */
/* Incoming-CSR graph on the device.  fr_pr_graph_rmat generates RMAT edges
 * (a,b,c = .57,.19,.19; counter-based, identical to oracle/sidetasks.c),
 * drops self loops and duplicates and builds the CSR sorted by (dst, src).
 * Synchronous (setup, not a step). */
typedef struct fr_pr_graph fr_pr_graph;
typedef struct fr_pr_state fr_pr_state;
int fr_pr_graph_rmat(int32_t scale, int32_t edge_factor, uint64_t seed, void* stream,
                     fr_pr_graph** out);
/* The caller's graph: E directed edges src[e] -> dst[e] (device int32 arrays,
 * read during the call), ids in [0, V) (else FR_ERR_VALIDATION); self loops
 * and duplicates dropped like the RMAT path.  Synchronous. */
int fr_pr_graph_from_edges(int32_t V, int64_t E, const int32_t* src, const int32_t* dst, void* stream,
                           fr_pr_graph** out);
int fr_pr_graph_destroy(fr_pr_graph* g);
int fr_pr_graph_info(const fr_pr_graph* g, int32_t* V, int64_t* E, int32_t* n_blocks);
/* device pointers: offsets[V+1], col_idx[E], outdeg[V] */
int fr_pr_graph_csr(const fr_pr_graph* g, const int32_t** offsets, const int32_t** col_idx,
                    const int32_t** outdeg);
int fr_pr_state_create(const fr_pr_graph* g, fr_pr_state** out);
int fr_pr_state_destroy(fr_pr_state* st);
/* iterations occupy at most `sms` SMs (0 = all): the persistent grid shrinks
 * and each CTA walks several of the build's split-row chunk lists */
int fr_pr_state_set_max_sms(fr_pr_state* st, int32_t sms);
/* r = 1/V, c = r * inv_outdeg */
int fr_pr_reset(fr_pr_state* st, void* stream);
/* `iters` pull iterations: r' = (1-d)/V + d * A_in^T c ; c' = r' * inv_outdeg */
int fr_pr_step(fr_pr_state* st, int32_t iters, float damping, void* stream);
/* ranks in original vertex ids (device pointer, V floats).  A readout point:
 * synchronises the device, then permutes the step's row-order ranks. */
int fr_pr_ranks(const fr_pr_state* st, const float** r, int64_t* iterations);

/* ------------------------------------------- K3/K4: Graph-SGD (rank k MF) */
/* Rating graph (u, v, r) with power-law endpoints (counter-based, identical
 * to oracle/sidetasks.c) and an fp32 latent matrix L[V][k], k in
 * {4,8,16,32,64,128}.  Hogwild updates: racy by design. */
typedef struct fr_sgd_problem fr_sgd_problem;
int fr_sgd_problem_generate(int32_t V, int64_t E, int32_t k, uint64_t edge_seed,
                            uint64_t init_seed, void* stream, fr_sgd_problem** out);
/* The caller's ratings: E edges (u, v, r) (host or device arrays, copied),
 * endpoints in [0, V) (else FR_ERR_VALIDATION), latent matrix seeded like the
 * generator's.  Synchronous. */
int fr_sgd_problem_from_edges(int32_t V, int64_t E, int32_t k, const int32_t* u, const int32_t* v,
                              const float* r, uint64_t init_seed, void* stream, fr_sgd_problem** out);
int fr_sgd_problem_destroy(fr_sgd_problem* p);
/* L ~ U(0, 1/sqrt(k)), seeded */
int fr_sgd_reinit(fr_sgd_problem* p, uint64_t init_seed, void* stream);
/* one step: edges [e_begin, e_end) */
int fr_sgd_step(fr_sgd_problem* p, int64_t e_begin, int64_t e_end, float eta, float lambda,
                void* stream);
/* Re-lays the edges out by user (Gardenia's CSR input order: ratings of one
 * user contiguous, generated order within a user); when the latent rows pass
 * 64 MiB, stable by item block (P = ceil(V k 4 B / 64 MiB) ranges of v, so a
 * step's L_v rows stay in L2); each (block, user) run cut into 64-edge pieces
 * dealt over R = ceil(E / window_edges) rounds inside its block (piece q of
 * np -> round (q R / np + h(u)) mod R, stable by block x R + round), so one
 * window-sized step holds at most ~one piece of any user per block.  Later steps run the
 * user-grouped kernel (L_u held in registers across a run, ~143 instead of
 * 268 B/edge at k = 16; k < 16 keeps the per-edge kernel).  Synchronous;
 * E < 2^31.  oracle/sidetasks.c orc_sgd_group_by_user is the same layout. */
int fr_sgd_group_by_user(fr_sgd_problem* p, int64_t window_edges, void* stream);
/* Pick the step kernel for the edges as they lie: 1 = user-grouped (L_u held
 * across each run of equal u -- correct for any order, fast when runs are
 * long), 0 = per-edge.  For callers that lay their ratings out themselves. */
int fr_sgd_problem_set_kernel(fr_sgd_problem* p, int32_t by_user);
/* Consecutive user-grouped steps may overlap (programmatic dependent launch:
 * a step's CTAs start while the previous step's last segments drain -- more
 * Hogwild concurrency, nothing else).  Only a step that directly follows
 * another user-grouped step of this problem on the same stream is made a
 * dependent: fr_sgd_reinit, fr_sgd_group_by_user, fr_sgd_sqerr/rmse, a
 * per-edge step or a call of this function restart the chain.  The caller
 * promises not to write the problem's buffers between two such steps.  The
 * built-in task sets it. */
int fr_sgd_problem_set_overlap(fr_sgd_problem* p, int32_t overlap);
/* steps occupy at most `sms` SMs (0 = all): fewer lane groups in flight */
int fr_sgd_problem_set_max_sms(fr_sgd_problem* p, int32_t sms);
/* K4: *d_acc (device fp64) += sum of squared errors over [e_begin, e_end) */
int fr_sgd_sqerr(const fr_sgd_problem* p, int64_t e_begin, int64_t e_end, double* d_acc,
                 void* stream);
/* synchronous RMSE over all edges */
int fr_sgd_rmse(const fr_sgd_problem* p, void* stream, double* rmse);
int fr_sgd_buffers(const fr_sgd_problem* p, const int32_t** u, const int32_t** v, const float** r,
                   float** L, int32_t* V, int64_t* E, int32_t* k);

/* ------------------------------------------------ side-task plugin surface */
/* The paper's overridable transition functions:
 * CreateSideTask / InitSideTask / StartSideTask / RunNextStep /
 * PauseSideTask / StopSideTask plus the loop-finished predicate.  Replaces
 * the reference's synthetic SideTaskSpec body (task.hpp:33-50) and its
 * TaskLookup callback (manager.hpp:52) with real GPU work.  Every hook
 * returns a status; init/run_next_step enqueue asynchronously on `stream`
 * (the worker's low-priority stream) and must not synchronise it. */
typedef struct fr_side_task_vtable {
  int (*create)(void* user);
  int (*init)(void* user, void* stream);
  int (*start)(void* user);
  int (*run_next_step)(void* user, void* stream);
  int (*pause)(void* user);
  int (*stop)(void* user);
  int (*finished)(void* user, int64_t steps_completed, int32_t* done);
  void (*destroy)(void* user);
  double work_units_per_step; /* px, edges, ... reported per completed step */
  /* Imperative interface (PAPER.md:484-499 RunGpuWorkload; task.hpp:93
   * imperative_run): interface_kind = FR_IMPERATIVE makes
   * the worker call run_gpu_workload from StartSideTask until the pause
   * instead of gated RunNextStep calls.  run_gpu_workload enqueues one
   * preemptible launch on `stream` (it returns when the work is done or the
   * preempt word fires, keeping its progress for the next call); work_done
   * reports cumulative completed work units (may synchronise `stream`). */
  int32_t interface_kind;     /* enum fr_interface: FR_ITERATIVE = 0, FR_IMPERATIVE = 1 */
  /* L1/shared split the task's kernels want on the SMs during its bubbles
   * (cudaFuncAttributePreferredSharedMemoryCarveout percent; -1 = no
   * preference).  The stage's resident dependency-wait kernel pins its SM's
   * split for the whole bubble, so the harness launches it with the split the
   * tasks want: max-L1 (0) only when every task asks for it (random-access
   * kernels whose loads in flight live in L1), else max-shared. */
  int32_t carveout_hint;
  int (*run_gpu_workload)(void* user, void* stream, const fr_preempt* preempt);
  int (*work_done)(void* user, void* stream, double* units);
  /* Framework-enforced kill (limits.hpp:34 framework_enforce, check_memory
   * :20): optional.  Called from the worker thread when the task is killed;
   * must make its in-flight GPU work end promptly (e.g. raise a word its
   * kernels poll) without synchronising.  The worker then drains the task's
   * stream, calls stop and releases the task's memory pool. */
  int (*cancel)(void* user);
  /* SM budget (optional): from now on the task's kernels occupy at most `sms`
   * SMs (0 = all).  On a power-capped B200 every joule a side task spends in
   * a bubble is taken from the boost the pipeline's GEMMs get from their idle
   * bubbles; the same bytes moved by fewer SMs cost far less power, so the
   * harness bounds the side task's SMs to hold the pipeline's ΔT (DESIGN.md
   * §5c).  The harness calls it before profiling and on every change. */
  int (*set_sm_budget)(void* user, int32_t sms);
} fr_side_task_vtable;

/* Built-in side tasks (kernels above) behind the vtable. */
typedef struct fr_image_task_config {
  int32_t sw, sh, dw, dh;       /* 3840x2160 -> 1920x1080 */
  int32_t batch;                /* images resident (device) or staged (host mode) */
  int32_t images_per_step;      /* one RunNextStep = this many images */
  int32_t host_io;              /* 1: inputs in pinned host memory, H2D/D2H per step */
  int32_t interface_kind;       /* FR_ITERATIVE: steps of images_per_step frames;
                                   FR_IMPERATIVE: one preemptible workload over the
                                   whole batch, paused on the device per output row */
  uint64_t seed;
  int64_t total_steps;          /* <= 0: unbounded */
  int32_t host_ring;            /* host_io: device staging slots, in steps (>= 2; 0 -> 2).
                                   The H2D of later steps' frames runs ahead on the copy
                                   engines -- also while the pipeline computes -- and each
                                   step's D2H leaves on its own stream */
} fr_image_task_config;
int fr_image_task_create(const fr_image_task_config* cfg, fr_side_task_vtable* vt, void** user);
/* bytes resident on the GPU once InitSideTask ran (memory_demand) */
int fr_image_task_memory(const fr_image_task_config* cfg, double* gib);
/* device pointers of the last processed batch slot (for checking) */
int fr_image_task_buffers(void* user, const uint8_t** src, uint8_t** dst, const uint8_t** wm,
                          int64_t* steps_done);
/* host_io = 1: the pinned host output batch [batch][dh][dw][3] (null before
 * the first InitSideTask); rows of frames not yet processed are undefined */
int fr_image_task_host_output(void* user, const uint8_t** h_dst);

/* Synthetic side task: the reference's SideTaskSpec (task.hpp:33-50) made
 * real -- each RunNextStep is a spin kernel occupying every SM for step_ns,
 * InitSideTask allocates memory_demand_gib, and the Fig. 9 misbehaviours
 * (task.hpp:26-31) are reproducible: MemoryLeak allocates leak_gib_per_step
 * more each step; a task whose steps run far longer than profiled
 * (step_ns >> profile_step_ns) overruns its bubbles like IgnoresPause.
 * cooperative = 1: the step kernel polls the task's cancel word, so a kill
 * ends it within ~1 us. */
typedef struct fr_synthetic_task_config {
  int64_t step_ns;
  int64_t profile_step_ns;      /* step length while being profiled (<= 0: step_ns) */
  double memory_demand_gib;
  double leak_gib_per_step;
  int64_t total_steps;          /* <= 0: unbounded */
  int32_t cooperative;
  int32_t reserved;
  int64_t init_ns;              /* InitSideTask: a GPU spin this long (0: none) -- an init
                                   that outlasts its bubble trips the init guard */
} fr_synthetic_task_config;
int fr_synthetic_task_create(const fr_synthetic_task_config* cfg, fr_side_task_vtable* vt,
                             void** user);

typedef struct fr_pagerank_task_config {
  int32_t scale;          /* RMAT scale: V = 2^scale */
  int32_t edge_factor;    /* edges generated = edge_factor * V (before dedup) */
  uint64_t seed;
  int32_t iters_per_step; /* pull iterations per RunNextStep */
  float damping;          /* 0.85 */
  int64_t total_steps;    /* <= 0: unbounded */
} fr_pagerank_task_config;
/* builds the graph immediately (work_units_per_step = E * iters_per_step) */
int fr_pagerank_task_create(const fr_pagerank_task_config* cfg, fr_side_task_vtable* vt,
                            void** user);
/* the same task over the caller's graph (fr_pr_graph_rmat / fr_pr_graph_from_edges):
 * the step arrays are copied at create, the caller keeps and frees `graph`;
 * cfg's scale / edge_factor / seed are ignored */
int fr_pagerank_task_create_from_graph(const fr_pagerank_task_config* cfg, const fr_pr_graph* graph,
                                       fr_side_task_vtable* vt, void** user);
int fr_pagerank_task_info(void* user, int32_t* V, int64_t* E, double* memory_gib,
                          const float** ranks, int64_t* iterations);

typedef struct fr_sgd_task_config {
  int32_t V;              /* 3,072,441 (Orkut shape) */
  int32_t k;              /* rank, 16 */
  int64_t E;              /* 117,185,083 */
  uint64_t edge_seed;
  uint64_t init_seed;
  int64_t edges_per_step; /* edges per RunNextStep (wraps into the next epoch) */
  float eta;              /* 0.01 */
  float lambda;           /* 0.05 */
  int64_t total_steps;    /* <= 0: unbounded */
  int32_t layout;         /* FR_SGD_LAYOUT_COO (generated order) or FR_SGD_LAYOUT_BY_USER */
  int32_t total_epochs;   /* > 0: stop after exactly this many passes over the edges (the
                             step that ends the last epoch is cut there); <= 0: unbounded */
} fr_sgd_task_config;
#define FR_SGD_LAYOUT_COO 0
#define FR_SGD_LAYOUT_BY_USER 1
/* generates the rating graph on the device immediately (setup) */
int fr_sgd_task_create(const fr_sgd_task_config* cfg, fr_side_task_vtable* vt, void** user);
/* the same task over the caller's ratings (fr_sgd_problem_from_edges): the task
 * takes `problem` over on success (freed with the task); V / E / k come from it,
 * cfg->layout BY_USER re-lays it out by user */
int fr_sgd_task_create_from_problem(const fr_sgd_task_config* cfg, fr_sgd_problem* problem,
                                    fr_side_task_vtable* vt, void** user);
int fr_sgd_task_problem(void* user, fr_sgd_problem** p, int64_t* epochs_done);

/* ------------------------------------------------------ the GPU runtime */
/* One GPU replaying stage `stage` of a p-stage 1F1B pipeline whose FP/BP
 * ops are real bf16 tensor-core GEMMs (the stand-in), with one side-task
 * worker: manager Alg. 1/2, the iterative interface and the program-directed
 * gate (the reference's missing run_experiment, engine.hpp:97) executed in
 * real time against device-clock bubble signals. */
typedef struct fr_harness fr_harness;

typedef struct fr_harness_config {
  int32_t num_stages;
  int32_t num_micro_batches;
  int32_t stage;              /* the stage this GPU replays (replica mode) */
  int32_t layers;             /* stand-in shape (per stage) */
  int32_t hidden;
  int32_t tokens;             /* micro-batch x sequence length */
  int32_t ffn_mult;
  int32_t profile_reps;       /* op timing repetitions (median) */
  int32_t max_inflight_steps; /* pipelined dispatch depth, >= 1 */
  int32_t gate_estimate;      /* 0 = profiled mean, 1 = max (config.hpp:17) */
  double gpu_memory_total;    /* GiB, memory model for Alg. 1 */
  double weight_mem;          /* GiB per stage; < 0 derive from the stand-in */
  double activation_mem;      /* GiB per in-flight micro-batch; < 0 derive */
  int64_t fp_ticks_override;  /* > 0: use instead of the measured op times */
  int64_t bp_ticks_override;
  int32_t profile_epochs;     /* dry-run epochs of the bubble profiler (0: from op times) */
  int32_t transport;          /* 0: replica (device-clock dependency waits, one GPU);
                                 1: peer-linked pipeline (stage s on its own GPU, real
                                 activation/gradient messages through neighbour mailboxes) */
  /* limits (limits.hpp:9-15): every task allocates from its own CUDA memory
   * pool; limit = profiled est_memory + headroom, checked (check_memory,
   * strict) after InitSideTask and every RunNextStep -> OOM kill; a pause not
   * observed within grace_ns -> pause-timeout kill (framework_enforce). */
  double memory_headroom_gib;
  int64_t grace_ns;           /* <= 0: 100 ms (LimitConfig::grace_period = 100 ticks of 1 ms) */
  int32_t step_group;         /* <= 1: timing events around every step; G > 1: up to G
                                 consecutive iterative steps between one pair of events
                                 (each still admitted by the gate), so they run back to
                                 back; timelines and reprofile then see step groups */
  double harvest_fraction;    /* (0, 1): the gate admits steps only in the first
                                 fraction of every bubble (the bubble end it is given is
                                 start + fraction x profiled duration); <= 0 or >= 1:
                                 the whole bubble */
  int64_t reclamation_delay_ns; /* LimitConfig::reclamation_delay (limits.hpp:12): a killed
                                   task's pool pages go back to the device this long after
                                   the kill (<= 0: at once) */
  int32_t side_sms;           /* SM budget of the side tasks' kernels (set_sm_budget;
                                 0 = all SMs); the starting point when dt_budget > 0 */
  int32_t min_side_sms;       /* floor of the ΔT controller (<= 0: 2) */
  double dt_budget;           /* > 0: ΔT-budgeted harvesting.  The worker times every op
                                 of the stage as it completes, compares it with the same
                                 op in the last run without side tasks, and sizes the side
                                 tasks' SM budget so the stage's ops run at most this
                                 fraction slower (e.g. 0.007); <= 0: fixed side_sms */
} fr_harness_config;

/* All durations in ns ticks (tick_seconds = 1e-9). */
typedef struct fr_harness_profile {
  fr_tick fp_ticks;
  fr_tick bp_ticks;
  fr_tick epoch_span;
  fr_tick stage_bubble_ticks;   /* sum of this stage's bubbles per epoch */
  double bubble_rate;           /* whole p-stage schedule (bubble_rate) */
  double available_memory;      /* GiB on this stage (PipelineConfig) */
  double fp_tflops;             /* stand-in tensor throughput, measured */
  double bp_tflops;
  int32_t n_bubbles;            /* this stage, per epoch */
  int32_t reserved;
  double clock_offset_err_ns;   /* host<->device clock calibration RTT/2 */
} fr_harness_profile;

typedef struct fr_run_report {
  int32_t epochs;
  int32_t with_tasks;
  double makespan_s;            /* device time, run start -> last epoch end */
  double bubble_s;              /* sum of actual bubbles on this run */
  double used_s;                /* step time inside bubbles */
  double overrun_s;             /* step time outside bubbles */
  double work_units;            /* completed steps x work_units_per_step */
  int64_t steps_launched;
  int64_t steps_completed;
  double dispatch_host_us;      /* mean host time per gate+launch */
  double max_step_overrun_s;    /* worst step tail past its bubble end */
  fr_stage_breakdown breakdown; /* bubble_breakdown (metrics.hpp:64), ns ticks */
  int64_t pauses;
  int64_t kills;                /* tasks killed in this run (both reasons) */
  int64_t kills_oom;            /* check_memory OomKill (limits.hpp:20) */
  int64_t kills_pause_timeout;  /* framework_enforce Kill (limits.hpp:34) */
  int64_t kills_init_timeout;   /* ArmInitGuard fired with InitSideTask still running
                                   (manager.hpp:58, KillReason::InitTimeout) */
  double op_growth;             /* mean (op duration / same op in the last run without
                                   side tasks) - 1 over this run's ops (0 if no reference) */
  double side_sms_mean;         /* side-task SM budget averaged over the run's ops */
  int32_t side_sms_final;       /* the budget at the run's end (ΔT controller state) */
  int32_t reserved2;
  /* transport 1: the stage-to-stage exchange (activation / gradient messages
   * this stage sent, copy engine into the neighbour's mailbox) */
  int64_t exchange_messages;
  double exchange_us;           /* mean device time per message copy */
  double exchange_gbps;         /* message bytes / copy time */
} fr_run_report;

int fr_harness_create(const fr_harness_config* cfg, fr_harness** out);
int fr_harness_destroy(fr_harness* h);
int fr_harness_get_profile(const fr_harness* h, fr_harness_profile* out);
/* this stage's bubbles of one epoch (profile, undelayed, relative ticks) */
int fr_harness_stage_bubbles(const fr_harness* h, fr_bubble* out, int32_t cap, int32_t* n);
/* Submits a side task: profile_task by running `profile_steps` steps
 * standalone (measured, CUDA events), then Alg. 1 over this GPU's worker.
 * Ownership of `user` passes to the harness (vtable destroy). */
int fr_harness_submit(fr_harness* h, const char* task_id, const fr_side_task_vtable* vt,
                      void* user, double memory_demand_gib, int32_t profile_steps,
                      fr_task_profile* profile, int32_t* assigned);
/* bubble profiler (profile_bubbles, profiler.hpp:45) from the last run's
 * measured bubbles: each of this stage's bubble durations := its median */
int fr_harness_reprofile_bubbles(fr_harness* h);
/* StopSideTask (task.hpp:21) between runs: releases the task's GPU state and
 * clears the worker's CurrentTask / queue entry (SURVEY.md Appendix B rule 8) */
int fr_harness_stop_task(fr_harness* h, const char* task_id);
/* profile_task from the task's steps in the last run (measured in bubbles,
 * under training load): est = mean, max = worst, as in profiler.cpp:50-78 */
int fr_harness_reprofile(fr_harness* h, const char* task_id, fr_task_profile* out);
/* harvest fraction for the next runs (fr_harness_config::harvest_fraction) */
int fr_harness_set_harvest_fraction(fr_harness* h, double fraction);
/* side-task SM budget for the next runs (fr_harness_config::side_sms); the
 * tasks' step estimates change with it: re-profile (fr_harness_reprofile)
 * after a run at the new budget */
int fr_harness_set_side_sms(fr_harness* h, int32_t sms);
/* ΔT budget of the next runs (fr_harness_config::dt_budget; 0 = off); the
 * controller restarts from side_sms */
int fr_harness_set_dt_budget(fr_harness* h, double budget);
/* Runs `epochs` epochs; with_tasks=0 is the ΔT baseline. Blocks. */
int fr_harness_run(fr_harness* h, int32_t epochs, int32_t with_tasks, fr_run_report* out);
/* a submitted task's state (enum fr_task_state), disposition (enum
 * fr_disposition; FR_DISP_ACTIVE while alive) and bytes in its memory pool */
int fr_harness_task_status(const fr_harness* h, const char* task_id, int32_t* state,
                           int32_t* disposition, double* memory_used_gib);
/* bytes the task's pool holds: in use, and reserved (kept mapped until the
 * task is stopped / killed and its reclamation delay has passed) */
int fr_harness_task_memory(const fr_harness* h, const char* task_id, double* used_gib,
                           double* reserved_gib);
/* The last run with tasks as the reference's parity object (RunTrace,
 * engine.hpp:75-92), recorded on the GPU: this stage's ops (CUDA events),
 * its bubbles, submits / assigns, every transition the worker applied, Init
 * and Step activities, kills and dispositions, in ns from the run's start
 * (ticks of 1e-9 s).  `measured` is set: fr_run_trace_check then skips the
 * simulated-only invariants (configured op durations, absent stages, op /
 * side-kernel exclusivity) and allows `tolerance` ns between the host-clock
 * transition stamps and the device-event activity times.  Caller destroys
 * it with fr_run_trace_destroy. */
int fr_harness_run_trace(const fr_harness* h, fr_run_trace** out);
/* Every program-directed gate decision of the last run (iterative_run,
 * task.cpp:89-100), in order: the inputs the worker gave it and its answer,
 * so the decisions can be replayed through the reference's function. */
typedef struct fr_gate_record {
  fr_tick now;          /* projected device start of the step, ns from run start */
  fr_tick bubble_end;   /* bubble end handed over at StartSideTask, ns from run start */
  double est_seconds;   /* the profiled estimate (GateEstimate) */
  fr_tick step_ticks;   /* actual_step_ticks argument (= the estimate in ticks) */
  int32_t run;          /* 1: admitted (RunNextStep dispatched) */
  int32_t signal;       /* index into the signal log of the BubbleStarted that started it */
  fr_tick step_end;     /* IterativeDecision::step_end */
  char task[FR_TASK_ID_MAX];
} fr_gate_record;
/* Every Alg. 2 call of the last run (on_bubble_started / on_bubble_ended,
 * manager.cpp:37-70), in call order, with the view of the task it looked up
 * and the actions it returned. */
typedef struct fr_signal_record {
  fr_tick t;            /* signal time (device clock), ns from run start */
  int32_t kind;         /* 0 BubbleStarted, 1 BubbleEnded */
  int32_t epoch;
  int32_t bubble;       /* index into fr_harness_stage_bubbles */
  int32_t looked_up;    /* 1: the manager consulted `task` (view below) */
  fr_tick duration;     /* profiled bubble duration carried by BubbleStarted */
  int32_t view_state;   /* enum fr_task_state of `task` at the call */
  int32_t view_initializing;
  int32_t n_actions;
  int32_t actions[4];   /* ManagerActionKind codes, in order */
  int32_t deferred;     /* 1: a BubbleStarted held until the previous pause landed */
  char task[FR_TASK_ID_MAX];
} fr_signal_record;
int fr_harness_gate_log(const fr_harness* h, fr_gate_record* out, int64_t cap, int64_t* n);
int fr_harness_signal_log(const fr_harness* h, fr_signal_record* out, int64_t cap, int64_t* n);
/* raw timelines of the last run, seconds from run start, (start, end) pairs */
int fr_harness_timeline(const fr_harness* h, int32_t which /*0 ops,1 bubbles,2 steps*/,
                        double* start_end, int64_t cap, int64_t* n);
/* Peer-linked pipeline (transport = 1), one harness per stage (normally one
 * per GPU/process).  Each stage owns a mailbox (device memory: flags + one
 * message slot per micro-batch and direction); a neighbour copies the op's
 * output (tokens x hidden bf16) into it with the copy engine over NVLink /
 * peer memory and raises the slot's flag; the stage's dependency wait spins
 * on its own flag (replaces NCCL send/recv).  Link the
 * neighbours' mailboxes (pointers valid in this process: same process, or
 * opened with fr_ipc_open) before running; both stages must run the same
 * epoch counts.  The bubble profiler does not dry-run at creation in this
 * mode: run without tasks, then fr_harness_reprofile_bubbles. */
int fr_harness_mailbox(const fr_harness* h, void** base, int64_t* bytes);
int fr_harness_link(fr_harness* h, void* prev_mailbox /* null on stage 0 */,
                    void* next_mailbox /* null on the last stage */);
/* CUDA IPC for mailboxes across processes (64-byte cudaIpcMemHandle_t) */
int fr_ipc_handle(void* dev_ptr, void* handle_out);
int fr_ipc_open(const void* handle, void** dev_ptr);
int fr_ipc_close(void* dev_ptr);
/* this GPU's kernel launch count in the last run (side-task steps + stand-in) */
int fr_harness_launches(const fr_harness* h, int64_t* side_steps, int64_t* training_ops);

#ifdef __cplusplus
}
#endif

#endif /* FREERIDE_GPU_H_ */
