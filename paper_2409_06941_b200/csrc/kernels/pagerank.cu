// K1/K2: PageRank pull step over the incoming CSR (Gardenia
// PR), one bounded step = `iters` power iterations.
//
//   r'[v] = (1-d)/V + d * sum_{u in in(v)} c[u],   c'[v] = r'[v] * inv_outdeg[v]
//   dangling vertices (out-degree 0) have inv_outdeg = 0: their mass is dropped.
//
// Graph build (once, on the GPU): RMAT edges with the oracle's counter-based
// generator, self-loops dropped, (dst,src) keys radix-sorted and de-duplicated
// (CUB), offsets by histogram + scan, out-degrees by atomics.
//
// Step kernel, binned CSR-vector: at graph build the rows are bucketed by
// in-degree into lane-group sizes g in {1..32} (~4 edges per lane); a warp
// serves 32/g rows of one bucket with no shared memory and no barriers, each
// lane keeping 4 independent L2 gathers in flight and accumulating in fp64,
// then an xor-shuffle reduction inside the g-lane group and a fused r'/c'
// epilogue.  Rows with more than kHubEdges in-edges (RMAT hubs, up to ~40k)
// get a whole CTA and are scheduled first.  (An earlier smem-staged
// "CSR-stream" variant lost ~2x to barrier and shared-atomic stalls on RMAT's
// skewed rows -- see DESIGN.md.)  At RMAT scale 20 the working set (~85 MB)
// is L2-resident on B200 (126 MB): the step is bound by L2 gather bandwidth
// (one 32 B sector per 4 B rank), not by HBM.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "freeride_gpu.h"
#include "kernels/common.cuh"

namespace {

constexpr int kPrThreads = 256;
constexpr uint32_t kRmatA = 2448131358u, kRmatAB = 3264175144u, kRmatABC = 4080218931u;
constexpr uint64_t kRmatPermMul = 0x9E3779B97F4A7C15ull;

__global__ void rmat_kernel(int scale, int64_t m, uint64_t seed, int32_t* __restrict__ src,
                            int32_t* __restrict__ dst) {
  const uint64_t mask = (1ull << scale) - 1;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < m;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t st = seed ^ (static_cast<uint64_t>(e) * 0xD1B54A32D192ED03ull);
    uint64_t u = 0, v = 0;
    for (int l = 0; l < scale; ++l) {
      st = frk::splitmix64(st);
      const uint32_t q = static_cast<uint32_t>(st >> 32);
      const uint64_t bit = 1ull << (scale - 1 - l);
      if (q >= kRmatA) {
        if (q < kRmatAB) {
          v |= bit;
        } else if (q < kRmatABC) {
          u |= bit;
        } else {
          u |= bit;
          v |= bit;
        }
      }
    }
    src[e] = static_cast<int32_t>((u * kRmatPermMul) & mask);
    dst[e] = static_cast<int32_t>((v * kRmatPermMul) & mask);
  }
}

// key = dst << 32 | src, self loops mapped to the all-ones sentinel (sorted last)
__global__ void edge_keys_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                 int64_t m, uint64_t* __restrict__ keys) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < m;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s = static_cast<uint32_t>(src[e]), d = static_cast<uint32_t>(dst[e]);
    keys[e] = s == d ? ~0ull : (static_cast<uint64_t>(d) << 32) | s;
  }
}

__global__ void split_keys_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                  int32_t* __restrict__ col, int32_t* __restrict__ indeg,
                                  int32_t* __restrict__ outdeg) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    const int32_t s = static_cast<int32_t>(k & 0xFFFFFFFFu), d = static_cast<int32_t>(k >> 32);
    col[i] = s;
    atomicAdd(&indeg[d], 1);
    atomicAdd(&outdeg[s], 1);
  }
}

__global__ void inv_deg_kernel(const int32_t* __restrict__ outdeg, int32_t V,
                               float* __restrict__ inv) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
    inv[v] = outdeg[v] > 0 ? 1.0f / static_cast<float>(outdeg[v]) : 0.0f;
}

__global__ void pr_reset_kernel(const float* __restrict__ inv, int32_t V, float* __restrict__ r,
                                float* __restrict__ c) {
  const float r0 = static_cast<float>(1.0 / static_cast<double>(V));
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    r[v] = r0;
    c[v] = r0 * inv[v];
  }
}

struct PrArgs {
  const int32_t* offsets;
  const int32_t* col;
  const float* inv;
  const int32_t* blk;  // work list: hub (row,-1) / item (start, g | count<<8) pairs
  const int32_t* rows; // binned row list (pr_binned_kernel)
  int32_t n_hub;
  const float* c_in;
  float* r_out;
  float* c_out;
  int32_t n_blk;
  double base;
  double damp;
};

__device__ __forceinline__ double block_sum(double x, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = x;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < kPrThreads / 32) t = red[threadIdx.x];
  if (w == 0) {
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

constexpr int kHubEdges = 2048;

// Binned CSR-vector pull: no shared memory, no barriers on the common path.
// Block b < n_hub: one hub row for the whole CTA.  Otherwise each warp takes
// one work item: 32/g rows of one degree bucket, g lanes per row striding the
// row's in-edges (coalesced col_idx within the group, 4 independent L2
// gathers in flight per lane), fp64 partials, xor-shuffle reduction inside
// the g-lane group, fused r'/c' epilogue by the group's first lane.
__global__ void __launch_bounds__(kPrThreads) pr_binned_kernel(PrArgs a) {
  __shared__ double red[kPrThreads / 32];
  const int tid = threadIdx.x;
  if (static_cast<int32_t>(blockIdx.x) < a.n_hub) {
    const int32_t r0 = a.blk[2 * blockIdx.x];
    const int32_t e0 = a.offsets[r0], e1 = a.offsets[r0 + 1];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int32_t i = e0 + tid;
    for (; i + 3 * kPrThreads < e1; i += 4 * kPrThreads) {
      const int32_t u0 = __ldg(&a.col[i]), u1 = __ldg(&a.col[i + kPrThreads]);
      const int32_t u2 = __ldg(&a.col[i + 2 * kPrThreads]), u3 = __ldg(&a.col[i + 3 * kPrThreads]);
      s0 += __ldg(&a.c_in[u0]);
      s1 += __ldg(&a.c_in[u1]);
      s2 += __ldg(&a.c_in[u2]);
      s3 += __ldg(&a.c_in[u3]);
    }
    for (; i < e1; i += kPrThreads) s0 += __ldg(&a.c_in[__ldg(&a.col[i])]);
    const double s = block_sum((s0 + s1) + (s2 + s3), red);
    if (tid == 0) {
      const float rv = static_cast<float>(a.base + a.damp * s);
      a.r_out[r0] = rv;
      a.c_out[r0] = rv * a.inv[r0];
    }
    return;
  }
  const int32_t item = a.n_hub + (static_cast<int32_t>(blockIdx.x) - a.n_hub) * (kPrThreads / 32) + (tid >> 5);
  if (item >= a.n_blk) return;
  const int32_t start = a.blk[2 * item], code = a.blk[2 * item + 1];
  const int lanes = code & 0xFF, count = code >> 8;
  const int lane = tid & 31, grp = lane / lanes, sub = lane % lanes;
  int32_t row = -1, e = 0, e1 = 0;
  if (grp < count) {
    row = a.rows[start + grp];
    e = a.offsets[row] + sub;
    e1 = a.offsets[row + 1];
  }
  // Predicated 4-wide chunks: all four col_idx loads, then all four gathers,
  // are in flight together even for rows shorter than 4 x lanes (the common
  // case), i.e. two dependent L2 round trips per chunk, not two per edge.
  double s0 = 0.0, s1 = 0.0;
  for (; e < e1; e += 4 * lanes) {
    int32_t u[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) u[j] = e + j * lanes < e1 ? __ldg(&a.col[e + j * lanes]) : -1;
    float c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j] = u[j] >= 0 ? __ldg(&a.c_in[u[j]]) : 0.0f;
    s0 += static_cast<double>(c[0]) + static_cast<double>(c[1]);
    s1 += static_cast<double>(c[2]) + static_cast<double>(c[3]);
  }
  double s = s0 + s1;
  for (int o = lanes >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (sub == 0 && row >= 0) {
    const float rv = static_cast<float>(a.base + a.damp * s);
    a.r_out[row] = rv;
    a.c_out[row] = rv * a.inv[row];
  }
}

int grid_for(int64_t work, int threads, int per_sm) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (work + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(sms) * per_sm)));
}

}  // namespace

struct fr_pr_graph {
  int32_t V = 0;
  int64_t E = 0;
  int32_t* offsets = nullptr;  // V + 1
  int32_t* col = nullptr;      // E
  int32_t* outdeg = nullptr;   // V
  float* inv = nullptr;        // V
  int32_t* blk = nullptr;      // work list: n_blk (a, b) pairs, then the binned row list
  int32_t n_blk = 0;           // hubs + warp items
  int32_t n_hub = 0;           // leading hub rows (one CTA each)
  int64_t blk_len = 0;         // int32 entries in blk
  int sms = 148;
};

struct fr_pr_state {
  const fr_pr_graph* g = nullptr;
  float* r = nullptr;
  float* c[2] = {nullptr, nullptr};
  int cur = 0;
  int64_t iterations = 0;
};

namespace {

void free_graph(fr_pr_graph* g) {
  for (void* p : {static_cast<void*>(g->offsets), static_cast<void*>(g->col),
                  static_cast<void*>(g->outdeg), static_cast<void*>(g->inv),
                  static_cast<void*>(g->blk)})
    if (p) cudaFree(p);
  delete g;
}

// Binned work list for pr_binned_kernel.  Rows with more than kHubEdges
// in-edges are hubs (one CTA each, listed first so they start in the first
// wave).  Every other row gets g lanes, g = the smallest power of two >=
// ceil(deg / 4) (so each lane gathers ~4 edges), 1 <= g <= 32; rows are
// bucketed by g and each warp item serves 32/g rows of one bucket.  Items are
// ordered by descending g (heavier work first).
// blk layout: n_blk pairs (a, b) then the bucketed row list:
//   hub  : (row, -1)
//   item : (start in row list, g | count << 8)
int build_bins(fr_pr_graph* g, cudaStream_t s) {
  std::vector<int32_t> off(static_cast<size_t>(g->V) + 1);
  FR_CUDA_TRY(cudaMemcpyAsync(off.data(), g->offsets, off.size() * sizeof(int32_t),
                              cudaMemcpyDeviceToHost, s));
  FR_CUDA_TRY(cudaStreamSynchronize(s));
  std::vector<int32_t> hubs, bucket[6];  // bucket k: g = 1 << k
  for (int32_t r = 0; r < g->V; ++r) {
    const int32_t d = off[r + 1] - off[r];
    if (d > kHubEdges) {
      hubs.push_back(r);
      continue;
    }
    int k = 0;
    while (k < 5 && (4 << k) < d) ++k;
    bucket[k].push_back(r);
  }
  std::sort(hubs.begin(), hubs.end(), [&](int32_t x, int32_t y) {
    return off[x + 1] - off[x] > off[y + 1] - off[y];
  });
  std::vector<int32_t> pairs, rows;
  for (int32_t h : hubs) {
    pairs.push_back(h);
    pairs.push_back(-1);
  }
  for (int k = 5; k >= 0; --k) {
    const int32_t lanes = 1 << k, per = 32 / lanes;
    for (size_t i = 0; i < bucket[k].size(); i += per) {
      const int32_t cnt = static_cast<int32_t>(std::min<size_t>(per, bucket[k].size() - i));
      pairs.push_back(static_cast<int32_t>(rows.size() + i));
      pairs.push_back(lanes | (cnt << 8));
    }
    rows.insert(rows.end(), bucket[k].begin(), bucket[k].end());
  }
  // item starts index the row list, which follows the pairs
  const int32_t n = static_cast<int32_t>(pairs.size() / 2);
  std::vector<int32_t> blk(pairs);
  blk.insert(blk.end(), rows.begin(), rows.end());
  g->n_blk = n;
  g->n_hub = static_cast<int32_t>(hubs.size());
  g->blk_len = static_cast<int64_t>(blk.size());
  FR_CUDA_TRY(cudaMalloc(&g->blk, blk.size() * sizeof(int32_t)));
  FR_CUDA_TRY(cudaMemcpyAsync(g->blk, blk.data(), blk.size() * sizeof(int32_t),
                              cudaMemcpyHostToDevice, s));
  FR_CUDA_TRY(cudaStreamSynchronize(s));
  return FR_OK;
}

int finish_graph(fr_pr_graph* g, cudaStream_t s) {
  FR_CUDA_TRY(cudaMalloc(&g->inv, sizeof(float) * static_cast<size_t>(g->V)));
  inv_deg_kernel<<<grid_for(g->V, 256, 8), 256, 0, s>>>(g->outdeg, g->V, g->inv);
  FR_CUDA_LAUNCHED("inv_deg");
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g->sms, cudaDevAttrMultiProcessorCount, dev);
  return build_bins(g, s);
}

}  // namespace

extern "C" {

int fr_pr_graph_rmat(int32_t scale, int32_t edge_factor, uint64_t seed, void* stream,
                     fr_pr_graph** out) {
  if (!out) return frcapi::fail(FR_ERR_ARGUMENT, "null graph out");
  if (scale < 1 || scale > 30 || edge_factor < 1)
    return frcapi::fail(FR_ERR_VALIDATION, "scale in [1,30], edge_factor >= 1", "scale");
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t m = static_cast<int64_t>(edge_factor) << scale;
  auto* g = new fr_pr_graph;
  g->V = 1 << scale;
  int32_t *src = nullptr, *dst = nullptr, *indeg = nullptr, *d_sel = nullptr;
  uint64_t *keys = nullptr, *sorted = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0, need = 0;
  int rc = FR_OK;
  auto step = [&](cudaError_t e, const char* what) {
    if (rc == FR_OK && e != cudaSuccess) rc = frcapi::cuda_status(e, what);
    return rc == FR_OK;
  };
  step(cudaMalloc(&src, m * sizeof(int32_t)), "rmat src");
  step(cudaMalloc(&dst, m * sizeof(int32_t)), "rmat dst");
  step(cudaMalloc(&keys, m * sizeof(uint64_t)), "keys");
  step(cudaMalloc(&sorted, m * sizeof(uint64_t)), "sorted");
  step(cudaMalloc(&d_sel, sizeof(int32_t)), "count");
  if (rc == FR_OK) {
    rmat_kernel<<<grid_for(m, 256, 16), 256, 0, s>>>(scale, m, seed, src, dst);
    edge_keys_kernel<<<grid_for(m, 256, 16), 256, 0, s>>>(src, dst, m, keys);
    step(cudaGetLastError(), "rmat / keys");
  }
  if (rc == FR_OK) {
    cub::DeviceRadixSort::SortKeys(nullptr, need, keys, sorted, static_cast<int>(m), 0, 64, s);
    tmp_bytes = need;
    cub::DeviceSelect::Unique(nullptr, need, sorted, keys, d_sel, static_cast<int>(m), s);
    tmp_bytes = std::max(tmp_bytes, need);
    step(cudaMalloc(&tmp, tmp_bytes), "cub temp");
  }
  int32_t n_unique = 0;
  if (rc == FR_OK) {
    step(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, sorted, static_cast<int>(m), 0, 64, s), "sort");
    step(cub::DeviceSelect::Unique(tmp, tmp_bytes, sorted, keys, d_sel, static_cast<int>(m), s), "unique");
    step(cudaMemcpyAsync(&n_unique, d_sel, sizeof(int32_t), cudaMemcpyDeviceToHost, s), "count");
    step(cudaStreamSynchronize(s), "sync");
  }
  if (rc == FR_OK) {
    // the self-loop sentinel sorts last and survives Unique once
    uint64_t last = 0;
    if (n_unique > 0)
      step(cudaMemcpy(&last, keys + n_unique - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost), "last key");
    g->E = (n_unique > 0 && last == ~0ull) ? n_unique - 1 : n_unique;
    step(cudaMalloc(&g->col, std::max<int64_t>(1, g->E) * sizeof(int32_t)), "col");
    step(cudaMalloc(&g->offsets, (static_cast<size_t>(g->V) + 1) * sizeof(int32_t)), "offsets");
    step(cudaMalloc(&g->outdeg, static_cast<size_t>(g->V) * sizeof(int32_t)), "outdeg");
    step(cudaMalloc(&indeg, static_cast<size_t>(g->V) * sizeof(int32_t)), "indeg");
  }
  if (rc == FR_OK) {
    step(cudaMemsetAsync(indeg, 0, static_cast<size_t>(g->V) * sizeof(int32_t), s), "memset");
    step(cudaMemsetAsync(g->outdeg, 0, static_cast<size_t>(g->V) * sizeof(int32_t), s), "memset");
    step(cudaMemsetAsync(g->offsets, 0, sizeof(int32_t), s), "memset");
    if (g->E > 0) split_keys_kernel<<<grid_for(g->E, 256, 16), 256, 0, s>>>(keys, g->E, g->col, indeg, g->outdeg);
    step(cudaGetLastError(), "split keys");
    size_t sb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, sb, indeg, g->offsets + 1, g->V, s);
    if (sb > tmp_bytes) {
      cudaFree(tmp);
      tmp = nullptr;
      step(cudaMalloc(&tmp, sb), "scan temp");
      tmp_bytes = sb;
    }
    step(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, indeg, g->offsets + 1, g->V, s), "scan");
  }
  for (void* p : {static_cast<void*>(src), static_cast<void*>(dst), static_cast<void*>(keys),
                  static_cast<void*>(sorted), static_cast<void*>(indeg), static_cast<void*>(d_sel), tmp})
    if (p) cudaFreeAsync(p, s);
  if (rc == FR_OK) rc = finish_graph(g, s);
  if (rc != FR_OK) {
    free_graph(g);
    return rc;
  }
  *out = g;
  return FR_OK;
}

int fr_pr_graph_destroy(fr_pr_graph* g) {
  if (g) free_graph(g);
  return FR_OK;
}

int fr_pr_graph_info(const fr_pr_graph* g, int32_t* V, int64_t* E, int32_t* n_blocks) {
  if (!g) return frcapi::fail(FR_ERR_ARGUMENT, "null graph");
  if (V) *V = g->V;
  if (E) *E = g->E;
  if (n_blocks) *n_blocks = g->n_blk;
  return FR_OK;
}

int fr_pr_graph_csr(const fr_pr_graph* g, const int32_t** offsets, const int32_t** col_idx,
                    const int32_t** outdeg) {
  if (!g) return frcapi::fail(FR_ERR_ARGUMENT, "null graph");
  if (offsets) *offsets = g->offsets;
  if (col_idx) *col_idx = g->col;
  if (outdeg) *outdeg = g->outdeg;
  return FR_OK;
}

int fr_pr_state_create(const fr_pr_graph* g, fr_pr_state** out) {
  if (!g || !out) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  auto* st = new fr_pr_state;
  st->g = g;
  const size_t b = sizeof(float) * static_cast<size_t>(std::max(1, g->V));
  cudaError_t e = cudaMalloc(&st->r, b);
  if (e == cudaSuccess) e = cudaMalloc(&st->c[0], b);
  if (e == cudaSuccess) e = cudaMalloc(&st->c[1], b);
  if (e != cudaSuccess) {
    for (float* p : {st->r, st->c[0], st->c[1]})
      if (p) cudaFree(p);
    delete st;
    return frcapi::cuda_status(e, "pagerank state");
  }
  *out = st;
  return FR_OK;
}

int fr_pr_state_destroy(fr_pr_state* st) {
  if (!st) return FR_OK;
  for (float* p : {st->r, st->c[0], st->c[1]})
    if (p) cudaFree(p);
  delete st;
  return FR_OK;
}

int fr_pr_reset(fr_pr_state* st, void* stream) {
  if (!st) return frcapi::fail(FR_ERR_ARGUMENT, "null state");
  st->cur = 0;
  st->iterations = 0;
  pr_reset_kernel<<<grid_for(st->g->V, 256, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      st->g->inv, st->g->V, st->r, st->c[0]);
  FR_CUDA_LAUNCHED("pr_reset");
  return FR_OK;
}

int fr_pr_step(fr_pr_state* st, int32_t iters, float damping, void* stream) {
  if (!st) return frcapi::fail(FR_ERR_ARGUMENT, "null state");
  if (iters < 0) return frcapi::fail(FR_ERR_VALIDATION, "iters must be >= 0", "iters");
  const fr_pr_graph* g = st->g;
  auto s = static_cast<cudaStream_t>(stream);
  PrArgs a{};
  a.offsets = g->offsets;
  a.col = g->col;
  a.inv = g->inv;
  a.blk = g->blk;
  a.n_blk = g->n_blk;
  a.n_hub = g->n_hub;
  a.rows = g->blk + 2 * static_cast<int64_t>(g->n_blk);
  a.r_out = st->r;
  a.damp = static_cast<double>(damping);
  a.base = (1.0 - static_cast<double>(damping)) / static_cast<double>(g->V);
  const int warps = kPrThreads / 32;
  const int grid = g->n_hub + (g->n_blk - g->n_hub + warps - 1) / warps;
  if (grid == 0) return FR_OK;
  for (int i = 0; i < iters; ++i) {
    a.c_in = st->c[st->cur];
    a.c_out = st->c[st->cur ^ 1];
    pr_binned_kernel<<<grid, kPrThreads, 0, s>>>(a);
    st->cur ^= 1;
    st->iterations++;
  }
  FR_CUDA_LAUNCHED("pr_pull");
  return FR_OK;
}

int fr_pr_ranks(const fr_pr_state* st, const float** r, int64_t* iterations) {
  if (!st) return frcapi::fail(FR_ERR_ARGUMENT, "null state");
  if (r) *r = st->r;
  if (iterations) *iterations = st->iterations;
  return FR_OK;
}

}  // extern "C"

// ------------------------------------------------------ built-in side task
// CreateSideTask builds the graph once and parks it in pinned host memory
// (the paper's CREATED state: context in main memory, not on the GPU);
// InitSideTask uploads it with stream-ordered allocations + async copies
// (nothing that synchronises the device inside a bubble); every
// RunNextStep runs `iters_per_step` pull iterations; StopSideTask frees the
// GPU copy.  Ranks restart from 1/V whenever the task is (re)initialised.
namespace {

struct PrTask {
  fr_pagerank_task_config cfg{};
  int32_t V = 0, n_blk = 0, n_hub = 0;
  int64_t blk_len = 0;
  int64_t E = 0;
  int32_t *h_off = nullptr, *h_col = nullptr, *h_outdeg = nullptr, *h_blk = nullptr;
  float* h_inv = nullptr;
  fr_pr_graph g;  // device view (owned through the task, freed with cudaFreeAsync)
  fr_pr_state st;
  bool on_gpu = false;
  cudaStream_t last = nullptr;
};

int pr_task_create(void* u) {
  auto* t = static_cast<PrTask*>(u);
  if (t->h_off) return FR_OK;
  cudaStream_t s = nullptr;
  FR_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  fr_pr_graph* g = nullptr;
  int rc = fr_pr_graph_rmat(t->cfg.scale, t->cfg.edge_factor, t->cfg.seed, s, &g);
  if (rc == FR_OK) {
    t->V = g->V;
    t->E = g->E;
    t->n_blk = g->n_blk;
    auto pin = [&](void** p, size_t bytes, const void* dev) {
      if (rc != FR_OK) return;
      cudaError_t e = cudaMallocHost(p, std::max<size_t>(bytes, 4));
      if (e == cudaSuccess && bytes) e = cudaMemcpy(*p, dev, bytes, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) rc = frcapi::cuda_status(e, "pagerank host copy");
    };
    pin(reinterpret_cast<void**>(&t->h_off), (size_t(t->V) + 1) * 4, g->offsets);
    pin(reinterpret_cast<void**>(&t->h_col), size_t(t->E) * 4, g->col);
    pin(reinterpret_cast<void**>(&t->h_outdeg), size_t(t->V) * 4, g->outdeg);
    pin(reinterpret_cast<void**>(&t->h_inv), size_t(t->V) * 4, g->inv);
    t->n_hub = g->n_hub;
    t->blk_len = g->blk_len;
    pin(reinterpret_cast<void**>(&t->h_blk), size_t(t->blk_len) * 4, g->blk);
    fr_pr_graph_destroy(g);
  }
  cudaStreamDestroy(s);
  return rc;
}

int pr_task_init(void* u, void* stream) {
  auto* t = static_cast<PrTask*>(u);
  auto s = static_cast<cudaStream_t>(stream);
  t->last = s;
  fr_pr_graph& g = t->g;
  g.V = t->V;
  g.E = t->E;
  g.n_blk = t->n_blk;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g.sms, cudaDevAttrMultiProcessorCount, dev);
  auto up = [&](void** d, const void* h, size_t bytes) -> cudaError_t {
    cudaError_t e = cudaMallocAsync(d, std::max<size_t>(bytes, 4), s);
    if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(*d, h, bytes, cudaMemcpyHostToDevice, s);
    return e;
  };
  FR_CUDA_TRY(up(reinterpret_cast<void**>(&g.offsets), t->h_off, (size_t(t->V) + 1) * 4));
  FR_CUDA_TRY(up(reinterpret_cast<void**>(&g.col), t->h_col, size_t(t->E) * 4));
  FR_CUDA_TRY(up(reinterpret_cast<void**>(&g.outdeg), t->h_outdeg, size_t(t->V) * 4));
  FR_CUDA_TRY(up(reinterpret_cast<void**>(&g.inv), t->h_inv, size_t(t->V) * 4));
  g.n_hub = t->n_hub;
  g.blk_len = t->blk_len;
  FR_CUDA_TRY(up(reinterpret_cast<void**>(&g.blk), t->h_blk, size_t(t->blk_len) * 4));
  t->st.g = &g;
  for (float** p : {&t->st.r, &t->st.c[0], &t->st.c[1]})
    FR_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(p), size_t(t->V) * 4, s));
  t->on_gpu = true;
  return fr_pr_reset(&t->st, s);
}

int pr_task_step(void* u, void* stream) {
  auto* t = static_cast<PrTask*>(u);
  t->last = static_cast<cudaStream_t>(stream);
  return fr_pr_step(&t->st, t->cfg.iters_per_step, t->cfg.damping, stream);
}

int pr_task_stop(void* u) {
  auto* t = static_cast<PrTask*>(u);
  if (!t->on_gpu) return FR_OK;
  for (void* p : {static_cast<void*>(t->g.offsets), static_cast<void*>(t->g.col),
                  static_cast<void*>(t->g.outdeg), static_cast<void*>(t->g.inv),
                  static_cast<void*>(t->g.blk), static_cast<void*>(t->st.r),
                  static_cast<void*>(t->st.c[0]), static_cast<void*>(t->st.c[1])})
    if (p) FR_CUDA_TRY(cudaFreeAsync(p, t->last));
  t->g = fr_pr_graph{};
  t->st = fr_pr_state{};
  t->on_gpu = false;
  return FR_OK;
}

int pr_task_finished(void* u, int64_t done, int32_t* out) {
  auto* t = static_cast<PrTask*>(u);
  *out = t->cfg.total_steps > 0 && done >= t->cfg.total_steps;
  return FR_OK;
}

void pr_task_destroy(void* u) {
  auto* t = static_cast<PrTask*>(u);
  if (t->last) cudaStreamSynchronize(t->last);
  pr_task_stop(t);
  if (t->last) cudaStreamSynchronize(t->last);
  for (void* p : {static_cast<void*>(t->h_off), static_cast<void*>(t->h_col),
                  static_cast<void*>(t->h_outdeg), static_cast<void*>(t->h_inv),
                  static_cast<void*>(t->h_blk)})
    if (p) cudaFreeHost(p);
  delete t;
}

}  // namespace

extern "C" {

int fr_pagerank_task_create(const fr_pagerank_task_config* c, fr_side_task_vtable* vt, void** user) {
  if (!c || !vt || !user) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (c->iters_per_step < 1) return frcapi::fail(FR_ERR_VALIDATION, "iters_per_step must be >= 1", "iters_per_step");
  auto* t = new PrTask;
  t->cfg = *c;
  const int rc = pr_task_create(t);  // build now: work units per step need E
  if (rc != FR_OK) {
    pr_task_destroy(t);
    return rc;
  }
  std::memset(vt, 0, sizeof(*vt));
  vt->create = pr_task_create;
  vt->init = pr_task_init;
  vt->run_next_step = pr_task_step;
  vt->stop = pr_task_stop;
  vt->finished = pr_task_finished;
  vt->destroy = pr_task_destroy;
  vt->work_units_per_step = static_cast<double>(t->E) * c->iters_per_step;  // edges
  *user = t;
  return FR_OK;
}

int fr_pagerank_task_info(void* user, int32_t* V, int64_t* E, double* memory_gib,
                          const float** ranks, int64_t* iterations) {
  auto* t = static_cast<PrTask*>(user);
  if (!t) return frcapi::fail(FR_ERR_ARGUMENT, "null task");
  if (V) *V = t->V;
  if (E) *E = t->E;
  if (memory_gib)
    *memory_gib = (4.0 * (t->V + 1) + 4.0 * t->E + 4.0 * t->V * 5 + 4.0 * t->blk_len) /
                  (1024.0 * 1024.0 * 1024.0);
  if (ranks) *ranks = t->on_gpu ? t->st.r : nullptr;
  if (iterations) *iterations = t->st.iterations;
  return FR_OK;
}

}  // extern "C"
