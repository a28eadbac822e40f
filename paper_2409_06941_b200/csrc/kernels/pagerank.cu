// K1/K2: PageRank pull step over the incoming CSR (Gardenia
// PR), one bounded step = `iters` power iterations.
//
//   r'[v] = (1-d)/V + d * sum_{u in in(v)} c[u],   c'[v] = r'[v] * inv_outdeg[v]
//   dangling vertices (out-degree 0) have inv_outdeg = 0: their mass is dropped.
//
// Graph build (once, on the GPU): RMAT edges with the oracle's counter-based
// generator, self-loops dropped, (dst,src) keys radix-sorted and de-duplicated
// (CUB), offsets by histogram + scan, out-degrees by atomics.  That original
// CSR is what the parity tests compare; the step reads a relabelled copy:
//
//  * columns (the c[] index space) are renumbered by out-degree descending,
//    so the sources of most in-edges sit in a short prefix of c[] (RMAT-20:
//    the top 48 Ki vertices feed ~78 % of all gathers).  Each CTA stages that
//    prefix in shared memory once per iteration; a warp gather from shared
//    memory costs its bank-conflict degree (~3) instead of one L1 wavefront
//    per distinct line (~32), which is what bounds a divergent L2 gather;
//  * rows are ordered by in-degree bucket (split rows, then lane-group sizes
//    g = 32..1, then the rows with no in-edges), so a work item is 32/g
//    consecutive rows whose offsets load coalesced, and the zero-in-degree
//    tail (r' = (1-d)/V forever) is written only by the first two iterations.
//
// r is kept in original vertex order (the scattered r' store goes through
// the row's original id), c in column order.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "freeride_gpu.h"
#include "kernels/common.cuh"

namespace {

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

__global__ void check_ids_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t m,
                                 int32_t V, int32_t* __restrict__ bad) {
  int32_t n = 0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < m;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    n += (static_cast<uint32_t>(src[e]) >= static_cast<uint32_t>(V)) + (static_cast<uint32_t>(dst[e]) >= static_cast<uint32_t>(V));
  if (n) atomicAdd(bad, n);
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

// Column order: out-degree descending, then original id.
__global__ void col_keys_kernel(const int32_t* __restrict__ outdeg, int32_t V,
                                uint64_t* __restrict__ keys) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
    keys[v] = (static_cast<uint64_t>(0x7FFFFFFF - outdeg[v]) << 32) | static_cast<uint32_t>(v);
}

__global__ void col_perm_kernel(const uint64_t* __restrict__ sorted, int32_t V,
                                int32_t* __restrict__ colid) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x)
    colid[static_cast<uint32_t>(sorted[i])] = i;
}

// In-degree bucket: 7 = split (> kSplitEdges), 6..1 = g = 32..1 lanes per
// row (smallest power of two with E g >= deg, E = lane_edges()), 0 = no in-edges.
int lane_edges() {
  static const int v = [] {
    const char* e = std::getenv("FR_PR_LANE_EDGES");  // tuning hook: 4, 8 (default) or 16
    const int x = e ? std::atoi(e) : 8;
    return x == 4 || x == 16 ? x : 8;
  }();
  return v;
}
__host__ __device__ __forceinline__ int row_bucket(int32_t d, int32_t split_edges, int32_t lane_e) {
  if (d > split_edges) return 7;
  if (d == 0) return 0;
  int k = 0;
  while (k < 5 && (lane_e << k) < d) ++k;
  return k + 1;
}

// Row order: bucket descending, then column id (keeps c' stores of a warp close).
__global__ void row_keys_kernel(const int32_t* __restrict__ indeg,
                                const int32_t* __restrict__ colid, int32_t V, int32_t split_edges,
                                int32_t lane_e, uint64_t* __restrict__ keys) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
    keys[v] = (static_cast<uint64_t>(7 - row_bucket(indeg[v], split_edges, lane_e)) << 40) |
              (static_cast<uint64_t>(static_cast<uint32_t>(colid[v])) << 8) |
              0u;  // low byte unused
}

// Per row i (vertex v): rowc = column id, rowr = original id, rinv, in-degree
__global__ void row_perm_kernel(const uint64_t* __restrict__ sorted, int32_t V,
                                const int32_t* __restrict__ colperm_inv,  // column id -> original
                                const int32_t* __restrict__ outdeg,
                                const int32_t* __restrict__ indeg, int32_t* __restrict__ rowof,
                                int32_t* __restrict__ rowc, int32_t* __restrict__ rowr,
                                float* __restrict__ rinv, int32_t* __restrict__ rindeg) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x) {
    const int32_t c = static_cast<int32_t>((sorted[i] >> 8) & 0xFFFFFFFFu);
    const int32_t v = colperm_inv[c];
    rowof[v] = i;
    rowc[i] = c;
    rowr[i] = v;
    rinv[i] = outdeg[v] > 0 ? 1.0f / static_cast<float>(outdeg[v]) : 0.0f;
    rindeg[i] = indeg[v];
  }
}

__global__ void col_inv_kernel(const uint64_t* __restrict__ sorted, int32_t V,
                               int32_t* __restrict__ colperm_inv) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x)
    colperm_inv[i] = static_cast<int32_t>(static_cast<uint32_t>(sorted[i]));
}

// (dst << 32 | src) in original ids -> (row of dst << 32 | column of src)
__global__ void relabel_edges_kernel(const uint64_t* __restrict__ keys, int64_t E,
                                     const int32_t* __restrict__ rowof,
                                     const int32_t* __restrict__ colid,
                                     uint64_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < E;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[e];
    out[e] = (static_cast<uint64_t>(rowof[k >> 32]) << 32) |
             static_cast<uint32_t>(colid[k & 0xFFFFFFFFu]);
  }
}

__global__ void low_word_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<int32_t>(keys[i] & 0xFFFFFFFFu);
}

// r = 1/V (original order); c[0][col] = r * inv (written through the rows),
// c[1] = 0 (rewritten by the first iteration).
__global__ void pr_reset_kernel(const int32_t* __restrict__ rowc, const float* __restrict__ rinv,
                                int32_t V, float* __restrict__ r, float* __restrict__ c0,
                                float* __restrict__ c1) {
  const float r0 = static_cast<float>(1.0 / static_cast<double>(V));
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x) {
    r[i] = r0;
    c0[rowc[i]] = r0 * rinv[i];
    c1[i] = 0.0f;
  }
}

// Persistent grid shape (tuning hook FR_PR_CFG): "1024x1" = one 1024-thread
// CTA per SM with a 48 Ki-column hot prefix (default), "768x2" = two
// 768-thread CTAs per SM (48 warps) with 27 Ki columns each.
struct PrCfg {
  int threads, ctas_per_sm, hot;
};
PrCfg pr_cfg() {
  static const PrCfg c = [] {
    const char* e = std::getenv("FR_PR_CFG");
    if (e && std::string(e) == "768x2") return PrCfg{768, 2, 27648};
    return PrCfg{1024, 1, 49152};
  }();
  return c;
}
constexpr int kSplitEdges = 256;     // default: rows with more in-edges are split into chunks
constexpr int kMaxCtas = 512;        // split-row chunk lists per CTA (grid = SMs x CTAs per SM)
constexpr int kMaxSlots = 256;       // split rows per CTA (shared-memory accumulators)

struct PrArgs {
  const int32_t* off;    // relabelled incoming CSR (row order)
  const int32_t* col;    // column ids
  const float* rinv;     // per row: 1 / out-degree (0 if dangling)
  const int32_t* rowc;   // per row: column id (c' store)
  // r is written in row order (coalesced); fr_pr_ranks permutes it back
  const int4* chunks;    // {row, e_begin, e_end, slot | chunks of the row << 8}, grouped by CTA
  const float* c_in;
  float* r_out;
  float* c_out;
  int32_t bstart[8];     // first row of bucket b (7 = split .. 1 = g 1), bstart[0] = tail
  int32_t istart[8];     // first item of bucket b = 6..1 (items of b-1 follow), istart[0] = total
  int32_t hot, V, do_tail;
  int32_t nlists;        // chunk lists (LPT at build, one per CTA of a full grid); a smaller
                         // grid (an SM budget) walks lists b, b + grid, ...
  double base, damp;
  int32_t cta_chunk[kMaxCtas + 1];  // list b owns chunks [cta_chunk[b], cta_chunk[b+1])
};

// N predicated gathers per lane, `stride` apart: hot sources from shared
// memory, the rest from L2.  The N values are summed in fp32 (N <= 8 terms,
// relative error <= N * 2^-24), the caller accumulates these partials in fp64.
// Predicated loads (no branch): written as C++ `?:` the hot/cold choice
// compiles to one divergent branch region per element, so each gather issues
// only after the previous element's branch resolved; as predicated LDS/LDG
// all 2N loads of a lane issue back to back.
__device__ __forceinline__ float ld_if_global(const float* p, bool pred) {
  float v = 0.0f;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.f32 %0, [%1];\n\t}"
      : "+f"(v) : "l"(p), "r"(static_cast<int>(pred)));
  return v;
}
__device__ __forceinline__ float ld_if_shared(const float* p, bool pred) {
  float v = 0.0f;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.f32 %0, [%1];\n\t}"
      : "+f"(v) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))), "r"(static_cast<int>(pred)));
  return v;
}

template <int N>
__device__ __forceinline__ void load_cols(const PrArgs& a, int32_t e, int32_t e1, int stride, int32_t (&u)[N]) {
#pragma unroll
  for (int j = 0; j < N; ++j) u[j] = e + j * stride < e1 ? __ldg(&a.col[e + j * stride]) : -1;
}

template <int N>
__device__ __forceinline__ double gather_cols(const PrArgs& a, const float* hot, const int32_t (&u)[N]) {
  float v[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const bool in = u[j] >= 0, h = u[j] < a.hot;
    const int32_t x = in ? u[j] : 0;
    v[j] = ld_if_shared(hot + (h ? x : 0), in && h) + ld_if_global(a.c_in + x, in && !h);
  }
  float s = 0.0f;
#pragma unroll
  for (int j = 0; j < N; ++j) s += v[j];
  return static_cast<double>(s);
}

template <int N>
__device__ __forceinline__ double gather(const PrArgs& a, const float* hot, int32_t e, int32_t e1,
                                         int stride) {
  int32_t u[N];
  load_cols<N>(a, e, e1, stride, u);
  return gather_cols<N>(a, hot, u);
}

// A bucket item as seen by one lane: its row, edge range and the row's
// output metadata, all loaded up front (one round trip).
struct Item {
  int32_t e, e1, rr, rc;
  float inv;
  int lanes;
  bool emit;
  int32_t u0[4];  // the first 4 column ids of this lane (loaded with the item)
};

__device__ __forceinline__ Item prep(const PrArgs& a, int it, bool valid, int lane) {
  int b = 6;
#pragma unroll
  for (int k = 6; k > 1; --k)
    if (it >= a.istart[k - 1]) b = k - 1;
  Item x;
  x.lanes = 1 << (b - 1);
  const int sub = lane & (x.lanes - 1);
  const int32_t row = a.bstart[b] + (it - a.istart[b]) * (32 >> (b - 1)) + (lane >> (b - 1));
  const bool live = valid && row < a.bstart[b - 1];
  x.e = x.e1 = 0;
  x.rr = x.rc = 0;
  x.inv = 0.0f;
  x.emit = live && sub == 0;
  if (live) {
    x.e = __ldg(&a.off[row]) + sub;
    x.e1 = __ldg(&a.off[row + 1]);
    if (sub == 0) {
      x.rr = row;
      x.rc = __ldg(&a.rowc[row]);
      x.inv = __ldg(&a.rinv[row]);
    }
  }
  return x;
}

// the item's first column ids, once its offsets are in (one item ahead)
__device__ __forceinline__ void prep_cols(const PrArgs& a, Item& x) { load_cols<4>(a, x.e, x.e1, x.lanes, x.u0); }

__device__ __forceinline__ void store(const PrArgs& a, int32_t rr, int32_t rc, float inv, double s) {
  const float rv = static_cast<float>(a.base + a.damp * s);
  a.r_out[rr] = rv;
  a.c_out[rc] = rv * inv;
}

__device__ __forceinline__ double group_sum(double s, int lanes) {
  for (int o = lanes >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// One pull iteration.  Persistent CTAs (one per SM, 32 warps) copy the hot
// prefix of c[] into shared memory, then
//  (1) split rows: each CTA owns whole split rows (LPT-balanced at graph
//      build), its warps take their 256-edge chunks (8 gathers in flight per
//      lane) and meet in shared-memory fp64 accumulators; the warp finishing
//      a row's last chunk stores r'/c' (CTA-scope fences only: no global
//      memory barrier, no L1 invalidation);
//  (2) bucket items (32/g consecutive rows, g lanes per row), two items per
//      warp interleaved so both items' loads are in flight together, in a
//      static round-robin over all warps (items are ordered heavy first and
//      carry ~64..256 edges each);
//  (3) the zero-in-degree tail, when asked.
// Registers (MINB CTAs of kPrThreads resident, and at 1024 x 1 room for the
// stage's 1-warp dependency-wait kernel inside a bubble: 56, allocated 8 at a
// time; 768 x 2: 40).
template <int kPrThreads, int MINB>
__global__ void __maxnreg__(kPrThreads >= 1024 ? 56 : 40) pr_pull_kernel(PrArgs a) {
  constexpr int kPrWarps = kPrThreads / 32;
  extern __shared__ float4 hot4[];
  __shared__ double sacc[kMaxSlots];
  __shared__ int scnt[kMaxSlots];
  const float* hot = reinterpret_cast<const float*>(hot4);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // launched as a programmatic dependent of the previous iteration: the CTA
  // is resident early, but reads c_in only once that grid completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  {
    const float4* src = reinterpret_cast<const float4*>(a.c_in);
    for (int i = tid; i < (a.hot >> 2); i += kPrThreads) hot4[i] = __ldg(&src[i]);
    if (tid < kMaxSlots) {
      sacc[tid] = 0.0;
      scnt[tid] = 0;
    }
  }
  __syncthreads();
  // split-row chunks, software-pipelined: the next chunk's descriptor and
  // first 8 column ids per lane load while this chunk gathers
  for (int lb = blockIdx.x; lb < a.nlists; lb += gridDim.x) {
  if (lb != static_cast<int>(blockIdx.x)) {  // the previous list's rows are all stored: reuse the slots
    __syncthreads();
    if (tid < kMaxSlots) {
      sacc[tid] = 0.0;
      scnt[tid] = 0;
    }
    __syncthreads();
  }
  const int c_end = a.cta_chunk[lb + 1];
  int c = a.cta_chunk[lb] + warp;
  int4 ch = c < c_end ? __ldg(&a.chunks[c]) : make_int4(0, 0, 0, 0);
  int32_t cu[8];
  load_cols<8>(a, ch.y + lane, ch.z, 32, cu);
  for (; c < c_end; c += kPrWarps) {
    const int cn = c + kPrWarps;
    const int4 chn = cn < c_end ? __ldg(&a.chunks[cn]) : make_int4(0, 0, 0, 0);
    double s = gather_cols<8>(a, hot, cu);
    for (int32_t e = ch.y + lane + 256; e < ch.z; e += 256) s += gather<8>(a, hot, e, ch.z, 32);
    load_cols<8>(a, chn.y + lane, chn.z, 32, cu);
    s = group_sum(s, 32);
    if (lane == 0) {
      const int slot = ch.w & 0xFF, need = ch.w >> 8;
      atomicAdd(&sacc[slot], s);
      __threadfence_block();
      if (atomicAdd(&scnt[slot], 1) + 1 == need) {
        __threadfence_block();
        const double tot = *static_cast<volatile double*>(&sacc[slot]);
        store(a, ch.x, __ldg(&a.rowc[ch.x]), __ldg(&a.rinv[ch.x]), tot);
      }
    }
    ch = chn;
  }
  }
  const int nw = gridDim.x * kPrWarps, gw = blockIdx.x * kPrWarps + warp, n = a.istart[0];
  // software-pipelined: the next pair's offsets and output metadata load
  // while this pair gathers
  Item x = prep(a, gw, gw < n, lane), y = prep(a, gw + nw, gw + nw < n, lane);
  prep_cols(a, x);
  prep_cols(a, y);
  for (int it = gw; it < n; it += 2 * nw) {
    const int nx = it + 2 * nw;
    Item px = prep(a, nx, nx < n, lane), py = prep(a, nx + nw, nx + nw < n, lane);
    double sx = gather_cols<4>(a, hot, x.u0), sy = gather_cols<4>(a, hot, y.u0);
    for (int32_t ex = x.e + 4 * x.lanes, ey = y.e + 4 * y.lanes; ex < x.e1 || ey < y.e1;
         ex += 4 * x.lanes, ey += 4 * y.lanes) {
      sx += gather<4>(a, hot, ex, x.e1, x.lanes);
      sy += gather<4>(a, hot, ey, y.e1, y.lanes);
    }
    prep_cols(a, px);  // next pair's first columns: in flight while this pair's sums and stores finish
    prep_cols(a, py);
    sx = group_sum(sx, x.lanes);
    sy = group_sum(sy, y.lanes);
    if (x.emit) store(a, x.rr, x.rc, x.inv, sx);
    if (y.emit) store(a, y.rr, y.rc, y.inv, sy);
    x = px;
    y = py;
  }
  asm volatile("griddepcontrol.launch_dependents;");
  if (a.do_tail) {
    for (int32_t i = a.bstart[0] + blockIdx.x * kPrThreads + tid; i < a.V; i += gridDim.x * kPrThreads)
      store(a, i, __ldg(&a.rowc[i]), __ldg(&a.rinv[i]), 0.0);
  }
}

// r is kept in row order by the step; readout permutes it to original ids
__global__ void pr_unpermute_kernel(const float* __restrict__ r_row, const int32_t* __restrict__ rowr,
                                    int32_t V, float* __restrict__ r_orig) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < V; i += gridDim.x * blockDim.x)
    r_orig[rowr[i]] = r_row[i];
}

int grid_for(int64_t work, int threads, int per_sm) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (work + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(sms) * per_sm)));
}

bool pr_pdl() {
  static const bool v = [] {
    const char* e = std::getenv("FR_PR_PDL");  // A/B override
    return !e || std::atoi(e) != 0;
  }();
  return v;
}

int split_edges() {
  static const int v = [] {
    const char* e = std::getenv("FR_PR_SPLIT");  // tuning hook, 32..256
    return e ? std::min(256, std::max(32, std::atoi(e))) : kSplitEdges;
  }();
  return v;
}

int chunk_edges() {
  static const int v = [] {
    // split-row chunk size (multiple of 256): 512 halves the per-chunk fp64
    // warp reductions and shared-memory atomics of 256 (37.7 -> 36.2 us per
    // back-to-back iteration; 1024: 36.2)
    const char* e = std::getenv("FR_PR_CHUNK");
    const int x = e ? std::atoi(e) : 512;
    return std::max(256, std::min(4096, x / 256 * 256));
  }();
  return v;
}

int hot_vertices(int32_t V) {
  static const int want = [] {
    const char* e = std::getenv("FR_PR_HOT");  // tuning hook
    return e ? std::max(0, std::atoi(e)) : pr_cfg().hot;
  }();
  return std::min(want, V) & ~3;
}

}  // namespace

// Device view of a graph.  The original CSR (offsets/col/outdeg) is what the
// parity tests compare with the oracle; the step kernel reads the relabelled
// copy (xoff/xcol + per-row rowc/rowr/rinv) and the split-row chunk list.
struct fr_pr_graph {
  int32_t V = 0;
  int64_t E = 0;
  int32_t* offsets = nullptr;  // V + 1, original ids
  int32_t* col = nullptr;      // E
  int32_t* outdeg = nullptr;   // V
  int32_t* xoff = nullptr;     // V + 1, row order
  int32_t* xcol = nullptr;     // E, column ids
  int32_t* rowc = nullptr;     // V
  int32_t* rowr = nullptr;     // V
  float* rinv = nullptr;       // V
  int4* chunks = nullptr;      // n_chunk, grouped by CTA
  int32_t n_chunk = 0, n_split = 0;
  int32_t cta_chunk[kMaxCtas + 1] = {};
  int32_t bstart[8] = {};      // see PrArgs
  int32_t istart[8] = {};
  int sms = 148;
};

struct fr_pr_state {
  const fr_pr_graph* g = nullptr;
  float* r = nullptr;       // row order (written by the step)
  float* r_orig = nullptr;  // original vertex order (filled by readout)
  float* c[2] = {nullptr, nullptr};
  int cur = 0;
  int64_t iterations = 0;
  int tail_pending = 2;        // launches that still write the zero-in-degree tail
  float tail_damping = -1.0f;  // damping the tail was written with
  int max_sms = 0;             // fr_pr_state_set_max_sms (0 = all)
};

namespace {

// Readout (a synchronisation point by contract): wait for the steps, then
// permute the row-order ranks to original vertex ids.
int pr_readout(const fr_pr_state* st) {
  FR_CUDA_TRY(cudaDeviceSynchronize());
  const fr_pr_graph* g = st->g;
  pr_unpermute_kernel<<<grid_for(g->V, 256, 8), 256>>>(st->r, g->rowr, g->V, st->r_orig);
  FR_CUDA_TRY(cudaGetLastError());
  FR_CUDA_TRY(cudaDeviceSynchronize());
  return FR_OK;
}

void free_graph(fr_pr_graph* g) {
  for (void* p : {static_cast<void*>(g->offsets), static_cast<void*>(g->col),
                  static_cast<void*>(g->outdeg), static_cast<void*>(g->xoff),
                  static_cast<void*>(g->xcol), static_cast<void*>(g->rowc),
                  static_cast<void*>(g->rowr), static_cast<void*>(g->rinv),
                  static_cast<void*>(g->chunks)})
    if (p) cudaFree(p);
  delete g;
}

// Bucket boundaries, item counts and the split-row chunk list (host, once).
int build_work(fr_pr_graph* g, cudaStream_t s) {
  std::vector<int32_t> off(static_cast<size_t>(g->V) + 1);
  FR_CUDA_TRY(cudaMemcpyAsync(off.data(), g->xoff, off.size() * sizeof(int32_t),
                              cudaMemcpyDeviceToHost, s));
  FR_CUDA_TRY(cudaStreamSynchronize(s));
  int32_t count[8] = {};
  const int split = split_edges();
  for (int32_t r = 0; r < g->V; ++r) ++count[row_bucket(off[r + 1] - off[r], split, lane_edges())];
  // rows are sorted by bucket descending: bucket 7 first
  int32_t at = 0;
  for (int b = 7; b >= 0; --b) {
    g->bstart[b] = at;
    at += count[b];
  }
  int32_t items = 0;
  for (int b = 6; b >= 1; --b) {
    g->istart[b] = items;
    const int per = 32 >> (b - 1);
    items += (count[b] + per - 1) / per;
  }
  g->istart[7] = 0;
  g->istart[0] = items;
  // split rows -> CTAs, longest first onto the least-loaded CTA (LPT), at
  // most kMaxSlots rows per CTA; each CTA's chunks are contiguous.
  const int ctas = std::min(g->sms * pr_cfg().ctas_per_sm, kMaxCtas);
  if (count[7] > ctas * kMaxSlots)
    return frcapi::fail(FR_ERR_UNSUPPORTED, "too many split rows for the per-CTA accumulators");
  std::vector<int32_t> order(count[7]);
  for (int32_t r = 0; r < count[7]; ++r) order[r] = r;
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
    return off[x + 1] - off[x] > off[y + 1] - off[y];
  });
  std::vector<int64_t> load(ctas, 0);
  std::vector<std::vector<int32_t>> owned(ctas);
  for (int32_t r : order) {
    int best = -1;
    for (int c = 0; c < ctas; ++c)
      if (static_cast<int>(owned[c].size()) < kMaxSlots && (best < 0 || load[c] < load[best])) best = c;
    owned[best].push_back(r);
    load[best] += off[r + 1] - off[r];
  }
  std::vector<int4> chunks;
  for (int c = 0; c < ctas; ++c) {
    g->cta_chunk[c] = static_cast<int32_t>(chunks.size());
    for (size_t slot = 0; slot < owned[c].size(); ++slot) {
      const int32_t r = owned[c][slot];
      const int32_t ce = chunk_edges();
      const int32_t n = (off[r + 1] - off[r] + ce - 1) / ce;
      for (int32_t e = off[r]; e < off[r + 1]; e += ce)
        chunks.push_back(make_int4(r, e, std::min(e + ce, off[r + 1]),
                                   static_cast<int32_t>(slot) | (n << 8)));
    }
  }
  for (int c = ctas; c <= kMaxCtas; ++c) g->cta_chunk[c] = static_cast<int32_t>(chunks.size());
  g->n_split = count[7];
  g->n_chunk = static_cast<int32_t>(chunks.size());
  FR_CUDA_TRY(cudaMalloc(&g->chunks, std::max<size_t>(1, chunks.size()) * sizeof(int4)));
  if (!chunks.empty()) {
    FR_CUDA_TRY(cudaMemcpyAsync(g->chunks, chunks.data(), chunks.size() * sizeof(int4),
                                cudaMemcpyHostToDevice, s));
    FR_CUDA_TRY(cudaStreamSynchronize(s));
  }
  return FR_OK;
}

// Builds the graph from m directed edges src[e] -> dst[e] (device): either
// RMAT-generated (gen_scale > 0, src/dst ignored) or the caller's (ids
// checked to lie in [0, V)).  Self loops and duplicates are dropped.
int build_graph(int32_t Vn, int64_t m, const int32_t* user_src, const int32_t* user_dst, int32_t gen_scale,
                uint64_t seed, cudaStream_t s, fr_pr_graph** out) {
  auto* g = new fr_pr_graph;
  g->V = Vn;
  int scale = 1;  // bits of a vertex id
  while (scale < 31 && (int64_t(1) << scale) < Vn) ++scale;
  const size_t V = static_cast<size_t>(g->V);
  int32_t *src = nullptr, *dst = nullptr, *indeg = nullptr, *d_sel = nullptr;
  int32_t *colid = nullptr, *colinv = nullptr, *rowof = nullptr, *rindeg = nullptr;
  uint64_t *keys = nullptr, *sorted = nullptr, *vkeys = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int rc = FR_OK;
  auto step = [&](cudaError_t e, const char* what) {
    if (rc == FR_OK && e != cudaSuccess) rc = frcapi::cuda_status(e, what);
    return rc == FR_OK;
  };
  auto temp = [&](size_t need) {  // grow the CUB scratch
    if (rc != FR_OK || need <= tmp_bytes) return;
    if (tmp) cudaFree(tmp);
    tmp = nullptr;
    tmp_bytes = 0;
    if (step(cudaMalloc(&tmp, need), "cub temp")) tmp_bytes = need;
  };
  const int gv = grid_for(g->V, 256, 8), gm = grid_for(m, 256, 16);
  const size_t mb = static_cast<size_t>(std::max<int64_t>(m, 1));
  if (gen_scale > 0) {
    step(cudaMalloc(&src, mb * sizeof(int32_t)), "rmat src");
    step(cudaMalloc(&dst, mb * sizeof(int32_t)), "rmat dst");
  }
  step(cudaMalloc(&keys, mb * sizeof(uint64_t)), "keys");
  step(cudaMalloc(&sorted, mb * sizeof(uint64_t)), "sorted");
  step(cudaMalloc(&d_sel, sizeof(int32_t)), "count");
  if (rc == FR_OK && gen_scale == 0 && m > 0) {  // caller's edges: every id in [0, V)
    int32_t bad = 0;
    step(cudaMemsetAsync(d_sel, 0, sizeof(int32_t), s), "memset");
    check_ids_kernel<<<gm, 256, 0, s>>>(user_src, user_dst, m, Vn, d_sel);
    step(cudaMemcpyAsync(&bad, d_sel, sizeof(int32_t), cudaMemcpyDeviceToHost, s), "id check");
    step(cudaStreamSynchronize(s), "id check");
    if (rc == FR_OK && bad)
      rc = frcapi::fail(FR_ERR_VALIDATION, std::to_string(bad) + " edge endpoints outside [0, V)", "edges");
  }
  if (rc == FR_OK && m > 0) {
    if (gen_scale > 0) rmat_kernel<<<gm, 256, 0, s>>>(gen_scale, m, seed, src, dst);
    edge_keys_kernel<<<gm, 256, 0, s>>>(gen_scale > 0 ? src : user_src, gen_scale > 0 ? dst : user_dst, m, keys);
    step(cudaGetLastError(), "rmat / keys");
  }
  size_t need = 0;
  if (rc == FR_OK && m > 0) {
    cub::DeviceRadixSort::SortKeys(nullptr, need, keys, sorted, static_cast<int>(m), 0, 64, s);
    temp(need);
    cub::DeviceSelect::Unique(nullptr, need, sorted, keys, d_sel, static_cast<int>(m), s);
    temp(need);
  }
  int32_t n_unique = 0;
  if (rc == FR_OK && m > 0) {
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
    const size_t Eb = std::max<int64_t>(1, g->E) * sizeof(int32_t);
    step(cudaMalloc(&g->col, Eb), "col");
    step(cudaMalloc(&g->xcol, Eb), "xcol");
    step(cudaMalloc(&g->offsets, (V + 1) * sizeof(int32_t)), "offsets");
    step(cudaMalloc(&g->xoff, (V + 1) * sizeof(int32_t)), "xoff");
    step(cudaMalloc(&g->outdeg, V * sizeof(int32_t)), "outdeg");
    step(cudaMalloc(&g->rowc, V * sizeof(int32_t)), "rowc");
    step(cudaMalloc(&g->rowr, V * sizeof(int32_t)), "rowr");
    step(cudaMalloc(&g->rinv, V * sizeof(float)), "rinv");
    step(cudaMalloc(&indeg, V * sizeof(int32_t)), "indeg");
    step(cudaMalloc(&colid, V * sizeof(int32_t)), "colid");
    step(cudaMalloc(&colinv, V * sizeof(int32_t)), "colinv");
    step(cudaMalloc(&rowof, V * sizeof(int32_t)), "rowof");
    step(cudaMalloc(&rindeg, V * sizeof(int32_t)), "rindeg");
    step(cudaMalloc(&vkeys, 2 * V * sizeof(uint64_t)), "vertex keys");
  }
  if (rc == FR_OK) {
    step(cudaMemsetAsync(indeg, 0, V * sizeof(int32_t), s), "memset");
    step(cudaMemsetAsync(g->outdeg, 0, V * sizeof(int32_t), s), "memset");
    step(cudaMemsetAsync(g->offsets, 0, sizeof(int32_t), s), "memset");
    step(cudaMemsetAsync(g->xoff, 0, sizeof(int32_t), s), "memset");
    if (g->E > 0) split_keys_kernel<<<grid_for(g->E, 256, 16), 256, 0, s>>>(keys, g->E, g->col, indeg, g->outdeg);
    step(cudaGetLastError(), "split keys");
    cub::DeviceScan::InclusiveSum(nullptr, need, indeg, g->offsets + 1, g->V, s);
    temp(need);
    step(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, indeg, g->offsets + 1, g->V, s), "scan");
  }
  // column order, then row order, then the relabelled CSR
  if (rc == FR_OK) {
    cub::DeviceRadixSort::SortKeys(nullptr, need, vkeys, vkeys + V, g->V, 0, 64, s);
    temp(need);
    col_keys_kernel<<<gv, 256, 0, s>>>(g->outdeg, g->V, vkeys);
    step(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, vkeys, vkeys + V, g->V, 0, 63, s), "column sort");
    col_perm_kernel<<<gv, 256, 0, s>>>(vkeys + V, g->V, colid);
    col_inv_kernel<<<gv, 256, 0, s>>>(vkeys + V, g->V, colinv);
    row_keys_kernel<<<gv, 256, 0, s>>>(indeg, colid, g->V, split_edges(), lane_edges(), vkeys);
    step(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, vkeys, vkeys + V, g->V, 8, 43, s), "row sort");
    row_perm_kernel<<<gv, 256, 0, s>>>(vkeys + V, g->V, colinv, g->outdeg, indeg, rowof, g->rowc,
                                       g->rowr, g->rinv, rindeg);
    step(cudaGetLastError(), "relabel");
    if (g->E > 0) {
      relabel_edges_kernel<<<grid_for(g->E, 256, 16), 256, 0, s>>>(keys, g->E, rowof, colid, sorted);
      step(cudaGetLastError(), "relabel edges");
      cub::DeviceRadixSort::SortKeys(nullptr, need, sorted, keys, static_cast<int>(g->E), 0, 32 + scale, s);
      temp(need);
      step(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, sorted, keys, static_cast<int>(g->E), 0,
                                          32 + scale, s), "relabelled edge sort");
      low_word_kernel<<<grid_for(g->E, 256, 16), 256, 0, s>>>(keys, g->E, g->xcol);
      step(cudaGetLastError(), "xcol");
    }
    cub::DeviceScan::InclusiveSum(nullptr, need, rindeg, g->xoff + 1, g->V, s);
    temp(need);
    step(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, rindeg, g->xoff + 1, g->V, s), "xscan");
  }
  for (void* p : {static_cast<void*>(src), static_cast<void*>(dst), static_cast<void*>(keys),
                  static_cast<void*>(sorted), static_cast<void*>(indeg), static_cast<void*>(d_sel),
                  static_cast<void*>(colid), static_cast<void*>(colinv), static_cast<void*>(rowof),
                  static_cast<void*>(rindeg), static_cast<void*>(vkeys), tmp})
    if (p) cudaFreeAsync(p, s);
  if (rc == FR_OK) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g->sms, cudaDevAttrMultiProcessorCount, dev);
    rc = build_work(g, s);
  }
  if (rc != FR_OK) {
    free_graph(g);
    return rc;
  }
  *out = g;
  return FR_OK;
}

}  // namespace

extern "C" {

int fr_pr_graph_rmat(int32_t scale, int32_t edge_factor, uint64_t seed, void* stream,
                     fr_pr_graph** out) {
  if (!out) return frcapi::fail(FR_ERR_ARGUMENT, "null graph out");
  if (scale < 1 || scale > 30 || edge_factor < 1)
    return frcapi::fail(FR_ERR_VALIDATION, "scale in [1,30], edge_factor >= 1", "scale");
  const int64_t m = static_cast<int64_t>(edge_factor) << scale;
  if (m > INT32_MAX) return frcapi::fail(FR_ERR_VALIDATION, "edge_factor << scale must be < 2^31", "edge_factor");
  return build_graph(1 << scale, m, nullptr, nullptr, scale, seed, static_cast<cudaStream_t>(stream), out);
}

int fr_pr_graph_from_edges(int32_t V, int64_t E, const int32_t* src, const int32_t* dst, void* stream,
                           fr_pr_graph** out) {
  if (!out) return frcapi::fail(FR_ERR_ARGUMENT, "null graph out");
  if (V < 1 || E < 0 || E > INT32_MAX) return frcapi::fail(FR_ERR_VALIDATION, "V >= 1, 0 <= E < 2^31", "V");
  if (E > 0 && (!src || !dst)) return frcapi::fail(FR_ERR_ARGUMENT, "null edge arrays");
  return build_graph(V, E, src, dst, 0, 0, static_cast<cudaStream_t>(stream), out);
}

int fr_pr_graph_destroy(fr_pr_graph* g) {
  if (g) free_graph(g);
  return FR_OK;
}

int fr_pr_graph_info(const fr_pr_graph* g, int32_t* V, int64_t* E, int32_t* n_blocks) {
  if (!g) return frcapi::fail(FR_ERR_ARGUMENT, "null graph");
  if (V) *V = g->V;
  if (E) *E = g->E;
  if (n_blocks) *n_blocks = g->n_chunk + g->istart[0];
  return FR_OK;
}

int fr_pr_graph_csr(const fr_pr_graph* g, const int32_t** offsets, const int32_t** col_idx,
                    const int32_t** outdeg) {
  if (!g) return frcapi::fail(FR_ERR_ARGUMENT, "null graph");
  if (!g->offsets) return frcapi::fail(FR_ERR_UNSUPPORTED, "graph holds only the relabelled CSR");
  if (offsets) *offsets = g->offsets;
  if (col_idx) *col_idx = g->col;
  if (outdeg) *outdeg = g->outdeg;
  return FR_OK;
}

int fr_pr_state_create(const fr_pr_graph* g, fr_pr_state** out) {
  if (!g || !out) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  auto* st = new fr_pr_state;
  st->g = g;
  const size_t b = sizeof(float) * static_cast<size_t>(std::max(4, g->V));
  cudaError_t e = cudaMalloc(&st->r, b);
  if (e == cudaSuccess) e = cudaMalloc(&st->r_orig, b);
  if (e == cudaSuccess) e = cudaMalloc(&st->c[0], b);
  if (e == cudaSuccess) e = cudaMalloc(&st->c[1], b);
  if (e != cudaSuccess) {
    for (void* p : {static_cast<void*>(st->r), static_cast<void*>(st->r_orig), static_cast<void*>(st->c[0]),
                    static_cast<void*>(st->c[1])})
      if (p) cudaFree(p);
    delete st;
    return frcapi::cuda_status(e, "pagerank state");
  }
  *out = st;
  return FR_OK;
}

int fr_pr_state_set_max_sms(fr_pr_state* st, int32_t sms) {
  if (!st) return frcapi::fail(FR_ERR_ARGUMENT, "null state");
  if (sms < 0) return frcapi::fail(FR_ERR_VALIDATION, "sms must be >= 0", "sms");
  st->max_sms = sms;
  return FR_OK;
}

int fr_pr_state_destroy(fr_pr_state* st) {
  if (!st) return FR_OK;
  for (void* p : {static_cast<void*>(st->r), static_cast<void*>(st->r_orig), static_cast<void*>(st->c[0]),
                  static_cast<void*>(st->c[1])})
    if (p) cudaFree(p);
  delete st;
  return FR_OK;
}

int fr_pr_reset(fr_pr_state* st, void* stream) {
  if (!st) return frcapi::fail(FR_ERR_ARGUMENT, "null state");
  auto s = static_cast<cudaStream_t>(stream);
  const fr_pr_graph* g = st->g;
  st->cur = 0;
  st->iterations = 0;
  st->tail_pending = 2;
  st->tail_damping = -1.0f;
  pr_reset_kernel<<<grid_for(g->V, 256, 8), 256, 0, s>>>(g->rowc, g->rinv, g->V, st->r, st->c[0],
                                                         st->c[1]);
  FR_CUDA_LAUNCHED("pr_reset");
  return FR_OK;
}

int fr_pr_step(fr_pr_state* st, int32_t iters, float damping, void* stream) {
  if (!st) return frcapi::fail(FR_ERR_ARGUMENT, "null state");
  if (iters < 0) return frcapi::fail(FR_ERR_VALIDATION, "iters must be >= 0", "iters");
  const fr_pr_graph* g = st->g;
  auto s = static_cast<cudaStream_t>(stream);
  PrArgs a{};
  a.off = g->xoff;
  a.col = g->xcol;
  a.rinv = g->rinv;
  a.rowc = g->rowc;
  a.chunks = g->chunks;
  a.r_out = st->r;
  std::memcpy(a.cta_chunk, g->cta_chunk, sizeof(a.cta_chunk));
  std::memcpy(a.bstart, g->bstart, sizeof(a.bstart));
  std::memcpy(a.istart, g->istart, sizeof(a.istart));
  a.hot = hot_vertices(g->V);
  a.V = g->V;
  a.damp = static_cast<double>(damping);
  a.base = (1.0 - static_cast<double>(damping)) / static_cast<double>(g->V);
  const size_t smem = static_cast<size_t>(a.hot) * sizeof(float);
  const PrCfg cfg = pr_cfg();
  auto kern = cfg.threads == 768 ? pr_pull_kernel<768, 2> : pr_pull_kernel<1024, 1>;
  static int smem_set = -1;  // per process; the attribute is per function
  if (static_cast<int>(smem) > smem_set) {
    FR_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
    smem_set = static_cast<int>(smem);
  }
  if (st->tail_damping != damping) {  // the tail's constant changed
    st->tail_damping = damping;
    st->tail_pending = 2;
  }
  for (int i = 0; i < iters; ++i) {
    a.c_in = st->c[st->cur];
    a.c_out = st->c[st->cur ^ 1];
    a.do_tail = st->tail_pending > 0;
    cudaLaunchConfig_t lc{};
    const int full = std::min(g->sms * cfg.ctas_per_sm, kMaxCtas);
    a.nlists = full;
    lc.gridDim = dim3(st->max_sms > 0 ? std::min(full, std::min(st->max_sms, g->sms) * cfg.ctas_per_sm) : full);
    lc.blockDim = dim3(cfg.threads);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;  // safe: the kernel waits before reading
    lc.attrs = at;
    lc.numAttrs = pr_pdl() ? 1 : 0;
    FR_CUDA_TRY(cudaLaunchKernelEx(&lc, kern, a));
    if (st->tail_pending > 0) --st->tail_pending;
    st->cur ^= 1;
    st->iterations++;
  }
  FR_CUDA_LAUNCHED("pr_pull");
  return FR_OK;
}

int fr_pr_ranks(const fr_pr_state* st, const float** r, int64_t* iterations) {
  if (!st) return frcapi::fail(FR_ERR_ARGUMENT, "null state");
  if (r) {
    const int rc = pr_readout(st);
    if (rc != FR_OK) return rc;
    *r = st->r_orig;
  }
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
  fr_pr_graph shape;  // sizes, buckets and counts of the built graph (no device pointers)
  int32_t *h_xoff = nullptr, *h_xcol = nullptr, *h_rowc = nullptr, *h_rowr = nullptr;
  float* h_rinv = nullptr;
  int4* h_chunks = nullptr;
  fr_pr_graph g;  // device view (owned through the task, freed with cudaFreeAsync)
  fr_pr_state st;
  bool on_gpu = false;
  cudaStream_t last = nullptr;
  int32_t max_sms = 0;  // set_sm_budget
};

// The task keeps only what the step reads (not the original-order CSR), in
// pinned host memory: StopSideTask frees the device copy, InitSideTask
// uploads it again.
int pin_graph(PrTask* t, const fr_pr_graph* g) {
  int rc = FR_OK;
  {
    fr_pr_graph& sh = t->shape;
    sh.V = g->V;
    sh.E = g->E;
    sh.n_chunk = g->n_chunk;
    sh.n_split = g->n_split;
    std::memcpy(sh.bstart, g->bstart, sizeof(sh.bstart));
    std::memcpy(sh.istart, g->istart, sizeof(sh.istart));
    std::memcpy(sh.cta_chunk, g->cta_chunk, sizeof(sh.cta_chunk));
    sh.sms = g->sms;
    auto pin = [&](void** p, size_t bytes, const void* dev) {
      if (rc != FR_OK) return;
      cudaError_t e = cudaMallocHost(p, std::max<size_t>(bytes, 16));
      if (e == cudaSuccess && bytes) e = cudaMemcpy(*p, dev, bytes, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) rc = frcapi::cuda_status(e, "pagerank host copy");
    };
    const size_t V = static_cast<size_t>(g->V);
    pin(reinterpret_cast<void**>(&t->h_xoff), (V + 1) * 4, g->xoff);
    pin(reinterpret_cast<void**>(&t->h_xcol), size_t(g->E) * 4, g->xcol);
    pin(reinterpret_cast<void**>(&t->h_rowc), V * 4, g->rowc);
    pin(reinterpret_cast<void**>(&t->h_rowr), V * 4, g->rowr);
    pin(reinterpret_cast<void**>(&t->h_rinv), V * 4, g->rinv);
    pin(reinterpret_cast<void**>(&t->h_chunks), size_t(g->n_chunk) * sizeof(int4), g->chunks);
  }
  return rc;
}

int pr_task_create(void* u) {
  auto* t = static_cast<PrTask*>(u);
  if (t->h_xoff) return FR_OK;
  cudaStream_t s = nullptr;
  FR_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  fr_pr_graph* g = nullptr;
  int rc = fr_pr_graph_rmat(t->cfg.scale, t->cfg.edge_factor, t->cfg.seed, s, &g);
  if (rc == FR_OK) rc = pin_graph(t, g);
  if (g) fr_pr_graph_destroy(g);
  cudaStreamDestroy(s);
  return rc;
}

int pr_task_init(void* u, void* stream) {
  auto* t = static_cast<PrTask*>(u);
  auto s = static_cast<cudaStream_t>(stream);
  t->last = s;
  fr_pr_graph& g = t->g;
  g = t->shape;
  const size_t V = static_cast<size_t>(g.V);
  auto up = [&](void** d, const void* h, size_t bytes) -> cudaError_t {
    cudaError_t e = cudaMallocAsync(d, std::max<size_t>(bytes, 16), s);
    if (e == cudaSuccess && bytes) e = cudaMemcpyAsync(*d, h, bytes, cudaMemcpyHostToDevice, s);
    return e;
  };
  FR_CUDA_TRY(up(reinterpret_cast<void**>(&g.xoff), t->h_xoff, (V + 1) * 4));
  FR_CUDA_TRY(up(reinterpret_cast<void**>(&g.xcol), t->h_xcol, size_t(g.E) * 4));
  FR_CUDA_TRY(up(reinterpret_cast<void**>(&g.rowc), t->h_rowc, V * 4));
  FR_CUDA_TRY(up(reinterpret_cast<void**>(&g.rowr), t->h_rowr, V * 4));
  FR_CUDA_TRY(up(reinterpret_cast<void**>(&g.rinv), t->h_rinv, V * 4));
  FR_CUDA_TRY(up(reinterpret_cast<void**>(&g.chunks), t->h_chunks, size_t(g.n_chunk) * sizeof(int4)));
  t->st = fr_pr_state{};
  t->st.g = &g;
  t->st.max_sms = t->max_sms;
  for (float** p : {&t->st.r, &t->st.r_orig, &t->st.c[0], &t->st.c[1]})
    FR_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(V, 4) * 4, s));
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
  for (void* p : {static_cast<void*>(t->g.xoff), static_cast<void*>(t->g.xcol),
                  static_cast<void*>(t->g.rowc), static_cast<void*>(t->g.rowr),
                  static_cast<void*>(t->g.rinv), static_cast<void*>(t->g.chunks),
                  static_cast<void*>(t->st.r), static_cast<void*>(t->st.r_orig), static_cast<void*>(t->st.c[0]),
                  static_cast<void*>(t->st.c[1])})
    if (p) FR_CUDA_TRY(cudaFreeAsync(p, t->last));
  t->g = fr_pr_graph{};
  t->st.r = nullptr;
  t->on_gpu = false;
  return FR_OK;
}

int pr_task_sm_budget(void* u, int32_t sms) {
  auto* t = static_cast<PrTask*>(u);
  t->max_sms = sms;
  t->st.max_sms = sms;
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
  for (void* p : {static_cast<void*>(t->h_xoff), static_cast<void*>(t->h_xcol),
                  static_cast<void*>(t->h_rowc), static_cast<void*>(t->h_rowr),
                  static_cast<void*>(t->h_rinv), static_cast<void*>(t->h_chunks)})
    if (p) cudaFreeHost(p);
  delete t;
}

}  // namespace

extern "C" {

int fr_pagerank_task_create(const fr_pagerank_task_config* c, fr_side_task_vtable* vt, void** user) {
  return fr_pagerank_task_create_from_graph(c, nullptr, vt, user);
}

int fr_pagerank_task_create_from_graph(const fr_pagerank_task_config* c, const fr_pr_graph* graph,
                                       fr_side_task_vtable* vt, void** user) {
  if (!c || !vt || !user) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (c->iters_per_step < 1) return frcapi::fail(FR_ERR_VALIDATION, "iters_per_step must be >= 1", "iters_per_step");
  auto* t = new PrTask;
  t->cfg = *c;
  int rc = FR_OK;
  if (graph) {  // the caller's graph: copy what the step reads, the caller keeps the graph
    rc = pin_graph(t, graph);
  } else {
    rc = pr_task_create(t);  // build now: work units per step need E
  }
  if (rc != FR_OK) {
    pr_task_destroy(t);
    return rc;
  }
  std::memset(vt, 0, sizeof(*vt));
  vt->carveout_hint = 100;
  vt->create = pr_task_create;
  vt->init = pr_task_init;
  vt->run_next_step = pr_task_step;
  vt->stop = pr_task_stop;
  vt->finished = pr_task_finished;
  vt->destroy = pr_task_destroy;
  vt->set_sm_budget = pr_task_sm_budget;
  vt->work_units_per_step = static_cast<double>(t->shape.E) * c->iters_per_step;  // edges
  *user = t;
  return FR_OK;
}

int fr_pagerank_task_info(void* user, int32_t* V, int64_t* E, double* memory_gib,
                          const float** ranks, int64_t* iterations) {
  auto* t = static_cast<PrTask*>(user);
  if (!t) return frcapi::fail(FR_ERR_ARGUMENT, "null task");
  const fr_pr_graph& g = t->shape;
  if (V) *V = g.V;
  if (E) *E = g.E;
  // xoff + xcol + rowc/rowr/rinv + r (row and original order) + 2 c + chunk list
  if (memory_gib)
    *memory_gib = (4.0 * (g.V + 1) + 4.0 * g.E + 4.0 * g.V * 7 + 16.0 * g.n_chunk) /
                  (1024.0 * 1024.0 * 1024.0);
  if (ranks) {
    *ranks = nullptr;
    if (t->on_gpu) {
      const int rc = pr_readout(&t->st);
      if (rc != FR_OK) return rc;
      *ranks = t->st.r_orig;
    }
  }
  if (iterations) *iterations = t->st.iterations;
  return FR_OK;
}

}  // extern "C"
