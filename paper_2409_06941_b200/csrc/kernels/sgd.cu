// K3/K4: Graph-SGD matrix factorisation (Gardenia SGD;
// SURVEY.md §8 a16), one bounded step = an edge chunk [e_begin, e_end).
//
//   per edge (u, v, r):  e = r - <L_u, L_v>
//                        L_u += eta (e L_v - lambda L_u)
//                        L_v += eta (e L_u - lambda L_v)      (old L_u)
//   Hogwild: concurrent edges race on shared vertices by design (lost
//   updates are part of the algorithm), so parity is on RMSE (north star:
//   |dRMSE| <= 1e-3 vs the sequential CPU oracle after a fixed epoch count).
//
// B200-first layout: L is fp32 [V][K] row-major, one 64 B row per vertex at
// K = 16 (HBM3e access granule); K/4 lanes own one edge, each lane one
// float4 of both rows (16-byte loads/stores), the dot product is an
// xor-shuffle inside the lane group.  Edge arrays are SoA (u, v, r).  The
// latent matrix (197 MB at the Orkut shape) does not fit the 126 MB L2, so a
// step streams 12 B of edge + 4 x 64 B of random rows per edge from HBM:
// 268 B/edge algorithmic.  Each lane carries two edges per iteration to keep
// enough 64 B requests in flight.
//
// User-grouped layout (fr_sgd_group_by_user): the edges stable-sorted by u,
// i.e. Gardenia's CSR input order (one row of ratings per user), with every
// user's row cut into 64-edge pieces dealt over rounds of about one step's
// edges (so a hub's thousands of ratings are never all in flight at once:
// at most ~one piece of a user per round).  Each lane group then walks a
// contiguous segment, keeps L_u of the current run of
// equal u in registers (updated edge by edge, exactly the sequential order
// within the run) and adds L_u's net change back with one vector atomic when
// the run (or the segment) ends; only L_v is read and atomically updated per
// edge.  148 B/edge instead of 268 (12 B of edge + 2 x 64 B of L_v + the L_u
// read/update once per run).
#include <cub/cub.cuh>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "freeride_gpu.h"
#include "kernels/common.cuh"

namespace {

constexpr int kSgdThreads = 256;
constexpr int kSgdEpi = 2;  // edges per lane group per iteration (4 was measured slower: register-capped occupancy)
constexpr int kSgdConflictDiv = 8;  // in-flight edges <= V / 8
constexpr uint64_t kSgdPermMul = 2654435761ull;
// by-user step: L_u is handed back and re-read at least every kSgdRefresh
// edges of a run.  Two groups holding the same hub row (pieces of it in one
// step) would otherwise each walk it through a long run and add both full
// moves -- an overshoot that diverges once the factors grow (measured: NaN
// after ~40 epochs with whole-run holds); refreshing bounds it to a
// mini-batch of a few x kSgdRefresh edges, like the per-edge kernel's
// (16: 88.6 us per 2^21-edge step at the Orkut shape; 8: 94.7; whole runs: 82.4).
#ifndef SGD_REFRESH
#define SGD_REFRESH 16
#endif
constexpr int kSgdRefresh = SGD_REFRESH;

__device__ __forceinline__ int32_t sgd_vertex(uint64_t h, int32_t V) {
  const double x = static_cast<double>(h >> 11) * (1.0 / 9007199254740992.0);
  double t = static_cast<double>(V) * x;
  t = t * sqrt(x);
  int64_t v = static_cast<int64_t>(t);
  if (v >= V) v = V - 1;
  return static_cast<int32_t>((static_cast<uint64_t>(v) * kSgdPermMul) % static_cast<uint64_t>(V));
}

__global__ void sgd_edges_kernel(int32_t V, int64_t E, uint64_t seed, int32_t* __restrict__ u,
                                 int32_t* __restrict__ v, float* __restrict__ r) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < E;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t a = sgd_vertex(frk::splitmix64(seed ^ (2 * static_cast<uint64_t>(e))), V);
    const int32_t b = sgd_vertex(frk::splitmix64(seed ^ (2 * static_cast<uint64_t>(e) + 1)), V);
    u[e] = a;
    v[e] = b;
    const uint64_t hr = frk::splitmix64((seed * 0x2545F4914F6CDD1Dull) ^
                                        (static_cast<uint64_t>(a) * static_cast<uint64_t>(V) +
                                         static_cast<uint64_t>(b)));
    r[e] = static_cast<float>(1 + static_cast<int>(hr % 5));
  }
}

__global__ void sgd_init_kernel(int64_t n, float scale, uint64_t seed, float* __restrict__ L) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    L[i] = static_cast<float>(frk::splitmix64(seed ^ (0x4C4154ull << 40) ^ static_cast<uint64_t>(i)) >> 40) * scale;
}

template <int K>
struct Row {
  static constexpr int kLanes = K / 4;  // lanes per edge, one float4 each
};

template <int K>
__device__ __forceinline__ float group_sum(float x) {
#pragma unroll
  for (int o = Row<K>::kLanes >> 1; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ float dot4(float4 a, float4 b) {
  return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
}

// The update as deltas: L_u += du, L_v += dv, both from the values read.
// eta (err x - lam y) as (eta err) x - (eta lam) y: one FMUL + one FFMA per
// component instead of two FMULs and an FFMA (the products round differently
// from the oracle's order; parity is RMSE within 1e-3, not bitwise)
__device__ __forceinline__ void deltas(const float4& a, const float4& b, float err, float eta,
                                       float lam, float4& da, float4& db) {
  const float e = eta * err, l = eta * lam;
  da = make_float4(e * b.x - l * a.x, e * b.y - l * a.y, e * b.z - l * a.z, e * b.w - l * a.w);
  db = make_float4(e * a.x - l * b.x, e * a.y - l * b.y, e * a.z - l * b.z, e * a.w - l * b.w);
}

// Deltas land with 16-byte vector atomics (red.global.add.v4.f32, sm_90+):
// with ~1e5 edges in flight a hub vertex sees tens of concurrent updates,
// and plain Hogwild stores would drop all but one of them (measured: RMSE
// 0.25 above the sequential oracle after one epoch).  With atomic deltas
// every update lands; concurrent ones act like a small mini-batch on the hub.
__device__ __forceinline__ void apply(float4* p, const float4& d) { atomicAdd(p, d); }

// Each lane group handles edges g, g + G, g + 2G, ..., EPI of them per
// iteration (EPI x 2 latent-row loads in flight per lane), and the next
// iteration's (u, v, r) load while this iteration's rows are in flight.
// Register cap (SGD_MAXNREG): registers are allocated in units of 8 per
// thread, so four 256-thread CTAs at 64 fill the register file and leave no
// room for the stage's resident 1-warp dependency-wait kernel inside a
// bubble; at 56 they do.
#ifndef SGD_MAXNREG
#define SGD_MAXNREG 56
#endif
template <int K, int EPI = kSgdEpi>
__global__ void __launch_bounds__(kSgdThreads) __maxnreg__(K >= 16 ? SGD_MAXNREG : 64) sgd_step_kernel(
    const int32_t* __restrict__ us, const int32_t* __restrict__ vs, const float* __restrict__ rs,
    float* __restrict__ L, int64_t e0, int64_t e1, float eta, float lam) {
  constexpr int LN = Row<K>::kLanes;
  const int lane = threadIdx.x & 31, sub = lane % LN;
  const int64_t group = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / LN;
  const int64_t G = static_cast<int64_t>(gridDim.x) * blockDim.x / LN;
  float4* L4 = reinterpret_cast<float4*>(L);
  // Warp-uniform trip count (the group shuffles need every lane present);
  // lanes whose edge is past the end ride along predicated off.
  const int64_t warp_first = group - lane / LN;
  auto fetch = [&](int64_t base, int32_t* a, int32_t* b, float* q) {
#pragma unroll
    for (int j = 0; j < EPI; ++j) {
      const int64_t e = base + lane / LN + j * G;
      const bool ok = e < e1;
      a[j] = ok ? __ldg(&us[e]) : (j ? a[0] : 0);
      b[j] = ok ? __ldg(&vs[e]) : (j ? b[0] : 0);
      q[j] = ok ? __ldg(&rs[e]) : 0.0f;
    }
  };
  int32_t u[EPI], v[EPI];
  float r[EPI];
  int64_t ew = e0 + warp_first;
  if (ew < e1) fetch(ew, u, v, r);
  for (; ew < e1; ew += EPI * G) {
    float4 a[EPI], b[EPI];
#pragma unroll
    for (int j = 0; j < EPI; ++j) {
      a[j] = L4[static_cast<int64_t>(u[j]) * LN + sub];
      b[j] = L4[static_cast<int64_t>(v[j]) * LN + sub];
    }
    int32_t nu[EPI], nv[EPI];
    float nr[EPI];
    if (ew + EPI * G < e1) {
      fetch(ew + EPI * G, nu, nv, nr);
    } else {
#pragma unroll
      for (int j = 0; j < EPI; ++j) nu[j] = nv[j] = 0, nr[j] = 0.0f;
    }
#pragma unroll
    for (int j = 0; j < EPI; ++j) {
      const float err = r[j] - group_sum<K>(dot4(a[j], b[j]));
      if (ew + lane / LN + j * G < e1) {
        float4 da, db;
        deltas(a[j], b[j], err, eta, lam, da, db);
        apply(&L4[static_cast<int64_t>(u[j]) * LN + sub], da);
        apply(&L4[static_cast<int64_t>(v[j]) * LN + sub], db);
      }
    }
#pragma unroll
    for (int j = 0; j < EPI; ++j) u[j] = nu[j], v[j] = nv[j], r[j] = nr[j];
  }
}

// User-grouped step (K >= 16: lane sub of a group fetches the metadata of
// edge c + (sub % D) of each D-edge chunk and the group shares it through
// shuffles).  Group g owns edges [e0 + g seg, e0 + (g + 1) seg); slot j of the
// D-slot ring holds the L_v row of the chunk's j-th edge, re-issued for the
// next chunk as soon as it is consumed (D rows in flight per group); the
// metadata runs two chunks ahead of the rows.  A run start (u differs from
// the previous edge) flushes the held L_u delta and loads the new row (a
// dependent load, ~1.7 per segment at the Orkut shape).
template <int K, int D = 4>
__global__ void __maxnreg__(SGD_MAXNREG) sgd_user_kernel(
    const int32_t* __restrict__ us, const int32_t* __restrict__ vs, const float* __restrict__ rs,
    float* __restrict__ L, int64_t e0, int64_t e1, int64_t seg, float eta, float lam) {
  constexpr int LN = Row<K>::kLanes;
  static_assert(LN >= D, "grouped step needs K / 4 >= D lanes per group");
  const int lane = threadIdx.x & 31, sub = lane % LN, base = lane - sub;
  const int64_t group = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / LN;
  if (e0 + (group - lane / LN) * seg >= e1) return;  // whole warp past the end (warp-uniform)
  float4* L4 = reinterpret_cast<float4*>(L);
  const int64_t s0 = e0 + group * seg, s1 = std::min<int64_t>(e1, s0 + seg);
  // metadata of edge c + (sub % D): (u, v, r) for chunks c, c + D, c + 2D
  auto meta = [&](int64_t c, int32_t& mu, int32_t& mv, float& mr) {
    const int64_t e = c + (sub % D);
    const bool ok = e < s1;
    mu = ok ? __ldg(&us[e]) : -1;
    mv = ok ? __ldg(&vs[e]) : 0;
    mr = ok ? __ldg(&rs[e]) : 0.0f;
  };
  int32_t mu0, mv0, mu1, mv1, mu2, mv2;
  float mr0, mr1, mr2;
  meta(s0, mu0, mv0, mr0);
  meta(s0 + D, mu1, mv1, mr1);
  float4 b[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const int32_t v = __shfl_sync(0xffffffffu, mv0, base + j);
    b[j] = s0 + j < s1 ? L4[static_cast<int64_t>(v) * LN + sub] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), a0 = a;
  int32_t cu = -1, held = 0;
  for (int64_t c = s0; c < s0 + seg; c += D) {  // same trip count for every group of the warp
    meta(c + 2 * D, mu2, mv2, mr2);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int32_t u = __shfl_sync(0xffffffffu, mu0, base + j);
      const int32_t v = __shfl_sync(0xffffffffu, mv0, base + j);
      const float r = __shfl_sync(0xffffffffu, mr0, base + j);
      const int32_t nv = __shfl_sync(0xffffffffu, mv1, base + j);
      const bool ok = u >= 0;
      if (ok && (u != cu || held >= kSgdRefresh)) {
        // run start (or kSgdRefresh edges held): hand the held row's change
        // back and (re)load the row, picking up concurrent updates of it
        if (cu >= 0)
          apply(&L4[static_cast<int64_t>(cu) * LN + sub],
                make_float4(a.x - a0.x, a.y - a0.y, a.z - a0.z, a.w - a0.w));
        cu = u;
        a = L4[static_cast<int64_t>(u) * LN + sub];
        a0 = a;
        held = 0;
      }
      const float4 bj = b[j];
      const float err = r - group_sum<K>(dot4(a, bj));
      if (ok) {
        float4 da, db;
        deltas(a, bj, err, eta, lam, da, db);
        a.x += da.x; a.y += da.y; a.z += da.z; a.w += da.w;
        ++held;
        apply(&L4[static_cast<int64_t>(v) * LN + sub], db);
      }
      b[j] = c + D + j < s1 ? L4[static_cast<int64_t>(nv) * LN + sub] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    mu0 = mu1; mv0 = mv1; mr0 = mr1;
    mu1 = mu2; mv1 = mv2; mr1 = mr2;
  }
  // segment done: a programmatic dependent launch (the next step) may start
  asm volatile("griddepcontrol.launch_dependents;");
  if (cu >= 0)
    apply(&L4[static_cast<int64_t>(cu) * LN + sub], make_float4(a.x - a0.x, a.y - a0.y, a.z - a0.z, a.w - a0.w));
}

__global__ void sgd_gather_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ v,
                                  const float* __restrict__ r, int64_t E, int32_t* __restrict__ v2,
                                  float* __restrict__ r2) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < E;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t e = __ldg(&perm[i]);
    v2[i] = __ldg(&v[e]);
    r2[i] = __ldg(&r[e]);
  }
}

constexpr int64_t kSgdPiece = 64;  // edges per piece of a user's run (by-user layout)

__global__ void sgd_count_kernel(const int32_t* __restrict__ u, int64_t n, int32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&cnt[__ldg(&u[i])], 1);
}

// round of the edge at sorted position i: piece k of np pieces of its user's
// run goes to round (k R / np + h(u)) mod R -- distinct rounds while np <= R,
// users spread over the rounds by a hash (mirrors oracle/sidetasks.c)
__host__ __device__ __forceinline__ int32_t sgd_round(int32_t u, int64_t rank, int64_t deg, int32_t R) {
  const int64_t np = (deg + kSgdPiece - 1) / kSgdPiece, k = rank / kSgdPiece;
  const uint64_t h = frk::splitmix64(0x5347445250ull ^ static_cast<uint64_t>(u)) % static_cast<uint64_t>(R);
  return static_cast<int32_t>((static_cast<uint64_t>(k * R / np) + h) % static_cast<uint64_t>(R));
}

// item blocks of the by-user layout: ceil(V k 4 B / 64 MiB) ranges of v
constexpr int64_t kSgdBlockBytes = int64_t(64) << 20;
int32_t sgd_item_blocks(int32_t V, int32_t k) {
  const int64_t bytes = int64_t(V) * k * 4;
  return static_cast<int32_t>(std::max<int64_t>(1, (bytes + kSgdBlockBytes - 1) / kSgdBlockBytes));
}
__host__ __device__ __forceinline__ int32_t sgd_block_of(int32_t v, int32_t V, int32_t P) {
  return static_cast<int32_t>(static_cast<int64_t>(v) * P / V);
}

__global__ void sgd_block_key_kernel(const int32_t* __restrict__ v, int64_t n, int32_t V, int32_t P,
                                     int32_t* __restrict__ key) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    key[i] = sgd_block_of(__ldg(&v[i]), V, P);
}

// 1 where a (block, user) run starts (edges sorted by block, then u)
__global__ void sgd_run_flag_kernel(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t n,
                                    int32_t V, int32_t P, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    flag[i] = i == 0 || __ldg(&u[i]) != __ldg(&u[i - 1]) ||
              sgd_block_of(__ldg(&v[i]), V, P) != sgd_block_of(__ldg(&v[i - 1]), V, P);
}

__global__ void sgd_fill_kernel(int32_t* __restrict__ x, int64_t n, int32_t value) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] = value;
}

// rst[run] = first edge of the run (runs numbered by the inclusive scan of flags, from 1)
__global__ void sgd_run_start_kernel(const int32_t* __restrict__ flag, const int32_t* __restrict__ rid,
                                     int64_t n, int32_t* __restrict__ rst) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (flag[i]) rst[rid[i] - 1] = static_cast<int32_t>(i);
}

__global__ void sgd_round_key_kernel(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t n,
                                     int32_t V, int32_t P, const int32_t* __restrict__ rid,
                                     const int32_t* __restrict__ rst, int32_t R, int32_t* __restrict__ key) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t run = __ldg(&rid[i]) - 1, b = __ldg(&rst[run]), len = __ldg(&rst[run + 1]) - b;
    key[i] = sgd_block_of(__ldg(&v[i]), V, P) * R + sgd_round(__ldg(&u[i]), i - b, len, R);
  }
}

__global__ void sgd_gather3_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ u,
                                   const int32_t* __restrict__ v, const float* __restrict__ r, int64_t E,
                                   int32_t* __restrict__ u2, int32_t* __restrict__ v2, float* __restrict__ r2) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < E;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t e = __ldg(&perm[i]);
    u2[i] = __ldg(&u[e]);
    v2[i] = __ldg(&v[e]);
    r2[i] = __ldg(&r[e]);
  }
}

__global__ void sgd_check_ids_kernel(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t n,
                                     int32_t V, int32_t* __restrict__ bad) {
  int32_t k = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    k += (static_cast<uint32_t>(u[i]) >= static_cast<uint32_t>(V)) + (static_cast<uint32_t>(v[i]) >= static_cast<uint32_t>(V));
  if (k) atomicAdd(bad, k);
}

__global__ void sgd_iota_kernel(int32_t* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] = static_cast<int32_t>(i);
}

// K4: sum of squared errors over [e0, e1) into *acc (fp64).
template <int K>
__global__ void __launch_bounds__(kSgdThreads) sgd_sqerr_kernel(
    const int32_t* __restrict__ us, const int32_t* __restrict__ vs, const float* __restrict__ rs,
    const float* __restrict__ L, int64_t e0, int64_t e1, double* __restrict__ acc) {
  constexpr int LN = Row<K>::kLanes;
  __shared__ double red[kSgdThreads / 32];
  const int lane = threadIdx.x & 31, sub = lane % LN;
  const int64_t group = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / LN;
  const int64_t G = static_cast<int64_t>(gridDim.x) * blockDim.x / LN;
  const float4* L4 = reinterpret_cast<const float4*>(L);
  double s = 0.0;
  const int64_t warp_first = group - lane / LN;
  for (int64_t ew = e0 + warp_first; ew < e1; ew += G) {  // warp-uniform (shuffles)
    const int64_t e = ew + lane / LN;
    const bool ok = e < e1;
    const float4 a = __ldg(&L4[static_cast<int64_t>(ok ? __ldg(&us[e]) : 0) * LN + sub]);
    const float4 b = __ldg(&L4[static_cast<int64_t>(ok ? __ldg(&vs[e]) : 0) * LN + sub]);
    double d = static_cast<double>(a.x) * b.x + static_cast<double>(a.y) * b.y +
               static_cast<double>(a.z) * b.z + static_cast<double>(a.w) * b.w;
#pragma unroll
    for (int o = LN >> 1; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    const double err = (ok ? static_cast<double>(__ldg(&rs[e])) : 0.0) - d;
    if (sub == 0 && ok) s += err * err;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kSgdThreads / 32; ++w) t += red[w];
    atomicAdd(acc, t);
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

struct fr_sgd_problem {
  int32_t V = 0, K = 0;
  int64_t E = 0;
  int32_t* u = nullptr;
  int32_t* v = nullptr;
  float* r = nullptr;
  float* L = nullptr;
  double* acc = nullptr;
  int sms = 148;
  int max_sms = 0;  // fr_sgd_problem_set_max_sms (0 = all)
  int64_t grid_sms() const { return max_sms > 0 ? std::min(max_sms, sms) : sms; }
  bool grouped = false;  // edges stable-sorted by u (fr_sgd_group_by_user)
  bool overlap = false;  // fr_sgd_problem_set_overlap: consecutive steps may overlap (Hogwild)
  // Programmatic dependent launch is only safe behind another user step of
  // this problem: any other launch that writes (init, re-layout) or reads
  // (sqerr) the problem's buffers breaks the chain, so the next step runs
  // fully serialised behind it.
  mutable bool chained = false;
  mutable cudaStream_t chain_stream = nullptr;
  void break_chain() const { chained = false; }
  int64_t max_deg = 0;   // largest number of ratings touching one vertex (u or v side)
};

namespace {

// Hub cap: with F edges in flight a vertex of degree d sees ~F d / E
// concurrent updates, applied from the same stale row -- a mini-batch whose
// effective step grows with it.  Keep that <= kSgdHubConc for the hottest
// vertex (no effect at the Orkut shape: d / E = 8.5e-5 allows 1.9e5 edges in
// flight; a Zipf(1.3) item with a quarter of all ratings would otherwise
// take thousands of simultaneous updates and diverge).
constexpr int64_t kSgdHubConc = 16;
int64_t hub_cap(const fr_sgd_problem* p) {
  if (p->max_deg <= 0 || p->E <= 0) return INT64_MAX;
  return std::max<int64_t>(64, kSgdHubConc * p->E / p->max_deg);
}

// degree histogram of both endpoints -> p->max_deg (setup, synchronous)
cudaError_t measure_max_degree(fr_sgd_problem* p, cudaStream_t s) {
  p->max_deg = 0;
  if (p->E == 0) return cudaSuccess;
  int32_t *cnt = nullptr, *mx = nullptr;
  void* tmp = nullptr;
  size_t need = 0;
  cub::DeviceReduce::Max(nullptr, need, cnt, mx, p->V, s);
  cudaError_t e = cudaMalloc(&cnt, size_t(p->V) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&mx, sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&tmp, std::max<size_t>(need, 1));
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, size_t(p->V) * 4, s);
  if (e == cudaSuccess) {
    sgd_count_kernel<<<grid_for(p->E, 256, 16), 256, 0, s>>>(p->u, p->E, cnt);
    sgd_count_kernel<<<grid_for(p->E, 256, 16), 256, 0, s>>>(p->v, p->E, cnt);
    e = cub::DeviceReduce::Max(tmp, need, cnt, mx, p->V, s);
  }
  int32_t h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, mx, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  for (void* q : {static_cast<void*>(cnt), static_cast<void*>(mx), tmp})
    if (q) cudaFree(q);
  if (e == cudaSuccess) p->max_deg = h;
  return e;
}

template <int K>
void launch_step(fr_sgd_problem* p, int64_t a, int64_t b, float eta, float lam, cudaStream_t s) {
  // persistent-style grid: exactly the resident CTAs (no second partial wave)
  static const int per_sm = [] {
    // The random latent-row loads land in L1: with the max-shared carveout
    // the pipeline's GEMMs leave behind (28 KB of L1) the loads in flight per
    // SM are capped and a step is ~45 % slower.  Ask for the max-L1 split so
    // the SMs are reconfigured when the step's CTAs arrive.
    cudaFuncSetAttribute(sgd_step_kernel<K>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxL1);
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sgd_step_kernel<K>, kSgdThreads, 0);
    return std::max(1, n);
  }();
  // Conflict-sparse Hogwild: at most V / kSgdConflictDiv edges in flight, so
  // concurrent updates of one vertex stay rare on small graphs (RMSE parity
  // with the sequential order); the Orkut shape is far from this cap.
  static const int div = [] {
    const char* e = std::getenv("FR_SGD_CONFLICT_DIV");  // tuning hook
    return e ? std::max(1, std::atoi(e)) : kSgdConflictDiv;
  }();
  const int64_t groups = (b - a + kSgdEpi - 1) / kSgdEpi;
  const int64_t cap_groups = std::max<int64_t>(1, std::min(int64_t(p->V) / div, hub_cap(p)) / kSgdEpi);
  const int64_t want = (std::min(groups, cap_groups) * Row<K>::kLanes + kSgdThreads - 1) / kSgdThreads;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, p->grid_sms() * per_sm)));
  sgd_step_kernel<K><<<grid, kSgdThreads, 0, s>>>(p->u, p->v, p->r, p->L, a, b, eta, lam);
}

// grouped layout: contiguous segments, D rows in flight per group
template <int K>
void launch_user_step(fr_sgd_problem* p, int64_t a, int64_t b, float eta, float lam, cudaStream_t s) {
  constexpr int D = 4, LN = Row<K>::kLanes;
  static const int per_sm = [] {
    cudaFuncSetAttribute(sgd_user_kernel<K, D>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxL1);
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sgd_user_kernel<K, D>, kSgdThreads, 0);
    return std::max(1, n);
  }();
  static const int div = [] {
    const char* e = std::getenv("FR_SGD_CONFLICT_DIV");
    return e ? std::max(1, std::atoi(e)) : kSgdConflictDiv;
  }();
  const int64_t n = b - a;
  const int64_t cap_groups = std::max<int64_t>(1, std::min(int64_t(p->V) / div, hub_cap(p)) / D);
  const int64_t max_groups = p->grid_sms() * per_sm * kSgdThreads / LN;
  const int64_t groups = std::min({(n + D - 1) / D, cap_groups, max_groups});
  const int64_t seg = ((n + groups - 1) / groups + D - 1) / D * D;
  const int64_t used = (n + seg - 1) / seg;
  const int grid = static_cast<int>((used * LN + kSgdThreads - 1) / kSgdThreads);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kSgdThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  static const int overlap_env = [] {
    const char* e = std::getenv("FR_SGD_OVERLAP");  // A/B override: 0 / 1
    return e ? std::atoi(e) : -1;
  }();
  const bool want = overlap_env >= 0 ? overlap_env != 0 : p->overlap;
  cfg.numAttrs = (want && p->chained && p->chain_stream == s) ? 1 : 0;
  p->chained = true;
  p->chain_stream = s;
  cudaLaunchKernelEx(&cfg, sgd_user_kernel<K, D>, static_cast<const int32_t*>(p->u), static_cast<const int32_t*>(p->v),
                     static_cast<const float*>(p->r), p->L, a, b, seg, eta, lam);
}

template <int K>
void launch_sqerr(const fr_sgd_problem* p, int64_t a, int64_t b, double* acc, cudaStream_t s) {
  const int grid = grid_for((b - a) * Row<K>::kLanes, kSgdThreads, 8);
  sgd_sqerr_kernel<K><<<grid, kSgdThreads, 0, s>>>(p->u, p->v, p->r, p->L, a, b, acc);
}

bool rank_supported(int k) { return k == 4 || k == 8 || k == 16 || k == 32 || k == 64 || k == 128; }

}  // namespace

extern "C" {

int fr_sgd_problem_generate(int32_t V, int64_t E, int32_t k, uint64_t edge_seed, uint64_t init_seed,
                            void* stream, fr_sgd_problem** out) {
  if (!out) return frcapi::fail(FR_ERR_ARGUMENT, "null problem out");
  if (V < 1 || E < 0) return frcapi::fail(FR_ERR_VALIDATION, "V >= 1, E >= 0", "V");
  if (!rank_supported(k)) return frcapi::fail(FR_ERR_UNSUPPORTED, "rank must be 4, 8, 16, 32, 64 or 128");
  auto s = static_cast<cudaStream_t>(stream);
  auto* p = new fr_sgd_problem;
  p->V = V;
  p->E = E;
  p->K = k;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaMalloc(&p->u, std::max<int64_t>(E, 1) * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&p->v, std::max<int64_t>(E, 1) * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&p->r, std::max<int64_t>(E, 1) * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&p->L, static_cast<size_t>(V) * k * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&p->acc, sizeof(double));
  if (e != cudaSuccess) {
    for (void* q : {static_cast<void*>(p->u), static_cast<void*>(p->v), static_cast<void*>(p->r),
                    static_cast<void*>(p->L), static_cast<void*>(p->acc)})
      if (q) cudaFree(q);
    delete p;
    return frcapi::cuda_status(e, "sgd problem allocation");
  }
  if (E > 0) sgd_edges_kernel<<<grid_for(E, 256, 16), 256, 0, s>>>(V, E, edge_seed, p->u, p->v, p->r);
  FR_CUDA_LAUNCHED("sgd_edges");
  if (const cudaError_t me = measure_max_degree(p, s); me != cudaSuccess) {
    fr_sgd_problem_destroy(p);
    return frcapi::cuda_status(me, "sgd degree histogram");
  }
  *out = p;
  return fr_sgd_reinit(p, init_seed, stream);
}

int fr_sgd_problem_from_edges(int32_t V, int64_t E, int32_t k, const int32_t* u, const int32_t* v,
                              const float* r, uint64_t init_seed, void* stream, fr_sgd_problem** out) {
  if (!out) return frcapi::fail(FR_ERR_ARGUMENT, "null problem out");
  if (V < 1 || E < 0) return frcapi::fail(FR_ERR_VALIDATION, "V >= 1, E >= 0", "V");
  if (E > 0 && (!u || !v || !r)) return frcapi::fail(FR_ERR_ARGUMENT, "null edge arrays");
  if (!rank_supported(k)) return frcapi::fail(FR_ERR_UNSUPPORTED, "rank must be 4, 8, 16, 32, 64 or 128");
  auto s = static_cast<cudaStream_t>(stream);
  // allocate through the generator with no edges, then take the caller's
  fr_sgd_problem* p = nullptr;
  int rc = fr_sgd_problem_generate(V, 0, k, 0, init_seed, stream, &p);
  if (rc != FR_OK) return rc;
  p->E = E;
  cudaError_t e = cudaSuccess;
  if (E > 0) {
    for (void* q : {static_cast<void*>(p->u), static_cast<void*>(p->v), static_cast<void*>(p->r)}) cudaFree(q);
    p->u = p->v = nullptr;
    p->r = nullptr;
    e = cudaMalloc(&p->u, size_t(E) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&p->v, size_t(E) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&p->r, size_t(E) * 4);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p->u, u, size_t(E) * 4, cudaMemcpyDefault, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p->v, v, size_t(E) * 4, cudaMemcpyDefault, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p->r, r, size_t(E) * 4, cudaMemcpyDefault, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(p->acc, 0, sizeof(double), s);
  }
  if (e == cudaSuccess && E > 0) {  // every endpoint in [0, V): count the bad ones on the device
    int32_t* bad = nullptr;
    int32_t h_bad = 0;
    e = cudaMalloc(&bad, sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemsetAsync(bad, 0, sizeof(int32_t), s);
    if (e == cudaSuccess) {
      sgd_check_ids_kernel<<<grid_for(E, 256, 16), 256, 0, s>>>(p->u, p->v, E, V, bad);
      e = cudaMemcpyAsync(&h_bad, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (bad) cudaFree(bad);
    if (e == cudaSuccess && h_bad) {
      fr_sgd_problem_destroy(p);
      return frcapi::fail(FR_ERR_VALIDATION, std::to_string(h_bad) + " endpoints outside [0, V)", "edges");
    }
  }
  if (e == cudaSuccess) e = measure_max_degree(p, s);
  if (e != cudaSuccess) {
    fr_sgd_problem_destroy(p);
    return frcapi::cuda_status(e, "sgd problem from edges");
  }
  *out = p;
  return FR_OK;
}

int fr_sgd_problem_destroy(fr_sgd_problem* p) {
  if (!p) return FR_OK;
  for (void* q : {static_cast<void*>(p->u), static_cast<void*>(p->v), static_cast<void*>(p->r),
                  static_cast<void*>(p->L), static_cast<void*>(p->acc)})
    if (q) cudaFree(q);
  delete p;
  return FR_OK;
}

int fr_sgd_reinit(fr_sgd_problem* p, uint64_t init_seed, void* stream) {
  if (!p) return frcapi::fail(FR_ERR_ARGUMENT, "null problem");
  const int64_t n = static_cast<int64_t>(p->V) * p->K;
  const float scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(p->K))) * (1.0f / 16777216.0f);
  p->break_chain();
  sgd_init_kernel<<<grid_for(n, 256, 16), 256, 0, static_cast<cudaStream_t>(stream)>>>(n, scale, init_seed, p->L);
  FR_CUDA_LAUNCHED("sgd_init");
  return FR_OK;
}

int fr_sgd_step(fr_sgd_problem* p, int64_t e_begin, int64_t e_end, float eta, float lambda,
                void* stream) {
  if (!p) return frcapi::fail(FR_ERR_ARGUMENT, "null problem");
  if (e_begin < 0 || e_end > p->E || e_begin > e_end)
    return frcapi::fail(FR_ERR_VALIDATION, "edge range outside [0, E]", "edges");
  if (e_begin == e_end) return FR_OK;
  auto s = static_cast<cudaStream_t>(stream);
  if (p->grouped && p->K >= 16) {
    switch (p->K) {
      case 16: launch_user_step<16>(p, e_begin, e_end, eta, lambda, s); break;
      case 32: launch_user_step<32>(p, e_begin, e_end, eta, lambda, s); break;
      case 64: launch_user_step<64>(p, e_begin, e_end, eta, lambda, s); break;
      default: launch_user_step<128>(p, e_begin, e_end, eta, lambda, s); break;
    }
    FR_CUDA_LAUNCHED("sgd_user_step");
    return FR_OK;
  }
  p->break_chain();
  switch (p->K) {
    case 4: launch_step<4>(p, e_begin, e_end, eta, lambda, s); break;
    case 8: launch_step<8>(p, e_begin, e_end, eta, lambda, s); break;
    case 16: launch_step<16>(p, e_begin, e_end, eta, lambda, s); break;
    case 32: launch_step<32>(p, e_begin, e_end, eta, lambda, s); break;
    case 64: launch_step<64>(p, e_begin, e_end, eta, lambda, s); break;
    default: launch_step<128>(p, e_begin, e_end, eta, lambda, s); break;
  }
  FR_CUDA_LAUNCHED("sgd_step");
  return FR_OK;
}

int fr_sgd_group_by_user(fr_sgd_problem* p, int64_t window_edges, void* stream) {
  if (!p) return frcapi::fail(FR_ERR_ARGUMENT, "null problem");
  if (window_edges < 1) return frcapi::fail(FR_ERR_VALIDATION, "window_edges >= 1", "window_edges");
  if (p->grouped || p->E == 0) {
    p->grouped = true;
    return FR_OK;
  }
  if (p->E > INT32_MAX) return frcapi::fail(FR_ERR_VALIDATION, "grouping needs E < 2^31", "E");
  p->break_chain();
  auto s = static_cast<cudaStream_t>(stream);
  const int n = static_cast<int>(p->E);
  const int32_t P = sgd_item_blocks(p->V, p->K);
  const int32_t R = static_cast<int32_t>(
      std::min<int64_t>((p->E + window_edges - 1) / window_edges, std::max<int64_t>(1, (int64_t(1) << 30) / P)));
  auto bits_for = [](int64_t x) {
    int b = 1;
    while (b < 31 && (int64_t(1) << b) < x) ++b;
    return b;
  };
  int32_t *u2 = nullptr, *v2 = nullptr, *idx = nullptr, *perm = nullptr, *key = nullptr, *key2 = nullptr;
  int32_t *flag = nullptr, *rid = nullptr, *rst = nullptr;
  float* r2 = nullptr;
  void* tmp = nullptr;
  size_t need = 0, need2 = 0, need3 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, p->u, u2, idx, perm, n, 0, bits_for(p->V), s);
  cub::DeviceRadixSort::SortPairs(nullptr, need2, key, key2, idx, perm, n, 0, bits_for(int64_t(P) * R), s);
  cub::DeviceScan::InclusiveSum(nullptr, need3, flag, rid, n, s);
  need = std::max({need, need2, need3, size_t(1)});
  cudaError_t e = cudaSuccess;
  for (auto [q, bytes] : {std::pair<void**, size_t>{reinterpret_cast<void**>(&u2), size_t(n) * 4},
                          {reinterpret_cast<void**>(&v2), size_t(n) * 4},
                          {reinterpret_cast<void**>(&r2), size_t(n) * 4},
                          {reinterpret_cast<void**>(&idx), size_t(n) * 4},
                          {reinterpret_cast<void**>(&perm), size_t(n) * 4},
                          {reinterpret_cast<void**>(&key), size_t(n) * 4},
                          {reinterpret_cast<void**>(&key2), size_t(n) * 4},
                          {reinterpret_cast<void**>(&flag), size_t(n) * 4},
                          {reinterpret_cast<void**>(&rid), size_t(n) * 4},
                          {reinterpret_cast<void**>(&rst), size_t(n + 1) * 4},
                          {&tmp, need}})
    if (e == cudaSuccess) e = cudaMalloc(q, bytes);
  const int gn = grid_for(n, 256, 16);
  auto swap3 = [&] {  // (u2, v2, r2) -> the problem's arrays
    std::swap(p->u, u2);
    std::swap(p->v, v2);
    std::swap(p->r, r2);
  };
  auto sort_by_key = [&](int bits) {  // stable: (u, v, r) reordered by key
    sgd_iota_kernel<<<gn, 256, 0, s>>>(idx, n);
    cudaError_t x = cub::DeviceRadixSort::SortPairs(tmp, need, key, key2, idx, perm, n, 0, bits, s);
    if (x == cudaSuccess) {
      sgd_gather3_kernel<<<gn, 256, 0, s>>>(perm, p->u, p->v, p->r, n, u2, v2, r2);
      x = cudaGetLastError();
    }
    if (x == cudaSuccess) swap3();
    return x;
  };
  // 1. stable sort by u (LSD radix keeps the generated order within a user)
  if (e == cudaSuccess) {
    sgd_iota_kernel<<<gn, 256, 0, s>>>(idx, n);
    e = cub::DeviceRadixSort::SortPairs(tmp, need, p->u, u2, idx, perm, n, 0, bits_for(p->V), s);
  }
  if (e == cudaSuccess) {
    sgd_gather_kernel<<<gn, 256, 0, s>>>(perm, p->v, p->r, n, v2, r2);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) swap3();
  // 2. item blocks: stable by block of v, so each block's L_v rows (<= 64
  //    MiB) stay in L2 while its ratings stream by
  if (e == cudaSuccess && P > 1) {
    sgd_block_key_kernel<<<gn, 256, 0, s>>>(p->v, n, p->V, P, key);
    e = sort_by_key(bits_for(P));
  }
  // 3. rounds: each (block, user) run cut into kSgdPiece-edge pieces dealt
  //    over R rounds inside its block (stable by block x R + round)
  if (e == cudaSuccess && R > 1) {
    sgd_run_flag_kernel<<<gn, 256, 0, s>>>(p->u, p->v, n, p->V, P, flag);
    e = cub::DeviceScan::InclusiveSum(tmp, need, flag, rid, n, s);
    if (e == cudaSuccess) {
      sgd_fill_kernel<<<gn, 256, 0, s>>>(rst, int64_t(n) + 1, n);
      sgd_run_start_kernel<<<gn, 256, 0, s>>>(flag, rid, n, rst);
      sgd_round_key_kernel<<<gn, 256, 0, s>>>(p->u, p->v, n, p->V, P, rid, rst, R, key);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = sort_by_key(bits_for(int64_t(P) * R));
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  for (void* q : {static_cast<void*>(u2), static_cast<void*>(v2), static_cast<void*>(r2),
                  static_cast<void*>(idx), static_cast<void*>(perm), static_cast<void*>(key),
                  static_cast<void*>(key2), static_cast<void*>(flag), static_cast<void*>(rid),
                  static_cast<void*>(rst), tmp})
    if (q) cudaFree(q);
  if (e != cudaSuccess) return frcapi::cuda_status(e, "sgd group by user");
  p->grouped = true;
  return FR_OK;
}

int fr_sgd_problem_set_overlap(fr_sgd_problem* p, int32_t overlap) {
  if (!p) return frcapi::fail(FR_ERR_ARGUMENT, "null problem");
  p->overlap = overlap != 0;
  p->break_chain();
  return FR_OK;
}

int fr_sgd_problem_set_max_sms(fr_sgd_problem* p, int32_t sms) {
  if (!p) return frcapi::fail(FR_ERR_ARGUMENT, "null problem");
  if (sms < 0) return frcapi::fail(FR_ERR_VALIDATION, "sms must be >= 0", "sms");
  p->max_sms = sms;
  return FR_OK;
}

int fr_sgd_problem_set_kernel(fr_sgd_problem* p, int32_t by_user) {
  if (!p) return frcapi::fail(FR_ERR_ARGUMENT, "null problem");
  p->grouped = by_user != 0;
  return FR_OK;
}

int fr_sgd_sqerr(const fr_sgd_problem* p, int64_t e_begin, int64_t e_end, double* d_acc, void* stream) {
  if (!p || !d_acc) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (e_begin < 0 || e_end > p->E || e_begin > e_end)
    return frcapi::fail(FR_ERR_VALIDATION, "edge range outside [0, E]", "edges");
  if (e_begin == e_end) return FR_OK;
  auto s = static_cast<cudaStream_t>(stream);
  p->break_chain();
  switch (p->K) {
    case 4: launch_sqerr<4>(p, e_begin, e_end, d_acc, s); break;
    case 8: launch_sqerr<8>(p, e_begin, e_end, d_acc, s); break;
    case 16: launch_sqerr<16>(p, e_begin, e_end, d_acc, s); break;
    case 32: launch_sqerr<32>(p, e_begin, e_end, d_acc, s); break;
    case 64: launch_sqerr<64>(p, e_begin, e_end, d_acc, s); break;
    default: launch_sqerr<128>(p, e_begin, e_end, d_acc, s); break;
  }
  FR_CUDA_LAUNCHED("sgd_sqerr");
  return FR_OK;
}

int fr_sgd_rmse(const fr_sgd_problem* p, void* stream, double* rmse) {
  if (!p || !rmse) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  auto s = static_cast<cudaStream_t>(stream);
  FR_CUDA_TRY(cudaMemsetAsync(p->acc, 0, sizeof(double), s));
  const int rc = fr_sgd_sqerr(p, 0, p->E, p->acc, stream);
  if (rc != FR_OK) return rc;
  double sum = 0.0;
  FR_CUDA_TRY(cudaMemcpyAsync(&sum, p->acc, sizeof(double), cudaMemcpyDeviceToHost, s));
  FR_CUDA_TRY(cudaStreamSynchronize(s));
  *rmse = p->E > 0 ? std::sqrt(sum / static_cast<double>(p->E)) : 0.0;
  return FR_OK;
}

int fr_sgd_buffers(const fr_sgd_problem* p, const int32_t** u, const int32_t** v, const float** r,
                   float** L, int32_t* V, int64_t* E, int32_t* k) {
  if (!p) return frcapi::fail(FR_ERR_ARGUMENT, "null problem");
  if (u) *u = p->u;
  if (v) *v = p->v;
  if (r) *r = p->r;
  if (L) *L = p->L;
  if (V) *V = p->V;
  if (E) *E = p->E;
  if (k) *k = p->K;
  return FR_OK;
}

}  // extern "C"

// ------------------------------------------------------ built-in side task
// The rating graph is the task's input and is generated at CreateSideTask
// directly on the device (1.4 GB at the Orkut shape; uploading it inside a
// bubble would overrun it); InitSideTask (re)initialises the latent model,
// every RunNextStep processes the next `edges_per_step` edges (wrapping into
// the next epoch), StopSideTask keeps nothing but the input graph.
namespace {

struct SgdTask {
  fr_sgd_task_config cfg{};
  fr_sgd_problem* p = nullptr;
  int64_t cursor = 0, epochs = 0;
  int64_t launched = 0;   // steps since InitSideTask
  int64_t last_step = 0;  // total_epochs: the step that ended the last epoch (1-based)
};

int sgd_task_create(void* u) {
  auto* t = static_cast<SgdTask*>(u);
  if (t->p) return FR_OK;
  int rc = fr_sgd_problem_generate(t->cfg.V, t->cfg.E, t->cfg.k, t->cfg.edge_seed,
                                   t->cfg.init_seed, nullptr, &t->p);
  if (rc == FR_OK && t->cfg.layout == FR_SGD_LAYOUT_BY_USER) rc = fr_sgd_group_by_user(t->p, t->cfg.edges_per_step, nullptr);
  if (rc == FR_OK) FR_CUDA_TRY(cudaDeviceSynchronize());
  return rc;
}

int sgd_task_init(void* u, void* stream) {
  auto* t = static_cast<SgdTask*>(u);
  t->cursor = 0;
  t->epochs = 0;
  t->launched = 0;
  t->last_step = 0;
  return fr_sgd_reinit(t->p, t->cfg.init_seed, stream);
}

int sgd_task_step(void* u, void* stream) {
  auto* t = static_cast<SgdTask*>(u);
  int64_t left = t->cfg.edges_per_step;
  ++t->launched;
  const bool bounded = t->cfg.total_epochs > 0;
  while (left > 0 && !(bounded && t->epochs >= t->cfg.total_epochs)) {
    const int64_t n = std::min<int64_t>(left, t->p->E - t->cursor);
    const int rc = fr_sgd_step(t->p, t->cursor, t->cursor + n, t->cfg.eta, t->cfg.lambda, stream);
    if (rc != FR_OK) return rc;
    t->cursor += n;
    left -= n;
    if (t->cursor == t->p->E) {
      t->cursor = 0;
      t->epochs++;
      if (bounded && t->epochs == t->cfg.total_epochs) t->last_step = t->launched;
    }
  }
  return FR_OK;
}

int sgd_task_finished(void* u, int64_t done, int32_t* out) {
  auto* t = static_cast<SgdTask*>(u);
  *out = (t->cfg.total_steps > 0 && done >= t->cfg.total_steps) ||
         (t->last_step > 0 && done >= t->last_step);
  return FR_OK;
}

int sgd_task_sm_budget(void* u, int32_t sms) {
  return fr_sgd_problem_set_max_sms(static_cast<SgdTask*>(u)->p, sms);
}

void sgd_task_destroy(void* u) {
  auto* t = static_cast<SgdTask*>(u);
  cudaDeviceSynchronize();
  fr_sgd_problem_destroy(t->p);
  delete t;
}

}  // namespace

extern "C" {

int fr_sgd_task_create(const fr_sgd_task_config* c, fr_side_task_vtable* vt, void** user) {
  return fr_sgd_task_create_from_problem(c, nullptr, vt, user);
}

int fr_sgd_task_create_from_problem(const fr_sgd_task_config* c, fr_sgd_problem* problem,
                                    fr_side_task_vtable* vt, void** user) {
  if (!c || !vt || !user) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (c->layout != FR_SGD_LAYOUT_COO && c->layout != FR_SGD_LAYOUT_BY_USER)
    return frcapi::fail(FR_ERR_VALIDATION, "layout must be FR_SGD_LAYOUT_COO or FR_SGD_LAYOUT_BY_USER", "layout");
  if (c->edges_per_step < 1 || (problem ? problem->E : c->E) < 1)
    return frcapi::fail(FR_ERR_VALIDATION, "E and edges_per_step must be >= 1", "edges_per_step");
  auto* t = new SgdTask;
  t->cfg = *c;
  int rc = FR_OK;
  if (problem) {  // the caller's ratings: the task takes the problem over (sizes from it)
    t->p = problem;
    t->cfg.V = problem->V;
    t->cfg.E = problem->E;
    t->cfg.k = problem->K;
    if (c->layout == FR_SGD_LAYOUT_BY_USER) rc = fr_sgd_group_by_user(problem, c->edges_per_step, nullptr);
  } else {
    rc = sgd_task_create(t);
  }
  // the task's steps follow each other (Hogwild: a step may start while the
  // previous one's last segments drain)
  if (rc == FR_OK) rc = fr_sgd_problem_set_overlap(t->p, 1);
  if (rc != FR_OK) {
    delete t;
    return rc;
  }
  std::memset(vt, 0, sizeof(*vt));
  vt->carveout_hint = 0;
  vt->create = sgd_task_create;
  vt->init = sgd_task_init;
  vt->run_next_step = sgd_task_step;
  vt->finished = sgd_task_finished;
  vt->destroy = sgd_task_destroy;
  vt->set_sm_budget = sgd_task_sm_budget;
  vt->work_units_per_step = static_cast<double>(c->edges_per_step);  // edges
  *user = t;
  return FR_OK;
}

int fr_sgd_task_problem(void* user, fr_sgd_problem** p, int64_t* epochs_done) {
  auto* t = static_cast<SgdTask*>(user);
  if (!t) return frcapi::fail(FR_ERR_ARGUMENT, "null task");
  if (p) *p = t->p;
  if (epochs_done) *epochs_done = t->epochs;
  return FR_OK;
}

}  // extern "C"
