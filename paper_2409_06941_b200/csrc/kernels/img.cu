// K5: bilinear resize + integer watermark alpha-blend, one bounded step of
// the image side task.
//
// Arithmetic (bit-exact with oracle/sidetasks.c and cv2 INTER_LINEAR_EXACT):
//   per axis: src = (d + 0.5) * S/D - 0.5, i0 = floor, w1 = rne(frac * 256)
//   px  = ((row_a * (256-wy) + row_b * wy) + 2^15) >> 16, rows pre-mixed in x
//   out = (px * (255 - alpha) + wm * alpha + 127) / 255
// At exactly 2x every weight is 128, so px = (a + b + c + d + 2) >> 2.
//
// Fast path (sw = 2 dw, sh = 2 dh, dw % 16 == 0), B200-first:
//  * the watermark is a task constant, so InitSideTask "prepares" it once:
//    per pixel (w*a + 127) for R,G,B and (255 - a), packed into 16-bit lanes
//    and laid out group-transposed so each thread's 64 B are one perfectly
//    coalesced 16 B load per warp-lane (L2-resident, evict-last);
//  * persistent CTAs (3 per SM) with a 2-stage smem ring; one elected
//    thread streams each output row's two contiguous source rows in with a
//    TMA bulk copy (cp.async.bulk -> UBLKCP) completing on an mbarrier
//    (expect_tx), and bulk-stores the finished output row from smem;
//  * the math runs two 16-bit lanes per 32-bit register: PRMT unpacks and
//    aligns byte pairs, one IADD3 forms (a+b+c+d+2), one IMAD blends R and G
//    together (they share alpha), /255 is (t + 1 + (t>>8)) >> 8 done with two
//    PRMTs and an IADD3, B uses umulhi(t, 2^32/255 rounded up).  Under the
//    pipeline's power-capped SM clock the kernel must stay HBM-bound, so the
//    instruction count per byte is what this layout minimises.
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include <cuda/atomic>

#include "freeride_gpu.h"
#include "kernels/common.cuh"

namespace {

constexpr int kImgThreads = 256;
// 2-stage ring x 3 CTAs per SM (63 registers): three CTAs computing rows
// side by side issue ~1.5x more per cycle than 3 stages x 2 CTAs, which is
// what bounded the kernel at in-bubble (power-capped) clocks; measured 64-frame
// launches 6.9 vs 6.0 TB/s, 8-frame in-bubble steps 52 vs 60 us.
constexpr int kImgStages = 2;
constexpr int kImgCtasPerSm = 3;
constexpr uint32_t kLaneMask = 0x00FF00FFu;
constexpr uint32_t kDiv255 = 16843010u;  // ceil(2^32 / 255): umulhi(t, .) = t / 255, t < 65408

__device__ __forceinline__ uint32_t blend255(uint32_t px, uint32_t wmc, uint32_t alpha) {
  return (px * (255u - alpha) + wmc * alpha + 127u) / 255u;
}

// Prepared watermark: for output row y, 8-pixel group g and pair j (0..3),
// uint4 {rg(p), bna(p), rg(p+1), bna(p+1)} at ((y*4 + j) * groups + g), p = 8g + 2j,
// rg = (wR*a + 127) | (wG*a + 127) << 16, bna = (wB*a + 127) | (255 - a) << 16.
__global__ void img_prepare_wm_kernel(const uint8_t* __restrict__ wm, uint4* __restrict__ out,
                                      int dw, int dh) {
  const int groups = dw >> 3;
  const int64_t total = static_cast<int64_t>(dh) * groups * 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % groups);
    const int64_t yj = i / groups;
    const int j = static_cast<int>(yj % 4);
    const int64_t y = yj / 4;
    uint32_t v[4];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint8_t* px = wm + (y * dw + 8 * g + 2 * j + q) * 4;
      const uint32_t a = px[3];
      v[2 * q] = (px[0] * a + 127u) | ((px[1] * a + 127u) << 16);
      v[2 * q + 1] = (px[2] * a + 127u) | ((255u - a) << 16);
    }
    out[(y * 4 + j) * groups + g] = make_uint4(v[0], v[1], v[2], v[3]);
  }
}

// One thread's 8 output pixels: the two source rows' 48 B each (ra/rb at the
// group's offset), the 16 prepared-watermark words, 24 B written to po.
__device__ __forceinline__ void img_group8(const uint8_t* __restrict__ ra, const uint8_t* __restrict__ rb,
                                       const uint32_t (&wv)[16], uint8_t* po8, int g) {
  uint32_t va[12], vb[12];
  const uint4* pa = reinterpret_cast<const uint4*>(ra + 48 * g);
  const uint4* pb = reinterpret_cast<const uint4*>(rb + 48 * g);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint4 x = pa[i], z = pb[i];
    va[4 * i + 0] = x.x; va[4 * i + 1] = x.y; va[4 * i + 2] = x.z; va[4 * i + 3] = x.w;
    vb[4 * i + 0] = z.x; vb[4 * i + 1] = z.y; vb[4 * i + 2] = z.z; vb[4 * i + 3] = z.w;
  }
  // vertical sums in 16-bit lanes: ev = bytes (0,2), od = bytes (1,3)
  uint32_t ev[12], od[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    ev[i] = (va[i] & kLaneMask) + (vb[i] & kLaneMask);
    od[i] = __byte_perm(va[i], 0u, 0x4341) + __byte_perm(vb[i], 0u, 0x4341);
  }
  uint32_t rgb[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // pixel pair (2q, 2q+1) = source words 3q..3q+2
    const uint32_t e0 = ev[3 * q], e1 = ev[3 * q + 1], e2 = ev[3 * q + 2];
    const uint32_t o0 = od[3 * q], o1 = od[3 * q + 1], o2 = od[3 * q + 2];
    uint32_t rg[2], bb;
    rg[0] = __byte_perm(e0, o0, 0x5410) + __byte_perm(o0, e1, 0x5432) + 0x00020002u;  // R0|G0
    rg[1] = __byte_perm(e1, o1, 0x7632) + __byte_perm(o2, e2, 0x7610) + 0x00020002u;  // R1|G1
    bb = __byte_perm(e0, e2, 0x5432) + __byte_perm(o1, o2, 0x7610) + 0x00020002u;     // B0|B1
    rg[0] = (rg[0] >> 2) & kLaneMask;
    rg[1] = (rg[1] >> 2) & kLaneMask;
    bb = (bb >> 2) & kLaneMask;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t wrg = wv[4 * q + 2 * j], wbna = wv[4 * q + 2 * j + 1];
      const uint32_t na = wbna >> 16;
      const uint32_t t = rg[j] * na + wrg;  // R,G lanes share alpha
      const uint32_t u = t + __byte_perm(t, 0u, 0x4341) + 0x00010001u;
      const uint32_t qrg = __byte_perm(u, 0u, 0x4341);  // (t + 1 + (t>>8)) >> 8 per lane
      const uint32_t b = j ? (bb >> 16) : (bb & 0xFFFFu);
      const uint32_t qb = __umulhi(b * na + (wbna & 0xFFFFu), kDiv255);
      rgb[2 * q + j] = __byte_perm(qrg, qb, 0x0420);  // R G B _
    }
  }
  uint2* po = reinterpret_cast<uint2*>(po8);
  po[0] = make_uint2(__byte_perm(rgb[0], rgb[1], 0x4210), __byte_perm(rgb[1], rgb[2], 0x5421));
  po[1] = make_uint2(__byte_perm(rgb[2], rgb[3], 0x6542), __byte_perm(rgb[4], rgb[5], 0x4210));
  po[2] = make_uint2(__byte_perm(rgb[5], rgb[6], 0x5421), __byte_perm(rgb[6], rgb[7], 0x6542));
    }

// ---- Math variant 1 (dot-product form; the default)
// The 2x2 sums come straight out of IDP.4A (dp4a): one dp4a sums the two
// bytes of a channel that lie in one source word, with weight 64, so
// 64 * (a + b + c + d + 2) < 2^16 carries floor((sum + 2) / 4) in its byte 1
// and zeros in bytes 2-3 -- the shift and the lane packing become one PRMT.
// A pixel pair (12 source bytes per row, words w0 w1 w2) gives channels
//   p0: R = w0.b0 + w0.b3, G = w0.b1 + w1.b0, B = w0.b2 + w1.b1
//   p1: R = w1.b2 + w2.b1, G = w1.b3 + w2.b2, B = w2.b0 + w2.b3
// (the cross-word pairs gathered into one word by a PRMT per row first),
// blended in three 16-bit-lane words X = [R0, B0] (alpha of p0),
// Z = [B1, G1] (p1) and Y = [G0, R1] (one IMAD per lane).  Prepared
// watermark: 5 words per pair {wX, wY, wZ, 255 - a0, 255 - a1}, wc = w*a + 127
// in the matching lane, group-transposed [y][5][groups] (uint4) like variant 0.
constexpr int kWmVecs1 = 5;  // uint4 per 8-pixel group
constexpr int kWsPipes = 3;  // producer/consumer pipelines per CTA of the warp-specialised kernel

__global__ void img_prepare_wm1_kernel(const uint8_t* __restrict__ wm, uint4* __restrict__ out,
                                       int dw, int dh) {
  const int groups = dw >> 3;
  const int64_t total = static_cast<int64_t>(dh) * groups;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(i % groups);
    const int64_t y = i / groups;
    uint32_t v[4 * kWmVecs1];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint8_t* p0 = wm + (y * dw + 8 * g + 2 * q) * 4;
      const uint8_t* p1 = p0 + 4;
      const uint32_t a0 = p0[3], a1 = p1[3];
      const auto wc = [](uint32_t w, uint32_t a) { return w * a + 127u; };
      v[5 * q + 0] = wc(p0[0], a0) | (wc(p0[2], a0) << 16);  // R0 | B0
      v[5 * q + 1] = wc(p0[1], a0) | (wc(p1[0], a1) << 16);  // G0 | R1
      v[5 * q + 2] = wc(p1[2], a1) | (wc(p1[1], a1) << 16);  // B1 | G1
      v[5 * q + 3] = 255u - a0;
      v[5 * q + 4] = 255u - a1;
    }
#pragma unroll
    for (int k = 0; k < kWmVecs1; ++k)
      out[(y * kWmVecs1 + k) * groups + g] = make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  }
}

__device__ __forceinline__ uint32_t dp4(uint32_t a, uint32_t w, uint32_t c) {
  return static_cast<uint32_t>(__dp4a(a, w, c));
}

// floor(t / 255) per 16-bit lane, t < 65408: (t + 1 + (t >> 8)) >> 8, the
// quotient left in bytes 1 and 3
__device__ __forceinline__ uint32_t div255_lanes(uint32_t t) {
  return t + __byte_perm(t, 0u, 0x4341) + 0x00010001u;
}

template <bool GLOBAL_OUT = false>
__device__ __forceinline__ void img_group8_dp(const uint8_t* __restrict__ ra, const uint8_t* __restrict__ rb,
                                          const uint32_t (&wv)[4 * kWmVecs1], uint8_t* po8, int g) {
  uint32_t va[12], vb[12];
  const uint4* pa = reinterpret_cast<const uint4*>(ra + 48 * g);
  const uint4* pb = reinterpret_cast<const uint4*>(rb + 48 * g);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint4 x = pa[i], z = pb[i];
    va[4 * i + 0] = x.x; va[4 * i + 1] = x.y; va[4 * i + 2] = x.z; va[4 * i + 3] = x.w;
    vb[4 * i + 0] = z.x; vb[4 * i + 1] = z.y; vb[4 * i + 2] = z.z; vb[4 * i + 3] = z.w;
  }
  constexpr uint32_t kW03 = 0x40000040u, kW02 = 0x00400040u, kW13 = 0x40004000u, kBias = 128u;
  uint32_t uX[4], uY[4], uZ[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t a0 = va[3 * q], a1 = va[3 * q + 1], a2 = va[3 * q + 2];
    const uint32_t b0 = vb[3 * q], b1 = vb[3 * q + 1], b2 = vb[3 * q + 2];
    const uint32_t ga = __byte_perm(a0, a1, 0x5421), gb = __byte_perm(b0, b1, 0x5421);  // G0 B0 G1 B1
    const uint32_t ha = __byte_perm(a1, a2, 0x6532), hb = __byte_perm(b1, b2, 0x6532);  // R2 G2 R3 G3
    const uint32_t sR0 = dp4(a0, kW03, dp4(b0, kW03, kBias));
    const uint32_t sG0 = dp4(ga, kW02, dp4(gb, kW02, kBias));
    const uint32_t sB0 = dp4(ga, kW13, dp4(gb, kW13, kBias));
    const uint32_t sR1 = dp4(ha, kW02, dp4(hb, kW02, kBias));
    const uint32_t sG1 = dp4(ha, kW13, dp4(hb, kW13, kBias));
    const uint32_t sB1 = dp4(a2, kW03, dp4(b2, kW03, kBias));
    const uint32_t wX = wv[5 * q], wY = wv[5 * q + 1], wZ = wv[5 * q + 2];
    const uint32_t na0 = wv[5 * q + 3], na1 = wv[5 * q + 4];
    const uint32_t X = __byte_perm(sR0, sB0, 0x6521);      // [R0, B0] lanes
    const uint32_t Z = __byte_perm(sB1, sG1, 0x6521);      // [B1, G1]
    const uint32_t Ylo = __byte_perm(sG0, 0u, 0x4441);     // [G0, 0]
    const uint32_t Yhi = __byte_perm(sR1, 0u, 0x4144);     // [0, R1]
    uX[q] = div255_lanes(X * na0 + wX);
    uZ[q] = div255_lanes(Z * na1 + wZ);
    uY[q] = div255_lanes(Yhi * na1 + (Ylo * na0 + wY));
  }
  uint32_t o[6];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int q = 2 * h;
    const uint32_t A0 = __byte_perm(uX[q], uY[q], 0x7351);          // R0 G0 B0 R1
    const uint32_t A1 = __byte_perm(uX[q + 1], uY[q + 1], 0x7351);  // R2 G2 B2 R3
    o[3 * h + 0] = A0;
    o[3 * h + 1] = __byte_perm(uZ[q], A1, 0x5413);      // G1 B1 R2 G2
    o[3 * h + 2] = __byte_perm(A1, uZ[q + 1], 0x5732);  // B2 R3 G3 B3
  }
  uint2* po = reinterpret_cast<uint2*>(po8);
  if constexpr (GLOBAL_OUT) {  // straight to HBM, evict-first (st.global.cs)
    __stcs(po + 0, make_uint2(o[0], o[1]));
    __stcs(po + 1, make_uint2(o[2], o[3]));
    __stcs(po + 2, make_uint2(o[4], o[5]));
  } else {
    po[0] = make_uint2(o[0], o[1]);
    po[1] = make_uint2(o[2], o[3]);
    po[2] = make_uint2(o[4], o[5]);
  }
}

// Rows are handed out dynamically (one atomicAdd per row by the elected
// thread) rather than statically strided: in a pipeline bubble some SMs may
// be unavailable (the stage's dependency-wait kernel, an NCCL receive, the
// tail of the previous GEMM), and with a static split the CTAs that could
// not become resident would run their whole share as a serial tail.  The
// last CTA to exit re-arms the counters for the next launch on the stream.
//
// PREEMPT (imperative interface): before taking a row the elected thread
// reads the stop word (gpu scope); once it reaches `token` no further row is
// taken, the rows already in the smem ring finish, and the CTA exits.  Rows
// are taken from a per-launch count t (counters[4]) as row (base + t) mod
// rows, base = counters[0], at most `budget` per launch, so one launch can
// loop over the batch several times; the last CTA out advances base by the
// rows taken, so the next launch resumes at the first untaken row, and adds
// them to counters[2..3] (every taken row is completed before exit).
template <int S, bool PREEMPT, int CPS, int MATH>
__global__ void __launch_bounds__(kImgThreads, CPS)
    img_resize2x_wm_tma(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                        const uint4* __restrict__ wmp, int dw, int dh, uint32_t rows,
                        uint32_t* __restrict__ counters, const uint32_t* __restrict__ stop_word,
                        uint32_t token, uint32_t budget, uint32_t /*fpu: rows are claimed one by one*/) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t row_of[S], y_of[S], next_of[S];
  const uint32_t src_row = 6u * static_cast<uint32_t>(dw);  // one source row, RGB
  const uint32_t out_row = 3u * static_cast<uint32_t>(dw);
  const uint32_t a_src = (2u * src_row + 127u) & ~127u;
  const uint32_t a_out = (out_row + 127u) & ~127u;
  const uint32_t stage_bytes = a_src + a_out;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);

  const int tid = threadIdx.x;
  const int groups = dw >> 3;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) frk::mbar_init(&full[s], 1);
    frk::fence_mbar_init();
  }

  uint64_t pol_stream = 0;
  if (tid == 0) pol_stream = frk::policy_evict_first();
  // Elected thread: grab the next row for stage s and start its TMA load.
  auto grab = [&](int s, uint32_t r) {
    row_of[s] = r;
    if (r >= rows) return;
    const uint32_t img = r / static_cast<uint32_t>(dh);
    const uint32_t y = r - img * static_cast<uint32_t>(dh);
    y_of[s] = y;
    frk::mbar_arrive_expect_tx(&full[s], 2u * src_row);
    frk::bulk_g2s(smem + s * stage_bytes,
                  src + (static_cast<uint64_t>(img) * 2 * dh + 2 * y) * src_row, 2u * src_row,
                  &full[s], pol_stream);
  };
  const uint32_t base = PREEMPT ? counters[0] : 0u;  // advanced only after this launch
  auto take = [&]() -> uint32_t {
    if (!PREEMPT) return atomicAdd(&counters[0], 1u);
    if (frk::ld_relaxed_gpu(stop_word) >= token) return rows;  // paused: no new row
    const uint32_t t = atomicAdd(&counters[4], 1u);
    if (t >= budget) return rows;
    const uint32_t r = base + t;  // base < rows, t < budget < 2^31
    return r % rows;
  };
  if (tid == 0)
    for (int s = 0; s < S; ++s) grab(s, take());
  __syncthreads();

  uint32_t k = 0;
  bool triggered = false;
  for (;; ++k) {
    const int s = static_cast<int>(k % S);
    const uint32_t row = row_of[s];  // written >= S-1 barriers ago (or before the first)
    if (row >= rows) break;          // rows are grabbed in increasing order: all done
    const uint32_t y = y_of[s];
    // the elected thread's next row: the atomic's round trip overlaps this
    // row's compute instead of delaying the refill after the barrier
    const uint32_t next_row = tid == 0 ? take() : 0u;
    if (tid == 0) next_of[s] = next_row;  // read after this row's barrier; rewritten S rows later
    uint8_t* st = smem + s * stage_bytes;
    const uint8_t* ra = st;
    const uint8_t* rb = st + src_row;
    uint8_t* orow = st + a_src;
    for (int g = tid; g < groups; g += kImgThreads) {
      // watermark first (L2): its latency overlaps the wait for the rows
      constexpr int kVecs = MATH == 1 ? kWmVecs1 : 4;
      uint32_t wv[4 * kVecs];
      const uint4* pw = wmp + (y * static_cast<uint32_t>(kVecs * groups) + static_cast<uint32_t>(g));
#pragma unroll
      for (int j = 0; j < kVecs; ++j) {
        const uint4 x = __ldg(pw + j * groups);
        wv[4 * j + 0] = x.x; wv[4 * j + 1] = x.y; wv[4 * j + 2] = x.z; wv[4 * j + 3] = x.w;
      }
      frk::mbar_wait(&full[s], (k / S) & 1u);
      if constexpr (MATH == 1)
        img_group8_dp(ra, rb, wv, orow + 24 * g, g);
      else
        img_group8(ra, rb, wv, orow + 24 * g, g);
    }
    frk::fence_proxy_async_smem();
    // Before anyone writes the next stage's output buffer, the bulk store
    // that last read it (issued S-1 rows ago) must have drained.
    if (tid == 0 && k + 1 >= S) frk::bulk_wait_read<S - 2>();
    __syncthreads();
    if (!PREEMPT && !triggered && next_of[s] >= rows) {
      // this CTA takes no further row: let a programmatic dependent launch
      // (the next step on the stream) start its CTAs on the SMs we free
      asm volatile("griddepcontrol.launch_dependents;");
      triggered = true;
    }
    if (tid == 0) {
      frk::bulk_s2g(dst + static_cast<uint64_t>(row) * out_row, orow, out_row, pol_stream);
      frk::bulk_commit();
      grab(s, next_row);
    }
  }
  if (tid == 0) {
    frk::bulk_wait<0>();
    if (PREEMPT) atomicAdd(reinterpret_cast<unsigned long long*>(counters + 2), k);
    __threadfence();
    if (atomicAdd(&counters[1], 1u) == gridDim.x - 1) {  // last CTA out re-arms
      if (PREEMPT) {
        const uint32_t taken = min(atomicAdd(&counters[4], 0u), budget);
        counters[0] = static_cast<uint32_t>((static_cast<uint64_t>(base) + taken) % rows);
        counters[4] = 0;
      } else {
        counters[0] = 0;
      }
      counters[1] = 0;
    }
  }
}

// Warp-specialised variant (the default exact-2x kernel).  The per-row CTA
// barrier of img_resize2x_wm_tma held every warp to the slowest one each row
// (36 % of the stall samples at a 16-SM budget once the dp4a math had cut
// the issue count).  Here no consumer warp waits for another:
//  * one producer warp (one lane) claims rows, one ahead (the claim's
//    global-atomic round trip overlaps the previous copy), and streams each
//    row's two source rows into one of S stages with a TMA bulk copy;
//  * it publishes the row id on meta[s] before the copy lands, so consumers
//    issue their watermark loads (L2) while the copy is in flight, then wait
//    on full[s] for the data;
//  * 8 consumer warps compute and store straight from registers to HBM
//    (st.global.cs, 24 B per thread, 768 B per warp), so the whole smem
//    budget is input (3 pipelines x 3 stages x 23 KB per SM); each warp
//    releases the stage on empty[s] (one arrival per warp) and moves on;
//  * a CTA holds G such pipelines (G x 9 warps, G x S stages).  Default G = 1:
//    up to 3 CTAs per SM, and an SM budget of n launches 3n CTAs, which the
//    block scheduler spreads one per SM (measured the better use of a ΔT
//    budget); G = 3 (FR_IMG_PIPES=3) packs one CTA per SM;
//  * claims are units of up to 16 frames' row y (fpu), so the consumers'
//    watermark stays in registers across a unit.
constexpr int kWsWarps = kImgThreads / 32 + 1;  // per pipeline: 8 consumers + the producer

// CHAOS (tests only, FR_IMG_CHAOS=1): pseudo-random nanosleeps at every
// hand-off (producer before publishing a row, consumers after taking one and
// before releasing the stage), so any ordering the mbarriers did not enforce
// would show up as a wrong byte.
__device__ __forceinline__ void chaos_sleep(uint32_t a, uint32_t b) {
  const uint32_t h = static_cast<uint32_t>(frk::splitmix64((static_cast<uint64_t>(a) << 32) ^ b ^ clock()));
  __nanosleep(h & 4095u);
}

template <int S, bool PREEMPT, int G, bool CHAOS = false>
__global__ void __launch_bounds__(G * kWsWarps * 32, kWsPipes / G)
    img_resize2x_wm_ws(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                       const uint4* __restrict__ wmp, int dw, int dh, uint32_t rows,
                       uint32_t* __restrict__ counters, const uint32_t* __restrict__ stop_word,
                       uint32_t token, uint32_t budget, uint32_t fpu) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t row_of_all[G][S], y_of_all[G][S];
  constexpr int kWarps = kWsWarps - 1;  // consumer warps; warp kWarps of a pipeline is its producer
  const uint32_t src_row = 6u * static_cast<uint32_t>(dw);  // one source row, RGB
  const uint32_t out_row = 3u * static_cast<uint32_t>(dw);
  const uint32_t stage_bytes = (2u * src_row + 127u) & ~127u;
  const int tid = threadIdx.x, lane = tid & 31;
  const int pipe = tid / (kWsWarps * 32), warp = (tid >> 5) - pipe * kWsWarps;
  const int ctid = tid - pipe * kWsWarps * 32;  // thread index within the pipeline
  uint8_t* stages = smem + static_cast<uint32_t>(pipe) * S * stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G * S * stage_bytes) + pipe * 3 * S;
  uint64_t* meta = full + S;
  uint64_t* empty = meta + S;
  uint32_t* row_of = row_of_all[pipe];
  uint32_t* y_of = y_of_all[pipe];  // the row's output y: consumers skip the division
  const int groups = dw >> 3;

  if (ctid == 0) {
    for (int s = 0; s < S; ++s) {
      frk::mbar_init(&full[s], 1);
      frk::mbar_init(&meta[s], 1);
      frk::mbar_init(&empty[s], kWarps);
    }
    frk::fence_mbar_init();
  }
  __syncthreads();

  if (warp == kWarps) {  // ---- producer
    if (lane == 0) {
      const uint64_t pol_stream = frk::policy_evict_first();
      const uint32_t base = PREEMPT ? counters[0] : 0u;  // advanced only after this launch
      // Claims are units of `fpu` rows with the same y in consecutive frames
      // (frames f0 .. f0+fpu-1), loaded into consecutive stages: consumers
      // keep that y's watermark in registers across them.  PREEMPT counts in
      // units too: base = counters[0] and the budget are units, unit
      // (base + t) mod units is the t-th taken.
      const uint32_t units = rows / fpu;
      auto take = [&]() -> uint32_t {
        if (!PREEMPT) return atomicAdd(&counters[0], 1u);
        if (frk::ld_relaxed_gpu(stop_word) >= token) return units;  // paused: no new unit
        const uint32_t t = atomicAdd(&counters[4], 1u);
        if (t >= budget) return units;
        return (base + t) % units;  // base < units, t < budget < 2^31
      };
      uint32_t unit = take(), next = take(), j = 0, done = 0;
      uint32_t fb = unit / static_cast<uint32_t>(dh), y = unit - fb * static_cast<uint32_t>(dh);
      for (uint32_t k = 0;; ++k) {
        const int s = static_cast<int>(k % S);
        if (k >= S) frk::mbar_wait(&empty[s], ((k / S) - 1) & 1u);
        if (CHAOS) chaos_sleep(blockIdx.x * 64 + pipe, k);
        if (unit >= units) {  // no more rows: this pipeline's consumers leave at this stage
          row_of[s] = rows;
          frk::mbar_arrive(&meta[s]);
          if (!PREEMPT) asm volatile("griddepcontrol.launch_dependents;");
          break;
        }
        const uint32_t img = fb * fpu + j;
        const uint32_t r = img * static_cast<uint32_t>(dh) + y;
        row_of[s] = r;
        y_of[s] = y;
        frk::mbar_arrive(&meta[s]);
        ++done;
        frk::mbar_arrive_expect_tx(&full[s], 2u * src_row);
        frk::bulk_g2s(stages + s * stage_bytes,
                      src + (static_cast<uint64_t>(img) * 2 * dh + 2 * y) * src_row, 2u * src_row,
                      &full[s], pol_stream);
        if (++j == fpu) {  // next unit (claimed one ahead: its round trip overlapped these copies)
          j = 0;
          unit = next;
          fb = unit / static_cast<uint32_t>(dh);
          y = unit - fb * static_cast<uint32_t>(dh);
          if (unit < units) next = take();
        }
      }
      if (PREEMPT) {
        // every claimed row was loaded (a claim after the stop returns no row)
        atomicAdd(reinterpret_cast<unsigned long long*>(counters + 2), done);
      }
    }
  } else {  // ---- consumers
    uint32_t wc[4 * kWmVecs1];  // the cached watermark of y == last_y (one group per thread)
    uint32_t last_y = 0xFFFFFFFFu;
    for (uint32_t k = 0;; ++k) {
      const int s = static_cast<int>(k % S);
      const uint32_t ph = (k / S) & 1u;
      frk::mbar_wait(&meta[s], ph);
      if (CHAOS) chaos_sleep(blockIdx.x * 64 + warp + 16 * pipe, k);
      const uint32_t row = row_of[s];
      if (row >= rows) break;
      const uint32_t y = y_of[s];
      const uint8_t* ra = stages + s * stage_bytes;
      const uint8_t* rb = ra + src_row;
      uint8_t* orow = dst + static_cast<uint64_t>(row) * out_row;
      bool waited = false;
      if (groups <= kImgThreads) {
        // one group per thread: the watermark stays in registers while the
        // producer's units keep y (consecutive frames, same output row)
        if (y != last_y && ctid < groups) {
          const uint4* pw = wmp + (y * static_cast<uint32_t>(kWmVecs1 * groups) + static_cast<uint32_t>(ctid));
#pragma unroll
          for (int j = 0; j < kWmVecs1; ++j) {
            const uint4 x = __ldg(pw + j * groups);
            wc[4 * j + 0] = x.x; wc[4 * j + 1] = x.y; wc[4 * j + 2] = x.z; wc[4 * j + 3] = x.w;
          }
        }
        last_y = y;
        frk::mbar_wait(&full[s], ph);
        waited = true;
        if (ctid < groups) img_group8_dp<true>(ra, rb, wc, orow + 24 * ctid, ctid);
      } else {
        for (int g = ctid; g < groups; g += kImgThreads) {  // wide rows: > 1 group per thread
          // watermark first (L2): its latency overlaps the copy still in flight
          uint32_t wv[4 * kWmVecs1];
          const uint4* pw = wmp + (y * static_cast<uint32_t>(kWmVecs1 * groups) + static_cast<uint32_t>(g));
#pragma unroll
          for (int j = 0; j < kWmVecs1; ++j) {
            const uint4 x = __ldg(pw + j * groups);
            wv[4 * j + 0] = x.x; wv[4 * j + 1] = x.y; wv[4 * j + 2] = x.z; wv[4 * j + 3] = x.w;
          }
          if (!waited) {
            frk::mbar_wait(&full[s], ph);
            waited = true;
          }
          img_group8_dp<true>(ra, rb, wv, orow + 24 * g, g);
        }
      }
      if (!waited) frk::mbar_wait(&full[s], ph);  // lanes with no group still release in order
      if (CHAOS) chaos_sleep(blockIdx.x * 64 + warp + 16 * pipe, k + 0x10000u);
      __syncwarp();
      if (lane == 0) frk::mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&counters[1], 1u) == gridDim.x - 1) {  // last CTA out re-arms
      if (PREEMPT) {
        const uint32_t base = counters[0];
        const uint32_t taken = min(atomicAdd(&counters[4], 0u), budget);
        counters[0] = static_cast<uint32_t>((static_cast<uint64_t>(base) + taken) % (rows / fpu));
        counters[4] = 0;
      } else {
        counters[0] = 0;
      }
      counters[1] = 0;
    }
  }
}

// General shapes: one thread per output pixel, coefficient tables from the
// plan (built on the host with the oracle's double-precision rule).
__global__ void img_resize_wm_general(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                      const uint8_t* __restrict__ wm,
                                      const int32_t* __restrict__ tab, int sw, int sh, int dw,
                                      int dh, int64_t total) {
  const int32_t* x0 = tab;
  const int32_t* x1 = tab + dw;
  const int32_t* xw = tab + 2 * dw;
  const int32_t* y0 = tab + 3 * dw;
  const int32_t* y1 = y0 + dh;
  const int32_t* yw = y0 + 2 * dh;
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < total;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t img = p / (static_cast<int64_t>(dw) * dh);
    const int64_t rem = p - img * dw * dh;
    const int y = static_cast<int>(rem / dw), x = static_cast<int>(rem % dw);
    const uint8_t* base = src + img * static_cast<int64_t>(sw) * sh * 3;
    const uint8_t* ra = base + static_cast<int64_t>(y0[y]) * sw * 3;
    const uint8_t* rb = base + static_cast<int64_t>(y1[y]) * sw * 3;
    const int a = x0[x] * 3, b = x1[x] * 3;
    const int32_t wx1 = xw[x], wx0 = 256 - wx1, wy1 = yw[y], wy0 = 256 - wy1;
    const uint8_t* w = wm + (static_cast<int64_t>(y) * dw + x) * 4;
    const uint32_t alpha = w[3];
    uint8_t* o = dst + p * 3;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int32_t ha = ra[a + c] * wx0 + ra[b + c] * wx1;
      const int32_t hb = rb[a + c] * wx0 + rb[b + c] * wx1;
      const uint32_t px = static_cast<uint32_t>((ha * wy0 + hb * wy1 + (1 << 15)) >> 16);
      o[c] = static_cast<uint8_t>(blend255(px, w[c], alpha));
    }
  }
}

__global__ void img_generate_kernel(uint8_t* __restrict__ dst, int64_t total_px, int w, int h,
                                    int ch, uint64_t seed, int first) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < total_px;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t hw = static_cast<int64_t>(h) * w;
    const int64_t i = p / hw + first;
    const int64_t rem = p % hw;
    const int64_t y = rem / w, x = rem % w;
    const uint64_t r = frk::splitmix64(seed ^ static_cast<uint64_t>((i * h + y) * w + x));
    for (int c = 0; c < ch; ++c) {
      const uint32_t g = static_cast<uint32_t>(x + 2 * y + 37 * i + 85 * c);
      dst[p * ch + c] = static_cast<uint8_t>((g + ((r >> (8 * c)) & 0x3f)) & 0xff);
    }
  }
}

__global__ void img_watermark_kernel(uint32_t* __restrict__ wm, int64_t n, uint64_t seed) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    wm[p] = static_cast<uint32_t>(
        frk::splitmix64(seed ^ (0x5741544552ull << 24) ^ static_cast<uint64_t>(p)));
}

// Host restatement of the oracle's coefficient rule (orc_img_coeffs).
void axis_coeffs(int S, int D, int32_t* i0, int32_t* i1, int32_t* w1) {
  const double scale = static_cast<double>(S) / static_cast<double>(D);
  for (int d = 0; d < D; ++d) {
    double f = (static_cast<double>(d) + 0.5) * scale - 0.5;
    const double fl = std::floor(f);
    int lo = static_cast<int>(fl);
    f -= fl;
    if (lo < 0) {
      lo = 0;
      f = 0.0;
    }
    if (lo >= S - 1) {
      lo = S - 1;
      f = 0.0;
    }
    i0[d] = lo;
    i1[d] = lo + 1 < S ? lo + 1 : S - 1;
    w1[d] = static_cast<int32_t>(std::nearbyint(f * 256.0));
  }
}

int grid_for(int64_t work, int threads, int per_sm) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (work + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(sms) * per_sm)));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

constexpr uint32_t kImgCtrSlots = 64;

namespace {
using ImgKernel = void (*)(const uint8_t*, uint8_t*, const uint4*, int, int, uint32_t, uint32_t*,
                           const uint32_t*, uint32_t, uint32_t, uint32_t);
template <bool PREEMPT>
ImgKernel img_kernel(int stages, int math, bool ws, int pipes, bool chaos = false) {
  if (ws && chaos) return img_resize2x_wm_ws<3, PREEMPT, 1, true>;
  if (ws) return pipes == 1 ? img_resize2x_wm_ws<3, PREEMPT, 1> : img_resize2x_wm_ws<3, PREEMPT, kWsPipes>;
  if (math == 1)
    return stages == 2 ? img_resize2x_wm_tma<2, PREEMPT, 3, 1> : img_resize2x_wm_tma<3, PREEMPT, 2, 1>;
  return stages == 2 ? img_resize2x_wm_tma<2, PREEMPT, 3, 0> : img_resize2x_wm_tma<3, PREEMPT, 2, 0>;
}
}  // namespace

struct fr_img_plan {
  int sw = 0, sh = 0, dw = 0, dh = 0;
  int stages = kImgStages, ctas_per_sm = kImgCtasPerSm;  // TMA path pipeline shape
  int path = FR_IMG_PATH_GENERAL;
  int math = 1;  // exact-2x math variant: 1 = dp4a sums (default), 0 = 16-bit lane sums (FR_IMG_MATH=0)
  bool ws = true;  // warp-specialised kernel (default); FR_IMG_CFG=bar|3x2: the per-row-barrier kernel
  // pipelines per CTA: 1 (default) = one-pipeline CTAs, up to 3 per SM, an SM
  // budget of n launching 3n of them (spread one per SM over 3n SMs while
  // 3n <= 148); FR_IMG_PIPES=3: one 3-pipeline CTA per SM, n CTAs on n SMs.
  // Spread CTAs harvest ~40 % more pixels at the same pipeline ΔT
  // (gpurun_out/r2s_ctrl_pipes.log).
  int pipes = 1;
  bool chaos = false;  // FR_IMG_CHAOS=1 (tests): the ws kernel with random sleeps at every hand-off
  int32_t* d_tab = nullptr;
  void* d_wm = nullptr;  // plan-owned prepared watermark for fr_img_resize_watermark
  uint32_t* d_ctr = nullptr;  // dynamic row scheduler {next row, CTAs done} x kImgCtrSlots; one stream at a time
  mutable uint32_t launches = 0;  // TMA launches so far: slot = launches % kImgCtrSlots
  bool overlap = false;           // fr_img_plan_set_overlap: consecutive launches may overlap
  // A launch is a programmatic dependent only directly behind another
  // exact-2x step of this plan on the same stream (nothing else of the plan
  // in between): the watermark preparation, a preemptible launch or a new
  // overlap setting break the chain, so the next step is fully serialised
  // behind whatever produced its inputs.
  mutable bool chained = false;
  mutable cudaStream_t chain_stream = nullptr;
  int smem = 0;
  int sms = 0;
  int max_sms = 0;  // fr_img_plan_set_max_sms: grid sized for this many SMs (0 = all)
  int64_t grid_sms() const { return max_sms > 0 ? std::min(max_sms, sms) : sms; }
  int block() const { return ws ? pipes * kWsWarps * 32 : kImgThreads; }
  size_t prepared_bytes() const {
    if (path != FR_IMG_PATH_TMA_2X) return static_cast<size_t>(dw) * dh * 4;
    return static_cast<size_t>(dw) * dh * (math == 1 ? 2 * kWmVecs1 : 8);
  }
};

namespace {
// rows per claimed unit of a preemptible launch over n frames (fixed by n,
// so every launch of one workload counts its cursor in the same unit)
uint32_t preemptible_fpu(const fr_img_plan* plan, int32_t n) {
  if (!plan->ws) return 1;  // the round-1 kernel claims single rows
  return n % 4 == 0 ? 4u : n % 2 == 0 ? 2u : 1u;
}
}  // namespace

extern "C" {

int fr_img_plan_create(int32_t sw, int32_t sh, int32_t dw, int32_t dh, fr_img_plan** out) {
  if (!out) return frcapi::fail(FR_ERR_ARGUMENT, "null plan out");
  if (sw < 1 || sh < 1 || dw < 1 || dh < 1)
    return frcapi::fail(FR_ERR_VALIDATION, "image sizes must be >= 1", "image.shape");
  auto* plan = new fr_img_plan;
  plan->sw = sw;
  plan->sh = sh;
  plan->dw = dw;
  plan->dh = dh;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&plan->sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) {
    delete plan;
    return frcapi::cuda_status(e, "cudaGetDevice");
  }
  const bool two_x = sw == 2 * dw && sh == 2 * dh && dw % 16 == 0;
  if (two_x) {
    auto al = [](int x) { return (x + 127) & ~127; };
    if (const char* e = std::getenv("FR_IMG_CFG")) {  // tuning hook: "bar" | "3x2" (barrier kernel)
      if (std::string(e) == "3x2") plan->stages = 3, plan->ctas_per_sm = 2;
      if (std::string(e) == "bar" || std::string(e) == "3x2") plan->ws = false;
    }
    if (const char* m = std::getenv("FR_IMG_MATH")) plan->math = std::atoi(m) == 0 ? 0 : 1;
    if (plan->math == 0) plan->ws = false;  // the warp-decoupled kernel has the dp4a math only
    if (const char* e = std::getenv("FR_IMG_PIPES")) plan->pipes = std::atoi(e) == kWsPipes ? kWsPipes : 1;
    if (const char* e = std::getenv("FR_IMG_CHAOS")) plan->chaos = std::atoi(e) != 0;
    if (plan->chaos) plan->pipes = 1;
    if (plan->ws) plan->stages = 3, plan->ctas_per_sm = kWsPipes / plan->pipes;
    plan->smem = plan->ws ? plan->pipes * plan->stages * (al(12 * dw) + 24)
                          : plan->stages * (al(12 * dw) + al(3 * dw)) + plan->stages * 8;
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (plan->smem <= optin) {
      for (const void* fn : {reinterpret_cast<const void*>(img_kernel<false>(plan->stages, plan->math, plan->ws, plan->pipes, plan->chaos)),
                             reinterpret_cast<const void*>(img_kernel<true>(plan->stages, plan->math, plan->ws, plan->pipes, plan->chaos))}) {
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, plan->smem);
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                   cudaSharedmemCarveoutMaxShared);
      }
      if (e != cudaSuccess) {
        delete plan;
        return frcapi::cuda_status(e, "cudaFuncSetAttribute(img_resize2x_wm_tma)");
      }
      plan->path = FR_IMG_PATH_TMA_2X;
    }
  }
  if (plan->path == FR_IMG_PATH_GENERAL) {
    std::vector<int32_t> tab(3 * static_cast<size_t>(dw) + 3 * static_cast<size_t>(dh));
    axis_coeffs(sw, dw, tab.data(), tab.data() + dw, tab.data() + 2 * dw);
    axis_coeffs(sh, dh, tab.data() + 3 * dw, tab.data() + 3 * dw + dh, tab.data() + 3 * dw + 2 * dh);
    e = cudaMalloc(&plan->d_tab, tab.size() * sizeof(int32_t));
    if (e == cudaSuccess)
      e = cudaMemcpy(plan->d_tab, tab.data(), tab.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) e = cudaMalloc(&plan->d_wm, plan->prepared_bytes());
  if (e == cudaSuccess) e = cudaMalloc(&plan->d_ctr, 2 * kImgCtrSlots * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(plan->d_ctr, 0, 2 * kImgCtrSlots * sizeof(uint32_t));
  if (e != cudaSuccess) {
    if (plan->d_tab) cudaFree(plan->d_tab);
    if (plan->d_wm) cudaFree(plan->d_wm);
    if (plan->d_ctr) cudaFree(plan->d_ctr);
    delete plan;
    return frcapi::cuda_status(e, "image plan setup");
  }
  *out = plan;
  return FR_OK;
}

int fr_img_plan_set_overlap(fr_img_plan* plan, int32_t overlap) {
  if (!plan) return frcapi::fail(FR_ERR_ARGUMENT, "null plan");
  plan->overlap = overlap != 0;
  plan->chained = false;
  return FR_OK;
}

int fr_img_plan_set_max_sms(fr_img_plan* plan, int32_t sms) {
  if (!plan) return frcapi::fail(FR_ERR_ARGUMENT, "null plan");
  if (sms < 0) return frcapi::fail(FR_ERR_VALIDATION, "sms must be >= 0", "sms");
  plan->max_sms = sms;
  return FR_OK;
}

int fr_img_plan_destroy(fr_img_plan* plan) {
  if (!plan) return FR_OK;
  if (plan->d_tab) cudaFree(plan->d_tab);
  if (plan->d_wm) cudaFree(plan->d_wm);
  if (plan->d_ctr) cudaFree(plan->d_ctr);
  delete plan;
  return FR_OK;
}

int fr_img_plan_path(const fr_img_plan* plan, int32_t* path) {
  if (!plan || !path) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  *path = plan->path;
  return FR_OK;
}

int fr_img_prepared_bytes(const fr_img_plan* plan, int64_t* bytes) {
  if (!plan || !bytes) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  *bytes = static_cast<int64_t>(plan->prepared_bytes());
  return FR_OK;
}

int fr_img_prepare_watermark(const fr_img_plan* plan, const uint8_t* wm_rgba, void* prepared,
                             void* stream) {
  if (!plan || !wm_rgba || !prepared) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  auto s = static_cast<cudaStream_t>(stream);
  plan->chained = false;
  if (plan->path == FR_IMG_PATH_TMA_2X) {
    if (!aligned16(prepared)) return frcapi::fail(FR_ERR_UNSUPPORTED, "prepared watermark must be 16-byte aligned");
    const int64_t groups = static_cast<int64_t>(plan->dh) * (plan->dw >> 3);
    if (plan->math == 1)
      img_prepare_wm1_kernel<<<grid_for(groups, 256, 8), 256, 0, s>>>(
          wm_rgba, static_cast<uint4*>(prepared), plan->dw, plan->dh);
    else
      img_prepare_wm_kernel<<<grid_for(groups * 4, 256, 8), 256, 0, s>>>(
          wm_rgba, static_cast<uint4*>(prepared), plan->dw, plan->dh);
  } else {
    FR_CUDA_TRY(cudaMemcpyAsync(prepared, wm_rgba, plan->prepared_bytes(), cudaMemcpyDeviceToDevice, s));
  }
  FR_CUDA_LAUNCHED("img_prepare_watermark");
  return FR_OK;
}

int fr_img_resize_watermark_prepared(const fr_img_plan* plan, const uint8_t* src, uint8_t* dst,
                                     const void* prepared, int32_t n, void* stream) {
  if (!plan || (n > 0 && (!src || !dst || !prepared))) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (n < 0) return frcapi::fail(FR_ERR_VALIDATION, "n must be >= 0", "n");
  if (n == 0) return FR_OK;
  auto s = static_cast<cudaStream_t>(stream);
  if (plan->path == FR_IMG_PATH_TMA_2X) {
    if (!aligned16(src) || !aligned16(dst) || !aligned16(prepared))
      return frcapi::fail(FR_ERR_UNSUPPORTED, "TMA path needs 16-byte aligned buffers");
    const int64_t rows = static_cast<int64_t>(n) * plan->dh;
    if (rows >= (int64_t{1} << 31)) return frcapi::fail(FR_ERR_UNSUPPORTED, "too many rows in one step");
    const int grid = static_cast<int>(std::min<int64_t>(rows, plan->grid_sms() * plan->ctas_per_sm));
    const ImgKernel k = img_kernel<false>(plan->stages, plan->math, plan->ws, plan->pipes, plan->chaos);
    // Consecutive steps overlap their tail and head (programmatic dependent
    // launch: a launch's CTAs start once every CTA of the previous one took
    // its last row).  Steps touch different frames; the row counters rotate
    // through kImgCtrSlots slots, so overlapping launches never share one.
    uint32_t* ctr = plan->d_ctr + 2 * (plan->launches++ % kImgCtrSlots);
    static const int pdl_env = [] {
      const char* e = std::getenv("FR_IMG_PDL");  // experiment override: 0 / 1
      return e ? std::atoi(e) : -1;
    }();
    const bool pdl = (pdl_env >= 0 ? pdl_env != 0 : plan->overlap) && plan->chained && plan->chain_stream == s;
    plan->chained = true;
    plan->chain_stream = s;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(plan->block());
    cfg.dynamicSmemBytes = plan->smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    // frames per claimed unit (same output row in consecutive frames: the
    // watermark is loaded once per unit): the largest of 16/8/4/2 that divides
    // the launch's frames and still leaves >= 8 units per CTA (load balance)
    uint32_t fpu = 1;
    for (uint32_t f : {16u, 8u, 4u, 2u})
      if (n % static_cast<int32_t>(f) == 0 && rows / f >= 8 * static_cast<int64_t>(grid)) {
        fpu = f;
        break;
      }
    FR_CUDA_TRY(cudaLaunchKernelEx(&cfg, k, src, dst, static_cast<const uint4*>(prepared), plan->dw, plan->dh,
                                   static_cast<uint32_t>(rows), ctr, static_cast<const uint32_t*>(nullptr), 0u, 0u,
                                   plan->ws ? fpu : 1u));
  } else {
    const int64_t total = static_cast<int64_t>(n) * plan->dw * plan->dh;
    img_resize_wm_general<<<grid_for(total, 256, 8), 256, 0, s>>>(
        src, dst, static_cast<const uint8_t*>(prepared), plan->d_tab, plan->sw, plan->sh, plan->dw,
        plan->dh, total);
  }
  FR_CUDA_LAUNCHED("img_resize_watermark");
  return FR_OK;
}

int fr_img_preemptible_unit_rows(const fr_img_plan* plan, int32_t n, int32_t* rows) {
  if (!plan || !rows) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  *rows = static_cast<int32_t>(preemptible_fpu(plan, n));
  return FR_OK;
}

int fr_img_resize_watermark_preemptible(const fr_img_plan* plan, const uint8_t* src, uint8_t* dst,
                                        const void* prepared, int32_t n, uint32_t* counters,
                                        int64_t max_rows, const fr_preempt* preempt, void* stream) {
  if (!plan || !counters || (n > 0 && (!src || !dst || !prepared)))
    return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (plan->path != FR_IMG_PATH_TMA_2X)
    return frcapi::fail(FR_ERR_UNSUPPORTED, "preemptible path needs the exact-2x TMA plan");
  if (n < 0) return frcapi::fail(FR_ERR_VALIDATION, "n must be >= 0", "n");
  if (n == 0) return FR_OK;
  if (!aligned16(src) || !aligned16(dst) || !aligned16(prepared) ||
      (reinterpret_cast<uintptr_t>(counters) & 7u))
    return frcapi::fail(FR_ERR_UNSUPPORTED, "TMA path needs 16-byte aligned buffers");
  const int64_t rows = static_cast<int64_t>(n) * plan->dh;
  if (rows >= (int64_t{1} << 31)) return frcapi::fail(FR_ERR_UNSUPPORTED, "too many rows in one launch");
  if (max_rows < 0 || max_rows >= (int64_t{1} << 31))
    return frcapi::fail(FR_ERR_VALIDATION, "max_rows in [0, 2^31)", "max_rows");
  if (max_rows == 0) return FR_OK;
  const int grid = static_cast<int>(std::min<int64_t>(max_rows, plan->grid_sms() * plan->ctas_per_sm));
  // no preempt: a stop word that never fires (counters[5] stays 0 < token)
  const uint32_t* word = preempt && preempt->stop_word ? preempt->stop_word : counters + 5;
  const uint32_t token = preempt && preempt->stop_word ? preempt->token : 0xFFFFFFFFu;
  const ImgKernel k = img_kernel<true>(plan->stages, plan->math, plan->ws, plan->pipes, plan->chaos);
  plan->chained = false;
  // units of fpu frames (the ws kernel; fixed by n alone, so every launch of
  // a workload counts its cursor in the same unit): max_rows is taken in
  // whole units
  const uint32_t fpu = preemptible_fpu(plan, n);
  if (max_rows < fpu) return FR_OK;
  k<<<grid, plan->block(), plan->smem, static_cast<cudaStream_t>(stream)>>>(
      src, dst, static_cast<const uint4*>(prepared), plan->dw, plan->dh, static_cast<uint32_t>(rows),
      counters, word, token, static_cast<uint32_t>(max_rows / fpu), fpu);
  FR_CUDA_LAUNCHED("img_resize_watermark_preemptible");
  return FR_OK;
}

int fr_img_resize_watermark(const fr_img_plan* plan, const uint8_t* src, uint8_t* dst,
                            const uint8_t* wm, int32_t n, void* stream) {
  if (!plan || (n > 0 && (!src || !dst || !wm))) return frcapi::fail(FR_ERR_ARGUMENT, "null argument");
  if (n < 0) return frcapi::fail(FR_ERR_VALIDATION, "n must be >= 0", "n");
  if (n == 0) return FR_OK;
  if (plan->path == FR_IMG_PATH_TMA_2X && (!aligned16(src) || !aligned16(dst)))
    return frcapi::fail(FR_ERR_UNSUPPORTED, "TMA path needs 16-byte aligned buffers");
  const int rc = fr_img_prepare_watermark(plan, wm, plan->d_wm, stream);
  if (rc != FR_OK) return rc;
  return fr_img_resize_watermark_prepared(plan, src, dst, plan->d_wm, n, stream);
}

int fr_img_generate(uint8_t* dst, int32_t n, int32_t w, int32_t h, int32_t ch, uint64_t seed,
                    int32_t first, void* stream) {
  if (n < 0 || w < 1 || h < 1 || ch < 1 || ch > 8)
    return frcapi::fail(FR_ERR_VALIDATION, "bad image generator shape", "image.shape");
  const int64_t total = static_cast<int64_t>(n) * w * h;
  if (total == 0) return FR_OK;
  img_generate_kernel<<<grid_for(total, 256, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      dst, total, w, h, ch, seed, first);
  FR_CUDA_LAUNCHED("img_generate");
  return FR_OK;
}

int fr_img_generate_watermark(uint8_t* wm, int32_t w, int32_t h, uint64_t seed, void* stream) {
  if (w < 1 || h < 1) return frcapi::fail(FR_ERR_VALIDATION, "bad watermark shape", "watermark.shape");
  if (reinterpret_cast<uintptr_t>(wm) & 3u) return frcapi::fail(FR_ERR_UNSUPPORTED, "watermark must be 4-byte aligned");
  const int64_t n = static_cast<int64_t>(w) * h;
  img_watermark_kernel<<<grid_for(n, 256, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<uint32_t*>(wm), n, seed);
  FR_CUDA_LAUNCHED("img_generate_watermark");
  return FR_OK;
}

}  // extern "C"
