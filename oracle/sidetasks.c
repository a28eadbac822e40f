/* ORACLE / TEST INFRASTRUCTURE ONLY.  See sidetasks.h for provenance.
 *
 * Every function here is the CPU statement of a side-task step the product
 * runs as an sm_100a kernel (paper_2409_06941_b200/csrc/kernels/).  The
 * generators are counter-based (splitmix64 of a per-element counter) so the
 * CPU and GPU produce identical inputs independently; integer paths are
 * bit-exact targets, floating paths carry the north-star tolerances.
 */
#include "sidetasks.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

static int nth(int n) { return n > 0 ? n : omp_get_max_threads(); }

uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* ------------------------------------------------------------------ images */
/* pixel (i,y,x,c) = gradient (x + 2y + 37i + 85c) + 6 bits of noise */
void orc_img_generate(uint8_t* dst, int n, int w, int h, int ch, uint64_t seed, int first,
                      int nthreads) {
#pragma omp parallel for num_threads(nth(nthreads)) schedule(static)
  for (int64_t row = 0; row < (int64_t)n * h; ++row) {
    const int64_t i = row / h + first;
    const int64_t y = row % h;
    uint8_t* out = dst + row * (int64_t)w * ch;
    for (int64_t x = 0; x < w; ++x) {
      const uint64_t r = orc_splitmix64(seed ^ (uint64_t)((i * h + y) * w + x));
      for (int c = 0; c < ch; ++c) {
        const uint32_t g = (uint32_t)(x + 2 * y + 37 * i + 85 * c);
        out[x * ch + c] = (uint8_t)((g + ((r >> (8 * c)) & 0x3f)) & 0xff);
      }
    }
  }
}

/* RGBA watermark: colour noise, alpha uniform in [0,255] */
void orc_img_generate_watermark(uint8_t* wm, int w, int h, uint64_t seed, int nthreads) {
#pragma omp parallel for num_threads(nth(nthreads)) schedule(static)
  for (int64_t p = 0; p < (int64_t)w * h; ++p) {
    const uint64_t r = orc_splitmix64(seed ^ (0x5741544552ull << 24) ^ (uint64_t)p);
    wm[4 * p + 0] = (uint8_t)(r);
    wm[4 * p + 1] = (uint8_t)(r >> 8);
    wm[4 * p + 2] = (uint8_t)(r >> 16);
    wm[4 * p + 3] = (uint8_t)(r >> 24);
  }
}

/* cv2.resize(..., INTER_LINEAR_EXACT) coefficient rule for one axis:
 * src = (d + 0.5) * (S/D) - 0.5 in double, i0 = floor(src), w1 = round-half-
 * even(frac * 256) in 8-bit fixed point; clamp to the border with w1 = 0. */
void orc_img_coeffs(int S, int D, int32_t* idx0, int32_t* idx1, int32_t* w1) {
  const double scale = (double)S / (double)D;
  for (int d = 0; d < D; ++d) {
    double f = ((double)d + 0.5) * scale - 0.5;
    double fl = floor(f);
    int i0 = (int)fl;
    f -= fl;
    if (i0 < 0) {
      i0 = 0;
      f = 0.0;
    }
    if (i0 >= S - 1) {
      i0 = S - 1;
      f = 0.0;
    }
    idx0[d] = i0;
    idx1[d] = i0 + 1 < S ? i0 + 1 : S - 1;
    w1[d] = (int32_t)nearbyint(f * 256.0);
  }
}

void orc_img_resize_watermark(const uint8_t* src, uint8_t* dst, const uint8_t* wm, int n,
                              int sw, int sh, int dw, int dh, int nthreads) {
  int32_t* x0 = malloc(sizeof(int32_t) * dw);
  int32_t* x1 = malloc(sizeof(int32_t) * dw);
  int32_t* xw = malloc(sizeof(int32_t) * dw);
  int32_t* y0 = malloc(sizeof(int32_t) * dh);
  int32_t* y1 = malloc(sizeof(int32_t) * dh);
  int32_t* yw = malloc(sizeof(int32_t) * dh);
  orc_img_coeffs(sw, dw, x0, x1, xw);
  orc_img_coeffs(sh, dh, y0, y1, yw);
#pragma omp parallel for num_threads(nth(nthreads)) schedule(static)
  for (int64_t row = 0; row < (int64_t)n * dh; ++row) {
    const int64_t i = row / dh;
    const int y = (int)(row % dh);
    const uint8_t* img = src + i * (int64_t)sw * sh * 3;
    const uint8_t* ra = img + (int64_t)y0[y] * sw * 3;
    const uint8_t* rb = img + (int64_t)y1[y] * sw * 3;
    const int32_t wy1 = yw[y], wy0 = 256 - yw[y];
    uint8_t* out = dst + row * (int64_t)dw * 3;
    const uint8_t* wrow = wm + (int64_t)y * dw * 4;
    for (int x = 0; x < dw; ++x) {
      const int32_t wx1 = xw[x], wx0 = 256 - xw[x];
      const int a = x0[x] * 3, b = x1[x] * 3;
      const uint32_t alpha = wrow[4 * x + 3];
      for (int c = 0; c < 3; ++c) {
        const int32_t ha = ra[a + c] * wx0 + ra[b + c] * wx1;
        const int32_t hb = rb[a + c] * wx0 + rb[b + c] * wx1;
        const uint32_t px = (uint32_t)((ha * wy0 + hb * wy1 + (1 << 15)) >> 16);
        out[3 * x + c] = (uint8_t)((px * (255u - alpha) + wrow[4 * x + c] * alpha + 127u) / 255u);
      }
    }
  }
  free(x0); free(x1); free(xw); free(y0); free(y1); free(yw);
}

/* --------------------------------------------------------------- PageRank */
/* RMAT quadrant thresholds a=0.57, a+b=0.76, a+b+c=0.95 on the top 32 bits */
#define RMAT_A 2448131358u  /* floor(0.57 * 2^32) */
#define RMAT_AB 3264175144u /* floor(0.76 * 2^32) */
#define RMAT_ABC 4080218931u /* floor(0.95 * 2^32) */
#define RMAT_PERM_MUL 0x9E3779B97F4A7C15ull

void orc_rmat_edges(int scale, int64_t m, uint64_t seed, int32_t* src, int32_t* dst,
                    int nthreads) {
  const uint64_t mask = (1ull << scale) - 1;
#pragma omp parallel for num_threads(nth(nthreads)) schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    uint64_t st = seed ^ ((uint64_t)e * 0xD1B54A32D192ED03ull);
    uint64_t u = 0, v = 0;
    for (int l = 0; l < scale; ++l) {
      st = orc_splitmix64(st);
      const uint32_t q = (uint32_t)(st >> 32);
      const uint64_t bit = 1ull << (scale - 1 - l);
      if (q >= RMAT_A) {
        if (q < RMAT_AB) {
          v |= bit;
        } else if (q < RMAT_ABC) {
          u |= bit;
        } else {
          u |= bit;
          v |= bit;
        }
      }
    }
    /* odd multiplier: a bijection on [0, 2^scale) that scatters hub labels */
    src[e] = (int32_t)((u * RMAT_PERM_MUL) & mask);
    dst[e] = (int32_t)((v * RMAT_PERM_MUL) & mask);
  }
}

void orc_pr_run(int32_t V, const int32_t* off, const int32_t* col, const int32_t* outdeg,
                double d, int iters, double* r, int nthreads) {
  double* c = malloc(sizeof(double) * (size_t)V);
  const double base = (1.0 - d) / (double)V;
  for (int it = 0; it < iters; ++it) {
#pragma omp parallel for num_threads(nth(nthreads)) schedule(static)
    for (int32_t u = 0; u < V; ++u) c[u] = outdeg[u] > 0 ? r[u] / (double)outdeg[u] : 0.0;
#pragma omp parallel for num_threads(nth(nthreads)) schedule(dynamic, 1024)
    for (int32_t v = 0; v < V; ++v) {
      double s = 0.0;
      for (int32_t j = off[v]; j < off[v + 1]; ++j) s += c[col[j]];
      r[v] = base + d * s;
    }
  }
  free(c);
}

/* -------------------------------------------------------------- Graph-SGD */
#define SGD_PERM_MUL 2654435761ull

static inline int32_t sgd_vertex(uint64_t h, int32_t V) {
  /* power-law-ish skew: density ~ v^(-1/3) from x^1.5 = x*sqrt(x) (IEEE
   * sqrt: bit-identical on CPU and GPU), max degree ~1e4 at the Orkut shape;
   * then a multiplicative bijection mod V scatters the hubs */
  const double x = (double)(h >> 11) * (1.0 / 9007199254740992.0);
  int64_t v = (int64_t)((double)V * x * sqrt(x));
  if (v >= V) v = V - 1;
  return (int32_t)(((uint64_t)v * SGD_PERM_MUL) % (uint64_t)V);
}

void orc_sgd_edges(int32_t V, int64_t E, uint64_t seed, int32_t* u, int32_t* v, float* r,
                   int nthreads) {
#pragma omp parallel for num_threads(nth(nthreads)) schedule(static)
  for (int64_t e = 0; e < E; ++e) {
    const int32_t a = sgd_vertex(orc_splitmix64(seed ^ (2 * (uint64_t)e)), V);
    const int32_t b = sgd_vertex(orc_splitmix64(seed ^ (2 * (uint64_t)e + 1)), V);
    u[e] = a;
    v[e] = b;
    const uint64_t hr = orc_splitmix64((seed * 0x2545F4914F6CDD1Dull) ^ ((uint64_t)a * (uint64_t)V + (uint64_t)b));
    r[e] = (float)(1 + (int)(hr % 5));
  }
}

/* fr_sgd_group_by_user's layout (paper_2409_06941_b200/csrc/kernels/sgd.cu):
 * Gardenia's CSR input order -- a stable counting sort by u -- then, when
 * the latent rows exceed 64 MiB, a stable sort by item block (P ranges of v,
 * P = ceil(V k 4 B / 64 MiB)), then each (block, user) run cut into 64-edge
 * pieces, piece q of np going to round (q R / np + h(u)) mod R inside its
 * block (R = ceil(E / window)), and a stable sort by block x R + round. */
#define SGD_PIECE 64
static int32_t sgd_round(int32_t u, int64_t rank, int64_t deg, int32_t R) {
  const int64_t np = (deg + SGD_PIECE - 1) / SGD_PIECE, k = rank / SGD_PIECE;
  const uint64_t h = orc_splitmix64(0x5347445250ull ^ (uint64_t)u) % (uint64_t)R;
  return (int32_t)(((uint64_t)(k * R / np) + h) % (uint64_t)R);
}

int32_t orc_sgd_item_blocks(int32_t V, int k) {
  const int64_t bytes = (int64_t)V * k * 4, blk = (int64_t)64 << 20;
  const int64_t P = (bytes + blk - 1) / blk;
  return (int32_t)(P < 1 ? 1 : P);
}

static int32_t sgd_block_of(int32_t v, int32_t V, int32_t P) { return (int32_t)((int64_t)v * P / V); }

/* stable counting sort of (u, v, r) by key[] in [0, nkeys) into (u2, v2, r2) */
static void sgd_counting_sort(int64_t E, const int32_t* key, int64_t nkeys, const int32_t* u,
                              const int32_t* v, const float* r, int32_t* u2, int32_t* v2, float* r2) {
  int64_t* start = (int64_t*)calloc((size_t)nkeys + 1, sizeof(int64_t));
  for (int64_t e = 0; e < E; ++e) start[key[e] + 1]++;
  for (int64_t i = 0; i < nkeys; ++i) start[i + 1] += start[i];
  for (int64_t e = 0; e < E; ++e) {
    const int64_t at = start[key[e]]++;
    u2[at] = u[e];
    v2[at] = v[e];
    r2[at] = r[e];
  }
  free(start);
}

void orc_sgd_group_by_user(int32_t V, int64_t E, int64_t window, int k, int32_t* u, int32_t* v, float* r) {
  const size_t n = (size_t)(E > 0 ? E : 1);
  const int32_t P = orc_sgd_item_blocks(V, k);
  int64_t R = window > 0 ? (E + window - 1) / window : 1;
  if (R < 1) R = 1;
  if (R > ((int64_t)1 << 30) / P) R = ((int64_t)1 << 30) / P;
  if (R < 1) R = 1;
  int32_t* key = (int32_t*)malloc(n * sizeof(int32_t));
  int32_t* u2 = (int32_t*)malloc(n * sizeof(int32_t));
  int32_t* v2 = (int32_t*)malloc(n * sizeof(int32_t));
  float* r2 = (float*)malloc(n * sizeof(float));
  /* 1. by u */
  sgd_counting_sort(E, u, V, u, v, r, u2, v2, r2);
  memcpy(u, u2, (size_t)E * sizeof(int32_t));
  memcpy(v, v2, (size_t)E * sizeof(int32_t));
  memcpy(r, r2, (size_t)E * sizeof(float));
  /* 2. by item block */
  if (P > 1) {
    for (int64_t e = 0; e < E; ++e) key[e] = sgd_block_of(v[e], V, P);
    sgd_counting_sort(E, key, P, u, v, r, u2, v2, r2);
    memcpy(u, u2, (size_t)E * sizeof(int32_t));
    memcpy(v, v2, (size_t)E * sizeof(int32_t));
    memcpy(r, r2, (size_t)E * sizeof(float));
  }
  /* 3. rounds inside each block */
  if (R > 1) {
    int64_t b = 0;
    for (int64_t e = 0; e < E; ++e) {
      if (e == 0 || u[e] != u[e - 1] || sgd_block_of(v[e], V, P) != sgd_block_of(v[e - 1], V, P)) b = e;
      int64_t end = b + 1;  /* run end: scan once per run start */
      if (e == b) {
        while (end < E && u[end] == u[b] && sgd_block_of(v[end], V, P) == sgd_block_of(v[b], V, P)) ++end;
        key[e] = (int32_t)end;  /* stash the end at the run's first edge */
      }
      (void)end;
    }
    int64_t run_b = 0, run_e = 0;
    for (int64_t e = 0; e < E; ++e) {
      if (e == run_e) {
        run_b = e;
        run_e = key[e];
      }
      key[e] = sgd_block_of(v[e], V, P) * (int32_t)R + sgd_round(u[e], e - run_b, run_e - run_b, (int32_t)R);
    }
    sgd_counting_sort(E, key, (int64_t)P * R, u, v, r, u2, v2, r2);
    memcpy(u, u2, (size_t)E * sizeof(int32_t));
    memcpy(v, v2, (size_t)E * sizeof(int32_t));
    memcpy(r, r2, (size_t)E * sizeof(float));
  }
  free(key);
  free(u2);
  free(v2);
  free(r2);
}

void orc_sgd_init(int32_t V, int k, uint64_t seed, float* L, int nthreads) {
  const float scale = (float)(1.0 / sqrt((double)k)) * (1.0f / 16777216.0f);
#pragma omp parallel for num_threads(nth(nthreads)) schedule(static)
  for (int64_t i = 0; i < (int64_t)V * k; ++i)
    L[i] = (float)(orc_splitmix64(seed ^ (0x4C4154ull << 40) ^ (uint64_t)i) >> 40) * scale;
}

static inline void sgd_update(float* lu, float* lv, float rating, int k, float eta, float lam) {
  float dot = 0.0f;
  for (int j = 0; j < k; ++j) dot += lu[j] * lv[j];
  const float err = rating - dot;
  for (int j = 0; j < k; ++j) {
    const float a = lu[j], b = lv[j];
    lu[j] = a + eta * (err * b - lam * a);
    lv[j] = b + eta * (err * a - lam * b);
  }
}

void orc_sgd_epoch(int64_t E, const int32_t* u, const int32_t* v, const float* r, float* L, int k,
                   float eta, float lam, int nthreads) {
  if (nthreads == 1) {
    for (int64_t e = 0; e < E; ++e)
      sgd_update(L + (int64_t)u[e] * k, L + (int64_t)v[e] * k, r[e], k, eta, lam);
    return;
  }
#pragma omp parallel for num_threads(nth(nthreads)) schedule(static, 4096)
  for (int64_t e = 0; e < E; ++e)
    sgd_update(L + (int64_t)u[e] * k, L + (int64_t)v[e] * k, r[e], k, eta, lam);
}

double orc_sgd_rmse(int64_t E, const int32_t* u, const int32_t* v, const float* r, const float* L,
                    int k, int nthreads) {
  double acc = 0.0;
#pragma omp parallel for num_threads(nth(nthreads)) reduction(+ : acc) schedule(static)
  for (int64_t e = 0; e < E; ++e) {
    const float* a = L + (int64_t)u[e] * k;
    const float* b = L + (int64_t)v[e] * k;
    double dot = 0.0;
    for (int j = 0; j < k; ++j) dot += (double)a[j] * (double)b[j];
    const double err = (double)r[e] - dot;
    acc += err * err;
  }
  return E > 0 ? sqrt(acc / (double)E) : 0.0;
}
