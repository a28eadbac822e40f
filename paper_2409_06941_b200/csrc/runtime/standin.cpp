#include "runtime/standin.hpp"

#include <cublasLt.h>

#include <stdexcept>

namespace freeride::rt {

void fill_random_bf16(void* p, std::size_t n, std::uint64_t seed, cudaStream_t s);  // timeline.cu

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

void ck(cublasStatus_t e, const char* what) {
  if (e != CUBLAS_STATUS_SUCCESS)
    throw std::runtime_error(std::string(what) + ": cublasLt status " + std::to_string(int(e)));
}

}  // namespace

StandIn::StandIn(const StandInShape& shape) : shape_(shape) {
  cublasLtHandle_t h = nullptr;
  ck(cublasLtCreate(&h), "cublasLtCreate");
  lt_ = h;
  ck(cudaMalloc(&workspace_, workspace_bytes_), "workspace");
  const std::size_t H = shape_.hidden, F = static_cast<std::size_t>(shape_.hidden) * shape_.ffn_mult,
                    T = shape_.tokens;
  const std::size_t per_layer[4] = {3 * H * H, H * H, F * H, H * F};
  cudaStream_t s = nullptr;
  ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  std::uint64_t seed = 1;
  for (int l = 0; l < shape_.layers; ++l)
    for (std::size_t n : per_layer) {
      void* w = nullptr;
      ck(cudaMalloc(&w, n * 2), "weights");
      fill_random_bf16(w, n, seed++, s);
      weights_.push_back(w);
    }
  const std::size_t wide = std::max<std::size_t>(3 * H, F) * T;
  for (void** p : {&act_, &out_, &gin_}) {
    ck(cudaMalloc(p, wide * 2), "activations");
    fill_random_bf16(*p, wide, seed++, s);
  }
  ck(cudaMalloc(&wgrad_, std::max<std::size_t>(3 * H * H, F * H) * 2), "wgrad");
  ck(cudaStreamSynchronize(s), "init sync");
  cudaStreamDestroy(s);
}

StandIn::~StandIn() {
  if (fp_graph_) cudaGraphExecDestroy(fp_graph_);
  if (bp_graph_) cudaGraphExecDestroy(bp_graph_);
  for (void* w : weights_) cudaFree(w);
  for (void* p : {act_, out_, gin_, wgrad_, workspace_})
    if (p) cudaFree(p);
  if (lt_) cublasLtDestroy(static_cast<cublasLtHandle_t>(lt_));
}

double StandIn::fp_flops() const {
  const double H = shape_.hidden, F = H * shape_.ffn_mult, T = shape_.tokens;
  return 2.0 * T * (3 * H * H + H * H + F * H + H * F) * shape_.layers;
}

std::size_t StandIn::weight_bytes() const {
  const std::size_t H = shape_.hidden, F = H * shape_.ffn_mult;
  return (3 * H * H + H * H + 2 * F * H) * 2 * shape_.layers;
}

std::size_t StandIn::activation_bytes() const {
  const std::size_t H = shape_.hidden, F = H * shape_.ffn_mult, T = shape_.tokens;
  return (3 * H + H + F + H) * T * 2 * shape_.layers;  // inputs each GEMM stashes for BP
}

void StandIn::run(const Gemm& g, cudaStream_t s) {
  auto lt = static_cast<cublasLtHandle_t>(lt_);
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, ld = nullptr;
  cublasLtMatmulPreference_t pref = nullptr;
  ck(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F), "desc");
  const cublasOperation_t ta = g.ta ? CUBLAS_OP_T : CUBLAS_OP_N, tb = g.tb ? CUBLAS_OP_T : CUBLAS_OP_N;
  ck(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)), "ta");
  ck(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)), "tb");
  ck(cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, g.ta ? g.k : g.m, g.ta ? g.m : g.k, g.lda), "la");
  ck(cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, g.tb ? g.n : g.k, g.tb ? g.k : g.n, g.ldb), "lb");
  ck(cublasLtMatrixLayoutCreate(&ld, CUDA_R_16BF, g.m, g.n, g.ldd), "ld");
  ck(cublasLtMatmulPreferenceCreate(&pref), "pref");
  ck(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES,
                                          &workspace_bytes_, sizeof(workspace_bytes_)),
     "pref ws");
  cublasLtMatmulHeuristicResult_t heur{};
  int found = 0;
  ck(cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, ld, ld, pref, 1, &heur, &found), "heuristic");
  if (found < 1) throw std::runtime_error("cublasLt: no algorithm for stand-in GEMM");
  const float alpha = 1.0f, beta = 0.0f;
  ck(cublasLtMatmul(lt, op, &alpha, g.a, la, g.b, lb, &beta, g.d, ld, g.d, ld, &heur.algo,
                    workspace_, workspace_bytes_, s),
     "cublasLtMatmul");
  cublasLtMatmulPreferenceDestroy(pref);
  cublasLtMatrixLayoutDestroy(la);
  cublasLtMatrixLayoutDestroy(lb);
  cublasLtMatrixLayoutDestroy(ld);
  cublasLtMatmulDescDestroy(op);
}

// Column-major view of row-major activations: Y^T[N x T] = W^T[N x K] X^T[K x T].
void StandIn::enqueue_fp(cudaStream_t s) {
  const int H = shape_.hidden, F = H * shape_.ffn_mult, T = shape_.tokens;
  const int mk[4][2] = {{3 * H, H}, {H, H}, {F, H}, {H, F}};
  for (int l = 0; l < shape_.layers; ++l)
    for (int j = 0; j < 4; ++j) {
      const int m = mk[j][0], k = mk[j][1];
      run(Gemm{m, T, k, false, false, weights_[4 * l + j], act_, out_, m, k, m}, s);
    }
}

// dX^T[K x T] = W[K x M] dY^T[M x T]  and  dW[M x K] = dY^T[M x T] X[T x K].
void StandIn::enqueue_bp(cudaStream_t s) {
  const int H = shape_.hidden, F = H * shape_.ffn_mult, T = shape_.tokens;
  const int mk[4][2] = {{3 * H, H}, {H, H}, {F, H}, {H, F}};
  for (int l = shape_.layers - 1; l >= 0; --l)
    for (int j = 3; j >= 0; --j) {
      const int m = mk[j][0], k = mk[j][1];
      run(Gemm{k, T, m, true, false, weights_[4 * l + j], gin_, out_, m, m, k}, s);
      run(Gemm{m, k, T, false, true, gin_, act_, wgrad_, m, k, m}, s);
    }
}

void StandIn::capture(cudaStream_t stream) {
  for (int which = 0; which < 2; ++which) {
    // warm the heuristics / lazy module loading outside the capture
    which == 0 ? enqueue_fp(stream) : enqueue_bp(stream);
    ck(cudaStreamSynchronize(stream), "stand-in warmup");
    cudaGraph_t g = nullptr;
    ck(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "begin capture");
    which == 0 ? enqueue_fp(stream) : enqueue_bp(stream);
    ck(cudaStreamEndCapture(stream, &g), "end capture");
    ck(cudaGraphInstantiate(which == 0 ? &fp_graph_ : &bp_graph_, g, 0), "instantiate");
    cudaGraphDestroy(g);
  }
}

void StandIn::launch_fp(cudaStream_t s) { ck(cudaGraphLaunch(fp_graph_, s), "fp graph"); }
void StandIn::launch_bp(cudaStream_t s) { ck(cudaGraphLaunch(bp_graph_, s), "bp graph"); }

}  // namespace freeride::rt
