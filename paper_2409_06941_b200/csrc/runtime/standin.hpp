// Synthetic pipeline-stage stand-in: per-stage FP/BP
// busy periods made of bf16 tensor-core GEMMs (cuBLASLt, fp32 accumulate)
// shaped like a GPT transformer stage, so the bubbles a stage exposes are
// real idle time between real tensor-core work.  FP = 4 GEMMs per layer
// (QKV, attention out-proj, MLP up, MLP down); BP = dgrad + wgrad of each
// (2x FP FLOPs).  Each op is captured once as a CUDA graph so a pipeline op
// is a single launch on the training stream.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace freeride::rt {

struct StandInShape {
  int layers = 6;       // layers held by this stage
  int hidden = 2048;    // h
  int tokens = 8192;    // micro-batch x sequence
  int ffn_mult = 4;
};

class StandIn {
 public:
  explicit StandIn(const StandInShape& shape);
  ~StandIn();
  StandIn(const StandIn&) = delete;
  StandIn& operator=(const StandIn&) = delete;

  // Captures the FP and BP op graphs for `stream` (must be called once).
  void capture(cudaStream_t stream);
  void launch_fp(cudaStream_t stream);
  void launch_bp(cudaStream_t stream);
  double fp_flops() const;
  double bp_flops() const { return 2.0 * fp_flops(); }
  std::size_t weight_bytes() const;
  std::size_t activation_bytes() const;  // one micro-batch's stashed activations
  // the activation / gradient a stage sends its neighbour per micro-batch:
  // tokens x hidden bf16, taken from the op's output buffer
  std::size_t message_bytes() const {
    return static_cast<std::size_t>(shape_.tokens) * shape_.hidden * 2;
  }
  const void* output() const { return out_; }

 private:
  struct Gemm {
    int m, n, k;
    bool ta, tb;
    const void* a;
    const void* b;
    void* d;
    int lda, ldb, ldd;
  };
  void enqueue_fp(cudaStream_t s);
  void enqueue_bp(cudaStream_t s);
  void run(const Gemm& g, cudaStream_t s);

  StandInShape shape_;
  void* lt_ = nullptr;  // cublasLtHandle_t
  void* workspace_ = nullptr;
  std::size_t workspace_bytes_ = 32u << 20;
  std::vector<void*> weights_;
  void* act_ = nullptr;   // input activations (T x max width)
  void* out_ = nullptr;   // outputs / grads
  void* gin_ = nullptr;   // incoming grads
  void* wgrad_ = nullptr; // weight-grad scratch (largest weight)
  cudaGraphExec_t fp_graph_ = nullptr;
  cudaGraphExec_t bp_graph_ = nullptr;
};

}  // namespace freeride::rt
