// engine.cuh -- device-resident client step: the decoder forward, the
// hand-ordered backward and the optimizer over one flat fp32 parameter buffer
// in the reference's canonical order (model.cpp:32-61).
#pragma once

#include <memory>
#include <vector>

#include "common.cuh"

namespace photon {

// One step's batch, already on the device.
struct StepBatch {
  const int32_t* tokens = nullptr;    // [B*S]
  const int32_t* targets = nullptr;   // [B*S]
  const int32_t* csr_off = nullptr;   // [V+1] rows per token (embedding backward)
  const int32_t* csr_rows = nullptr;  // [B*S] row ids sorted by (token, row)
  int B = 0, S = 0;
  float inv_count = 0.f;              // 1 / #targets >= 0
  const float* inv_count_dev = nullptr;  // the same on the device (graph-captured rounds)
};

// Per-kernel-class device time accumulated when timing is enabled.
struct KernelTimes {
  double gemm_ms = 0, attn_ms = 0, other_ms = 0, optim_ms = 0;
  double gemm_flops = 0, attn_flops = 0;
  int gemm_launches = 0, attn_launches = 0, launches = 0;
};

class Engine {
 public:
  static std::unique_ptr<Engine> create(const photon_model_cfg& cfg, int precision,
                                        uint64_t max_batch, cudaStream_t st);
  virtual ~Engine() = default;

  const photon_model_cfg cfg;
  const int precision;
  const uint64_t max_batch;
  const uint64_t P;
  cudaStream_t stream;

  float* master = nullptr;  // fp32 [P] client parameters (theta during local steps)
  float* grads = nullptr;   // fp32 [P]
  float* mom = nullptr;     // fp32 [P] AdamW m
  float* vel2 = nullptr;    // fp32 [P] AdamW v
  bf16* shadow = nullptr;   // bf16 [P] GEMM operand copy (BF16 precision only)
  // scratch
  double* red_part = nullptr;   // reduction partials
  float* cf = nullptr;          // clip factor
  double* norm = nullptr;
  int* bad_step = nullptr;      // first step (1-based) with a non-finite grad norm

  // timing instrumentation (per kernel class, CUDA events on `stream`)
  bool timing = false;
  KernelTimes times;
  int gemm_mode = 1;  // 1: tcgen05 for bf16 operands, 0: SIMT everywhere
  int attn_mode = 1;  // 1: tensor-core attention for bf16, 0: SIMT

  // master -> shadow (bf16 mode)
  virtual void refresh_shadow() = 0;
  // loss (scaled mean) to *loss_dev; grads when backward
  virtual void forward_backward(const StepBatch& b, double* loss_dev, bool backward) = 0;
  // AdamW / SGD with the global-norm clip (optim.cpp:50-103); scalars from host
  // lr_dev (optional): lr read from device memory (graph-captured rounds)
  void adamw(double clip, double lr, double b1, double b2, double bc1, double bc2, double eps,
             double wd, int step, const double* lr_dev = nullptr);
  void sgd(double clip, double lr, int step, const double* lr_dev = nullptr);

 protected:
  Engine(const photon_model_cfg& c, int prec, uint64_t mb, cudaStream_t st);
};

// Deterministic CSR of rows by token for the embedding backward (host side).
void build_token_csr(const int32_t* tokens, int M, int V, int32_t* off, int32_t* rows);

}  // namespace photon
