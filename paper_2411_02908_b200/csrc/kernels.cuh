// kernels.cuh -- launch wrappers for the non-GEMM kernels of the client step,
// the optimizer and the aggregation.  Reference citations are in kernels.cu /
// optim.cu next to each kernel.
#pragma once

#include <vector>

#include "common.cuh"

namespace photon {
namespace k {

// ---- deferred column reductions -------------------------------------------------
// The bias / LayerNorm-gain gradients are column sums of per-block partials.
// With a ReduceJobs list the producers below write their partials and append a
// job instead of launching the reduction; run_reduce_jobs then runs every
// first-level row reduction in ONE launch and every final column reduction in
// a second, each element summed in exactly the order of the one-job kernels
// (the gradients are bitwise those of the immediate path).  The partial
// buffers must stay distinct until run_reduce_jobs.
struct RowJob {
  const float* part;
  int nparts, per, n, nseg;
  size_t seg_stride;
  float* out;
  int used;
};
struct ColJob {
  const float* part;
  int nparts, n, stride, split, split2;
  float *out, *out1, *out2;
  int acc;
};
struct ReduceJobs {
  std::vector<RowJob> rows;
  std::vector<ColJob> cols;
};
void run_reduce_jobs(ReduceJobs& jobs, cudaStream_t st);

// ---- embedding (gather_rows + add, tensor.cpp:209-223, 290-320) ------------
void embed_fwd(const int32_t* tokens, const float* tok, const float* pos, float* x, int M, int S,
               int d, cudaStream_t st);
// deterministic scatter-add: rows sorted by token (CSR), ascending row order.
// dx holds rows [row0, row0 + M) of the CSR's batch (one micro-batch); acc adds
// onto dtok / dpos instead of overwriting them (micro-batches after the first).
void embed_bwd(const float* dx, const int32_t* csr_off, const int32_t* csr_rows, float* dtok,
               float* dpos, int V, int M, int S, int d, cudaStream_t st, int row0 = 0,
               bool acc = false);

// ---- layer norm (tensor.cpp:322-394) ---------------------------------------
template <typename T>
void ln_fwd(const float* x, const float* gain, const float* bias, T* y, float* mean, float* rstd,
            int M, int d, cudaStream_t st);
// dx_out = dres + LN'(dy) (dy in the activation type T: bf16 on the tensor-core
// path, where the dX GEMMs write it); dx_T = bf16/f32 copy (optional); gain/bias grads
// written to dgain/dbias via per-block partials in `part` (>= ln_bwd_parts()*3*d
// floats).  dsum (optional) receives the column sums of dx_out: the bias
// gradient of the linear layer whose output is this residual-stream gradient
// (add_bias backward, tensor.cpp:279-285), without a second pass over dx_out.
template <typename T>
void ln_bwd(const T* dy, const float* x, const float* mean, const float* rstd,
            const float* gain, const float* dres, float* dx_out, T* dx_T, float* part,
            float* dgain, float* dbias, int M, int d, cudaStream_t st, float* dsum = nullptr,
            bool acc = false,  // acc: add dgain / dbias / dsum onto the existing values
            ReduceJobs* defer = nullptr);
int ln_bwd_parts();

// ---- column sums (add_bias backward, tensor.cpp:279-285) -------------------
template <typename T>
void colsum(const T* x, int M, int N, float* part, float* out, cudaStream_t st, bool acc = false);
size_t colsum_part_floats(int M, int N);
// Column sums from caller-written partials part[nparts][N] (e.g. the per-32-row
// sums a GEMM epilogue emits): fixed-order two-level reduction through
// `scratch` (colsum_parts_scratch_floats(N) floats) into out[N].
constexpr int kColsumPartGroups = 64;
size_t colsum_parts_scratch_floats(int N);
void colsum_parts(const float* part, int nparts, int N, float* scratch, float* out, cudaStream_t st,
                  bool acc = false, ReduceJobs* defer = nullptr);
// three same-shaped partial arrays (part + i * seg_stride) into out0..out2 in
// two launches (the q / k / v bias gradients); scratch >= 3 x colsum_parts_scratch_floats(N)
void colsum_parts3(const float* part, size_t seg_stride, int nparts, int N, float* scratch,
                   float* out0, float* out1, float* out2, cudaStream_t st, bool acc = false,
                   ReduceJobs* defer = nullptr);

// ---- softmax cross-entropy fwd+bwd (tensor.cpp:544-603) --------------------
// logits [M,V] overwritten with dlogits = (softmax - onehot) * inv_count;
// rowloss[m] = logsumexp - logit[target] (0 for target < 0)
// With write_grad and dbias / part (>= ce_bias_part_floats(V) floats), the
// bf16 pipelined kernel also produces the head-bias gradient dbias[V] (the
// column sums of dlogits; acc adds onto dbias) and returns true; false: the
// caller takes the column sums itself.
// inv_dev (optional): 1 / #targets read from device memory instead of inv_count.
template <typename T>
bool ce_fwd_bwd(T* logits, const int32_t* targets, int M, int V, float inv_count,
                double* rowloss, bool write_grad, cudaStream_t st, float* dbias = nullptr,
                float* part = nullptr, bool acc = false, const float* inv_dev = nullptr,
                ReduceJobs* defer = nullptr);
size_t ce_bias_part_floats(int V);
// out = inv_count * sum(rowloss) (fixed-order tree); acc: out += ...
void sum_scaled(const double* x, int n, double scale, double* out, cudaStream_t st,
                bool acc = false, const float* scale_dev = nullptr);

// ---- causal attention (tensor.cpp:436-542), SIMT fp32 math ------------------
template <typename T>
void attn_fwd_simt(const T* q, const T* k, const T* v, T* o, float* lse, int B, int S, int H,
                   int d, cudaStream_t st);
template <typename T>
void attn_bwd_simt(const T* q, const T* k, const T* v, const T* o, const T* dO, const float* lse,
                   float* Dvec, T* dq, T* dk, T* dv, int B, int S, int H, int d, cudaStream_t st);

// ---- causal attention on tensor cores (bf16, mma.sync m16n8k16), attn_mma.cu ----
bool attn_mma_supported(int dh);
void attn_fwd_mma(const bf16* q, const bf16* k, const bf16* v, bf16* o, float* lse, int B, int S,
                  int H, int d, cudaStream_t st);
void attn_bwd_mma(const bf16* q, const bf16* k, const bf16* v, const bf16* o, const bf16* dO,
                  const float* lse, float* Dvec, bf16* dq, bf16* dk, bf16* dv, int B, int S, int H,
                  int d, cudaStream_t st);

// ---- causal attention on tcgen05/TMEM/TMA (dh = 64), attn_tc.cu ----
bool attn_tc_supported(int dh, int d);
void attn_fwd_tc(const bf16* q, const bf16* k, const bf16* v, bf16* o, float* lse, int B, int S,
                 int H, int d, cudaStream_t st);
// Fused deterministic backward; ws = attn_bwd_tc_ws_floats() floats of device
// workspace owned by the caller (nullptr: a per-device scratch, debug use only).
size_t attn_bwd_tc_ws_floats(int B, int S, int H, int d);
void attn_bwd_tc(const bf16* q, const bf16* k, const bf16* v, const bf16* o, const bf16* dO,
                 const float* lse, bf16* dq, bf16* dk, bf16* dv, int B, int S, int H, int d,
                 float* ws, cudaStream_t st, float* sums = nullptr);
// sums (optional): the kernels also write per-32-row column sums of dq, dk, dv
// (the q / k / v bias gradients' partials) as three consecutive
// [B * ceil(S / 32)][d] blocks, for colsum_parts
inline size_t attn_bwd_sums_floats(int B, int S, int d) { return (size_t)3 * B * ((S + 31) / 32) * d; }

// ---- casts -------------------------------------------------------------------
void f64_to_f32(const double* in, float* out, uint64_t n, cudaStream_t st);
void f32_to_f64(const float* in, double* out, uint64_t n, cudaStream_t st);
void f32_to_bf16(const float* in, bf16* out, uint64_t n, cudaStream_t st);
// out[c][r] = in[r][c], [rows][cols] bf16
void transpose_bf16(const bf16* in, int rows, int cols, bf16* out, cudaStream_t st);

// ---- optimizer (optim.cu, compiled without FMA contraction) ---------------------
// global-norm clip (optim.cpp:50-57): parts -> norm, cf; bad[0] set to step+1
// on a non-finite norm (first one wins)
void sumsq_parts(const float* g, uint64_t n, double* part, cudaStream_t st);
int sumsq_nparts();
void clip_finalize(const double* part, double clip, double* norm_out, float* cf_out,
                   int* bad_step, int step, cudaStream_t st);
// AdamW (optim.cpp:61-90) in f64 arithmetic over fp32 storage
// lr_dev (optional): the learning rate read from device memory instead of `lr`
// (CUDA-graph replays of a local round, whose lr changes every round)
void adamw_f32(float* p, const float* g, float* m, float* v, bf16* shadow, uint64_t n,
               const float* cf, double lr, double b1, double b2, double bc1, double bc2,
               double eps, double wd, cudaStream_t st, const double* lr_dev = nullptr);
void sgd_f32(float* p, const float* g, bf16* shadow, uint64_t n, const float* cf, double lr,
             cudaStream_t st, const double* lr_dev = nullptr);
// exact f64 variants for the f64 C-ABI (bit-exact vs the reference)
void sumsq_sequential_f64(const double* g, uint64_t n, double* out, cudaStream_t st);
void adamw_f64(double* p, const double* g, double* m, double* v, uint64_t n, const double* norm,
               double clip, double lr, double b1, double b2, double bc1, double bc2, double eps,
               double wd, cudaStream_t st);
void sgd_f64(double* p, const double* g, uint64_t n, const double* norm, double clip, double lr,
             cudaStream_t st);

// ---- aggregation (param_vector.cpp:120-152, optim.cpp:124-159) -----------------
// kind: 0 FedAvg, 1 momentum.  models: device array of k device pointers.
// Round boundary over peer memory (optim.cu): models[c] = surviving client c's
// full model (ascending slot, IPC-mapped or local), replicas[g] = rank g's
// theta buffer; this rank updates [off, off+len) of every replica.
using photon::kMaxPeerModels;  // host.hpp: the boundary plan
using photon::kMaxPeerWorld;
struct PeerBoundaryArgs {
  const float* models[kMaxPeerModels];
  float* replicas[kMaxPeerWorld];
  float* vel;  // this rank's velocity shard [len]
  const int* abort;  // nonzero: a peer never reached the boundary -- do nothing
  uint64_t off, len;
  int n, world, rank, kind, nesterov;
  float eta, mu;
};
void boundary_p2p(const PeerBoundaryArgs& a, cudaStream_t st);

template <typename T>
void aggregate(const T* const* models, int k, uint64_t n, T* theta, T* velocity, int kind,
               double eta, double mu, int nesterov, cudaStream_t st);
template <typename T>
void mean_only(const T* const* models, int k, uint64_t n, T* out, cudaStream_t st);
template <typename T>
void sub_only(const T* a, const T* b, uint64_t n, T* out, cudaStream_t st);
template <typename T>
void server_step_only(const T* theta, const T* delta, const T* mean, T* velocity, T* out,
                      uint64_t n, int kind, double eta, double mu, int nesterov, cudaStream_t st);
// post_process clip (client.cpp:96-110): out = ref + min(1, thr/|k-ref|) (k - ref)
void clip_update_f32(const float* ref, float* theta_k, uint64_t n, double threshold,
                     double* part, cudaStream_t st);

}  // namespace k
}  // namespace photon
