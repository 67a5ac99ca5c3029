// engine.cu -- the client step on one GPU.
//
// Forward = model.cpp:98-158; backward = the reverse topological order the
// reference's autodiff produces for that graph (tensor.cpp:605-647), written
// out as a static schedule; optimizer = optim.cpp:50-103.  Activations that
// feed tensor-core contractions are stored as T (fp32 or bf16); the residual
// stream, LayerNorm statistics, softmax statistics and every gradient
// accumulator stay fp32.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "engine.cuh"
#include "gemm.cuh"
#include "kernels.cuh"

namespace photon {

void build_token_csr(const int32_t* tokens, int M, int V, int32_t* off, int32_t* rows) {
  std::fill(off, off + V + 1, 0);
  for (int m = 0; m < M; ++m) off[tokens[m] + 1] += 1;
  for (int v = 0; v < V; ++v) off[v + 1] += off[v];
  std::vector<int32_t> fill(off, off + V);
  for (int m = 0; m < M; ++m) rows[fill[tokens[m]]++] = m;  // ascending rows per token
}

Engine::Engine(const photon_model_cfg& c, int prec, uint64_t mb, cudaStream_t st)
    : cfg(c), precision(prec), max_batch(mb), P(param_count(c)), stream(st) {}

void Engine::adamw(double clip, double lr, double b1, double b2, double bc1, double bc2,
                   double eps, double wd, int step, const double* lr_dev) {
  if (timing) times.launches += 3;
  k::sumsq_parts(grads, P, red_part, stream);
  k::clip_finalize(red_part, clip, norm, cf, bad_step, step, stream);
  k::adamw_f32(master, grads, mom, vel2, shadow, P, cf, lr, b1, b2, bc1, bc2, eps, wd, stream,
               lr_dev);
}

void Engine::sgd(double clip, double lr, int step, const double* lr_dev) {
  if (timing) times.launches += 3;
  k::sumsq_parts(grads, P, red_part, stream);
  k::clip_finalize(red_part, clip, norm, cf, bad_step, step, stream);
  k::sgd_f32(master, grads, shadow, P, cf, lr, stream, lr_dev);
}

namespace {

template <typename T>
constexpr DT dt_of() {
  return sizeof(T) == 4 ? DT::F32 : DT::BF16;
}

template <typename T>
class EngineT final : public Engine {
 public:
  EngineT(const photon_model_cfg& c, int prec, uint64_t mb, cudaStream_t st)
      : Engine(c, prec, mb, st), off_(model_offsets(c)) {
    d_ = c.d_model;
    H_ = c.n_heads;
    hid_ = c.expansion_ratio * d_;
    V_ = c.vocab_size;
    L_ = c.n_blocks;
    Smax_ = c.seq_len;
    Mmax_ = mb * Smax_;
    if (const char* e = std::getenv("PHOTON_GEMM")) gemm_mode = std::string(e) == "simt" ? 0 : 1;
    if (const char* e = std::getenv("PHOTON_ATTN"))
      attn_mode = std::string(e) == "simt" ? 0 : (std::string(e) == "mma" ? 2 : 1);
    allocate();
  }
  ~EngineT() override {
    if (pool_) cudaFree(pool_);
    if (master_alloc_) cudaFree(master_alloc_);
    for (auto& e : ev_pool_) cudaEventDestroy(e);
  }

  void refresh_shadow() override {
    if (shadow) k::f32_to_bf16(master, shadow, P, stream);
  }

  void forward_backward(const StepBatch& b, double* loss_dev, bool backward) override;
  // one micro-batch: rows [row0, row0 + bt.B * S) of the step's batch; acc adds
  // every gradient (and the loss) onto the previous micro-batches'
  void micro(const StepBatch& bt, double* loss_dev, bool backward, bool acc, int row0);

 private:
  ModelOffsets off_;
  uint64_t d_, H_, hid_, V_, L_, Smax_, Mmax_;
  char* pool_ = nullptr;
  // master is its own allocation: the multi-GPU boundary exports it through
  // CUDA IPC, and peers then map P * 4 bytes rather than the whole pool
  float* master_alloc_ = nullptr;
  // activations
  float *x_, *xmid_, *mean1_, *rstd1_, *mean2_, *rstd2_, *meanf_, *rstdf_, *lse_;
  T *h_, *q_, *k_, *v_, *o_, *h2_, *pre_, *u_, *xf_, *logits_;
  // backward scratch
  float *dx_, *dy_, *Dvec_, *part_, *attn_ws_, *gemm_ws_;
  // deferred column reductions: every bias / LayerNorm-gain partial of a
  // backward pass in its own slice of defer_, reduced by two batched launches
  // at the end of the pass (k::run_reduce_jobs)
  float* defer_ = nullptr;
  size_t defer_ln_ = 0, defer_b1_ = 0, defer_qkv_ = 0, defer_head_ = 0;
  k::ReduceJobs jobs_;
  // the LayerNorm backwards' input gradient in the activation type (bf16 on the
  // tensor-core path: the dX GEMMs write it directly; fp32 mode: dy_ itself)
  T* dyT_;
  T *dxT_, *dpre_, *dq_, *dk_, *dv_, *dO_;
  double* rowloss_;
  // timing
  std::vector<cudaEvent_t> ev_pool_;
  struct Span { int cat; cudaEvent_t a, b; double flops; };
  std::vector<Span> spans_;
  size_t ev_next_ = 0;

  const T* W(uint64_t offset) const {
    if constexpr (sizeof(T) == 4) return reinterpret_cast<const T*>(master + offset);
    else return reinterpret_cast<const T*>(shadow + offset);
  }
  const float* Pm(uint64_t offset) const { return master + offset; }
  float* G(uint64_t offset) { return grads + offset; }

  template <typename U>
  U* carve(char*& p, uint64_t n) {
    U* r = reinterpret_cast<U*>(p);
    p += ((n * sizeof(U) + 255) / 256) * 256;
    return r;
  }

  void allocate() {
    const uint64_t M = Mmax_, d = d_, L = L_, hid = hid_;
    const uint64_t rows_bhs = max_batch * H_ * Smax_;
    size_t part_floats = std::max<size_t>((size_t)k::ln_bwd_parts() * 3 * d,
                                          std::max({k::colsum_part_floats((int)M, (int)V_),
                                                    k::ce_bias_part_floats((int)V_),
                                                    k::colsum_part_floats((int)M, (int)hid),
                                                    k::colsum_part_floats((int)M, (int)d),
                                                    // b1 partials of the GeluBwd epilogue
                                                    (size_t)(M / 32) * hid +
                                                        k::colsum_parts_scratch_floats((int)hid),
                                                    // q / k / v partials of the attention backward
                                                    k::attn_bwd_sums_floats((int)max_batch,
                                                                            (int)Smax_, (int)d) +
                                                        3 * k::colsum_parts_scratch_floats((int)d)}));
    defer_ln_ = (size_t)k::ln_bwd_parts() * 3 * d;
    defer_b1_ = (size_t)(M / 32) * hid + k::colsum_parts_scratch_floats((int)hid);
    defer_qkv_ = k::attn_bwd_sums_floats((int)max_batch, (int)Smax_, (int)d) +
                 3 * k::colsum_parts_scratch_floats((int)d);
    defer_head_ = k::ce_bias_part_floats((int)V_);
    const size_t defer_floats = L * (2 * defer_ln_ + defer_b1_ + defer_qkv_) + defer_ln_ + defer_head_;
    auto plan = [&](char* p) {
      char* s = p;
      // master: separate allocation (see master_alloc_)
      grads = carve<float>(p, P);
      mom = carve<float>(p, P);
      vel2 = carve<float>(p, P);
      shadow = sizeof(T) == 2 ? carve<bf16>(p, P) : nullptr;
      red_part = carve<double>(p, 4096);
      cf = carve<float>(p, 1);
      norm = carve<double>(p, 1);
      bad_step = carve<int>(p, 1);
      x_ = carve<float>(p, (L + 1) * M * d);
      xmid_ = carve<float>(p, L * M * d);
      mean1_ = carve<float>(p, L * M);
      rstd1_ = carve<float>(p, L * M);
      mean2_ = carve<float>(p, L * M);
      rstd2_ = carve<float>(p, L * M);
      meanf_ = carve<float>(p, M);
      rstdf_ = carve<float>(p, M);
      lse_ = carve<float>(p, L * rows_bhs);
      h_ = carve<T>(p, L * M * d);
      q_ = carve<T>(p, L * M * d);
      k_ = carve<T>(p, L * M * d);
      v_ = carve<T>(p, L * M * d);
      o_ = carve<T>(p, L * M * d);
      h2_ = carve<T>(p, L * M * d);
      pre_ = carve<T>(p, L * M * hid);
      u_ = carve<T>(p, L * M * hid);
      xf_ = carve<T>(p, M * d);
      logits_ = carve<T>(p, M * V_);
      dx_ = carve<float>(p, M * d);
      dy_ = carve<float>(p, M * d);
      dyT_ = sizeof(T) == 4 ? reinterpret_cast<T*>(dy_) : carve<T>(p, M * d);
      Dvec_ = carve<float>(p, rows_bhs);
      gemm_ws_ = sizeof(T) == 2 ? carve<float>(p, kGemmWsFloats) : nullptr;
      attn_ws_ = sizeof(T) == 2 && k::attn_tc_supported((int)(d_ / H_), (int)d_)
                     ? carve<float>(p, k::attn_bwd_tc_ws_floats((int)max_batch, (int)Smax_, (int)H_, (int)d_))
                     : nullptr;
      part_ = carve<float>(p, part_floats);
      defer_ = carve<float>(p, defer_floats);
      dxT_ = carve<T>(p, M * d);
      dpre_ = carve<T>(p, M * hid);
      dq_ = carve<T>(p, M * d);
      dk_ = carve<T>(p, M * d);
      dv_ = carve<T>(p, M * d);
      dO_ = carve<T>(p, M * d);
      rowloss_ = carve<double>(p, M);
      return (size_t)(p - s);
    };
    const size_t bytes = plan(reinterpret_cast<char*>(256));  // dry run for the size
    // + 64: a runner with one local client aggregates straight out of master,
    // reading whole boundary shards (up to Ppad = P rounded to 4 * world <= P + 31)
    PH_CUDA(cudaMalloc(&master_alloc_, (P + 64) * sizeof(float)));
    master = master_alloc_;
    PH_CUDA(cudaMemsetAsync(master, 0, (P + 64) * sizeof(float), stream));
    PH_CUDA(cudaMalloc(&pool_, bytes + 256));
    plan(pool_);
    PH_CUDA(cudaMemsetAsync(pool_, 0, bytes, stream));
  }

  // ---- timing helpers ----
  cudaEvent_t next_event() {
    if (ev_next_ == ev_pool_.size()) {
      cudaEvent_t e;
      PH_CUDA(cudaEventCreate(&e));
      ev_pool_.push_back(e);
    }
    return ev_pool_[ev_next_++];
  }
  struct Scope {
    EngineT* e;
    int cat;
    double flops;
    cudaEvent_t a = nullptr;
    Scope(EngineT* eng, int c, double f) : e(eng), cat(c), flops(f) {
      if (e->timing) {
        a = e->next_event();
        PH_CUDA(cudaEventRecord(a, e->stream));
      }
    }
    ~Scope() noexcept(false) {
      if (e->timing) {
        cudaEvent_t b = e->next_event();
        PH_CUDA(cudaEventRecord(b, e->stream));
        e->spans_.push_back(Span{cat, a, b, flops});
      }
    }
  };
  void collect_times() {
    if (!timing) return;
    PH_CUDA(cudaStreamSynchronize(stream));
    for (auto& s : spans_) {
      float ms = 0.f;
      PH_CUDA(cudaEventElapsedTime(&ms, s.a, s.b));
      if (s.cat == 0) { times.gemm_ms += ms; times.gemm_flops += s.flops; ++times.gemm_launches; }
      else if (s.cat == 1) { times.attn_ms += ms; times.attn_flops += s.flops; ++times.attn_launches; }
      else times.other_ms += ms;
      ++times.launches;
    }
    spans_.clear();
    ev_next_ = 0;
  }

  bool use_mma_attn() const {
    return sizeof(T) == 2 && attn_mode >= 1 && k::attn_mma_supported((int)(d_ / H_));
  }
  void attn_fwd(const T* q, const T* k, const T* v, T* o, float* lse, int B, int S, int H, int d) {
    if constexpr (sizeof(T) == 2) {
      if (attn_mode == 1 && k::attn_tc_supported((int)(d_ / H_), d)) {
        k::attn_fwd_tc(q, k, v, o, lse, B, S, H, d, stream);
        return;
      }
      if (use_mma_attn()) {
        k::attn_fwd_mma(q, k, v, o, lse, B, S, H, d, stream);
        return;
      }
    }
    k::attn_fwd_simt<T>(q, k, v, o, lse, B, S, H, d, stream);
  }
  // true when the q / k / v column sums came with it (attn_bwd_sums_floats in sums)
  bool attn_bwd(const T* q, const T* k, const T* v, const T* o, const T* dO, const float* lse,
                int B, int S, int H, int d, float* sums) {
    if constexpr (sizeof(T) == 2) {
      if (attn_mode == 1 && k::attn_tc_supported((int)(d_ / H_), d)) {
        k::attn_bwd_tc(q, k, v, o, dO, lse, dq_, dk_, dv_, B, S, H, d, attn_ws_, stream, sums);
        return true;
      }
      if (use_mma_attn()) {
        k::attn_bwd_mma(q, k, v, o, dO, lse, Dvec_, dq_, dk_, dv_, B, S, H, d, stream);
        return false;
      }
    }
    k::attn_bwd_simt<T>(q, k, v, o, dO, lse, Dvec_, dq_, dk_, dv_, B, S, H, d, stream);
    return false;
  }

  void mm(int M, int N, int K, const void* A, int64_t lda, bool ak, const void* B, int64_t ldb,
          bool bk, void* C, int64_t ldc, DT cdt, Epi epi, const float* bias = nullptr,
          const float* resid = nullptr, void* aux = nullptr, float* colsum_part = nullptr) {
    GemmArgs g;
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.lda = lda; g.a_kmajor = ak;
    g.B = B; g.ldb = ldb; g.b_kmajor = bk;
    g.ab = dt_of<T>();
    g.C = C; g.ldc = ldc; g.c = cdt;
    g.epi = epi; g.bias = bias; g.resid = resid; g.aux = aux;
    g.ws = gemm_ws_; g.ws_floats = gemm_ws_ ? kGemmWsFloats : 0;
    g.colsum_part = colsum_part;
    Scope sc(this, 0, 2.0 * M * N * (double)K);
    if (sizeof(T) == 2 && gemm_mode == 1) {
      if (!gemm_tc(g, stream))
        throw Error(PHOTON_ERR_CONFIG, "tcgen05 GEMM does not support this shape/layout");
    } else {
      gemm_simt(g, stream);
    }
  }
};

// A step's batch larger than the activation capacity (max_batch rows) runs as
// micro-batches of at most max_batch rows: every gradient write of the later
// micro-batches adds onto the earlier ones (GEMM Accum epilogues, accumulating
// column reductions), the cross-entropy scale stays 1 / #targets of the whole
// batch, so the step's loss and gradient are those of the full batch
// (client.cpp:135-154: one mean over all local-batch targets).
template <typename T>
void EngineT<T>::forward_backward(const StepBatch& bt, double* loss_dev, bool backward) {
  PdlScope pdl(d_ <= kPdlMaxWidth);  // launch-bound small models only (common.cuh)
  if ((uint64_t)bt.S > Smax_)
    throw Error(PHOTON_ERR_SHAPE, "sequence exceeds the context's seq_len");
  const int mb = (int)max_batch;
  for (int r0 = 0, j = 0; r0 < bt.B; r0 += mb, ++j) {
    StepBatch sb = bt;
    sb.B = std::min(mb, bt.B - r0);
    sb.tokens = bt.tokens + (size_t)r0 * bt.S;
    sb.targets = bt.targets + (size_t)r0 * bt.S;
    micro(sb, loss_dev, backward, j > 0, r0 * bt.S);
  }
}

template <typename T>
void EngineT<T>::micro(const StepBatch& bt, double* loss_dev, bool backward, bool acc, int row0) {
  jobs_.rows.clear();  // (a pass that threw left its jobs behind)
  jobs_.cols.clear();
  const int B = bt.B, S = bt.S, M = B * S;
  const int d = (int)d_, hid = (int)hid_, V = (int)V_, H = (int)H_, L = (int)L_;
  // weight gradients: stored by the first micro-batch, accumulated by the rest
  const Epi WG = acc ? Epi::Accum : Epi::Store;
  bool head_b_done = false;
  const size_t Md = (size_t)M * d, Mh = (size_t)M * hid;
  const double attn_fwd_flops = 4.0 * B * H * (d / H) * (double)S * (S + 1) / 2.0;
  const DT TT = dt_of<T>();

  // ---------------- forward (model.cpp:140-156) ----------------
  {
    Scope sc(this, 2, 0);
    k::embed_fwd(bt.tokens, Pm(off_.tok), Pm(off_.pos), x_, M, S, d, stream);
  }
  for (int l = 0; l < L; ++l) {
    const BlockOffsets& o = off_.blocks[l];
    float* x = x_ + (size_t)l * Md;
    float* xm = xmid_ + (size_t)l * Md;
    T *h = h_ + l * Md, *q = q_ + l * Md, *kk = k_ + l * Md, *v = v_ + l * Md, *ao = o_ + l * Md;
    T *h2 = h2_ + l * Md, *pre = pre_ + l * Mh, *u = u_ + l * Mh;
    {
      Scope sc(this, 2, 0);
      k::ln_fwd<T>(x, Pm(o.ln1g), Pm(o.ln1b), h, mean1_ + (size_t)l * M, rstd1_ + (size_t)l * M, M,
                   d, stream);
    }
    mm(M, d, d, h, d, true, W(o.wq), d, false, q, d, TT, Epi::Bias, Pm(o.bq));
    mm(M, d, d, h, d, true, W(o.wk), d, false, kk, d, TT, Epi::Bias, Pm(o.bk));
    mm(M, d, d, h, d, true, W(o.wv), d, false, v, d, TT, Epi::Bias, Pm(o.bv));
    {
      Scope sc(this, 1, attn_fwd_flops);
      attn_fwd(q, kk, v, ao, lse_ + (size_t)l * B * H * S, B, S, H, d);
    }
    mm(M, d, d, ao, d, true, W(o.wo), d, false, xm, d, DT::F32, Epi::ResidBias, Pm(o.bo), x);
    {
      Scope sc(this, 2, 0);
      k::ln_fwd<T>(xm, Pm(o.ln2g), Pm(o.ln2b), h2, mean2_ + (size_t)l * M, rstd2_ + (size_t)l * M,
                   M, d, stream);
    }
    mm(M, hid, d, h2, d, true, W(o.w1), hid, false, u, hid, TT, Epi::GeluBias, Pm(o.b1), nullptr,
       pre);
    mm(M, d, hid, u, hid, true, W(o.w2), d, false, x + Md, d, DT::F32, Epi::ResidBias, Pm(o.b2),
       xm);
  }
  float* xL = x_ + (size_t)L * Md;
  {
    Scope sc(this, 2, 0);
    k::ln_fwd<T>(xL, Pm(off_.lnfg), Pm(off_.lnfb), xf_, meanf_, rstdf_, M, d, stream);
  }
  mm(M, V, d, xf_, d, true, W(off_.head_w), V, false, logits_, V, TT, Epi::Bias, Pm(off_.head_b));
  {
    Scope sc(this, 2, 0);
    // the head-bias gradient (column sums of dlogits) comes out of the
    // cross-entropy pass where the kernel supports the shape
    head_b_done = k::ce_fwd_bwd<T>(logits_, bt.targets, M, V, bt.inv_count, rowloss_, backward,
                                   stream, backward ? G(off_.head_b) : nullptr,
                                   defer_ + L_ * (2 * defer_ln_ + defer_b1_ + defer_qkv_) + defer_ln_,
                                   acc, bt.inv_count_dev, &jobs_);
    k::sum_scaled(rowloss_, M, (double)bt.inv_count, loss_dev, stream, acc, bt.inv_count_dev);
  }
  if (!backward) {
    collect_times();
    return;
  }

  // ---------------- backward (reverse topological order) ----------------
  // every gradient entry is written (stored, never accumulated) by exactly one
  // kernel below -- except the position embeddings of positions this batch
  // does not reach (S < seq_len), which are zero
  if ((uint64_t)S < Smax_ && !acc)
    PH_CUDA(cudaMemsetAsync(G(off_.pos) + (size_t)S * d, 0, (Smax_ - S) * d * sizeof(float),
                            stream));
  // logits = add_bias(xf W_head, b_head)
  if (!head_b_done) {
    Scope sc(this, 2, 0);
    k::colsum<T>(logits_, M, V, part_, G(off_.head_b), stream, acc);
  }
  mm(M, d, V, logits_, V, true, W(off_.head_w), V, true, dyT_, d, TT, Epi::Store);
  if (sizeof(T) == 2 && gemm_mode == 1 && M % 8 == 0) {
    // K-major A for the head weight gradient: xf transposed into dq_ (free until
    // the last block's attention backward); 4.3 -> 3.6 ms for the contraction
    {
      Scope sc(this, 2, 0);
      k::transpose_bf16(reinterpret_cast<const bf16*>(xf_), M, d, reinterpret_cast<bf16*>(dq_), stream);
    }
    mm(d, V, M, dq_, M, true, logits_, V, false, G(off_.head_w), V, DT::F32, WG);
  } else {
    mm(d, V, M, xf_, d, false, logits_, V, false, G(off_.head_w), V, DT::F32, WG);
  }
  {
    Scope sc(this, 2, 0);
    // the column sums of its output are the last block's b2 gradient
    k::ln_bwd<T>(dyT_, xL, meanf_, rstdf_, Pm(off_.lnfg), nullptr, dx_, dxT_,
                 defer_ + L_ * (2 * defer_ln_ + defer_b1_ + defer_qkv_), G(off_.lnfg),
                 G(off_.lnfb), M, d, stream, G(off_.blocks[L - 1].b2), acc, &jobs_);
  }
  for (int l = L - 1; l >= 0; --l) {
    const BlockOffsets& o = off_.blocks[l];
    // this layer's slices of the deferred-reduction partials
    float* pl = defer_ + (size_t)l * (2 * defer_ln_ + defer_b1_ + defer_qkv_);
    float *p_ln2 = pl, *p_b1 = pl + defer_ln_, *p_qkv = p_b1 + defer_b1_, *p_ln1 = p_qkv + defer_qkv_;
    float* x = x_ + (size_t)l * Md;
    float* xm = xmid_ + (size_t)l * Md;
    T *h = h_ + l * Md, *q = q_ + l * Md, *kk = k_ + l * Md, *v = v_ + l * Md, *ao = o_ + l * Md;
    T *h2 = h2_ + l * Md, *pre = pre_ + l * Mh, *u = u_ + l * Mh;
    // x_out = x_mid + (u W2 + b2); db2 came with the LayerNorm backward above
    // pre = h2 W1 + b1: on the tensor-core path the GeluBwd epilogue also emits
    // the column sums of every 32-row block of dpre (fp32, before rounding)
    bool fuse_b1 = false;
    if (sizeof(T) == 2 && gemm_mode == 1 && M % 32 == 0) {
      GemmArgs ga;
      ga.M = M; ga.N = hid; ga.K = d;
      ga.A = dxT_; ga.lda = d; ga.a_kmajor = true;
      ga.B = W(o.w2); ga.ldb = d; ga.b_kmajor = true;
      ga.ab = TT; ga.C = dpre_; ga.ldc = hid; ga.c = TT;
      ga.epi = Epi::GeluBwd; ga.aux = pre;
      fuse_b1 = gemm_tc_single_pass(ga);
    }
    mm(M, hid, d, dxT_, d, true, W(o.w2), d, true, dpre_, hid, TT, Epi::GeluBwd, nullptr, nullptr,
       pre, fuse_b1 ? p_b1 : nullptr);
    mm(hid, d, M, u, hid, false, dxT_, d, false, G(o.w2), d, DT::F32, WG);
    {
      Scope sc(this, 2, 0);
      if (fuse_b1)
        k::colsum_parts(p_b1, M / 32, hid, p_b1 + (size_t)(M / 32) * hid, G(o.b1), stream, acc,
                        &jobs_);
      else
        k::colsum<T>(dpre_, M, hid, part_, G(o.b1), stream, acc);
    }
    mm(M, d, hid, dpre_, hid, true, W(o.w1), hid, true, dyT_, d, TT, Epi::Store);
    mm(d, hid, M, h2, d, false, dpre_, hid, false, G(o.w1), hid, DT::F32, WG);
    {
      Scope sc(this, 2, 0);
      // x_mid = x + (o Wo + bo): dbo = column sums of this output
      k::ln_bwd<T>(dyT_, xm, mean2_ + (size_t)l * M, rstd2_ + (size_t)l * M, Pm(o.ln2g), dx_, dx_,
                   dxT_, p_ln2, G(o.ln2g), G(o.ln2b), M, d, stream, G(o.bo), acc, &jobs_);
    }
    mm(M, d, d, dxT_, d, true, W(o.wo), d, true, dO_, d, TT, Epi::Store);
    mm(d, d, M, ao, d, false, dxT_, d, false, G(o.wo), d, DT::F32, WG);
    bool qkv_sums;
    {
      Scope sc(this, 1, 2.5 * attn_fwd_flops);
      qkv_sums = attn_bwd(q, kk, v, ao, dO_, lse_ + (size_t)l * B * H * S, B, S, H, d, p_qkv);
    }
    // q,k,v = h W{q,k,v} + b{q,k,v}; LN1's output grad sums v, k, q in that order
    {
      Scope sc(this, 2, 0);
      if (qkv_sums) {  // partials from the attention backward's stores
        const int np = B * ((S + 31) / 32);
        const size_t P = (size_t)np * d;
        float* scr = p_qkv + 3 * P;
        k::colsum_parts3(p_qkv, P, np, d, scr, G(o.bq), G(o.bk), G(o.bv), stream, acc, &jobs_);
      } else {
        k::colsum<T>(dv_, M, d, part_, G(o.bv), stream, acc);
        k::colsum<T>(dk_, M, d, part_, G(o.bk), stream, acc);
        k::colsum<T>(dq_, M, d, part_, G(o.bq), stream, acc);
      }
    }
    // dy = dv Wv^T + dk Wk^T + dq Wq^T: one K-concatenated contraction on the
    // tensor-core path (one fp32 pass over dy instead of a store + two RMWs)
    if (sizeof(T) == 2 && gemm_mode == 1 && d % 64 == 0) {
      GemmArgs g;
      g.M = M; g.N = d; g.K = d;
      g.A = dv_; g.lda = d; g.a_kmajor = true;
      g.B = W(o.wv); g.ldb = d; g.b_kmajor = true;
      g.ab = dt_of<T>();
      g.C = dyT_; g.ldc = d; g.c = dt_of<T>();
      g.epi = Epi::Store;
      g.nseg = 3;
      g.A_seg[1] = dk_; g.B_seg[1] = W(o.wk);
      g.A_seg[2] = dq_; g.B_seg[2] = W(o.wq);
      g.ws = gemm_ws_; g.ws_floats = kGemmWsFloats;
      Scope sc(this, 0, 2.0 * M * d * 3.0 * d);
      if (!gemm_tc(g, stream)) throw Error(PHOTON_ERR_CONFIG, "tcgen05 GEMM: K-concatenated dX");
    } else {
      mm(M, d, d, dv_, d, true, W(o.wv), d, true, dy_, d, DT::F32, Epi::Store);
      mm(M, d, d, dk_, d, true, W(o.wk), d, true, dy_, d, DT::F32, Epi::Accum);
      mm(M, d, d, dq_, d, true, W(o.wq), d, true, dy_, d, DT::F32, Epi::Accum);
      if (sizeof(T) == 2) k::f32_to_bf16(dy_, reinterpret_cast<bf16*>(dyT_), (uint64_t)M * d, stream);
    }
    mm(d, d, M, h, d, false, dv_, d, false, G(o.wv), d, DT::F32, WG);
    mm(d, d, M, h, d, false, dk_, d, false, G(o.wk), d, DT::F32, WG);
    mm(d, d, M, h, d, false, dq_, d, false, G(o.wq), d, DT::F32, WG);
    {
      Scope sc(this, 2, 0);
      // the output is block l-1's x_out gradient: its column sums are db2 of l-1
      k::ln_bwd<T>(dyT_, x, mean1_ + (size_t)l * M, rstd1_ + (size_t)l * M, Pm(o.ln1g), dx_, dx_,
                   dxT_, p_ln1, G(o.ln1g), G(o.ln1b), M, d, stream,
                   l > 0 ? G(off_.blocks[l - 1].b2) : nullptr, acc, &jobs_);
    }
  }
  {
    Scope sc(this, 2, 0);
    // every deferred bias / LayerNorm-gain reduction of the pass: two launches
    k::run_reduce_jobs(jobs_, stream);
    k::embed_bwd(dx_, bt.csr_off, bt.csr_rows, G(off_.tok), G(off_.pos), V, M, S, d, stream, row0,
                 acc);
  }
  collect_times();
}

}  // namespace

std::unique_ptr<Engine> Engine::create(const photon_model_cfg& cfg, int precision,
                                       uint64_t max_batch, cudaStream_t st) {
  validate_model(cfg);
  if (max_batch == 0) throw Error(PHOTON_ERR_CONFIG, "max_batch must be >= 1");
  if (precision == PHOTON_PREC_F32) return std::make_unique<EngineT<float>>(cfg, precision, max_batch, st);
  if (precision == PHOTON_PREC_BF16) return std::make_unique<EngineT<bf16>>(cfg, precision, max_batch, st);
  throw Error(PHOTON_ERR_CONFIG, "unknown precision");
}

}  // namespace photon
