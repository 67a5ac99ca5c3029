// ctx.cpp -- device context and the device-resident client update.
#include "ctx.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include <cmath>

#include "kernels.cuh"

namespace photon {

void RoundBatches::prepare(int tau_, int B_, int S_, int V) {
  tau = tau_;
  B = B_;
  S = S_;
  const size_t M = (size_t)B * S;
  tokens.reserve(tau * M);
  targets.reserve(tau * M);
  csr_off.reserve((size_t)tau * (V + 1));
  csr_rows.reserve(tau * M);
  inv_count.assign(tau, 0.f);
}

void RoundBatches::finalize(int V) {
  const int M = B * S;
  for (int i = 0; i < tau; ++i) {
    const int32_t* tk = tokens.ptr + (size_t)i * M;
    for (int m = 0; m < M; ++m)
      if (tk[m] < 0 || tk[m] >= V)
        throw Error(PHOTON_ERR_INDEX, "gather_rows: index " + std::to_string(tk[m]) +
                                          " out of range [0," + std::to_string(V) + ")");
    build_token_csr(tk, M, V, csr_off.ptr + (size_t)i * (V + 1), csr_rows.ptr + (size_t)i * M);
    const int32_t* tg = targets.ptr + (size_t)i * M;
    int count = 0;
    for (int m = 0; m < M; ++m) {
      if (tg[m] >= V) throw Error(PHOTON_ERR_INDEX, "cross_entropy: target out of vocab");
      count += tg[m] >= 0;
    }
    if (count == 0) throw Error(PHOTON_ERR_USAGE, "cross_entropy: no target tokens");
    inv_count[i] = (float)(1.0 / (double)count);
  }
}

Ctx::Ctx(int dev, const photon_model_cfg& m, int prec, uint64_t mb)
    : device(dev), cfg(m), precision(prec), max_batch(mb) {
  validate_model(m);
  if (const char* g = std::getenv("PHOTON_GRAPHS")) graphs_on = std::string(g) != "0";
  PH_CUDA(cudaSetDevice(dev));
  PH_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  PH_CUDA(cudaEventCreate(&ev0));
  PH_CUDA(cudaEventCreate(&ev1));
  eng = Engine::create(m, prec, mb, stream);
  h_flag.reserve(4);
}

Ctx::~Ctx() {
  for (auto& kv : graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  eng.reset();
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (stream) cudaStreamDestroy(stream);
}

void Ctx::begin_timing() { PH_CUDA(cudaEventRecord(ev0, stream)); }

double Ctx::end_timing() {
  PH_CUDA(cudaEventRecord(ev1, stream));
  PH_CUDA(cudaEventSynchronize(ev1));
  float ms = 0.f;
  PH_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
  last_ms = ms;
  return ms;
}

void DeviceBatches::upload(const RoundBatches& rb, int V, cudaStream_t st) {
  const size_t M = (size_t)rb.B * rb.S;
  tau = rb.tau;
  B = rb.B;
  S = rb.S;
  inv_count = rb.inv_count;
  tokens.reserve(rb.tau * M);
  targets.reserve(rb.tau * M);
  csr_off.reserve(rb.tau * (size_t)(V + 1));
  csr_rows.reserve(rb.tau * M);
  PH_CUDA(cudaMemcpyAsync(tokens.ptr, rb.tokens.ptr, rb.tau * M * 4, cudaMemcpyHostToDevice, st));
  PH_CUDA(cudaMemcpyAsync(targets.ptr, rb.targets.ptr, rb.tau * M * 4, cudaMemcpyHostToDevice, st));
  PH_CUDA(cudaMemcpyAsync(csr_off.ptr, rb.csr_off.ptr, rb.tau * (size_t)(V + 1) * 4,
                          cudaMemcpyHostToDevice, st));
  PH_CUDA(cudaMemcpyAsync(csr_rows.ptr, rb.csr_rows.ptr, rb.tau * M * 4, cudaMemcpyHostToDevice, st));
  // pageable source: staged by the call, so the host vector may change after it returns
  inv_dev.reserve(std::max(rb.tau, 1));
  PH_CUDA(cudaMemcpyAsync(inv_dev.ptr, rb.inv_count.data(), rb.tau * sizeof(float),
                          cudaMemcpyHostToDevice, st));
}

void Ctx::upload(const RoundBatches& rb) { dev_batches.upload(rb, (int)cfg.vocab_size, stream); }

// optim.cpp:20-35, 105-113 validation of the client hyper-parameters
void check_train_cfg(const photon_train_cfg& t) {
  validate_model(t.model);
  const auto& a = t.adamw;
  if (a.beta1 < 0.0 || a.beta1 >= 1.0 || a.beta2 < 0.0 || a.beta2 >= 1.0)
    throw Error(PHOTON_ERR_CONFIG, "adamw: betas must be in [0,1)");
  if (!(a.eps > 0.0)) throw Error(PHOTON_ERR_CONFIG, "adamw: eps must be > 0");
  if (a.weight_decay < 0.0) throw Error(PHOTON_ERR_CONFIG, "adamw: weight_decay must be >= 0");
  if (t.opt != 0 && t.opt != 1) throw Error(PHOTON_ERR_CONFIG, "unknown client optimizer");
  if (t.batch_size == 0) throw Error(PHOTON_ERR_CONFIG, "stream: batch_size must be >= 1");
  if (t.post_kind == 1 && !(t.post_threshold > 0.0))
    throw Error(PHOTON_ERR_CONFIG, "clip post-process needs a positive threshold");
  (void)lr_at(t.schedule, 0);  // validates the schedule
}

// run_local_round (client.cpp:125-158) on the device: theta copy, fresh AdamW
// state, tau x {forward, backward, clip, AdamW/SGD}, post-process.  Losses stay
// on the device until the caller reads them once per round.  lr_dev (optional):
// the per-step learning rates on the device, read instead of the host values.
static void enqueue_local_round(Ctx& c, const photon_train_cfg& t, const DeviceBatches& db,
                                const float* d_theta_in, float* d_theta_out, uint64_t step_base,
                                double* d_loss, int* d_flag, const double* lr_dev) {
  Engine& e = *c.eng;
  cudaStream_t stream = c.stream;
  const uint64_t P = e.P;
  if (d_theta_in != e.master)
    PH_CUDA(cudaMemcpyAsync(e.master, d_theta_in, P * 4, cudaMemcpyDeviceToDevice, stream));
  e.refresh_shadow();
  PH_CUDA(cudaMemsetAsync(e.mom, 0, P * 4, stream));
  PH_CUDA(cudaMemsetAsync(e.vel2, 0, P * 4, stream));
  PH_CUDA(cudaMemsetAsync(e.bad_step, 0, sizeof(int), stream));
  const size_t M = (size_t)db.B * db.S, V = c.cfg.vocab_size;
  const double b1 = t.adamw.beta1, b2 = t.adamw.beta2;
  for (int i = 0; i < db.tau; ++i) {
    StepBatch sb;
    sb.tokens = db.tokens.ptr + i * M;
    sb.targets = db.targets.ptr + i * M;
    sb.csr_off = db.csr_off.ptr + i * (V + 1);
    sb.csr_rows = db.csr_rows.ptr + i * M;
    sb.B = db.B;
    sb.S = db.S;
    sb.inv_count = db.inv_count[i];
    sb.inv_count_dev = lr_dev ? db.inv_dev.ptr + i : nullptr;
    e.forward_backward(sb, d_loss + i, true);
    const double lr = lr_at(t.schedule, step_base + i);
    if (t.opt == 0) {
      const double stepc = (double)(i + 1);  // fresh state each round: step_count = i+1
      e.adamw(t.adamw.clip_norm, lr, b1, b2, 1.0 - std::pow(b1, stepc), 1.0 - std::pow(b2, stepc),
              t.adamw.eps, t.adamw.weight_decay, i, lr_dev ? lr_dev + i : nullptr);
    } else {
      e.sgd(t.sgd_clip_norm, lr, i, lr_dev ? lr_dev + i : nullptr);
    }
  }
  if (t.post_kind == 1)
    k::clip_update_f32(d_theta_in, e.master, P, t.post_threshold, e.red_part, stream);
  if (d_theta_out != e.master)
    PH_CUDA(cudaMemcpyAsync(d_theta_out, e.master, P * 4, cudaMemcpyDeviceToDevice, stream));
  PH_CUDA(cudaMemcpyAsync(d_flag, e.bad_step, sizeof(int), cudaMemcpyDeviceToDevice, stream));
}

void Ctx::launch_local_round(const photon_train_cfg& t, const DeviceBatches& db,
                             const float* d_theta_in, float* d_theta_out, uint64_t step_base,
                             double* d_loss, int* d_flag) {
  PdlScope pdl(cfg.d_model <= kPdlMaxWidth);  // launch-bound small models only (common.cuh)
  if (!graphs_on || eng->timing || db.tau < 1) {
    enqueue_local_round(*this, t, db, d_theta_in, d_theta_out, step_base, d_loss, d_flag, nullptr);
    return;
  }
  d_lr.reserve(std::max(db.tau, 64));  // before the key: a reserve that moves it re-keys
  // everything the captured launches depend on, except the per-round data that
  // lives in device memory (tokens, targets, CSR, 1/#targets, lr)
  char key[512];
  std::snprintf(key, sizeof(key), "%p %p %p %p %p %p %p %p %p %p %d %d %d %d %d %.17g %.17g %.17g "
                "%.17g %.17g %.17g %.17g %d %.17g",
                (const void*)d_lr.ptr,
                (const void*)db.tokens.ptr, (const void*)db.targets.ptr, (const void*)db.csr_off.ptr,
                (const void*)db.csr_rows.ptr, (const void*)db.inv_dev.ptr, (const void*)d_theta_in,
                (const void*)d_theta_out, (const void*)d_loss, (const void*)d_flag, db.tau, db.B,
                db.S, (int)t.opt, (int)t.post_kind, t.adamw.beta1, t.adamw.beta2, t.adamw.eps,
                t.adamw.weight_decay, t.adamw.clip_norm, t.sgd_clip_norm, t.post_threshold,
                (int)max_batch, t.schedule.eta_max);
  std::vector<double> lr(db.tau);
  for (int i = 0; i < db.tau; ++i) lr[i] = lr_at(t.schedule, step_base + i);
  RoundGraph& g = graphs[key];
  // per-round device scalars: pageable source, staged by the call
  PH_CUDA(cudaMemcpyAsync(d_lr.ptr, lr.data(), db.tau * sizeof(double), cudaMemcpyHostToDevice,
                          stream));
  if (!g.exec && g.seen++ >= 1) {
    cudaGraph_t graph = nullptr;
    const uint64_t n0 = launch_counter().load();
    PH_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_local_round(*this, t, db, d_theta_in, d_theta_out, step_base, d_loss, d_flag,
                          d_lr.ptr);
    } catch (...) {
      cudaStreamEndCapture(stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
      graphs_on = false;  // this context stays eager from here on
      throw;
    }
    PH_CUDA(cudaStreamEndCapture(stream, &graph));
    // captured launches did not run: count the graph's kernel nodes per replay
    launch_counter().fetch_sub(launch_counter().load() - n0);
    size_t nn = 0;
    PH_CUDA(cudaGraphGetNodes(graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    if (nn) PH_CUDA(cudaGraphGetNodes(graph, nodes.data(), &nn));
    g.kernels = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType ty;
      PH_CUDA(cudaGraphNodeGetType(nd, &ty));
      g.kernels += ty == cudaGraphNodeTypeKernel;
    }
    const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      cudaGetLastError();
      g.exec = nullptr;
      graphs_on = false;
    }
  }
  if (g.exec) {
    PH_CUDA(cudaGraphLaunch(g.exec, stream));
    launch_counter().fetch_add(g.kernels);
  } else
    enqueue_local_round(*this, t, db, d_theta_in, d_theta_out, step_base, d_loss, d_flag,
                           d_lr.ptr);
}

constexpr uint64_t kStageChunk = 1ull << 24;  // 16 M values = 128 MB of f64 staging

void Ctx::h2d_f64_to_f32(const double* host, float* dev, uint64_t n) {
  d_f64a.reserve(std::min(n, kStageChunk));
  for (uint64_t o = 0; o < n; o += kStageChunk) {
    const uint64_t c = std::min(kStageChunk, n - o);
    PH_CUDA(cudaMemcpyAsync(d_f64a.ptr, host + o, c * 8, cudaMemcpyHostToDevice, stream));
    k::f64_to_f32(d_f64a.ptr, dev + o, c, stream);
  }
}

void Ctx::d2h_f32_to_f64(const float* dev, double* host, uint64_t n) {
  d_f64a.reserve(std::min(n, kStageChunk));
  for (uint64_t o = 0; o < n; o += kStageChunk) {
    const uint64_t c = std::min(kStageChunk, n - o);
    k::f32_to_f64(dev + o, d_f64a.ptr, c, stream);
    PH_CUDA(cudaMemcpyAsync(host + o, d_f64a.ptr, c * 8, cudaMemcpyDeviceToHost, stream));
  }
  PH_CUDA(cudaStreamSynchronize(stream));
}

LocalResult classify(const double* losses, int tau, int bad) {
  LocalResult r;
  r.losses.assign(losses, losses + tau);
  for (int i = 0; i < tau; ++i) {
    if (!std::isfinite(r.losses[i])) {
      r.error = PHOTON_ERR_DIVERGENCE;
      r.error_step = i;
      break;
    }
    if (bad == i + 1) {
      r.error = PHOTON_ERR_NUMERIC;
      r.error_step = i;
      break;
    }
  }
  return r;
}

LocalResult Ctx::local_round(const photon_train_cfg& t, const float* d_theta_in,
                             float* d_theta_out, uint64_t step_base) {
  const int tau = dev_batches.tau;
  d_losses.reserve(std::max(tau, 1));
  h_losses.reserve(std::max(tau, 1));
  d_flags.reserve(1);
  launch_local_round(t, dev_batches, d_theta_in, d_theta_out, step_base, d_losses.ptr, d_flags.ptr);
  PH_CUDA(cudaMemcpyAsync(h_losses.ptr, d_losses.ptr, tau * sizeof(double), cudaMemcpyDeviceToHost, stream));
  PH_CUDA(cudaMemcpyAsync(h_flag.ptr, d_flags.ptr, sizeof(int), cudaMemcpyDeviceToHost, stream));
  PH_CUDA(cudaStreamSynchronize(stream));
  return classify(h_losses.ptr, tau, h_flag.ptr[0]);
}

}  // namespace photon
