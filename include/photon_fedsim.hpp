// photon_fedsim.hpp -- header-only adapter: the reference's client-update,
// aggregator and outer-optimizer C++ interfaces implemented over photon.h.
//
// A maintainer of fedsim::core adds this header and links libphoton.so; call
// sites keep the reference signatures:
//   client.h:97-99        run_local_round(theta_t, stream, cfg, round, client, step_base)
//   param_vector.h:50-54  ParamVector::mean(vs) / ParamVector::sub(a, b)
//   optim.h:78            server_step(state, theta, delta, client_mean)
//   optim.h:46-52         adamw_step / sgd_step
// Errors come back as the same fedsim:: exception types (errors.h:9-72).
#pragma once

#include <cstring>
#include <memory>
#include <stdexcept>
#include <vector>

#include "fedsim/client.h"
#include "fedsim/data.h"
#include "fedsim/errors.h"
#include "fedsim/optim.h"
#include "fedsim/param_vector.h"
#include "photon.h"

namespace photon_fedsim {

inline void check(int rc, const photon_err& e) {
  if (rc == PHOTON_OK) return;
  switch (rc) {
    case PHOTON_ERR_CAPACITY: throw fedsim::CapacityError(e.msg);
    case PHOTON_ERR_CONFIG: throw fedsim::ConfigError(e.msg);
    case PHOTON_ERR_SHAPE: throw fedsim::ShapeError(e.msg);
    case PHOTON_ERR_INDEX: throw fedsim::IndexError(e.msg);
    case PHOTON_ERR_USAGE: throw fedsim::UsageError(e.msg);
    case PHOTON_ERR_LOOKUP: throw fedsim::LookupError(e.msg);
    case PHOTON_ERR_NUMERIC: throw fedsim::NumericError(e.msg);
    case PHOTON_ERR_DIVERGENCE:
      throw fedsim::DivergenceError(e.msg, e.round, e.client, e.step);
    case PHOTON_ERR_IO: throw fedsim::IoError(e.msg);
    case PHOTON_ERR_INTEGRITY: throw fedsim::IntegrityError(e.msg);
    case PHOTON_ERR_ROUND_FAILURE: throw fedsim::RoundFailureError(e.msg);
    case PHOTON_ERR_PARSE: throw fedsim::ParseError(e.msg);
    default: throw std::runtime_error(std::string("photon: ") + e.msg);
  }
}

inline photon_model_cfg to_c(const fedsim::ModelConfig& m) {
  return photon_model_cfg{m.n_blocks, m.d_model, m.n_heads, m.expansion_ratio, m.vocab_size,
                          m.seq_len};
}

inline photon_train_cfg to_c(const fedsim::LocalTrainConfig& c) {
  photon_train_cfg t{};
  t.model = to_c(c.model);
  t.adamw = photon_adamw_cfg{c.adamw.beta1, c.adamw.beta2, c.adamw.eps, c.adamw.weight_decay,
                             c.adamw.clip_norm};
  t.schedule = photon_lr_schedule{c.schedule.eta_max, c.schedule.warmup_steps,
                                  c.schedule.decay_steps, c.schedule.alpha};
  t.opt = c.opt == fedsim::ClientOptKind::kAdamW ? 0 : 1;
  t.sgd_clip_norm = c.sgd_clip_norm;
  t.local_steps = c.local_steps;
  t.batch_size = c.batch_size;
  t.throughput_bps = c.throughput_bps;
  t.post_kind = c.post.kind == fedsim::PostProcessPolicy::Kind::kIdentity ? 0 : 1;
  t.post_threshold = c.post.threshold;
  return t;
}

inline photon_server_cfg to_c(const fedsim::ServerOptConfig& s) {
  return photon_server_cfg{s.kind == fedsim::ServerOptKind::FedAvg ? 0 : 1, s.eta, s.momentum,
                           s.nesterov ? 1 : 0};
}

// A GPU engine for one model shape (one client slot).
class Device {
 public:
  Device(int device, const fedsim::ModelConfig& m, std::size_t max_batch,
         int precision = PHOTON_PREC_BF16) {
    photon_err e{};
    const photon_model_cfg c = to_c(m);
    check(photon_ctx_create(device, &c, precision, max_batch, &ctx_, &e), e);
  }
  ~Device() { photon_ctx_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  photon_ctx* get() const { return ctx_; }

 private:
  photon_ctx* ctx_ = nullptr;
};

// client.h:97-99 -- the stream stays the reference's own BatchStream (host,
// unchanged); its tau batches are handed to the device in one call.
inline fedsim::ClientResult run_local_round(Device& dev, const fedsim::ParamVector& theta_t,
                                            fedsim::BatchStream& stream,
                                            const fedsim::LocalTrainConfig& cfg,
                                            std::size_t round, std::size_t client_id,
                                            std::size_t step_base) {
  const std::size_t tau = cfg.local_steps, B = cfg.batch_size, S = cfg.model.seq_len;
  std::vector<int32_t> inputs(tau * B * S), targets(tau * B * S);
  for (std::size_t i = 0; i < tau; ++i) {
    fedsim::Batch b = stream.next();
    std::memcpy(inputs.data() + i * B * S, b.inputs.data(), B * S * 4);
    std::memcpy(targets.data() + i * B * S, b.targets.data(), B * S * 4);
  }
  const std::vector<double> flat = theta_t.flatten();
  std::vector<double> out(flat.size());
  std::vector<photon_step_metric> metrics(tau);
  const photon_train_cfg c = to_c(cfg);
  photon_err e{};
  check(photon_client_round(dev.get(), &c, flat.data(), inputs.data(), targets.data(), round,
                            client_id, step_base, out.data(), metrics.data(), &e),
        e);
  fedsim::ClientResult r;
  r.theta = theta_t.clone();
  r.theta.assign_flat(out);
  for (const auto& m : metrics) r.steps.push_back(fedsim::StepMetric{m.loss, m.tokens, m.sim_seconds});
  r.cursor = stream.cursor();
  return r;
}

// param_vector.cpp:127-152 (anchored, ascending order; bit-exact)
inline fedsim::ParamVector mean(Device& dev, const std::vector<const fedsim::ParamVector*>& vs) {
  if (vs.empty()) throw fedsim::UsageError("mean of zero param vectors");
  std::vector<std::vector<double>> flats;
  std::vector<const double*> ptrs;
  for (const auto* v : vs) {
    vs[0]->check_combinable(*v);
    flats.push_back(v->flatten());
    ptrs.push_back(flats.back().data());
  }
  std::vector<double> out(flats[0].size());
  photon_err e{};
  check(photon_mean(dev.get(), ptrs.data(), ptrs.size(), out.size(), out.data(), &e), e);
  fedsim::ParamVector r = vs[0]->clone();
  r.assign_flat(out);
  return r;
}

// optim.cpp:124-159 (bit-exact); state.velocity updated in place
inline fedsim::ParamVector server_step(Device& dev, fedsim::ServerOptState& state,
                                       const fedsim::ParamVector& theta,
                                       const fedsim::ParamVector& delta,
                                       const fedsim::ParamVector& client_mean) {
  const std::vector<double> t = theta.flatten(), d = delta.flatten(), m = client_mean.flatten();
  std::vector<double> v = state.velocity.flatten(), out(t.size());
  const photon_server_cfg c = to_c(state.cfg);
  photon_err e{};
  check(photon_server_step(dev.get(), &c, t.data(), d.data(), m.data(), v.data(), t.size(),
                           out.data(), &e),
        e);
  state.velocity.assign_flat(v);
  fedsim::ParamVector r = theta.clone();
  r.assign_flat(out);
  return r;
}

// optim.cpp:61-90 (bit-exact)
inline void adamw_step(Device& dev, fedsim::ParamVector& params, const fedsim::ParamVector& grads,
                       fedsim::AdamWState& state, double lr) {
  params.check_combinable(grads);
  std::vector<double> p = params.flatten(), m = state.m.flatten(), v = state.v.flatten();
  const std::vector<double> g = grads.flatten();
  uint64_t sc = state.step_count;
  const photon_adamw_cfg a{state.cfg.beta1, state.cfg.beta2, state.cfg.eps,
                           state.cfg.weight_decay, state.cfg.clip_norm};
  photon_err e{};
  check(photon_adamw_step(dev.get(), p.data(), g.data(), m.data(), v.data(), p.size(), &sc, &a,
                          lr, &e),
        e);
  params.assign_flat(p);
  state.m.assign_flat(m);
  state.v.assign_flat(v);
  state.step_count = sc;
}

}  // namespace photon_fedsim
