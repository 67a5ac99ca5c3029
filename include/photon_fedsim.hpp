// photon_fedsim.hpp -- header-only adapter: the reference's client-update,
// aggregator and outer-optimizer C++ interfaces implemented over photon.h.
//
// A maintainer of fedsim::core adds this header and links libphoton.so; call
// sites keep the reference signatures:
//   client.h:97-99        run_local_round(theta_t, stream, cfg, round, client, step_base)
//   param_vector.h:50-54  ParamVector::mean(vs) / ParamVector::sub(a, b)
//   optim.h:78            server_step(state, theta, delta, client_mean)
//   optim.h:46-52         adamw_step / sgd_step
//   aggregator.h:70-102   FederationRunner (device-resident rounds: run_round,
//                         theta, server_state, client_cursor, restore, done)
//   baselines.h:48-52     run_centralized (the DDP baseline on the device)
// Errors come back as the same fedsim:: exception types (errors.h:9-72).
#pragma once

#include <cstring>
#include <memory>
#include <stdexcept>
#include <vector>

#include <cmath>
#include <limits>
#include <set>
#include <utility>

#include "fedsim/aggregator.h"
#include "fedsim/baselines.h"
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

// ---- data.h:33-62: a reference ShardPlan, imported as is -------------------------
class Plan {
 public:
  explicit Plan(const fedsim::ShardPlan& plan) {
    std::vector<const uint16_t*> corpora;
    std::vector<uint64_t> lens;
    for (std::size_t s = 0; s < plan.n_sources(); ++s) {
      corpora.push_back(plan.corpus(s).tokens.data());
      lens.push_back(plan.corpus(s).tokens.size());
    }
    std::vector<uint64_t> counts;
    std::vector<uint32_t> sources;
    std::vector<uint64_t> offsets;
    for (std::size_t c = 0; c < plan.n_clients(); ++c) {
      const auto& blocks = plan.client_blocks(c);
      counts.push_back(blocks.size());
      for (const auto& b : blocks) {
        sources.push_back(b.source);
        offsets.push_back(b.offset);
      }
    }
    photon_err e{};
    check(photon_plan_from_blocks(corpora.data(), lens.data(), lens.size(), plan.seq_len(),
                                  counts.data(), counts.size(), sources.data(), offsets.data(),
                                  &plan_, &e),
          e);
  }
  ~Plan() { photon_plan_free(plan_); }
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;
  const photon_plan* get() const { return plan_; }

 private:
  photon_plan* plan_ = nullptr;
};

inline photon_fed_cfg to_c(const fedsim::FederationConfig& f) {
  photon_fed_cfg c{};
  c.population = f.population;
  c.clients_per_round = f.clients_per_round;
  c.rounds = f.rounds;
  c.topology = f.topology == fedsim::Topology::kParameterServer ? 0
               : f.topology == fedsim::Topology::kAllReduce     ? 1
                                                                 : 2;
  c.seed = f.seed;
  return c;
}

// aggregator.h:70-102 -- the round runs on the device (client steps, anchored
// mean, outer step); theta_t and the velocity stay in HBM between rounds.
// CostModelParams and RunnerOptions::{n_threads, eval_fn, checkpoint paths} are
// accepted for signature compatibility; simulated-time fields of RoundRecord
// stay zero (the cost model is not part of the device path).  Dropouts apply.
class FederationRunner {
 public:
  FederationRunner(Device& dev, fedsim::FederationConfig fed, fedsim::LocalTrainConfig local,
                   fedsim::ServerOptConfig server, fedsim::CostModelParams /*cost*/,
                   std::shared_ptr<const fedsim::ShardPlan> plan, fedsim::ParamVector theta0,
                   fedsim::RunnerOptions opts = {})
      : fed_(fed), server_cfg_(server), plan_(*plan), theta_(std::move(theta0)) {
    const photon_fed_cfg f = to_c(fed);
    const photon_train_cfg t = to_c(local);
    const photon_server_cfg s = to_c(server);
    const std::vector<double> flat = theta_.flatten();
    photon_err e{};
    check(photon_runner_create(dev.get(), &f, &t, &s, plan_.get(), flat.data(), 0, 1, nullptr,
                               &r_, &e),
          e);
    for (const auto& d : opts.dropouts) photon_runner_add_dropout(r_, d.first, d.second);
  }
  ~FederationRunner() { photon_runner_destroy(r_); }
  FederationRunner(const FederationRunner&) = delete;
  FederationRunner& operator=(const FederationRunner&) = delete;

  fedsim::RoundRecord run_round() {
    photon_round_record rec{};
    photon_err e{};
    check(photon_runner_run_round(r_, &rec, &e), e);
    fedsim::RoundRecord out;
    out.round = rec.round;
    for (uint64_t i = 0; i < rec.n_sampled && i < 64; ++i) out.sampled_ids.push_back(rec.sampled_ids[i]);
    if (rec.n_sampled > 64)  // ids past the record's inline array: the same deterministic draw
      out.sampled_ids = fedsim::sample_clients(fed_.population, fed_.clients_per_round, fed_.seed,
                                               rec.round);
    out.mean_client_loss = rec.mean_client_loss;
    out.min_client_loss = rec.min_client_loss;
    out.max_client_loss = rec.max_client_loss;
    out.eval_ppl = rec.eval_ppl;
    fresh_ = false;
    return out;
  }
  bool done() const { return next_round() >= fed_.rounds; }
  std::size_t next_round() const { return photon_runner_next_round(r_); }
  const fedsim::ParamVector& theta() const {
    if (!fresh_) sync();
    return theta_;
  }
  const fedsim::ServerOptState& server_state() const {
    if (!fresh_) sync();
    return state_;
  }
  const fedsim::FederationConfig& federation() const { return fed_; }
  std::uint64_t client_cursor(std::size_t client) const { return photon_runner_cursor(r_, client); }
  void restore(fedsim::ParamVector theta, fedsim::ParamVector velocity, std::size_t next_round,
               double /*t_cum*/, const std::vector<std::uint64_t>& cursors) {
    const std::vector<double> t = theta.flatten(), v = velocity.flatten();
    photon_err e{};
    check(photon_runner_restore(r_, t.data(), v.data(), next_round, cursors.data(),
                                cursors.size(), &e),
          e);
    fresh_ = false;
  }

 private:
  void sync() const {
    std::vector<double> t(theta_.total_len()), v(theta_.total_len());
    photon_err e{};
    check(photon_runner_theta(r_, t.data(), &e), e);
    check(photon_runner_velocity(r_, v.data(), &e), e);
    theta_.assign_flat(t);
    state_ = fedsim::ServerOptState::init(server_cfg_, theta_);
    state_.velocity.assign_flat(v);
    fresh_ = true;
  }
  fedsim::FederationConfig fed_;
  fedsim::ServerOptConfig server_cfg_;
  Plan plan_;
  mutable fedsim::ParamVector theta_;
  mutable fedsim::ServerOptState state_;
  mutable bool fresh_ = false;
  photon_runner* r_ = nullptr;
};

// baselines.h:48-52 -- the centralized / DDP baseline on the device; the
// observer sees theta after every step (read back from the device).
inline fedsim::CentralizedResult run_centralized(Device& dev, const fedsim::CentralizedConfig& cfg,
                                                 std::shared_ptr<const fedsim::ShardPlan> plan,
                                                 std::uint64_t seed,
                                                 const fedsim::ParamVector& theta0,
                                                 std::size_t /*n_threads*/ = 1,
                                                 const fedsim::StepObserver& observer = {}) {
  Plan p(*plan);
  photon_central_cfg c{};
  c.model = to_c(cfg.model);
  c.adamw = photon_adamw_cfg{cfg.adamw.beta1, cfg.adamw.beta2, cfg.adamw.eps,
                             cfg.adamw.weight_decay, cfg.adamw.clip_norm};
  c.schedule = photon_lr_schedule{cfg.schedule.eta_max, cfg.schedule.warmup_steps,
                                  cfg.schedule.decay_steps, cfg.schedule.alpha};
  c.opt = cfg.opt == fedsim::ClientOptKind::kAdamW ? 0 : 1;
  c.sgd_clip_norm = cfg.sgd_clip_norm;
  c.n_workers = cfg.n_workers;
  c.global_batch = cfg.global_batch;
  c.total_steps = cfg.total_steps;
  c.opt_reset_interval = cfg.opt_reset_interval;
  c.throughput_bps = cfg.throughput_bps;
  const std::vector<double> flat = theta0.flatten();
  photon_central* h = nullptr;
  photon_err e{};
  check(photon_central_create(dev.get(), &c, p.get(), seed, flat.data(), 0, 1, nullptr, &h, &e), e);
  struct Guard {
    photon_central* h;
    ~Guard() { photon_central_destroy(h); }
  } guard{h};
  fedsim::CentralizedResult r;
  std::vector<double> th(flat.size());
  fedsim::ParamVector cur = theta0.clone();
  for (std::size_t t = 0; t < cfg.total_steps; ++t) {
    photon_step_metric m{};
    check(photon_central_step(h, &m, &e), e);
    r.steps.push_back(fedsim::StepMetric{m.loss, m.tokens, m.sim_seconds});
    if (observer) {
      check(photon_central_theta(h, th.data(), &e), e);
      cur.assign_flat(th);
      observer(t, cur);
    }
  }
  check(photon_central_theta(h, th.data(), &e), e);
  r.theta = theta0.clone();
  r.theta.assign_flat(th);
  r.sync_events = cfg.n_workers > 1 ? cfg.total_steps : 0;
  for (std::size_t w = 0; w < cfg.n_workers; ++w) r.cursors.push_back(photon_central_cursor(h, w));
  return r;
}

}  // namespace photon_fedsim
