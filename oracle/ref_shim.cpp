// ref_shim.cpp -- flat C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// /root/reference/proj/core/src/*.cpp (never copied into this repo) into
// oracle/_ref/libfedsim_ref.so.  Tests use it to pin the C restatement
// (fedsim_oracle.c) bit-for-bit, and bench.py --impl reference times it as the
// reference's own CPU implementation of the federated round.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "fedsim/checkpoint.h"
#include "fedsim/aggregator.h"
#include "fedsim/baselines.h"
#include "fedsim/client.h"
#include "fedsim/data.h"
#include "fedsim/errors.h"
#include "fedsim/harness.h"
#include "fedsim/model.h"
#include "fedsim/optim.h"
#include "fedsim/param_vector.h"
#include "fedsim/rng.h"
#include "fedsim/tensor.h"

using namespace fedsim;

namespace {

int code_of(const std::exception_ptr& e) {
  try {
    std::rethrow_exception(e);
  } catch (const CapacityError&) { return 2; }
  catch (const ConfigError&) { return 1; }
  catch (const ShapeError&) { return 3; }
  catch (const IndexError&) { return 4; }
  catch (const UsageError&) { return 5; }
  catch (const LookupError&) { return 6; }
  catch (const DivergenceError&) { return 8; }
  catch (const NumericError&) { return 7; }
  catch (const RoundFailureError&) { return 11; }
  catch (const IntegrityError&) { return 10; }
  catch (const IoError&) { return 9; }
  catch (const ParseError&) { return 12; }
  catch (...) { return 99; }
}

#define GUARD(body)                                  \
  try {                                              \
    body;                                            \
    return 0;                                        \
  } catch (...) {                                    \
    return code_of(std::current_exception());        \
  }

ModelConfig mcfg(const uint64_t* m) {
  ModelConfig c;
  c.n_blocks = m[0];
  c.d_model = m[1];
  c.n_heads = m[2];
  c.expansion_ratio = m[3];
  c.vocab_size = m[4];
  c.seq_len = m[5];
  return c;
}

ParamVector to_pv(const TransformerModel& model, const double* flat) {
  ParamVector pv = model.init_params(0);
  std::vector<double> v(flat, flat + pv.total_len());
  pv.assign_flat(v);
  return pv;
}

ParamVector flat_pv(const double* x, std::size_t n) {
  ParamVector pv;
  pv.add("w", Shape{n}, std::vector<double>(x, x + n));
  return pv;
}

void copy_out(const ParamVector& pv, double* out) {
  auto f = pv.flatten();
  std::memcpy(out, f.data(), f.size() * sizeof(double));
}

// train cfg layout (doubles): eta_max, warmup, decay, alpha, beta1, beta2, eps,
// wd, clip, opt, sgd_clip, local_steps, batch, post_kind, post_threshold
LocalTrainConfig tcfg(const uint64_t* m, const double* t) {
  LocalTrainConfig c;
  c.model = mcfg(m);
  c.schedule.eta_max = t[0];
  c.schedule.warmup_steps = static_cast<std::size_t>(t[1]);
  c.schedule.decay_steps = static_cast<std::size_t>(t[2]);
  c.schedule.alpha = t[3];
  c.adamw.beta1 = t[4];
  c.adamw.beta2 = t[5];
  c.adamw.eps = t[6];
  c.adamw.weight_decay = t[7];
  c.adamw.clip_norm = t[8];
  c.opt = t[9] == 0.0 ? ClientOptKind::kAdamW : ClientOptKind::kSgd;
  c.sgd_clip_norm = t[10];
  c.local_steps = static_cast<std::size_t>(t[11]);
  c.batch_size = static_cast<std::size_t>(t[12]);
  c.post.kind = t[13] == 0.0 ? PostProcessPolicy::Kind::kIdentity
                             : PostProcessPolicy::Kind::kClipUpdateNorm;
  c.post.threshold = t[14];
  return c;
}

ServerOptConfig scfg(const double* s) {
  ServerOptConfig c;
  c.kind = s[0] == 0.0 ? ServerOptKind::FedAvg : ServerOptKind::FedMomentum;
  c.eta = s[1];
  c.momentum = s[2];
  c.nesterov = s[3] != 0.0;
  return c;
}

std::shared_ptr<const ShardPlan> make_plan(int32_t policy, int32_t style, uint64_t tokens,
                                           uint64_t data_seed, uint32_t vocab,
                                           uint64_t shards, uint64_t seq_len) {
  if (policy == 0) {
    const auto styles = known_styles();
    return std::make_shared<const ShardPlan>(partition_iid(
        generate_corpus(styles[style], tokens, data_seed, vocab), shards, seq_len, data_seed));
  }
  std::vector<Corpus> cs;
  for (const auto& s : known_styles()) cs.push_back(generate_corpus(s, tokens, data_seed, vocab));
  return std::make_shared<const ShardPlan>(
      partition_by_source(std::move(cs), shards / 4, seq_len));
}

}  // namespace

extern "C" {

uint64_t ref_mix64(uint64_t x) { return mix64(x); }

int ref_rng_normals(uint64_t seed, uint64_t n, double* out) {
  Rng r(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = r.normal();
  return 0;
}

int ref_init_params(const uint64_t* m, uint64_t seed, double* out) {
  GUARD(TransformerModel model(mcfg(m)); copy_out(model.init_params(seed), out))
}

uint64_t ref_param_count(const uint64_t* m) { return mcfg(m).param_count(); }

int ref_generate_corpus(int32_t style, uint64_t length, uint64_t seed, uint32_t vocab,
                        uint16_t* out) {
  GUARD(auto c = generate_corpus(known_styles()[style], length, seed, vocab);
        std::memcpy(out, c.tokens.data(), length * sizeof(uint16_t)))
}

int ref_sample_clients(uint64_t p, uint64_t k, uint64_t seed, uint64_t round, uint64_t* out) {
  GUARD(auto s = sample_clients(p, k, seed, round);
        for (std::size_t i = 0; i < s.size(); ++i) out[i] = s[i])
}

int ref_lr_at(const double* sched, uint64_t step, double* out) {
  GUARD(LrSchedule s; s.eta_max = sched[0]; s.warmup_steps = (std::size_t)sched[1];
        s.decay_steps = (std::size_t)sched[2]; s.alpha = sched[3]; *out = lr_at(s, step))
}

// batches: n_steps consecutive stream.next() calls; writes inputs/targets and
// the final cursor.
int ref_stream(int32_t policy, int32_t style, uint64_t tokens, uint64_t data_seed,
               uint32_t vocab, uint64_t shards, uint64_t seq_len, uint64_t client,
               uint64_t batch, uint64_t seed, uint64_t cursor, uint64_t n_steps,
               int32_t* inputs, int32_t* targets, uint64_t* cursor_out) {
  GUARD(auto plan = make_plan(policy, style, tokens, data_seed, vocab, shards, seq_len);
        BatchStream s(plan, client, batch, seq_len, stream_seed(seed, client), cursor);
        for (uint64_t i = 0; i < n_steps; ++i) {
          Batch b = s.next();
          std::memcpy(inputs + i * batch * seq_len, b.inputs.data(), b.inputs.size() * 4);
          std::memcpy(targets + i * batch * seq_len, b.targets.data(), b.targets.size() * 4);
        } *cursor_out = s.cursor())
}

int ref_forward_backward(const uint64_t* m, const double* params, const int32_t* inputs,
                         const int32_t* targets, uint64_t batch, uint64_t seq, double* loss,
                         double* grads) {
  GUARD(TransformerModel model(mcfg(m)); ParamVector pv = to_pv(model, params); Batch b;
        b.batch_size = batch; b.seq_len = seq;
        b.inputs.assign(inputs, inputs + batch * seq);
        b.targets.assign(targets, targets + batch * seq);
        auto fwd = model.forward_loss(pv, b, grads != nullptr); *loss = fwd.loss.item();
        if (grads) {
          backward(fwd.loss);
          copy_out(model.collect_grads(fwd), grads);
        })
}

int ref_adamw_step(double* p, const double* g, double* mm, double* vv, uint64_t n,
                   uint64_t* step_count, const double* t, double lr) {
  GUARD(ParamVector P = flat_pv(p, n); ParamVector G = flat_pv(g, n); AdamWConfig c;
        c.beta1 = t[4]; c.beta2 = t[5]; c.eps = t[6]; c.weight_decay = t[7];
        c.clip_norm = t[8]; AdamWState st = AdamWState::fresh(c, P);
        st.m = flat_pv(mm, n); st.v = flat_pv(vv, n); st.step_count = *step_count;
        adamw_step(P, G, st, lr); copy_out(P, p); copy_out(st.m, mm); copy_out(st.v, vv);
        *step_count = st.step_count)
}

int ref_mean(const double* const* vs, uint64_t k, uint64_t n, double* out) {
  GUARD(std::vector<ParamVector> pvs; for (uint64_t i = 0; i < k; ++i)
            pvs.push_back(flat_pv(vs[i], n));
        std::vector<const ParamVector*> ptrs; for (auto& p : pvs) ptrs.push_back(&p);
        copy_out(ParamVector::mean(ptrs), out))
}

int ref_server_step(const double* s, const double* theta, const double* delta,
                    const double* mean, double* velocity, uint64_t n, double* out) {
  GUARD(ServerOptState st = ServerOptState::init(scfg(s), flat_pv(theta, n));
        st.velocity = flat_pv(velocity, n);
        ParamVector r = server_step(st, flat_pv(theta, n), flat_pv(delta, n), flat_pv(mean, n));
        copy_out(r, out); copy_out(st.velocity, velocity))
}

// One client round through the reference's run_local_round.
int ref_local_round(const uint64_t* m, const double* t, int32_t policy, int32_t style,
                    uint64_t tokens, uint64_t data_seed, uint64_t shards, uint64_t client,
                    uint64_t seed, uint64_t cursor, uint64_t round, uint64_t step_base,
                    const double* theta_in, double* theta_out, double* losses,
                    uint64_t* cursor_out) {
  GUARD(LocalTrainConfig c = tcfg(m, t); TransformerModel model(c.model);
        auto plan = make_plan(policy, style, tokens, data_seed, (uint32_t)c.model.vocab_size,
                              shards, c.model.seq_len);
        BatchStream s(plan, client, c.batch_size, c.model.seq_len, stream_seed(seed, client),
                      cursor);
        ClientResult r = run_local_round(to_pv(model, theta_in), s, c, round, client, step_base);
        copy_out(r.theta, theta_out);
        for (std::size_t i = 0; i < r.steps.size(); ++i) losses[i] = r.steps[i].loss;
        *cursor_out = r.cursor)
}

// R rounds of FederationRunner (no eval, no checkpoints).  theta in/out,
// velocity out, per-round mean client loss out, per-round wall seconds out.
int ref_run_rounds(const uint64_t* m, const double* t, const double* s, int32_t policy,
                   int32_t style, uint64_t tokens, uint64_t data_seed, uint64_t population,
                   uint64_t k, uint64_t rounds, uint64_t seed, int32_t topology,
                   uint64_t n_threads, const double* theta0, double* theta_out,
                   double* velocity_out, double* round_losses, double* round_seconds) {
  GUARD(LocalTrainConfig c = tcfg(m, t); TransformerModel model(c.model);
        auto plan = make_plan(policy, style, tokens, data_seed, (uint32_t)c.model.vocab_size,
                              population, c.model.seq_len);
        FederationConfig fed; fed.population = population; fed.clients_per_round = k;
        fed.rounds = rounds; fed.seed = seed;
        fed.topology = topology == 0 ? Topology::kParameterServer
                                     : (topology == 1 ? Topology::kAllReduce
                                                      : Topology::kRingAllReduce);
        CostModelParams cost; cost.payload_mb = c.model.payload_mib();
        RunnerOptions opts; opts.n_threads = n_threads; opts.eval_every = 0;
        FederationRunner runner(fed, c, scfg(s), cost, plan, to_pv(model, theta0), opts);
        for (uint64_t r = 0; r < rounds; ++r) {
          const auto t0 = std::chrono::steady_clock::now();
          RoundRecord rec = runner.run_round();
          const auto t1 = std::chrono::steady_clock::now();
          if (round_losses) round_losses[r] = rec.mean_client_loss;
          if (round_seconds) round_seconds[r] = std::chrono::duration<double>(t1 - t0).count();
        } copy_out(runner.theta(), theta_out);
        if (velocity_out) copy_out(runner.server_state().velocity, velocity_out))
}

// c7-style experiment (acceptance_main.cpp:467-534): returns initial and final
// eval perplexity of the federated run.
int ref_run_experiment_fed(const uint64_t* m, const double* t, const double* s,
                           uint64_t corpus_tokens, uint64_t population, uint64_t rounds,
                           uint64_t seed, uint64_t model_seed, uint64_t data_seed,
                           uint64_t eval_sequences, uint64_t eval_batch, const char* out_dir,
                           double* ppl_out /* [initial, final] */) {
  GUARD(ExperimentSpec f; f.name = "ref"; f.mode = RunMode::kFederated;
        f.model = mcfg(m); f.corpus_tokens = corpus_tokens; f.population = population;
        f.participation = 1.0; f.rounds = rounds; f.local_steps = (std::size_t)t[11];
        f.batch_size = (std::size_t)t[12]; f.topology = Topology::kRingAllReduce;
        f.schedule.eta_max = t[0]; f.schedule.warmup_steps = (std::size_t)t[1];
        f.schedule.decay_steps = (std::size_t)t[2]; f.schedule.alpha = t[3];
        f.server_opt = scfg(s); f.seed = seed; f.model_seed = model_seed;
        f.data_seed = data_seed; f.eval_every = 1; f.eval_sequences = eval_sequences;
        f.eval_batch = eval_batch;
        RunOutcome o = run_experiment(f, out_dir); ppl_out[0] = o.initial_ppl;
        ppl_out[1] = o.final_ppl)
}

// Bounded CPU sample of the reference client step (client.cpp:135-154):
// `threads` independent clients, each `steps` x {forward_loss, backward,
// collect_grads, lr_at, adamw_step} on [batch, seq] token blocks drawn from the
// reference's own corpus generator.  Wall seconds of the step loop only.
int ref_train_sample(const uint64_t* m, const double* t, uint64_t batch, uint64_t seq,
                     uint64_t steps, uint64_t threads, double* seconds_out, double* loss_out) {
  GUARD(LocalTrainConfig c = tcfg(m, t); TransformerModel model(c.model);
        const ParamVector theta0 = model.init_params(1);
        std::vector<double> losses(threads, 0.0);
        std::vector<std::exception_ptr> errs(threads);
        auto body = [&](uint64_t w) {
          try {
            Corpus corp = generate_corpus("web", steps * batch * (seq + 1) + 1, 7 + w,
                                          (uint32_t)c.model.vocab_size);
            ParamVector theta = theta0.clone();
            AdamWState opt = AdamWState::fresh(c.adamw, theta);
            for (uint64_t i = 0; i < steps; ++i) {
              Batch b;
              b.batch_size = batch;
              b.seq_len = seq;
              for (uint64_t r = 0; r < batch; ++r)
                for (uint64_t q = 0; q < seq; ++q) {
                  const std::size_t o = (i * batch + r) * (seq + 1) + q;
                  b.inputs.push_back(corp.tokens[o]);
                  b.targets.push_back(corp.tokens[o + 1]);
                }
              ForwardResult fwd = model.forward_loss(theta, b);
              losses[w] = fwd.loss.item();
              backward(fwd.loss);
              ParamVector grads = model.collect_grads(fwd);
              adamw_step(theta, grads, opt, lr_at(c.schedule, i));
            }
          } catch (...) {
            errs[w] = std::current_exception();
          }
        };
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (uint64_t w = 0; w < threads; ++w) pool.emplace_back(body, w);
        for (auto& th : pool) th.join();
        const auto t1 = std::chrono::steady_clock::now();
        for (auto& e : errs) if (e) std::rethrow_exception(e);
        *seconds_out = std::chrono::duration<double>(t1 - t0).count();
        if (loss_out) *loss_out = losses[0])
}

// baselines.cpp:25-127: the reference's centralized / DDP baseline on an IID
// plan built like ref_run_rounds'; t[12] is the global batch
int ref_run_centralized(const uint64_t* m, const double* t, int32_t style, uint64_t tokens,
                        uint64_t data_seed, uint64_t n_workers, uint64_t total_steps,
                        uint64_t reset, uint64_t seed, const double* theta0, double* theta_out,
                        double* step_losses, uint64_t* cursors) {
  GUARD(LocalTrainConfig lc = tcfg(m, t); TransformerModel model(lc.model);
        auto plan = make_plan(0, style, tokens, data_seed, (uint32_t)lc.model.vocab_size,
                              n_workers, lc.model.seq_len);
        CentralizedConfig cc; cc.model = lc.model; cc.adamw = lc.adamw; cc.schedule = lc.schedule;
        cc.opt = lc.opt; cc.sgd_clip_norm = lc.sgd_clip_norm; cc.n_workers = n_workers;
        cc.global_batch = lc.batch_size; cc.total_steps = total_steps;
        cc.opt_reset_interval = reset;
        CentralizedResult r = run_centralized(cc, plan, seed, to_pv(model, theta0), 1);
        copy_out(r.theta, theta_out);
        for (uint64_t i = 0; i < total_steps; ++i) step_losses[i] = r.steps[i].loss;
        for (uint64_t w = 0; w < n_workers; ++w) cursors[w] = r.cursors[w])
}

// checkpoint.cpp: the reference's PHCK writer / reader on a model-layout ParamVector
int ref_write_checkpoint(const uint64_t* m, const double* params, uint64_t round,
                         const char* path) {
  GUARD(TransformerModel model(mcfg(m)); CheckpointMeta meta; meta.round = round;
        write_checkpoint(path, to_pv(model, params), meta))
}

int ref_read_checkpoint(const char* path, double* params, uint64_t n, uint64_t* round) {
  GUARD(Checkpoint ck = read_checkpoint(path);
        if (ck.params.total_len() != n) throw ShapeError("size");
        const std::vector<double> flat = ck.params.flatten();
        std::copy(flat.begin(), flat.end(), params); *round = ck.meta.round)
}

}  // extern "C"
