// runner.cpp -- FederationRunner::run_round (aggregator.cpp:93-220) on B200s.
//
// Each rank runs the sampled clients whose slot % world == rank, each from the
// replicated theta_t.  The round boundary is the only communication:
//   1. every rank scatters 1/world shards of its client models to the shard
//      owners (ncclSend/ncclRecv in ascending slot order -> the owner holds its
//      shard of every surviving model in canonical ascending client order);
//   2. the owner runs the fused anchored-mean -> pseudo-gradient -> outer
//      update kernel on its shard (theta_t and velocity shards stay resident);
//   3. ncclAllGather rebuilds theta_{t+1} on every rank.
// Per-GPU wire bytes = 2 (G-1)/G * P * 4, the ring all-reduce volume; the
// arithmetic is bit-identical to the single-GPU path for any world size.
#include "runner.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <fstream>

#include "kernels.cuh"
#include "nccl_api.hpp"

namespace photon {

#define PH_NCCL(call)                                                                    \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess)                                                               \
      throw Error(PHOTON_ERR_NCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

bool boundary_prefers_peer(uint64_t replica_bytes) {
  const char* e = std::getenv("PHOTON_BOUNDARY");
  if (e && std::string(e) == "nccl") return false;
  if (e && std::string(e) == "p2p") return true;
  return replica_bytes <= kPeerMaxBytes;
}
bool use_peer_boundary(uint64_t replica_bytes) { return boundary_prefers_peer(replica_bytes); }

// optim.cpp:105-113
void validate_server(const photon_server_cfg& s) {
  if (!(s.eta > 0.0)) throw Error(PHOTON_ERR_CONFIG, "server opt: eta must be > 0");
  if (s.momentum < 0.0 || s.momentum >= 1.0)
    throw Error(PHOTON_ERR_CONFIG, "server opt: momentum must be in [0,1)");
  if (s.kind != 0 && s.kind != 1) throw Error(PHOTON_ERR_CONFIG, "server opt: unknown kind");
  if (s.kind == 0 && (s.eta != 1.0 || s.momentum != 0.0))
    throw Error(PHOTON_ERR_CONFIG, "server opt: fedavg is eta=1, momentum=0 by definition");
}

Runner::Runner(Ctx* c, const photon_fed_cfg& f, const photon_train_cfg& t,
               const photon_server_cfg& s, const Plan* p, const double* theta0, int rk, int ws,
               const uint8_t* nccl_id)
    : ctx(c), fed(f), train(t), server(s), plan(p), rank(rk), world(ws) {
  // FederationConfig::validate (aggregator.cpp:16-23) + runner guards (:50-71)
  if (f.population < 1) throw Error(PHOTON_ERR_CONFIG, "federation: population must be >= 1");
  if (f.clients_per_round < 1 || f.clients_per_round > f.population)
    throw Error(PHOTON_ERR_CONFIG, "federation: need 1 <= K <= P");
  if (f.rounds < 1) throw Error(PHOTON_ERR_CONFIG, "federation: rounds must be >= 1");
  if (!p) throw Error(PHOTON_ERR_USAGE, "runner: null shard plan");
  if (p->blocks.size() < f.population)
    throw Error(PHOTON_ERR_CONFIG, "shard plan covers " + std::to_string(p->blocks.size()) +
                                       " clients, federation needs " +
                                       std::to_string(f.population));
  if (p->seq_len != t.model.seq_len)
    throw Error(PHOTON_ERR_USAGE, "stream: seq_len does not match the plan's block size");
  if (std::memcmp(&t.model, &c->cfg, sizeof(photon_model_cfg)) != 0)
    throw Error(PHOTON_ERR_CONFIG, "runner: train model differs from the context's model");
  if (ws < 1 || rk < 0 || rk >= ws) throw Error(PHOTON_ERR_USAGE, "runner: bad rank/world");
  check_train_cfg(t);
  validate_server(s);
  P = c->eng->P;
  shard = shard_len(P, ws);
  Ppad = shard * ws;
  cursors.assign(f.population, 0);
  PH_CUDA(cudaSetDevice(c->device));
  d_theta.reserve(Ppad);
  d_vel.reserve(ws > 1 ? shard : Ppad);  // the outer velocity is sharded across ranks
  PH_CUDA(cudaMemsetAsync(d_theta.ptr, 0, Ppad * 4, c->stream));
  PH_CUDA(cudaMemsetAsync(d_vel.ptr, 0, d_vel.n * 4, c->stream));
  c->h2d_f64_to_f32(theta0, d_theta.ptr, P);
  h_stats.reserve(4 * f.clients_per_round + 4);
  d_stats.reserve(4 * f.clients_per_round + 4);
  PH_CUDA(cudaEventCreate(&ev_a));
  PH_CUDA(cudaEventCreate(&ev_b));
  PH_CUDA(cudaEventCreate(&ev_c));
  PH_CUDA(cudaEventCreate(&ev_b2));
  PH_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
  PH_CUDA(cudaEventCreateWithFlags(&copied[0], cudaEventDisableTiming));
  PH_CUDA(cudaEventCreateWithFlags(&copied[1], cudaEventDisableTiming));
  if (ws > 1) {
    if (!nccl_id) throw Error(PHOTON_ERR_USAGE, "runner: world > 1 needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    PH_NCCL(nccl().CommInitRank(&comm, ws, id, rk));
    if (use_peer_boundary(Ppad * 4)) p2p = std::make_unique<PeerBoundary>(comm, rk, ws, c->device);
  }
  PH_CUDA(cudaStreamSynchronize(c->stream));
}

Runner::~Runner() {
  p2p.reset();
  if (comm) nccl().CommDestroy(comm);
  if (ev_a) cudaEventDestroy(ev_a);
  if (ev_b) cudaEventDestroy(ev_b);
  if (ev_c) cudaEventDestroy(ev_c);
  if (ev_b2) cudaEventDestroy(ev_b2);
  if (copy_stream) cudaStreamSynchronize(copy_stream);
  for (cudaEvent_t e : copied)
    if (e) cudaEventDestroy(e);
  if (copy_stream) cudaStreamDestroy(copy_stream);
}

// Stage round `round`'s batches for this rank's slots into set `set`: host
// BatchStream port into pinned buffers, then async H2D on copy_stream.  `cur`
// are the client cursors at the start of that round.  Returns host ms.
double Runner::stage(uint64_t round, int set, const std::vector<uint64_t>& cur) {
  const auto t0 = std::chrono::steady_clock::now();
  // the set's previous H2D (if any) must have read its pinned buffers
  PH_CUDA(cudaEventSynchronize(copied[set]));
  const auto sampled = sample_clients(fed.population, fed.clients_per_round, fed.seed, round);
  const int K = (int)sampled.size();
  const int tau = (int)train.local_steps, B = (int)train.batch_size, S = (int)plan->seq_len;
  const int V = (int)train.model.vocab_size;
  std::vector<int> mine;
  for (int si = 0; si < K; ++si)
    if (slot_owner(si, world) == rank) mine.push_back(si);
  if (host_batches[set].size() < mine.size()) {
    host_batches[set].resize(mine.size());
    dev_batches[set].resize(mine.size());
  }
  for (size_t j = 0; j < mine.size(); ++j) {
    const uint64_t client = sampled[mine[j]];
    RoundBatches& hb = host_batches[set][j];
    hb.prepare(tau, B, S, V);
    const uint64_t seed = derive(fed.seed, kPurposeStream, client);
    for (int i = 0; i < tau; ++i)
      stream_rows(*plan, client, seed, cur[client] + (uint64_t)i * B, B,
                  hb.tokens.ptr + (size_t)i * B * S, hb.targets.ptr + (size_t)i * B * S);
    hb.finalize(V);
    dev_batches[set][j].upload(hb, V, copy_stream);
  }
  PH_CUDA(cudaEventRecord(copied[set], copy_stream));
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

void Runner::run_round(photon_round_record* rec) {
  if (next_round >= fed.rounds) throw Error(PHOTON_ERR_USAGE, "run_round called after the final round");
  PH_CUDA(cudaSetDevice(ctx->device));
  const uint64_t round = next_round;
  const auto sampled = sample_clients(fed.population, fed.clients_per_round, fed.seed, round);
  const int K = (int)sampled.size();
  const int tau = (int)train.local_steps, B = (int)train.batch_size, S = (int)plan->seq_len;
  const int V = (int)train.model.vocab_size;
  const uint64_t step_base = round * train.local_steps;
  cudaStream_t st = ctx->stream;

  std::vector<int> mine;
  for (int si = 0; si < K; ++si)
    if (slot_owner(si, world) == rank) mine.push_back(si);
  // one local client trains in (and is aggregated from) the engine's master;
  // several keep their results in dedicated slots
  const bool in_master = mine.size() == 1;
  if (!in_master && d_models.n < mine.size() * Ppad) {
    d_models.reserve(mine.size() * Ppad);
    PH_CUDA(cudaMemsetAsync(d_models.ptr, 0, d_models.n * 4, st));
  }
  auto model_ptr = [&](size_t j) -> float* {
    return in_master ? ctx->eng->master : d_models.ptr + j * Ppad;
  };

  // ---- this round's batches: already staged by the previous round, or now
  double host_ms = 0.0;
  if (staged_round != round) host_ms = stage(round, buf, cursors);
  PH_CUDA(cudaStreamWaitEvent(st, copied[buf], 0));
  std::vector<DeviceBatches>& dev = dev_batches[buf];

  // ---- device: the local phase, inputs resident in HBM
  const size_t nm = std::max<size_t>(mine.size(), 1);
  d_loss.reserve(nm * std::max(tau, 1));
  d_flag.reserve(nm);
  h_loss.reserve(nm * std::max(tau, 1));
  h_flag.reserve(nm);
  PH_CUDA(cudaEventRecord(ev_a, st));
  for (size_t j = 0; j < mine.size(); ++j)
    ctx->launch_local_round(train, dev[j], d_theta.ptr, model_ptr(j), step_base,
                            d_loss.ptr + j * tau, d_flag.ptr + j);
  PH_CUDA(cudaEventRecord(ev_b, st));
  // ---- prefetch round t+1 into the other set while the GPU trains round t
  // (its cursors are known: every sampled client advances, dropped or not)
  bool prefetched = false;
  if (round + 1 < fed.rounds) {
    std::vector<uint64_t> next_cur = cursors;
    for (int si = 0; si < K; ++si) next_cur[sampled[si]] += (uint64_t)tau * B;
    stage(round + 1, buf ^ 1, next_cur);
    prefetched = true;
  }
  if (!mine.empty()) {
    PH_CUDA(cudaMemcpyAsync(h_loss.ptr, d_loss.ptr, mine.size() * tau * sizeof(double),
                            cudaMemcpyDeviceToHost, st));
    PH_CUDA(cudaMemcpyAsync(h_flag.ptr, d_flag.ptr, mine.size() * sizeof(int),
                            cudaMemcpyDeviceToHost, st));
  }
  PH_CUDA(cudaStreamSynchronize(st));
  // stats layout: [0,K) mean loss, [K,2K) error code, [2K,3K) error step
  std::fill(h_stats.ptr, h_stats.ptr + 3 * K, 0.0);
  for (size_t j = 0; j < mine.size(); ++j) {
    const int si = mine[j];
    LocalResult lr = classify(h_loss.ptr + j * tau, tau, h_flag.ptr[j]);
    double acc = 0.0;
    for (double l : lr.losses) acc += l;
    h_stats.ptr[si] = tau ? acc / tau : 0.0;  // ClientResult::mean_loss (client.cpp:112-117)
    if (lr.error) {
      h_stats.ptr[K + si] = lr.error;
      h_stats.ptr[2 * K + si] = (double)lr.error_step;
    }
  }
  if (world > 1) {
    PH_CUDA(cudaMemcpyAsync(d_stats.ptr, h_stats.ptr, 3 * K * 8, cudaMemcpyHostToDevice, st));
    PH_NCCL(nccl().AllReduce(d_stats.ptr, d_stats.ptr, 3 * K, ncclDouble, ncclSum, comm, st));
    PH_CUDA(cudaMemcpyAsync(h_stats.ptr, d_stats.ptr, 3 * K * 8, cudaMemcpyDeviceToHost, st));
    PH_CUDA(cudaStreamSynchronize(st));
  }
  // errors surface in ascending client order (aggregator.cpp:141-144)
  for (int si = 0; si < K; ++si) {
    const int code = (int)h_stats.ptr[K + si];
    if (code) {
      Error e(code, code == PHOTON_ERR_DIVERGENCE
                        ? "client " + std::to_string(sampled[si]) + " diverged at round " +
                              std::to_string(round) + ", step " +
                              std::to_string((uint64_t)h_stats.ptr[2 * K + si])
                        : "gradient norm is not finite");
      e.round = round;
      e.client = sampled[si];
      e.step = (uint64_t)h_stats.ptr[2 * K + si];
      throw e;
    }
  }
  // a dropped client trains and advances its cursor but never reports
  std::vector<int> surv;
  for (int si = 0; si < K; ++si) {
    cursors[sampled[si]] += (uint64_t)tau * B;
    if (!dropouts.count({round, sampled[si]})) surv.push_back(si);
  }
  // from here a failed round leaves the cursors advanced (aggregator.cpp:146-151):
  // a retry must stream from them, not reuse this round's staged batches
  if (surv.empty() || ((int)surv.size() < K && fed.topology == 2)) staged_round = ~0ULL;
  if (surv.empty())
    throw Error(PHOTON_ERR_ROUND_FAILURE, "round " + std::to_string(round) + ": no surviving clients");
  if ((int)surv.size() < K && fed.topology == 2)
    throw Error(PHOTON_ERR_ROUND_FAILURE,
                "round " + std::to_string(round) + ": ring all-reduce cannot tolerate dropouts");

  // ---- round boundary: mean -> pseudo-gradient -> outer step ----
  const int n = (int)surv.size();
  std::vector<const float*> local_models(mine.size());
  for (size_t j = 0; j < mine.size(); ++j) local_models[j] = model_ptr(j);
  float* recv = nullptr;
  if (world > 1) {
    // received shards land in the AdamW moments when they fit: m and v are dead
    // between rounds (the next round re-zeroes them) and adjacent in the pool
    Engine& e = *ctx->eng;
    const size_t span = (size_t)(e.vel2 - e.mom) + P;
    recv = e.mom;
    if ((size_t)n * shard > span) {
      d_recv.reserve((size_t)n * shard);
      recv = d_recv.ptr;
    }
  }
  // every rank must take the same path (host.hpp peer_round_ok)
  const bool peer = p2p && peer_round_ok((uint64_t)n, (uint64_t)K, world);
  if (peer) {
    p2p->publish(local_models.data(), (int)local_models.size(), d_theta.ptr, st);
    p2p->run(surv, shard, d_vel.ptr, server, st);
  } else {
    PH_CUDA(cudaEventRecord(ev_b2, st));
    round_boundary(comm, rank, world, P, shard, surv, local_models.data(), recv, d_model_ptrs,
                   d_theta.ptr, d_vel.ptr, server, st);
  }
  PH_CUDA(cudaEventRecord(ev_c, st));
  PH_CUDA(cudaEventSynchronize(ev_c));
  if (peer) p2p->check();  // a peer that never arrived: a host-side error, not a trap
  float bnd_ms = 0.f;
  if (peer) bnd_ms = p2p->last_kernel_ms();
  else PH_CUDA(cudaEventElapsedTime(&bnd_ms, ev_b2, ev_c));
  if (K >= 2) ++sync_events;

  if (rec) {
    std::memset(rec, 0, sizeof(*rec));
    rec->round = round;
    rec->n_sampled = K;
    for (int si = 0; si < K && si < 64; ++si) rec->sampled_ids[si] = sampled[si];
    double acc = 0.0, lo = std::numeric_limits<double>::infinity(), hi = -lo;
    for (int si : surv) {
      const double l = h_stats.ptr[si];
      acc += l;
      lo = std::min(lo, l);
      hi = std::max(hi, l);
    }
    rec->mean_client_loss = acc / (double)n;
    rec->min_client_loss = lo;
    rec->max_client_loss = hi;
    float ms = 0.f;
    PH_CUDA(cudaEventElapsedTime(&ms, ev_a, ev_b));
    rec->local_ms = ms;
    PH_CUDA(cudaEventElapsedTime(&ms, ev_b, ev_c));
    rec->aggregate_ms = ms;
    PH_CUDA(cudaEventElapsedTime(&ms, ev_a, ev_c));
    rec->round_ms = ms;
    rec->tokens = (uint64_t)mine.size() * tau * B * S;
    rec->host_ms = host_ms;
    rec->h2d_bytes = 0;
    for (size_t j = 0; j < mine.size(); ++j)
      rec->h2d_bytes += (uint64_t)tau * ((uint64_t)B * S * 3 + V + 1) * 4;
    rec->d2h_bytes = (uint64_t)mine.size() * (tau * sizeof(double) + sizeof(int));
    rec->eval_ppl = std::numeric_limits<double>::quiet_NaN();
    rec->boundary_ms = bnd_ms;
  }
  next_round = round + 1;
  buf ^= 1;  // the prefetched set holds round t+1
  staged_round = prefetched ? round + 1 : ~0ULL;
  // aggregator.cpp:207-212: after the boundary, outside the timed round
  if (eval_every > 0 && (round % eval_every == eval_every - 1 || next_round == fed.rounds)) {
    const double ppl = eval_theta();
    if (rec) rec->eval_ppl = ppl;
  }
}

void round_boundary(ncclComm_t comm, int rank, int world, uint64_t P, uint64_t shard,
                    const std::vector<int>& surv, const float* const* local_models,
                    float* recv, DevBuf<const float*>& d_ptrs, float* d_theta, float* d_vel,
                    const photon_server_cfg& server, cudaStream_t st) {
  const int n = (int)surv.size();
  std::vector<const float*> ptrs(n);
  if (world == 1) {
    for (int r = 0; r < n; ++r) ptrs[r] = local_models[surv[r]];
  } else {
    PH_NCCL(nccl().GroupStart());
    for (int r = 0; r < n; ++r) {
      const int si = surv[r], owner = slot_owner(si, world);
      if (owner == rank) {
        const float* model = local_models[si / world];
        for (int q = 0; q < world; ++q)
          PH_NCCL(nccl().Send(model + (size_t)q * shard, shard, ncclFloat, q, comm, st));
      }
      PH_NCCL(nccl().Recv(recv + (size_t)r * shard, shard, ncclFloat, owner, comm, st));
    }
    PH_NCCL(nccl().GroupEnd());
    for (int r = 0; r < n; ++r) ptrs[r] = recv + (size_t)r * shard;
  }
  d_ptrs.reserve(n);
  PH_CUDA(cudaMemcpyAsync(d_ptrs.ptr, ptrs.data(), n * sizeof(float*), cudaMemcpyHostToDevice, st));
  const uint64_t off = world == 1 ? 0 : (uint64_t)rank * shard;
  const uint64_t len = world == 1 ? P : shard;
  k::aggregate<float>(d_ptrs.ptr, n, len, d_theta + off, d_vel, server.kind, server.eta,
                      server.momentum, server.nesterov, st);
  if (world > 1) PH_NCCL(nccl().AllGather(d_theta + off, d_theta, shard, ncclFloat, comm, st));
}

void Runner::set_eval(const EvalSet& es, uint64_t every) {
  PH_CUDA(cudaSetDevice(ctx->device));
  const int S = (int)es.seq_len, V = (int)train.model.vocab_size;
  if (es.seq_len != train.model.seq_len)
    throw Error(PHOTON_ERR_SHAPE, "eval set: seq_len does not match the model");
  eval_every = every;
  eval_n = es.batch_sizes.size();
  eval_dev.clear();
  eval_ids.clear();
  eval_valid.assign(eval_n, 0);
  uint64_t row = 0;
  for (uint64_t b = 0; b < eval_n; ++b) {
    const uint64_t B = es.batch_sizes[b];
    const int32_t* in = es.inputs.data() + row * S;
    const int32_t* tg = es.targets.data() + row * S;
    for (uint64_t i = 0; i < B * S; ++i) eval_valid[b] += tg[i] >= 0;
    if ((int)(b % world) == rank) {
      RoundBatches rb;
      rb.prepare(1, (int)B, S, V);
      std::memcpy(rb.tokens.ptr, in, B * S * 4);
      std::memcpy(rb.targets.ptr, tg, B * S * 4);
      rb.finalize(V);
      eval_dev.emplace_back();
      eval_dev.back().upload(rb, V, ctx->stream);
      PH_CUDA(cudaStreamSynchronize(ctx->stream));  // rb's pinned buffers die here
      eval_ids.push_back(b);
    }
    row += B;
  }
  d_eval.reserve(std::max<uint64_t>(eval_n, 1));
  h_eval.reserve(std::max<uint64_t>(eval_n, 1));
}

// model.cpp:176-192: exp(sum_b loss_b * valid_b / sum_b valid_b), batches in order
double Runner::eval_theta() {
  if (eval_n == 0) throw Error(PHOTON_ERR_USAGE, "runner: no evaluation set");
  PH_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  Engine& e = *ctx->eng;
  PH_CUDA(cudaMemcpyAsync(e.master, d_theta.ptr, P * 4, cudaMemcpyDeviceToDevice, st));
  e.refresh_shadow();
  PH_CUDA(cudaMemsetAsync(d_eval.ptr, 0, eval_n * sizeof(double), st));
  for (size_t j = 0; j < eval_dev.size(); ++j) {
    const DeviceBatches& db = eval_dev[j];
    StepBatch sb{db.tokens.ptr, db.targets.ptr, db.csr_off.ptr, db.csr_rows.ptr, db.B, db.S,
                 db.inv_count[0]};
    e.forward_backward(sb, d_eval.ptr + eval_ids[j], false);
  }
  // every batch loss sits on exactly one rank: the sum reassembles them exactly
  if (world > 1) PH_NCCL(nccl().AllReduce(d_eval.ptr, d_eval.ptr, eval_n, ncclDouble, ncclSum, comm, st));
  PH_CUDA(cudaMemcpyAsync(h_eval.ptr, d_eval.ptr, eval_n * sizeof(double), cudaMemcpyDeviceToHost, st));
  PH_CUDA(cudaStreamSynchronize(st));
  double nll = 0.0;
  uint64_t tokens = 0;
  for (uint64_t b = 0; b < eval_n; ++b) {
    nll += h_eval.ptr[b] * (double)eval_valid[b];
    tokens += eval_valid[b];
  }
  if (tokens == 0) throw Error(PHOTON_ERR_USAGE, "eval_perplexity: no target tokens");
  return std::exp(nll / (double)tokens);
}

// harness.cpp:845-905: checkpoint.phck (theta, meta.round = next round), velocity.phck
// for a momentum server, state.json
void Runner::save(const std::string& dir) {
  std::vector<double> th(P), vel;
  theta_f64(th.data());
  if (server.kind == 1) {
    vel.resize(P);
    velocity_f64(vel.data());  // collective for world > 1
  }
  if (rank != 0) return;
  write_phck(dir + "/checkpoint.phck", train.model, th.data(), next_round);
  if (server.kind == 1) write_phck(dir + "/velocity.phck", train.model, vel.data(), next_round);
  ResumeState s;
  s.next_round = next_round;
  s.initial_ppl = initial_ppl;
  s.sync_events = sync_events;
  s.cursors = cursors;
  write_state_json(dir + "/state.json", s);
}

void Runner::resume(const std::string& dir) {
  const ResumeState s = read_state_json(dir + "/state.json");
  if (s.cursors.size() != fed.population) throw Error(PHOTON_ERR_INTEGRITY, "resume: population changed");
  std::vector<double> th(P), vel(P, 0.0);
  const uint64_t r = read_phck(dir + "/checkpoint.phck", train.model, th.data());
  if (r != s.next_round)
    throw Error(PHOTON_ERR_INTEGRITY, "resume: checkpoint round disagrees with state.json");
  if (server.kind == 1 && s.next_round > 0) {
    std::ifstream probe(dir + "/velocity.phck");
    if (!probe) throw Error(PHOTON_ERR_INTEGRITY, "resume: velocity.phck missing");
    read_phck(dir + "/velocity.phck", train.model, vel.data());
  }
  restore(th.data(), vel.data(), s.next_round, s.cursors.data(), s.cursors.size());
  initial_ppl = s.initial_ppl;
  sync_events = s.sync_events;
}

void Runner::theta_f64(double* out) {
  PH_CUDA(cudaSetDevice(ctx->device));
  ctx->d2h_f32_to_f64(d_theta.ptr, out, P);
}

void Runner::velocity_f64(double* out) {
  PH_CUDA(cudaSetDevice(ctx->device));
  if (world == 1) {
    ctx->d2h_f32_to_f64(d_vel.ptr, out, P);
    return;
  }
  // gather the shards chunk by chunk (bounded scratch): chunk c of every
  // rank's shard lands at [q][chunk] in d_f32a
  const uint64_t chunk = std::min<uint64_t>(shard, 1ull << 22);
  ctx->d_f32a.reserve((size_t)world * chunk);
  std::vector<double> tmp;
  for (uint64_t c0 = 0; c0 < shard; c0 += chunk) {
    const uint64_t len = std::min(chunk, shard - c0);
    PH_NCCL(nccl().AllGather(d_vel.ptr + c0, ctx->d_f32a.ptr, len, ncclFloat, comm, ctx->stream));
    tmp.resize((size_t)world * len);
    // ranks' pieces are len apart in the gather buffer
    ctx->d2h_f32_to_f64(ctx->d_f32a.ptr, tmp.data(), (uint64_t)world * len);
    for (int q = 0; q < world; ++q) {
      const uint64_t dst = (uint64_t)q * shard + c0;
      if (dst >= P) continue;
      const uint64_t m = std::min(len, P - dst);
      std::copy(tmp.begin() + (size_t)q * len, tmp.begin() + (size_t)q * len + m, out + dst);
    }
  }
}

// FederationRunner::restore (aggregator.cpp:78-91)
void Runner::restore(const double* theta, const double* velocity, uint64_t nr,
                     const uint64_t* cur, uint64_t n) {
  if (n != cursors.size()) throw Error(PHOTON_ERR_USAGE, "restore: cursor vector has wrong length");
  PH_CUDA(cudaSetDevice(ctx->device));
  ctx->h2d_f64_to_f32(theta, d_theta.ptr, P);
  if (world == 1) {
    ctx->h2d_f64_to_f32(velocity, d_vel.ptr, P);
  } else {  // this rank's shard only
    const uint64_t o = (uint64_t)rank * shard;
    PH_CUDA(cudaMemsetAsync(d_vel.ptr, 0, shard * 4, ctx->stream));
    if (o < P) ctx->h2d_f64_to_f32(velocity + o, d_vel.ptr, std::min(shard, P - o));
  }
  PH_CUDA(cudaStreamSynchronize(ctx->stream));
  next_round = nr;
  cursors.assign(cur, cur + n);
  staged_round = ~0ULL;  // any prefetched batches were for the old cursors
}

}  // namespace photon
