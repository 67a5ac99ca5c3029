// host.hpp -- host-side determinism layer of the Photon round: seeding, RNG
// draw conversions, synthetic corpora, shard plans, batch streams, client
// sampling, LR schedule, canonical layout and parameter init.  All integer
// results are bit-exact with the reference (/root/reference/proj/core); the
// f64 ones (init, lr) are bit-exact given the same libm.
#pragma once

#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "photon.h"

namespace photon {

// Exception carrying a photon status code; converted to photon_err at the
// C-ABI boundary (capi.cpp).
struct Error : std::runtime_error {
  int code;
  uint64_t round = 0, client = 0, step = 0;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// rng.h:14-32 -- splitmix64 finalizer; seeds are functions of (seed, purpose, ids)
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline uint64_t derive(uint64_t seed, uint64_t a) { return mix64(seed ^ mix64(a)); }
inline uint64_t derive(uint64_t seed, uint64_t a, uint64_t b) { return derive(derive(seed, a), b); }
inline uint64_t derive(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  return derive(derive(seed, a, b), c);
}

// seeding purposes
constexpr uint64_t kPurposeSample = 0x53616d70ULL;  // "Samp" aggregator.cpp:31
constexpr uint64_t kPurposeShard = 0x53686172ULL;   // "Shar" data.cpp:149
constexpr uint64_t kPurposeCorpus = 0x436f7270ULL;  // "Corp" data.cpp:59
constexpr uint64_t kPurposeStream = 0x44617461ULL;  // "Data" data.cpp:202
constexpr uint64_t kPurposeEpoch = 0x45706f63ULL;   // "Epoc" data.cpp:226
constexpr uint64_t kPurposeEval = 0x4576616cULL;    // "Eval" harness.cpp:453

// rng.h:37-84 -- mt19937_64 with the reference's pinned draw conversions.
class Draws {
 public:
  explicit Draws(uint64_t seed) : eng_(seed) {}
  uint64_t u64() { return eng_(); }
  double unit() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) { return eng_() % n; }
  double gauss();  // Box-Muller with cached spare
  template <typename T>
  void permute(std::vector<T>& v) {  // Fisher-Yates from the top
    for (size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[below(i)]);
  }

 private:
  std::mt19937_64 eng_;
  double spare_ = 0.0;
  bool has_spare_ = false;
};

// ---- model ------------------------------------------------------------------
struct Entry {
  std::string name;
  uint64_t offset, rows, cols;  // cols == 0: rank-1
  uint64_t numel() const { return cols ? rows * cols : rows; }
};

void validate_model(const photon_model_cfg& m);
uint64_t param_count(const photon_model_cfg& m);
std::vector<Entry> layout(const photon_model_cfg& m);
std::vector<double> init_params(const photon_model_cfg& m, uint64_t seed);

// Offsets of one block's entries in the flat canonical buffer.
struct BlockOffsets {
  uint64_t ln1g, ln1b, wq, bq, wk, bk, wv, bv, wo, bo, ln2g, ln2b, w1, b1, w2, b2;
};
struct ModelOffsets {
  uint64_t tok, pos, lnfg, lnfb, head_w, head_b;
  std::vector<BlockOffsets> blocks;
};
ModelOffsets model_offsets(const photon_model_cfg& m);

// ---- schedule / sampling --------------------------------------------------------
double lr_at(const photon_lr_schedule& s, uint64_t step);
std::vector<uint64_t> sample_clients(uint64_t population, uint64_t k, uint64_t seed,
                                     uint64_t round);

// ---- data -----------------------------------------------------------------------
int style_index(const std::string& style);
std::vector<uint16_t> generate_corpus(int style, uint64_t length, uint64_t seed, uint32_t vocab);

struct Plan {
  uint64_t seq_len = 0;
  std::vector<std::vector<uint16_t>> corpora;
  // per client: packed (source << 48 | token offset) of each (seq_len+1)-token block
  std::vector<std::vector<uint64_t>> blocks;

  static Plan iid(std::vector<uint16_t> tokens, uint64_t n_shards, uint64_t seq_len,
                  uint64_t seed);
  static Plan by_source(std::vector<std::vector<uint16_t>> corpora, uint64_t cps,
                        uint64_t seq_len);
  const std::vector<uint64_t>& client(uint64_t c) const;
};

// BatchStream::next without hidden state: rows [cursor, cursor+batch) of the
// client's epoch-shuffled block sequence.  Writes batch*S inputs/targets.
void stream_rows(const Plan& p, uint64_t client, uint64_t seed, uint64_t cursor,
                 uint64_t batch, int32_t* inputs, int32_t* targets);

// ---- evaluation set / checkpoints (checkpoint.cpp) ---------------------------------
struct EvalSet {  // build_eval_batches (harness.cpp:440-472)
  uint64_t seq_len = 0;
  std::vector<int32_t> inputs, targets;  // concatenated rows
  std::vector<uint64_t> batch_sizes;
};
EvalSet build_eval_set(const std::vector<std::string>& styles, uint64_t eval_sequences,
                       uint64_t data_seed, uint64_t vocab, uint64_t seq_len, uint64_t eval_batch);

uint64_t crc64(const void* data, size_t len);  // CRC-64/XZ (checkpoint.h:14-16)
void write_phck(const std::string& path, const photon_model_cfg& m, const double* params,
                uint64_t round);
uint64_t read_phck(const std::string& path, const photon_model_cfg& m, double* params);

struct ResumeState {  // PersistedState (harness.cpp:527-535), federated fields
  uint64_t next_round = 0;
  double initial_ppl = 0.0;
  uint64_t sync_events = 0;
  std::vector<uint64_t> cursors;
};
void write_state_json(const std::string& path, const ResumeState& st);
ResumeState read_state_json(const std::string& path);

// ---- the multi-GPU round boundary's plan (runner.cpp, central.cpp, p2p.cpp) ----
// The flat parameter vector is cut into `world` contiguous shards of
// shard_len elements (a multiple of 4 for 128-bit access; world * shard_len >=
// P).  Slot si of a round's ascending sampled clients (worker w of the
// centralized baseline) trains on rank si % world, so each shard owner sees its
// shard of every model in the canonical ascending order (aggregator.cpp:177).
inline uint64_t shard_len(uint64_t P, int world) {
  return ((P + (uint64_t)world - 1) / (uint64_t)world + 3) / 4 * 4;
}
inline int slot_owner(uint64_t si, int world) { return (int)(si % (uint64_t)world); }
// The NVLink peer-memory boundary kernel takes at most this many surviving
// models and ranks (its pointer tables), and replicas up to kPeerMaxBytes: on
// 4 B200s 27.5 GB replicas (6.87B fp32) collapse to ~200 GB/s once remote loads
// and stores run together (remote address translation over very large
// mappings), where the NCCL path keeps ~500 GB/s.
constexpr int kMaxPeerModels = 16;
constexpr int kMaxPeerWorld = 16;
constexpr uint64_t kPeerMaxBytes = 24000000000ull;
// Whether a runner sets the peer boundary up at all (PHOTON_BOUNDARY=nccl|p2p
// forces either), from the padded fp32 replica size.
bool boundary_prefers_peer(uint64_t replica_bytes);
// Whether a round of k sampled clients with n_surv survivors takes it: decided
// from quantities every rank shares -- the survivor count and the busiest
// rank's local model count ceil(k / world) -- so all ranks take the same path.
inline bool peer_round_ok(uint64_t n_surv, uint64_t k, int world) {
  return n_surv <= (uint64_t)kMaxPeerModels && world <= kMaxPeerWorld &&
         (k + (uint64_t)world - 1) / (uint64_t)world <= (uint64_t)kMaxPeerModels;
}

}  // namespace photon
