// host.cpp -- see host.hpp.  Reference citations: /root/reference/proj/core.
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace photon {

// rng.h:53-67
double Draws::gauss() {
  if (has_spare_) {
    has_spare_ = false;
    return spare_;
  }
  double u1;
  do {
    u1 = unit();
  } while (u1 <= 0.0);
  const double u2 = unit();
  const double radius = std::sqrt(-2.0 * std::log(u1));
  const double angle = 6.283185307179586476925286766559 * u2;
  spare_ = radius * std::sin(angle);
  has_spare_ = true;
  return radius * std::cos(angle);
}

// model.cpp:10-19
void validate_model(const photon_model_cfg& m) {
  if (m.n_blocks == 0) throw Error(PHOTON_ERR_CONFIG, "model: n_blocks must be >= 1");
  if (m.d_model == 0) throw Error(PHOTON_ERR_CONFIG, "model: d_model must be >= 1");
  if (m.n_heads == 0 || m.d_model % m.n_heads != 0)
    throw Error(PHOTON_ERR_CONFIG, "model: d_model must be divisible by n_heads");
  if (m.expansion_ratio == 0) throw Error(PHOTON_ERR_CONFIG, "model: expansion_ratio must be >= 1");
  if (m.vocab_size < 2) throw Error(PHOTON_ERR_CONFIG, "model: vocab_size must be >= 2");
  if (m.seq_len == 0) throw Error(PHOTON_ERR_CONFIG, "model: seq_len must be >= 1");
}

// model.cpp:21-26
uint64_t param_count(const photon_model_cfg& m) {
  const uint64_t d = m.d_model, e = m.expansion_ratio;
  return m.vocab_size * d + m.seq_len * d + m.n_blocks * ((4 + 2 * e) * d * d + (9 + e) * d) +
         2 * d + d * m.vocab_size + m.vocab_size;
}

// model.cpp:32-61: the canonical entry order is the wire format of every buffer.
std::vector<Entry> layout(const photon_model_cfg& m) {
  const uint64_t d = m.d_model, hid = m.expansion_ratio * d;
  std::vector<Entry> out;
  uint64_t off = 0;
  auto push = [&](std::string name, uint64_t r, uint64_t c) {
    out.push_back(Entry{std::move(name), off, r, c});
    off += c ? r * c : r;
  };
  push("token_embedding", m.vocab_size, d);
  push("position_embedding", m.seq_len, d);
  for (uint64_t b = 0; b < m.n_blocks; ++b) {
    const std::string p = "block" + std::to_string(b) + ".";
    push(p + "ln1.gain", d, 0);
    push(p + "ln1.bias", d, 0);
    for (const char* w : {"q", "k", "v", "o"}) {
      push(p + "attn.w" + w, d, d);
      push(p + "attn.b" + w, d, 0);
    }
    push(p + "ln2.gain", d, 0);
    push(p + "ln2.bias", d, 0);
    push(p + "mlp.w1", d, hid);
    push(p + "mlp.b1", hid, 0);
    push(p + "mlp.w2", hid, d);
    push(p + "mlp.b2", d, 0);
  }
  push("final_ln.gain", d, 0);
  push("final_ln.bias", d, 0);
  push("head.w", d, m.vocab_size);
  push("head.b", m.vocab_size, 0);
  return out;
}

ModelOffsets model_offsets(const photon_model_cfg& m) {
  const auto lay = layout(m);
  ModelOffsets o{};
  o.tok = lay[0].offset;
  o.pos = lay[1].offset;
  for (uint64_t b = 0; b < m.n_blocks; ++b) {
    const Entry* e = &lay[2 + 16 * b];
    o.blocks.push_back(BlockOffsets{e[0].offset, e[1].offset, e[2].offset, e[3].offset,
                                    e[4].offset, e[5].offset, e[6].offset, e[7].offset,
                                    e[8].offset, e[9].offset, e[10].offset, e[11].offset,
                                    e[12].offset, e[13].offset, e[14].offset, e[15].offset});
  }
  const size_t t = 2 + 16 * m.n_blocks;
  o.lnfg = lay[t].offset;
  o.lnfb = lay[t + 1].offset;
  o.head_w = lay[t + 2].offset;
  o.head_b = lay[t + 3].offset;
  return o;
}

namespace {
bool has_suffix(const std::string& s, const char* suf) {
  const size_t n = std::char_traits<char>::length(suf);
  return s.size() >= n && s.compare(s.size() - n, n, suf) == 0;
}
}  // namespace

// model.cpp:72-96: gains 1, biases 0 (no draws), weights N(0, 0.02) in entry
// order; residual projections (attn.wo, mlp.w2) scaled by 1/sqrt(2L).
std::vector<double> init_params(const photon_model_cfg& m, uint64_t seed) {
  validate_model(m);
  Draws rng(seed);
  const double sd = 0.02;
  const double sd_resid = sd / std::sqrt(2.0 * static_cast<double>(m.n_blocks));
  std::vector<double> out(param_count(m), 0.0);
  for (const Entry& e : layout(m)) {
    double* v = out.data() + e.offset;
    if (has_suffix(e.name, ".gain")) {
      std::fill(v, v + e.numel(), 1.0);
    } else if (e.cols == 0 || e.name == "head.b") {
      // every rank-1 non-gain entry is a bias: zeros, no draws
    } else {
      const double s =
          (has_suffix(e.name, "attn.wo") || has_suffix(e.name, "mlp.w2")) ? sd_resid : sd;
      for (uint64_t j = 0; j < e.numel(); ++j) v[j] = rng.gauss() * s;
    }
  }
  return out;
}

// optim.cpp:10-27
double lr_at(const photon_lr_schedule& s, uint64_t step) {
  if (!(s.eta_max > 0.0)) throw Error(PHOTON_ERR_CONFIG, "schedule: eta_max must be > 0");
  if (s.decay_steps == 0) throw Error(PHOTON_ERR_CONFIG, "schedule: decay_steps must be >= 1");
  if (s.alpha < 0.0 || s.alpha > 1.0) throw Error(PHOTON_ERR_CONFIG, "schedule: alpha in [0,1]");
  if (s.warmup_steps > 0 && step < s.warmup_steps)
    return s.eta_max * static_cast<double>(step) / static_cast<double>(s.warmup_steps);
  const double p = std::min(
      1.0, static_cast<double>(step - s.warmup_steps) / static_cast<double>(s.decay_steps));
  const double lo = s.alpha * s.eta_max;
  return lo + (s.eta_max - lo) * 0.5 * (1.0 + std::cos(3.14159265358979323846 * p));
}

// aggregator.cpp:25-41: partial Fisher-Yates, first k slots, ascending.
std::vector<uint64_t> sample_clients(uint64_t population, uint64_t k, uint64_t seed,
                                     uint64_t round) {
  if (k > population) throw Error(PHOTON_ERR_CONFIG, "sample_clients: K > P");
  if (k == 0) throw Error(PHOTON_ERR_CONFIG, "sample_clients: K must be >= 1");
  std::vector<uint64_t> ids(population);
  std::iota(ids.begin(), ids.end(), 0);
  Draws rng(derive(seed, kPurposeSample, round));
  for (uint64_t i = 0; i < k; ++i) std::swap(ids[i], ids[i + rng.below(population - i)]);
  ids.resize(k);
  std::sort(ids.begin(), ids.end());
  return ids;
}

// data.cpp:24-71: four band-separated affine Markov styles.
int style_index(const std::string& style) {
  static const char* kNames[4] = {"academic", "web", "reference", "prose"};
  for (int i = 0; i < 4; ++i)
    if (style == kNames[i]) return i;
  throw Error(PHOTON_ERR_CONFIG, "unknown data style: " + style);
}

std::vector<uint16_t> generate_corpus(int style, uint64_t length, uint64_t seed, uint32_t vocab) {
  static const uint32_t kMul[4] = {1, 3, 5, 7}, kAdd[4] = {1, 1, 2, 3};
  if (style < 0 || style > 3) throw Error(PHOTON_ERR_CONFIG, "unknown data style");
  if (vocab < 8 || vocab % 4 != 0)
    throw Error(PHOTON_ERR_CONFIG, "corpus vocab_size must be a multiple of 4, >= 8");
  if (length == 0) throw Error(PHOTON_ERR_CONFIG, "corpus length must be > 0");
  const uint32_t band = vocab / 4, base = static_cast<uint32_t>(style) * band;
  Draws rng(derive(seed, kPurposeCorpus, static_cast<uint64_t>(style)));
  std::vector<uint16_t> out(length);
  uint32_t state = static_cast<uint32_t>(rng.below(band));
  out[0] = static_cast<uint16_t>(base + state);
  for (uint64_t i = 1; i < length; ++i) {
    state = rng.unit() < 0.8 ? (kMul[style] * state + kAdd[style]) % band
                             : static_cast<uint32_t>(rng.below(band));
    out[i] = static_cast<uint16_t>(base + state);
  }
  return out;
}

// data.cpp:137-164: shuffle block order once, deal round-robin.
Plan Plan::iid(std::vector<uint16_t> tokens, uint64_t n_shards, uint64_t seq_len, uint64_t seed) {
  if (n_shards == 0) throw Error(PHOTON_ERR_CONFIG, "partition: n_shards must be >= 1");
  if (seq_len == 0) throw Error(PHOTON_ERR_CONFIG, "partition: seq_len must be >= 1");
  const uint64_t bl = seq_len + 1, n_blocks = tokens.size() / bl;
  if (n_blocks < n_shards)
    throw Error(PHOTON_ERR_CONFIG, "corpus too short: " + std::to_string(n_blocks) +
                                       " blocks for " + std::to_string(n_shards) + " shards");
  std::vector<uint32_t> order(n_blocks);
  std::iota(order.begin(), order.end(), 0u);
  Draws rng(derive(seed, kPurposeShard));
  rng.permute(order);
  Plan p;
  p.seq_len = seq_len;
  p.corpora.push_back(std::move(tokens));
  p.blocks.assign(n_shards, {});
  for (uint64_t i = 0; i < n_blocks; ++i)
    p.blocks[i % n_shards].push_back(static_cast<uint64_t>(order[i]) * bl);
  return p;
}

// data.cpp:166-199: source-major contiguous runs, remainder dropped.
Plan Plan::by_source(std::vector<std::vector<uint16_t>> corpora, uint64_t cps, uint64_t seq_len) {
  if (corpora.empty()) throw Error(PHOTON_ERR_CONFIG, "partition: no corpora");
  if (cps == 0) throw Error(PHOTON_ERR_CONFIG, "partition: clients_per_source must be >= 1");
  if (seq_len == 0) throw Error(PHOTON_ERR_CONFIG, "partition: seq_len must be >= 1");
  const uint64_t bl = seq_len + 1;
  Plan p;
  p.seq_len = seq_len;
  p.blocks.assign(corpora.size() * cps, {});
  for (uint64_t s = 0; s < corpora.size(); ++s) {
    const uint64_t per = (corpora[s].size() / bl) / cps;
    if (per == 0) throw Error(PHOTON_ERR_CONFIG, "source too short for clients_per_source");
    for (uint64_t c = 0; c < cps; ++c)
      for (uint64_t b = 0; b < per; ++b)
        p.blocks[s * cps + c].push_back((s << 48) | ((c * per + b) * bl));
  }
  p.corpora = std::move(corpora);
  return p;
}

const std::vector<uint64_t>& Plan::client(uint64_t c) const {
  if (c >= blocks.size()) throw Error(PHOTON_ERR_LOOKUP, "unknown client id " + std::to_string(c));
  return blocks[c];
}

// data.cpp:222-253: row idx of the stream is block perm_epoch[idx % n] with
// perm_epoch a Fisher-Yates shuffle seeded by (seed, "Epoc", client, epoch).
void stream_rows(const Plan& p, uint64_t client, uint64_t seed, uint64_t cursor, uint64_t batch,
                 int32_t* inputs, int32_t* targets) {
  const auto& blocks = p.client(client);
  if (batch == 0) throw Error(PHOTON_ERR_CONFIG, "stream: batch_size must be >= 1");
  const uint64_t n = blocks.size(), S = p.seq_len;
  std::vector<uint32_t> perm;
  uint64_t epoch_cached = ~0ULL;
  for (uint64_t r = 0; r < batch; ++r) {
    const uint64_t idx = cursor + r, epoch = idx / n;
    if (epoch != epoch_cached) {
      perm.resize(n);
      std::iota(perm.begin(), perm.end(), 0u);
      Draws rng(derive(seed, kPurposeEpoch, client, epoch));
      rng.permute(perm);
      epoch_cached = epoch;
    }
    const uint64_t ref = blocks[perm[idx % n]];
    const uint16_t* tok = p.corpora[ref >> 48].data() + (ref & ((1ULL << 48) - 1));
    for (uint64_t t = 0; t < S; ++t) {
      inputs[r * S + t] = tok[t];
      targets[r * S + t] = tok[t + 1];
    }
  }
}

}  // namespace photon
