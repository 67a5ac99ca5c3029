// checkpoint.cpp -- PHCK model snapshots (checkpoint.h:17-45) and the runner's
// resume state (harness.cpp:527-570), host side.
//
//   "PHCK" | u32 version=1 | u64 round | u64 param_count | u64 crc64 |
//   entry table (u32 name_len, name, u32 rank, u64 dims...) | f64 payload
// little-endian; the CRC-64/XZ covers table + payload; written to <path>.tmp
// and renamed into place.  Byte-identical to the reference writer for the same
// (params, round) (tests/test_checkpoint.py).
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <sstream>

#include "host.hpp"

namespace photon {

namespace {

const uint64_t* crc_table() {  // reflected 0x42F0E1EBA9EA3693
  static uint64_t table[256];
  static bool init = [] {
    for (uint64_t i = 0; i < 256; ++i) {
      uint64_t c = i;
      for (int b = 0; b < 8; ++b) c = (c >> 1) ^ ((c & 1) ? 0xC96C5795D7870F42ULL : 0);
      table[i] = c;
    }
    return true;
  }();
  (void)init;
  return table;
}

template <typename T>
void put(std::vector<uint8_t>& buf, T v) {
  const auto* p = reinterpret_cast<const uint8_t*>(&v);
  buf.insert(buf.end(), p, p + sizeof(T));
}

template <typename T>
T take(const std::vector<uint8_t>& buf, size_t& off) {
  if (off + sizeof(T) > buf.size()) throw Error(PHOTON_ERR_INTEGRITY, "checkpoint truncated");
  T v;
  std::memcpy(&v, buf.data() + off, sizeof(T));
  off += sizeof(T);
  return v;
}

void write_file_atomic(const std::string& path, const std::vector<uint8_t>& a,
                       const std::vector<uint8_t>& b) {
  const std::string tmp = path + ".tmp";
  {
    std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
    if (!f) throw Error(PHOTON_ERR_IO, "cannot open " + tmp + " for writing");
    f.write(reinterpret_cast<const char*>(a.data()), (std::streamsize)a.size());
    f.write(reinterpret_cast<const char*>(b.data()), (std::streamsize)b.size());
    f.flush();
    if (!f.good()) throw Error(PHOTON_ERR_IO, "short write to " + tmp);
  }
  if (std::rename(tmp.c_str(), path.c_str()) != 0)
    throw Error(PHOTON_ERR_IO, "rename " + tmp + " -> " + path + " failed");
}

}  // namespace

uint64_t crc64(const void* data, size_t len) {
  const uint64_t* t = crc_table();
  const auto* p = static_cast<const uint8_t*>(data);
  uint64_t c = ~0ULL;
  for (size_t i = 0; i < len; ++i) c = (c >> 8) ^ t[(c ^ p[i]) & 0xFF];
  return ~c;
}

void write_phck(const std::string& path, const photon_model_cfg& m, const double* params,
                uint64_t round) {
  const std::vector<Entry> lay = layout(m);
  const uint64_t P = param_count(m);
  std::vector<uint8_t> body;
  for (const Entry& e : lay) {
    put<uint32_t>(body, (uint32_t)e.name.size());
    body.insert(body.end(), e.name.begin(), e.name.end());
    put<uint32_t>(body, e.cols ? 2u : 1u);
    put<uint64_t>(body, e.rows);
    if (e.cols) put<uint64_t>(body, e.cols);
  }
  const auto* pp = reinterpret_cast<const uint8_t*>(params);
  body.insert(body.end(), pp, pp + P * sizeof(double));
  std::vector<uint8_t> head;
  const char magic[4] = {'P', 'H', 'C', 'K'};
  head.insert(head.end(), magic, magic + 4);
  put<uint32_t>(head, 1u);
  put<uint64_t>(head, round);
  put<uint64_t>(head, P);
  put<uint64_t>(head, crc64(body.data(), body.size()));
  write_file_atomic(path, head, body);
}

uint64_t read_phck(const std::string& path, const photon_model_cfg& m, double* params) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw Error(PHOTON_ERR_IO, "cannot open " + path);
  std::vector<uint8_t> raw((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  if (raw.size() < 4 || std::memcmp(raw.data(), "PHCK", 4) != 0)
    throw Error(PHOTON_ERR_INTEGRITY, "not a checkpoint file: " + path);
  size_t off = 4;
  const uint32_t version = take<uint32_t>(raw, off);
  if (version != 1)
    throw Error(PHOTON_ERR_INTEGRITY, "unsupported checkpoint version " + std::to_string(version));
  const uint64_t round = take<uint64_t>(raw, off);
  const uint64_t count = take<uint64_t>(raw, off);
  const uint64_t crc = take<uint64_t>(raw, off);
  if (crc64(raw.data() + off, raw.size() - off) != crc)
    throw Error(PHOTON_ERR_INTEGRITY, "checkpoint checksum mismatch: " + path);
  // entry table (checkpoint.cpp: ends when the declared scalar count is reached)
  const std::vector<Entry> lay = layout(m);
  uint64_t seen = 0;
  size_t i = 0;
  bool match = true;
  while (seen < count) {
    const uint32_t nl = take<uint32_t>(raw, off);
    if (off + nl > raw.size()) throw Error(PHOTON_ERR_INTEGRITY, "checkpoint truncated");
    const std::string name(reinterpret_cast<const char*>(raw.data() + off), nl);
    off += nl;
    const uint32_t rank = take<uint32_t>(raw, off);
    uint64_t numel = 1, dims[8] = {0};
    for (uint32_t r = 0; r < rank; ++r) {
      const uint64_t d = take<uint64_t>(raw, off);
      if (r < 8) dims[r] = d;
      numel *= d;
    }
    seen += numel;
    if (i >= lay.size() || lay[i].name != name || rank != (lay[i].cols ? 2u : 1u) ||
        dims[0] != lay[i].rows || (lay[i].cols && dims[1] != lay[i].cols))
      match = false;
    ++i;
  }
  if (seen != count)
    throw Error(PHOTON_ERR_INTEGRITY, "checkpoint entry table does not sum to param_count");
  if (off + count * sizeof(double) != raw.size())
    throw Error(PHOTON_ERR_INTEGRITY, off + count * sizeof(double) > raw.size()
                                          ? "checkpoint truncated"
                                          : "checkpoint has trailing bytes");
  // combinable with the model layout (param_vector.cpp:69-84 -> ShapeError)
  if (!match || i != lay.size() || count != param_count(m))
    throw Error(PHOTON_ERR_SHAPE, "checkpoint layout does not match the model: " + path);
  std::memcpy(params, raw.data() + off, count * sizeof(double));
  return round;
}

// state.json (harness.cpp:527-570), format 1.  The simulated-time fields of
// the cost model are out of scope and written as zeros.
void write_state_json(const std::string& path, const ResumeState& st) {
  std::ostringstream o;
  o.precision(17);
  o << "{\n  \"cursors\": [";
  for (size_t i = 0; i < st.cursors.size(); ++i) o << (i ? ",\n    " : "\n    ") << st.cursors[i];
  o << (st.cursors.empty() ? "]" : "\n  ]") << ",\n";
  o << "  \"format\": 1,\n";
  o << "  \"initial_ppl\": " << st.initial_ppl << ",\n";
  o << "  \"next_round\": " << st.next_round << ",\n";
  o << "  \"opt_step_count\": 0,\n";
  o << "  \"sync_events\": " << st.sync_events << ",\n";
  o << "  \"t_cum\": 0.0,\n";
  o << "  \"total_bytes\": 0.0\n}\n";
  const std::string s = o.str();
  write_file_atomic(path, std::vector<uint8_t>(s.begin(), s.end()), {});
}

namespace {
// minimal reader for the fields above: "key": number | [numbers]
size_t find_key(const std::string& s, const char* key) {
  const std::string k = std::string("\"") + key + "\"";
  const size_t p = s.find(k);
  if (p == std::string::npos) throw Error(PHOTON_ERR_PARSE, std::string("state.json: missing ") + key);
  const size_t c = s.find(':', p + k.size());
  if (c == std::string::npos) throw Error(PHOTON_ERR_PARSE, std::string("state.json: bad ") + key);
  return c + 1;
}
}  // namespace

ResumeState read_state_json(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw Error(PHOTON_ERR_IO, "cannot open " + path + " (nothing to resume?)");
  const std::string s((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  ResumeState st;
  try {
    st.next_round = std::stoull(s.substr(find_key(s, "next_round")));
    st.initial_ppl = std::stod(s.substr(find_key(s, "initial_ppl")));
    st.sync_events = std::stoull(s.substr(find_key(s, "sync_events")));
    size_t p = s.find('[', find_key(s, "cursors"));
    const size_t e = s.find(']', p);
    if (p == std::string::npos || e == std::string::npos)
      throw Error(PHOTON_ERR_PARSE, "state.json: bad cursors");
    std::istringstream in(s.substr(p + 1, e - p - 1));
    std::string tok;
    while (std::getline(in, tok, ','))
      if (tok.find_first_of("0123456789") != std::string::npos) st.cursors.push_back(std::stoull(tok));
  } catch (const std::logic_error&) {
    throw Error(PHOTON_ERR_PARSE, "state.json: malformed " + path);
  }
  return st;
}

// build_eval_batches (harness.cpp:440-472): per style a held-out corpus from
// mix_seed(data_seed, "Eval"), eval_sequences / n_styles sequences each, cut
// into batches of eval_batch rows (the last one may be short).
EvalSet build_eval_set(const std::vector<std::string>& styles, uint64_t eval_sequences,
                       uint64_t data_seed, uint64_t vocab, uint64_t seq_len, uint64_t eval_batch) {
  if (styles.empty()) throw Error(PHOTON_ERR_CONFIG, "eval set: no styles");
  if (eval_batch == 0) throw Error(PHOTON_ERR_CONFIG, "eval set: eval_batch must be >= 1");
  EvalSet es;
  es.seq_len = seq_len;
  const uint64_t per_style = eval_sequences / styles.size();
  const uint64_t bl = seq_len + 1;
  uint64_t cur = 0;
  for (const std::string& style : styles) {
    const std::vector<uint16_t> c =
        generate_corpus(style_index(style), per_style * bl, derive(data_seed, kPurposeEval),
                        (uint32_t)vocab);
    for (uint64_t s = 0; s < per_style; ++s) {
      for (uint64_t t = 0; t < seq_len; ++t) {
        es.inputs.push_back((int32_t)c[s * bl + t]);
        es.targets.push_back((int32_t)c[s * bl + t + 1]);
      }
      if (++cur == eval_batch) {
        es.batch_sizes.push_back(cur);
        cur = 0;
      }
    }
  }
  if (cur) es.batch_sizes.push_back(cur);
  return es;
}

}  // namespace photon
