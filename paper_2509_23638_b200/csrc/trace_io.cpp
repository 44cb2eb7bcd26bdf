// Trace file format v1 — write_trace / read_trace (workload.cpp:290-436), so the B200
// driver consumes traces the reference produced (and the reference reads ours).
//
// Layout: one JSON header line, keys in nlohmann's (sorted) order
//   {"batch_size":B,"checksum":FNV1a64(body),"format_version":1,"seed":S,"spec":{...}}
// then one body line per (token, layer) step in (token, layer) order (Trace::step,
// workload.cpp:81-83):
//   layer \t hidden[H] \t gate_weights[E] \t active[k] \t e:m e:m ...
// doubles as "%.17g" (round-trip exact), token map in ascending expert order
// (std::map iteration). The reader returns dense arrays; the writer reproduces the
// reference's bytes exactly for the same trace (tests/test_trace_io.py).
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

#include "common.hpp"

struct ps_trace_s {
  ps_model_spec spec{};
  int32_t batch = 0;
  uint64_t seed = 0, checksum = 0;
  std::vector<double> hidden, gate_weights;  // [B*L*H], [B*L*E]
  std::vector<int32_t> active, tokens;        // [B*L*k], [B*L*E]
};

namespace ps {
namespace {

// TraceFormatError / TraceChecksumError (workload.hpp:106-111) are runtime_errors.
[[noreturn]] void format_error(const std::string& m) { fail(PS_ERUNTIME, "TraceFormatError: " + m); }

// Minimal JSON reader for the header: objects of unsigned integers / nested objects.
struct JsonValue {
  bool is_object = false;
  uint64_t number = 0;
  std::map<std::string, JsonValue> members;
};

struct JsonParser {
  const std::string& s;
  size_t p = 0;
  void ws() {
    while (p < s.size() && (s[p] == ' ' || s[p] == '\t' || s[p] == '\r' || s[p] == '\n')) ++p;
  }
  void expect(char c) {
    ws();
    if (p >= s.size() || s[p] != c) format_error(std::string("read_trace: bad header: expected '") + c + "'");
    ++p;
  }
  std::string str() {
    expect('"');
    std::string out;
    while (p < s.size() && s[p] != '"') {
      if (s[p] == '\\') format_error("read_trace: bad header: escapes unsupported");
      out += s[p++];
    }
    expect('"');
    return out;
  }
  JsonValue value() {
    ws();
    JsonValue v;
    if (p < s.size() && s[p] == '{') {
      ++p;
      v.is_object = true;
      ws();
      if (p < s.size() && s[p] == '}') {
        ++p;
        return v;
      }
      while (true) {
        std::string k = str();
        expect(':');
        v.members[k] = value();
        ws();
        if (p < s.size() && s[p] == ',') {
          ++p;
          continue;
        }
        expect('}');
        return v;
      }
    }
    const size_t b = p;
    while (p < s.size() && s[p] >= '0' && s[p] <= '9') ++p;
    if (b == p) format_error("read_trace: bad header: expected a non-negative integer");
    errno = 0;
    v.number = std::strtoull(s.c_str() + b, nullptr, 10);
    if (errno == ERANGE) format_error("read_trace: bad header: integer overflow");
    return v;
  }
};

uint64_t at_num(const JsonValue& o, const char* key) {
  auto it = o.members.find(key);
  if (it == o.members.end() || it->second.is_object)
    fail(PS_ERUNTIME, std::string("read_trace: header key missing or not a number: ") + key);
  return it->second.number;
}

std::string fmt_double(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

std::vector<std::string> split(const std::string& line, char sep) {
  std::vector<std::string> out;
  size_t pos = 0;
  while (true) {
    size_t q = line.find(sep, pos);
    out.push_back(line.substr(pos, q == std::string::npos ? q : q - pos));
    if (q == std::string::npos) break;
    pos = q + 1;
  }
  return out;
}

// Whitespace-separated doubles / ints of one field into out[0..want). Returns "" or the
// problem (unparsable value or a count other than `want`); the caller decides whether it
// is fatal now (syntax the reference parser also rejects) or after the checksum check.
template <typename T>
std::string parse_list(const std::string& f, size_t want, T* out, const char* what) {
  const char* c = f.c_str();
  size_t n = 0;
  while (true) {
    while (*c == ' ') ++c;
    if (!*c) break;
    char* end = nullptr;
    errno = 0;
    T v;
    if constexpr (std::is_same_v<T, double>) v = std::strtod(c, &end);
    else v = static_cast<T>(std::strtol(c, &end, 10));
    if (end == c || errno == ERANGE || (*end && *end != ' ')) return std::string("trace body line: bad ") + what;
    if (n >= want) return std::string("trace body line: too many ") + what;
    out[n++] = v;
    c = end;
  }
  if (n != want) return std::string("trace body line: wrong number of ") + what;
  return {};
}

std::string header_line(const ps_model_spec& s, int batch, uint64_t seed, uint64_t checksum) {
  std::ostringstream h;
  h << "{\"batch_size\":" << batch << ",\"checksum\":" << checksum << ",\"format_version\":1,\"seed\":" << seed
    << ",\"spec\":{\"expert_bytes\":" << s.expert_bytes << ",\"experts_per_layer\":" << s.experts_per_layer
    << ",\"group_begin_middle\":" << s.group_begin_middle << ",\"group_begin_output\":" << s.group_begin_output
    << ",\"hidden_dim\":" << s.hidden_dim << ",\"num_layers\":" << s.num_layers << ",\"top_k\":" << s.top_k << "}}";
  return h.str();
}

uint64_t fnv1a64(const char* data, size_t n) {  // workload.cpp:290-297
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= static_cast<unsigned char>(data[i]);
    h *= 0x100000001b3ull;
  }
  return h;
}

void read_trace(const char* path, ps_trace_s& t) {
  require(path != nullptr, "read_trace: null path");
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(PS_ERUNTIME, std::string("read_trace: cannot open ") + path);
  std::string line;
  if (!std::getline(in, line)) format_error("read_trace: missing header");
  JsonParser jp{line};
  JsonValue hdr = jp.value();
  if (!hdr.is_object) format_error("read_trace: bad header: not an object");
  if (at_num(hdr, "format_version") != 1) format_error("read_trace: unsupported format version");
  auto sp = hdr.members.find("spec");
  if (sp == hdr.members.end() || !sp->second.is_object) fail(PS_ERUNTIME, "read_trace: header key missing: spec");
  const JsonValue& js = sp->second;
  ps_model_spec& s = t.spec;
  s.num_layers = static_cast<int32_t>(at_num(js, "num_layers"));
  s.experts_per_layer = static_cast<int32_t>(at_num(js, "experts_per_layer"));
  s.top_k = static_cast<int32_t>(at_num(js, "top_k"));
  s.expert_bytes = at_num(js, "expert_bytes");
  s.hidden_dim = static_cast<int32_t>(at_num(js, "hidden_dim"));
  s.group_begin_middle = static_cast<int32_t>(at_num(js, "group_begin_middle"));
  s.group_begin_output = static_cast<int32_t>(at_num(js, "group_begin_output"));
  if (ps_spec_validate(&s) != PS_OK) fail(PS_EINVAL, ps_last_error());  // spec_from_json -> validate()
  t.batch = static_cast<int32_t>(at_num(hdr, "batch_size"));
  t.seed = at_num(hdr, "seed");
  t.checksum = at_num(hdr, "checksum");
  require(t.batch >= 1, "read_trace: batch_size must be >= 1");

  const int L = s.num_layers, E = s.experts_per_layer, K = s.top_k, H = s.hidden_dim;
  const size_t n_steps = static_cast<size_t>(t.batch) * L;
  t.hidden.assign(n_steps * H, 0.0);
  t.gate_weights.assign(n_steps * E, 0.0);
  t.active.assign(n_steps * K, 0);
  t.tokens.assign(n_steps * E, 0);
  // Syntax errors the reference's parse_step also throws on (field count, token map
  // without ':') are raised at once; anything the reference would accept silently but a
  // dense trace cannot hold (vector sizes, expert ids, step order/count) is deferred until
  // after the checksum, so a corrupted file reports TraceChecksumError like the reference.
  std::string deferred;
  auto note = [&](const std::string& m) {
    if (deferred.empty()) deferred = m;
  };
  uint64_t h = 0xcbf29ce484222325ull;
  size_t i = 0;
  while (std::getline(in, line)) {
    for (unsigned char c : line) {
      h ^= c;
      h *= 0x100000001b3ull;
    }
    h ^= static_cast<unsigned char>('\n');
    h *= 0x100000001b3ull;
    auto f = split(line, '\t');
    if (f.size() != 5) format_error("trace body line: expected 5 fields");
    for (const std::string& pr : split(f[4], ' '))
      if (!pr.empty() && pr.find(':') == std::string::npos) format_error("trace body line: bad token map");
    if (i >= n_steps) note("read_trace: more steps than batch_size * num_layers");
    if (deferred.empty()) {
      int32_t layer = 0;
      std::string err = parse_list(f[0], 1, &layer, "layer");
      if (err.empty() && layer != static_cast<int32_t>(i % L)) err = "read_trace: steps not in (token, layer) order";
      if (err.empty()) err = parse_list(f[1], H, t.hidden.data() + i * H, "hidden");
      if (err.empty()) err = parse_list(f[2], E, t.gate_weights.data() + i * E, "gate weights");
      if (err.empty()) err = parse_list(f[3], K, t.active.data() + i * K, "active experts");
      for (const std::string& pr : split(f[4], ' ')) {
        if (pr.empty() || !err.empty()) continue;
        const size_t colon = pr.find(':');
        int32_t e = 0, m = 0;
        err = parse_list(pr.substr(0, colon), 1, &e, "token map expert");
        if (err.empty()) err = parse_list(pr.substr(colon + 1), 1, &m, "token map count");
        if (err.empty() && (e < 0 || e >= E)) err = "trace body line: token map expert out of range";
        if (err.empty()) t.tokens[i * E + e] = m;
      }
      if (!err.empty()) note(err);
    }
    ++i;
  }
  if (h != t.checksum) fail(PS_ERUNTIME, std::string("TraceChecksumError: read_trace: checksum mismatch in ") + path);
  if (!deferred.empty()) format_error(deferred);
  if (i != n_steps) format_error("read_trace: fewer steps than batch_size * num_layers");
}

void write_trace(const char* path, const ps_model_spec& s, int batch, uint64_t seed, const double* hidden,
                 const double* gw, const int32_t* active, const int32_t* tokens) {
  require(path && hidden && gw && active && tokens, "write_trace: null argument");
  if (ps_spec_validate(&s) != PS_OK) fail(PS_EINVAL, ps_last_error());
  require(batch >= 1, "write_trace: batch must be >= 1");
  const int L = s.num_layers, E = s.experts_per_layer, K = s.top_k, H = s.hidden_dim;
  std::string body;
  const size_t n_steps = static_cast<size_t>(batch) * L;
  for (size_t i = 0; i < n_steps; ++i) {
    body += std::to_string(i % L);
    body += '\t';
    for (int d = 0; d < H; ++d) {
      if (d) body += ' ';
      body += fmt_double(hidden[i * H + d]);
    }
    body += '\t';
    for (int e = 0; e < E; ++e) {
      if (e) body += ' ';
      body += fmt_double(gw[i * E + e]);
    }
    body += '\t';
    for (int j = 0; j < K; ++j) {
      if (j) body += ' ';
      body += std::to_string(active[i * K + j]);
    }
    body += '\t';
    bool first = true;
    for (int e = 0; e < E; ++e) {
      if (tokens[i * E + e] == 0) continue;
      if (!first) body += ' ';
      first = false;
      body += std::to_string(e) + ':' + std::to_string(tokens[i * E + e]);
    }
    body += '\n';
  }
  std::ofstream out(path, std::ios::binary);
  if (!out) fail(PS_ERUNTIME, std::string("write_trace: cannot open ") + path);
  out << header_line(s, batch, seed, fnv1a64(body.data(), body.size())) << '\n' << body;
  if (!out) fail(PS_ERUNTIME, std::string("write_trace: write failed on ") + path);
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

uint64_t ps_fnv1a64(const void* data, size_t n) { return fnv1a64(static_cast<const char*>(data), n); }

ps_status ps_trace_read(const char* path, ps_trace* out) {
  return guarded([&] {
    require(out != nullptr, "ps_trace_read: null out");
    auto t = std::make_unique<ps_trace_s>();
    read_trace(path, *t);
    *out = t.release();
  });
}

ps_status ps_trace_shape(ps_trace t, ps_model_spec* spec, int32_t* batch, uint64_t* seed, uint64_t* checksum) {
  return guarded([&] {
    require(t != nullptr, "ps_trace_shape: null trace");
    if (spec) *spec = t->spec;
    if (batch) *batch = t->batch;
    if (seed) *seed = t->seed;
    if (checksum) *checksum = t->checksum;
  });
}

ps_status ps_trace_arrays(ps_trace t, double* hidden, double* gate_weights, int32_t* active, int32_t* tokens) {
  return guarded([&] {
    require(t != nullptr, "ps_trace_arrays: null trace");
    if (hidden) std::memcpy(hidden, t->hidden.data(), sizeof(double) * t->hidden.size());
    if (gate_weights) std::memcpy(gate_weights, t->gate_weights.data(), sizeof(double) * t->gate_weights.size());
    if (active) std::memcpy(active, t->active.data(), sizeof(int32_t) * t->active.size());
    if (tokens) std::memcpy(tokens, t->tokens.data(), sizeof(int32_t) * t->tokens.size());
  });
}

ps_status ps_trace_free(ps_trace t) {
  delete t;
  return PS_OK;
}

ps_status ps_trace_write(const char* path, const ps_model_spec* spec, int batch, uint64_t seed, const double* hidden,
                         const double* gate_weights, const int32_t* active, const int32_t* tokens) {
  return guarded([&] {
    require(spec != nullptr, "ps_trace_write: null spec");
    write_trace(path, *spec, batch, seed, hidden, gate_weights, active, tokens);
  });
}

}  // extern "C"
