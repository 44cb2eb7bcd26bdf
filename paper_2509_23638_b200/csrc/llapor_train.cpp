// LLaPor host model: LLPC v1 checkpoint read/write (predictor.cpp:733-929) and the
// online fine_tune step (predictor.cpp:654-663: AdamW passes of run_epoch, 565-592,
// over observed samples). f64 on the host — the nets are 10^4-10^5 parameters — then
// re-uploaded to the GPU for inference (ps_llapor_fine_tune in k4_llapor.cu).
//
// Bit-exactness with the reference: every double is formed with the reference's operand
// order (forward 166-183/205-247, loss 363-403, backward 185-203/263-297, AdamW 317-338),
// randomness comes from the same libstdc++ engine and distributions in the same draw
// order (std::shuffle of the sample order, one uniform per dropout unit), and this file
// is compiled with -ffp-contract=off like the reference build (oracle/Makefile). A model
// fine-tuned here and saved with write_llpc is byte-identical to the reference's
// save_checkpoint after its fine_tune (tests/test_llapor_train.py).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <numeric>
#include <random>

#include "common.hpp"
#include "llapor_model.hpp"

namespace ps {
namespace {

// ------------------------------------------------------------------ LLPC v1 I/O
struct In {
  std::ifstream f;
  template <typename T> T get() {
    T v{};
    f.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!f) fail(PS_ERUNTIME, "checkpoint: truncated file");
    return v;
  }
  std::vector<double> vec() {
    const uint64_t n = get<uint64_t>();
    if (n > (1ull << 31)) fail(PS_ERUNTIME, "checkpoint: corrupt vector length");
    std::vector<double> v(n);
    f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(double)));
    if (!f) fail(PS_ERUNTIME, "checkpoint: truncated file");
    return v;
  }
  void mat(int& r, int& c, std::vector<double>& a) {
    r = get<int32_t>();
    c = get<int32_t>();
    a = vec();
    if (a.size() != static_cast<size_t>(r) * c) fail(PS_ERUNTIME, "checkpoint: corrupt matrix");
  }
  HostBlk blk() {
    HostBlk b;
    mat(b.rows, b.cols, b.w);
    b.b = vec();
    return b;
  }
  GroupHyperH hyper() {
    GroupHyperH h;
    h.base_lr = get<double>();
    h.weight_decay = get<double>();
    h.pca_dim = get<int32_t>();
    h.width = get<int32_t>();
    h.num_blocks = get<int32_t>();
    return h;
  }
};

struct Out {
  std::ofstream f;
  template <typename T> void put(const T& v) { f.write(reinterpret_cast<const char*>(&v), sizeof(T)); }
  void vec(const std::vector<double>& v) {
    put<uint64_t>(v.size());
    f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(double)));
  }
  void mat(int r, int c, const std::vector<double>& a) {
    put<int32_t>(r);
    put<int32_t>(c);
    vec(a);
  }
  void blk(const HostBlk& b) {
    mat(b.rows, b.cols, b.w);
    vec(b.b);
  }
  void hyper(const GroupHyperH& h) {
    put(h.base_lr);
    put(h.weight_decay);
    put<int32_t>(h.pca_dim);
    put<int32_t>(h.width);
    put<int32_t>(h.num_blocks);
  }
};

// ------------------------------------------------------------------ f64 net
double gelu(double x) { return 0.5 * x * (1.0 + std::erf(x / std::sqrt(2.0))); }
double gelu_grad(double x) {
  constexpr double inv_sqrt2pi = 0.3989422804014327;
  return 0.5 * (1.0 + std::erf(x / std::sqrt(2.0))) + x * inv_sqrt2pi * std::exp(-0.5 * x * x);
}
double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }

void affine(const HostBlk& b, const std::vector<double>& x, std::vector<double>& z) {
  z.assign(b.rows, 0.0);
  for (int r = 0; r < b.rows; ++r) {
    double s = 0.0;
    const double* row = b.w.data() + static_cast<size_t>(r) * b.cols;
    for (int c = 0; c < b.cols; ++c) s += row[c] * x[c];
    z[r] = s;
  }
}

struct BlkTape {  // what the backward pass of one GELU block needs
  std::vector<double> x, z, mask;
};

// GELU block with training-mode dropout (one uniform draw per output unit).
std::vector<double> block_train(const HostBlk& b, const std::vector<double>& x, double dropout, std::mt19937_64& rng,
                                BlkTape& t) {
  t.x = x;
  affine(b, x, t.z);
  for (size_t i = 0; i < t.z.size(); ++i) t.z[i] += b.b[i];
  std::vector<double> out(t.z.size());
  for (size_t i = 0; i < t.z.size(); ++i) out[i] = gelu(t.z[i]);
  const double keep = 1.0 - dropout;
  std::uniform_real_distribution<double> unif(0.0, 1.0);
  t.mask.resize(out.size());
  for (size_t i = 0; i < out.size(); ++i) {
    t.mask[i] = (keep > 0.0 && unif(rng) < keep) ? 1.0 / keep : 0.0;
    out[i] *= t.mask[i];
  }
  return out;
}

std::vector<double> block_back(const HostBlk& b, const BlkTape& t, const std::vector<double>& d_out, HostBlk& g) {
  std::vector<double> dz(t.z.size());
  for (size_t i = 0; i < dz.size(); ++i) {
    double dh = d_out[i];
    if (!t.mask.empty()) dh *= t.mask[i];
    dz[i] = dh * gelu_grad(t.z[i]);
  }
  for (int r = 0; r < b.rows; ++r) {
    g.b[r] += dz[r];
    for (int c = 0; c < b.cols; ++c) g.w[static_cast<size_t>(r) * b.cols + c] += dz[r] * t.x[c];
  }
  std::vector<double> dx(b.cols, 0.0);
  for (int r = 0; r < b.rows; ++r)
    for (int c = 0; c < b.cols; ++c) dx[c] += b.w[static_cast<size_t>(r) * b.cols + c] * dz[r];
  return dx;
}

struct NetTape {
  std::vector<double> reduced;
  std::vector<BlkTape> blocks, res;
  std::vector<double> res_in, res_u, y, logits;
  double gate = 1.0;
};

void forward_train(const HostNet& n, const HostSample& s, std::mt19937_64& rng, NetTape& t) {
  if (static_cast<int>(s.reduced.size()) != n.eff_dim || static_cast<int>(s.onehot.size()) != n.E ||
      static_cast<int>(s.gate.size()) != n.E)
    fail(PS_EINVAL, "forward: feature shape mismatch");
  t.reduced = s.reduced;
  std::vector<double> x = s.reduced;
  x.insert(x.end(), s.onehot.begin(), s.onehot.end());
  x.insert(x.end(), s.gate.begin(), s.gate.end());
  t.blocks.resize(n.blocks.size());
  for (size_t i = 0; i < n.blocks.size(); ++i) x = block_train(n.blocks[i], x, n.dropout, rng, t.blocks[i]);
  if (!n.res.empty()) {
    t.res_in = x;
    std::vector<double> u = x;
    t.res.resize(n.res.size());
    for (size_t i = 0; i < n.res.size(); ++i) u = block_train(n.res[i], u, n.dropout, rng, t.res[i]);
    t.res_u = u;
    double d = 0.0;
    for (size_t i = 0; i < n.gate_w.size(); ++i) d += n.gate_w[i] * t.reduced[i];
    t.gate = sigmoid(d + n.gate_b);
    for (size_t i = 0; i < x.size(); ++i) x[i] = u[i] * t.gate + t.res_in[i];
  }
  t.y = x;
  affine(n.out, x, t.logits);
  for (size_t i = 0; i < t.logits.size(); ++i) t.logits[i] += n.out.b[i];
}

void backward(const HostNet& n, const NetTape& t, const std::vector<double>& dl, HostNet& g) {
  for (int r = 0; r < n.out.rows; ++r) {
    g.out.b[r] += dl[r];
    for (int c = 0; c < n.out.cols; ++c) g.out.w[static_cast<size_t>(r) * n.out.cols + c] += dl[r] * t.y[c];
  }
  std::vector<double> dy(n.out.cols, 0.0);
  for (int r = 0; r < n.out.rows; ++r)
    for (int c = 0; c < n.out.cols; ++c) dy[c] += n.out.w[static_cast<size_t>(r) * n.out.cols + c] * dl[r];
  if (!n.res.empty()) {
    std::vector<double> du(dy.size());
    double dg = 0.0;
    for (size_t i = 0; i < dy.size(); ++i) {
      du[i] = dy[i] * t.gate;
      dg += dy[i] * t.res_u[i];
    }
    std::vector<double> dskip = dy;
    for (int i = static_cast<int>(n.res.size()) - 1; i >= 0; --i) du = block_back(n.res[i], t.res[i], du, g.res[i]);
    for (size_t i = 0; i < dskip.size(); ++i) dskip[i] += du[i];
    const double dzg = dg * t.gate * (1.0 - t.gate);
    for (size_t i = 0; i < g.gate_w.size(); ++i) g.gate_w[i] += dzg * t.reduced[i];
    g.gate_b += dzg;
    dy = std::move(dskip);
  }
  for (int i = static_cast<int>(n.blocks.size()) - 1; i >= 0; --i)
    dy = block_back(n.blocks[i], t.blocks[i], dy, g.blocks[i]);
}

// L = L_expert + lambda * L_focal gradient w.r.t. the logits (hybrid_loss).
std::vector<double> loss_grad(const std::vector<double>& p, const std::vector<double>& y,
                              const std::vector<double>& freqs, double lambda, double gamma) {
  const size_t n = p.size();
  constexpr double eps = 1e-7;
  std::vector<double> gl(n, 0.0);
  for (size_t i = 0; i < n; ++i) {
    const double pc = std::clamp(p[i], eps, 1.0 - eps);
    const bool pos = y[i] > 0.5;
    const double pt = pos ? pc : 1.0 - pc;
    const double mod = gamma == 0.0 ? 1.0 : std::pow(1.0 - pt, gamma);
    const double dbce = pc - (pos ? 1.0 : 0.0);
    double dfp;
    if (pos)
      dfp = (gamma == 0.0 ? 0.0 : gamma * std::pow(1.0 - pc, gamma - 1.0) * std::log(pc)) - mod / pc;
    else
      dfp = (gamma == 0.0 ? 0.0 : -gamma * std::pow(pc, gamma - 1.0) * std::log(1.0 - pc)) + mod / (1.0 - pc);
    const double dfz = dfp * pc * (1.0 - pc);
    gl[i] = (dbce / freqs[i] + lambda * dfz) / static_cast<double>(n);
  }
  return gl;
}

HostNet zeros_like(const HostNet& n) {
  HostNet g = n;
  auto zero = [](HostBlk& b) {
    std::fill(b.w.begin(), b.w.end(), 0.0);
    std::fill(b.b.begin(), b.b.end(), 0.0);
  };
  for (HostBlk& b : g.blocks) zero(b);
  for (HostBlk& b : g.res) zero(b);
  std::fill(g.gate_w.begin(), g.gate_w.end(), 0.0);
  g.gate_b = 0.0;
  zero(g.out);
  return g;
}

// Trainable parameters as (pointer, length) spans, in the reference's collect_params order.
std::vector<std::pair<double*, size_t>> spans(HostNet& n) {
  std::vector<std::pair<double*, size_t>> v;
  auto blk = [&](HostBlk& b) {
    v.emplace_back(b.w.data(), b.w.size());
    v.emplace_back(b.b.data(), b.b.size());
  };
  for (HostBlk& b : n.blocks) blk(b);
  for (HostBlk& b : n.res) blk(b);
  if (!n.gate_w.empty()) v.emplace_back(n.gate_w.data(), n.gate_w.size());
  v.emplace_back(&n.gate_b, 1);
  blk(n.out);
  return v;
}

struct Adam {  // AdamW with bias correction and decoupled weight decay
  HostNet m, v;
  long t = 0;
  explicit Adam(const HostNet& n) : m(zeros_like(n)), v(zeros_like(n)) {}
  void step(HostNet& n, HostNet& g, double lr, double wd) {
    constexpr double b1 = 0.9, b2 = 0.999, eps = 1e-8;
    ++t;
    auto pn = spans(n), pg = spans(g), pm = spans(m), pv = spans(v);
    const double c1 = 1.0 - std::pow(b1, t), c2 = 1.0 - std::pow(b2, t);
    for (size_t s = 0; s < pn.size(); ++s)
      for (size_t i = 0; i < pn[s].second; ++i) {
        const double gi = pg[s].first[i];
        double& mi = pm[s].first[i];
        double& vi = pv[s].first[i];
        mi = b1 * mi + (1.0 - b1) * gi;
        vi = b2 * vi + (1.0 - b2) * gi * gi;
        const double upd = (mi / c1) / (std::sqrt(vi / c2) + eps);
        pn[s].first[i] -= lr * (upd + wd * pn[s].first[i]);
      }
  }
};

}  // namespace

HostModel read_llpc(const char* path) {
  In in;
  in.f.open(path, std::ios::binary);
  if (!in.f) fail(PS_ERUNTIME, std::string("load_checkpoint: cannot open ") + path);
  char magic[4];
  in.f.read(magic, 4);
  if (!in.f || std::memcmp(magic, "LLPC", 4) != 0) fail(PS_ERUNTIME, "load_checkpoint: bad magic");
  if (in.get<uint32_t>() != 1) fail(PS_ERUNTIME, "load_checkpoint: unsupported version");
  HostModel m;
  m.checksum = in.get<uint64_t>();
  ps_model_spec& s = m.spec;
  s.num_layers = in.get<int32_t>();
  s.experts_per_layer = in.get<int32_t>();
  s.top_k = in.get<int32_t>();
  s.expert_bytes = in.get<uint64_t>();
  s.hidden_dim = in.get<int32_t>();
  s.group_begin_middle = in.get<int32_t>();
  s.group_begin_output = in.get<int32_t>();
  TrainCfgH& c = m.cfg;
  c.lambda = in.get<double>();
  c.gamma = in.get<double>();
  c.epochs = in.get<int32_t>();
  c.warmup = in.get<int32_t>();
  c.input = in.hyper();
  c.middle = in.hyper();
  c.output = in.hyper();
  c.dropout = in.get<double>();
  c.noise = in.get<double>();
  c.mask = in.get<double>();
  c.batch_size = in.get<int32_t>();
  c.seed = in.get<uint64_t>();
  const uint32_t num = in.get<uint32_t>();
  m.nets.resize(num);
  for (HostNet& n : m.nets) {
    n.target = in.get<int32_t>();
    n.group = in.get<uint8_t>();
    n.E = in.get<int32_t>();
    n.dropout = in.get<double>();
    n.mean = in.vec();
    in.mat(n.p_rows, n.p_cols, n.comp);
    n.eigen = in.vec();
    n.req_dim = in.get<int32_t>();
    n.eff_dim = in.get<int32_t>();
    n.blocks.resize(in.get<uint32_t>());
    for (HostBlk& b : n.blocks) b = in.blk();
    n.res.resize(in.get<uint32_t>());
    for (HostBlk& b : n.res) b = in.blk();
    n.gate_w = in.vec();
    n.gate_b = in.get<double>();
    n.out = in.blk();
  }
  return m;
}

void write_llpc(const HostModel& m, const char* path) {
  Out o;
  o.f.open(path, std::ios::binary);
  if (!o.f) fail(PS_ERUNTIME, std::string("save_checkpoint: cannot open ") + path);
  o.f.write("LLPC", 4);
  o.put<uint32_t>(1);
  o.put<uint64_t>(m.checksum);
  const ps_model_spec& s = m.spec;
  o.put<int32_t>(s.num_layers);
  o.put<int32_t>(s.experts_per_layer);
  o.put<int32_t>(s.top_k);
  o.put<uint64_t>(s.expert_bytes);
  o.put<int32_t>(s.hidden_dim);
  o.put<int32_t>(s.group_begin_middle);
  o.put<int32_t>(s.group_begin_output);
  const TrainCfgH& c = m.cfg;
  o.put(c.lambda);
  o.put(c.gamma);
  o.put<int32_t>(c.epochs);
  o.put<int32_t>(c.warmup);
  o.hyper(c.input);
  o.hyper(c.middle);
  o.hyper(c.output);
  o.put(c.dropout);
  o.put(c.noise);
  o.put(c.mask);
  o.put<int32_t>(c.batch_size);
  o.put<uint64_t>(c.seed);
  o.put<uint32_t>(static_cast<uint32_t>(m.nets.size()));
  for (const HostNet& n : m.nets) {
    o.put<int32_t>(n.target);
    o.put<uint8_t>(static_cast<uint8_t>(n.group));
    o.put<int32_t>(n.E);
    o.put(n.dropout);
    o.vec(n.mean);
    o.mat(n.p_rows, n.p_cols, n.comp);
    o.vec(n.eigen);
    o.put<int32_t>(n.req_dim);
    o.put<int32_t>(n.eff_dim);
    o.put<uint32_t>(static_cast<uint32_t>(n.blocks.size()));
    for (const HostBlk& b : n.blocks) o.blk(b);
    o.put<uint32_t>(static_cast<uint32_t>(n.res.size()));
    for (const HostBlk& b : n.res) o.blk(b);
    o.vec(n.gate_w);
    o.put(n.gate_b);
    o.blk(n.out);
  }
  if (!o.f) fail(PS_ERUNTIME, std::string("save_checkpoint: write failed on ") + path);
}

std::vector<double> host_pca_apply(const HostNet& n, const double* v) {
  const int H = n.p_cols;
  std::vector<double> centered(H);
  for (int i = 0; i < H; ++i) centered[i] = v[i] - n.mean[i];
  std::vector<double> out(n.p_rows, 0.0);
  for (int r = 0; r < n.p_rows; ++r) {
    double s = 0.0;
    const double* row = n.comp.data() + static_cast<size_t>(r) * H;
    for (int c = 0; c < H; ++c) s += row[c] * centered[c];
    out[r] = s;
  }
  return out;
}

void host_fine_tune(HostNet& net, const std::vector<HostSample>& samples, int steps, double lr, const TrainCfgH& cfg) {
  if (samples.empty()) fail(PS_EINVAL, "fine_tune: empty sample set");
  require(cfg.batch_size >= 1, "fine_tune: batch_size must be >= 1");
  const std::vector<double> freqs(net.E, 1.0 / net.E);  // uniform expert prior
  std::mt19937_64 rng(cfg.seed ^ 0xf1e2d3c4b5a69788ull ^ static_cast<uint64_t>(static_cast<int64_t>(net.target)));
  Adam opt(net);
  const double wd = cfg.for_group(net.group).weight_decay;
  for (int pass = 0; pass < steps; ++pass) {  // run_epoch without augmentation
    std::vector<size_t> order(samples.size());
    std::iota(order.begin(), order.end(), 0);
    std::shuffle(order.begin(), order.end(), rng);
    for (size_t pos = 0; pos < order.size();) {
      const size_t count = std::min<size_t>(static_cast<size_t>(cfg.batch_size), order.size() - pos);
      HostNet grad = zeros_like(net);
      for (size_t b = 0; b < count; ++b) {
        const HostSample& s = samples[order[pos + b]];
        NetTape tape;
        forward_train(net, s, rng, tape);
        std::vector<double> probs(tape.logits.size());
        for (size_t i = 0; i < probs.size(); ++i) probs[i] = sigmoid(tape.logits[i]);
        std::vector<double> gl = loss_grad(probs, s.labels, freqs, cfg.lambda, cfg.gamma);
        for (double& g : gl) g /= static_cast<double>(count);
        backward(net, tape, gl, grad);
      }
      opt.step(net, grad, lr, wd);
      pos += count;
    }
  }
}

}  // namespace ps
