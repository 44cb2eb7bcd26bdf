// K4 — LLaPor layer-group predictor, inference only.
//
// Reference (fp64 CPU): pca_apply (predictor.cpp:116-124), block_forward =
// affine + erf-GELU (166-183), net_forward with the middle-group gated residual
// (205-247), forward (344-352), predict_topk on LOGITS (669-672), and the per-layer
// predicted histogram of predict_loads (experiment.cpp:104-112).
//
// Two launches per predicted layer:
//  pca_partial_kernel — HBM-bound skinny GEMM over the [P, H] component matrix (the
//               dominant bytes, 8 MiB at P=512, H=4096): grid (P/16, H/512), two rows per
//               warp, the centred x chunk staged once per CTA; partial sums per H chunk
//               (deterministic, summed in fixed order by the MLP kernel).
//  mlp_kernel — 16 tokens per CTA: feature concat [pca | onehot(prev top-k) | prev
//               gate weights], GELU blocks, gated residual, logits, top-k, histogram;
//               every weight row is read once per CTA and applied to all its tokens.
// fp32 throughout (the reference is fp64: logits within rel 1e-4, top-k bit-exact
// against topk_indices on the kernel's own logits).
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <random>
#include <vector>

#include "device_common.cuh"
#include "llapor_model.hpp"

namespace ps {

constexpr int kMaxBlocks = 6;
constexpr int kMaxE = 256;

struct NetDev {  // device pointers into one allocation; kernel parameter
  int P, in_dim, width, E, n_blocks, n_res, valid;
  int mlp_floats;  // contiguous MLP parameters from w[0] to the end of out_b (staged in smem)
  int dims[kMaxBlocks + 1];
  const float* mean;
  const float* comp;
  const float* w[kMaxBlocks];
  const float* b[kMaxBlocks];
  const float* rw[kMaxBlocks];
  const float* rb[kMaxBlocks];
  const float* gate_w;
  float gate_b;
  const float* out_w;
  const float* out_b;
  // float offsets of the MLP parameters from w[0] (addresses into the smem-staged copy)
  int o_w[kMaxBlocks], o_b[kMaxBlocks], o_rw[kMaxBlocks], o_rb[kMaxBlocks], o_gate, o_ow, o_ob;
};

}  // namespace ps

struct ps_llapor_s {
  ps_model_spec spec{};
  ps::HostModel host;            // f64 checkpoint model (fine_tune / save operate on it)
  std::vector<ps::NetDev> nets;  // index = target layer; nets[0] unused
  std::vector<uint8_t> stale;    // host net changed since its device copy (or never uploaded)
  std::vector<std::pair<float*, size_t>> net_buf;  // per net: its device buffer and size (floats)
  std::vector<void*> allocs;
  int max_p = 0, max_in = 0, max_width = 0;
  uint64_t generation = 0;       // bumped by every upload (a captured forward holds NetDev by value)
};

namespace ps {
namespace {

constexpr int kPcaWarps = 8;     // warps per CTA (two component rows each)
constexpr int kPcaChunk = 512;   // H elements per CTA (grid.y splits H)
constexpr int kPcaTok = 16;      // tokens per pass
constexpr int kMlpTokBig = 16;   // tokens per MLP CTA (batches > 64)
constexpr int kMlpTokSmall = 4;  // tokens per MLP CTA (decode batches <= 64)
constexpr int kMlpThreads = 512;

// Stage 1 of pca_apply: part[s][t][p] = sum_{h in chunk s} comp[p][h] * (x[t][h] - mean[h]).
// grid = (ceil(P/16), ceil(H/512)): 256 CTAs at P=512, H=4096, so the 8 MiB component
// matrix streams at HBM rate. The centred x chunk is staged once per CTA in smem; each
// warp owns two component rows and each lane four consecutive columns per step, so one
// 16-byte activation load from smem feeds eight FMAs. The 2 x 16 partial sums per lane
// are reduced with one transpose-reduce (lane L owns row L / 16, token L % 16).
__global__ void __launch_bounds__(kPcaWarps * 32)
pca_partial_kernel(const float* __restrict__ comp, const float* __restrict__ mean, const float* __restrict__ x,
                   int B, int H, int P, float* __restrict__ part) {
  static_assert(2 * kPcaTok == 32, "transpose-reduce maps (2 rows x kPcaTok tokens) onto the 32 lanes");
  static_assert((kPcaWarps * 32) % (kPcaChunk / 4) == 0, "each thread stages one fixed column quad");
  __shared__ __align__(16) float s_x[kPcaTok][kPcaChunk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p0 = (blockIdx.x * kPcaWarps + warp) * 2;
  const int h0 = blockIdx.y * kPcaChunk;
  const int hn = min(kPcaChunk, H - h0);
  const bool vec = (H & 3) == 0 && (hn & 3) == 0;
  const int my_c4 = (threadIdx.x % (kPcaChunk / 4)) * 4;  // fixed column quad of this thread
  const float4 my_mean = vec && my_c4 < hn ? __ldg(reinterpret_cast<const float4*>(mean + h0 + my_c4))
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int tb = 0; tb < B; tb += kPcaTok) {
    __syncthreads();
    // Stage the x chunk with asynchronous copies (all of a thread's copies in flight at
    // once), then the copying thread centres its own elements in place.
    if (vec) {
      for (int t = threadIdx.x / (kPcaChunk / 4); t < kPcaTok; t += blockDim.x / (kPcaChunk / 4)) {
        if (tb + t < B && my_c4 < hn) cp_async16(&s_x[t][my_c4], x + static_cast<size_t>(tb + t) * H + h0 + my_c4);
        else *reinterpret_cast<float4*>(&s_x[t][my_c4]) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      cp_async_wait_all();
      for (int t = threadIdx.x / (kPcaChunk / 4); t < kPcaTok; t += blockDim.x / (kPcaChunk / 4)) {
        if (tb + t < B && my_c4 < hn) {
          float4& v = *reinterpret_cast<float4*>(&s_x[t][my_c4]);
          v.x -= my_mean.x; v.y -= my_mean.y; v.z -= my_mean.z; v.w -= my_mean.w;
        }
      }
    } else {
      for (int i = threadIdx.x; i < kPcaTok * kPcaChunk; i += blockDim.x) {
        const int t = i / kPcaChunk, c = i % kPcaChunk;
        s_x[t][c] = (tb + t < B && c < hn) ? x[static_cast<size_t>(tb + t) * H + h0 + c] - mean[h0 + c] : 0.f;
      }
    }
    __syncthreads();
    if (p0 >= P) continue;
    const bool two = p0 + 1 < P;
    float acc[2 * kPcaTok];
#pragma unroll
    for (int i = 0; i < 2 * kPcaTok; ++i) acc[i] = 0.f;
    const float* r0 = comp + static_cast<size_t>(p0) * H + h0;
    const float* r1 = two ? r0 + H : r0;
    if (vec) {
      float4 c0[kPcaChunk / 128], c1[kPcaChunk / 128];
#pragma unroll
      for (int j = 0; j < kPcaChunk / 128; ++j) {
        const int c = 4 * lane + 128 * j;
        const bool ok = c < hn;
        c0[j] = ok ? __ldg(reinterpret_cast<const float4*>(r0 + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
        c1[j] = ok && two ? __ldg(reinterpret_cast<const float4*>(r1 + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < kPcaChunk / 128; ++j) {
        const int c = 4 * lane + 128 * j;
#pragma unroll
        for (int t = 0; t < kPcaTok; ++t) {
          const float4 a = *reinterpret_cast<const float4*>(&s_x[t][c]);
          acc[t] += c0[j].x * a.x; acc[t] += c0[j].y * a.y; acc[t] += c0[j].z * a.z; acc[t] += c0[j].w * a.w;
          acc[kPcaTok + t] += c1[j].x * a.x; acc[kPcaTok + t] += c1[j].y * a.y;
          acc[kPcaTok + t] += c1[j].z * a.z; acc[kPcaTok + t] += c1[j].w * a.w;
        }
      }
    } else {
      for (int c = lane; c < hn; c += 32) {
        const float v0 = r0[c], v1 = two ? r1[c] : 0.f;
#pragma unroll
        for (int t = 0; t < kPcaTok; ++t) { acc[t] += v0 * s_x[t][c]; acc[kPcaTok + t] += v1 * s_x[t][c]; }
      }
    }
    const float sum = warp_transpose_sum(acc);
    const int t = lane % kPcaTok, p = p0 + lane / kPcaTok;
    if (tb + t < B && p < P) part[(static_cast<size_t>(blockIdx.y) * B + tb + t) * P + p] = sum;
  }
}

__device__ __forceinline__ float gelu_erf(float v) { return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f)); }

// out[t][r] = act(W[r,:] . in[t,:] + b[r]) for the TOK tokens of the CTA. A warp owns
// R = 32 / TOK rows; lanes stride the columns so every activation read from shared memory
// feeds R FMAs, and the R x TOK partial sums are reduced with one transpose-reduce (lane L
// ends up owning row r0 + L / TOK, token L % TOK and applies bias + activation itself).
// TOK = 16 (two rows per warp) for big batches; TOK = 4 (eight rows per warp, four CTAs
// for a 16-token decode batch) halves the per-layer rounds and spreads a decode batch
// over more SMs.
template <int TOK>
__device__ __forceinline__ void affine_tokens(const float* __restrict__ W, const float* __restrict__ bvec, int rows,
                                              int cols, const float* in, int in_stride, float* out, int out_stride,
                                              int nt, bool gelu) {
  constexpr int R = 32 / TOK;
  static_assert(R * TOK == 32, "transpose-reduce maps (R rows x TOK tokens) onto the 32 lanes");
  constexpr int kU = TOK >= 16 ? 4 : 2;  // weight loads in flight per lane and row
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int r0 = R * warp; r0 < rows; r0 += R * nw) {
    float acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.f;
    for (int c0 = 0; c0 < cols; c0 += 32 * kU) {
      float w[R][kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int c = c0 + lane + 32 * u;
#pragma unroll
        for (int ri = 0; ri < R; ++ri) w[ri][u] = c < cols && r0 + ri < rows ? W[(r0 + ri) * cols + c] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int c = c0 + lane + 32 * u;
        if (c < cols) {
#pragma unroll
          for (int t = 0; t < TOK; ++t) {
            const float a = in[t * in_stride + c];
#pragma unroll
            for (int ri = 0; ri < R; ++ri) acc[ri * TOK + t] += w[ri][u] * a;
          }
        }
      }
    }
    const float s = warp_transpose_sum(acc);
    const int t = lane % TOK, r = r0 + lane / TOK;
    if (t < nt && r < rows) {
      const float v = s + bvec[r];
      out[t * out_stride + r] = gelu ? gelu_erf(v) : v;
    }
  }
}

// Feature concat [pca | onehot(prev top-k) | prev gate weights] (predictor.cpp:214-220),
// GELU blocks, middle-group gated residual (229-240), logits (242-245), top-k on
// logits (669-672), predicted histogram (experiment.cpp:104-112). TOK tokens/CTA.
// kStage: every MLP parameter is staged in shared memory first (one L2 round trip) and
// addressed as smem + offset, so the layer loops issue LDS rather than generic loads.
template <int TOK, bool kStage>
__global__ void __launch_bounds__(kMlpThreads)
mlp_kernel(const __grid_constant__ NetDev net, const float* __restrict__ part, int n_part,
           const int32_t* __restrict__ prev_ids, int k_prev, const float* __restrict__ prev_w, int B, int k,
           float* __restrict__ logits_out, int32_t* __restrict__ ids_out, int32_t* __restrict__ pred_counts) {
  extern __shared__ __align__(16) float smem[];
  const int P = net.P, E = net.E, D = net.in_dim, Wd = net.width;
  const int t0 = blockIdx.x * TOK, nt = min(TOK, B - t0);
  int maxh = Wd;
  for (int j = 1; j <= net.n_blocks; ++j) maxh = max(maxh, net.dims[j]);
  float* wsm = smem;                                       // [mlp_floats] staged parameters
  float* feat = smem + (kStage ? (net.mlp_floats + 3) / 4 * 4 : 0);  // [TOK][D]
  float* h1 = feat + TOK * D;                          // [TOK][maxh]
  float* h2 = h1 + TOK * maxh;
  float* h3 = h2 + TOK * maxh;
  float* lg = h3 + TOK * maxh;                         // [TOK][E]
  const float* base = kStage ? wsm : net.w[0];

  if (kStage) {
    const float4* src = reinterpret_cast<const float4*>(net.w[0]);
    float4* dst = reinterpret_cast<float4*>(wsm);
    for (int i = threadIdx.x; i < net.mlp_floats / 4; i += blockDim.x) cp_async16(dst + i, src + i);
  }

  // PCA features: partial sums in fixed part order (0 + p0 + p1 + ...), all of a quad's
  // partial loads in flight together.
  constexpr int kMaxParts = 16;
  const bool vecP = (P & 3) == 0;
  const int Pq = vecP ? P / 4 : P;
  for (int i = threadIdx.x; i < TOK * Pq; i += blockDim.x) {
    const int t = i / Pq, q = i % Pq;
    if (vecP) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < nt) {
        const float4* src = reinterpret_cast<const float4*>(part + static_cast<size_t>(t0 + t) * P) + q;
        const size_t stride = static_cast<size_t>(B) * P / 4;
        float4 pv[kMaxParts];
#pragma unroll
        for (int s = 0; s < kMaxParts; ++s) if (s < n_part) pv[s] = __ldg(src + s * stride);
#pragma unroll
        for (int s = 0; s < kMaxParts; ++s)
          if (s < n_part) { a.x += pv[s].x; a.y += pv[s].y; a.z += pv[s].z; a.w += pv[s].w; }
      }
      float* f = feat + t * D + 4 * q;
      f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    } else {
      float a = 0.f;
      if (t < nt)
        for (int s = 0; s < n_part; ++s) a += part[(static_cast<size_t>(s) * B + t0 + t) * P + q];
      feat[t * D + q] = a;
    }
  }
  // onehot(prev top-k) | prev gate weights
  for (int i = threadIdx.x; i < TOK * 2 * E; i += blockDim.x) {
    const int t = i / (2 * E), j = i % (2 * E);
    float v = 0.f;
    if (t < nt) {
      if (j < E) {
        for (int r = 0; r < k_prev; ++r)
          if (prev_ids[static_cast<size_t>(t0 + t) * k_prev + r] == j) v = 1.0f;
      } else {
        v = prev_w[static_cast<size_t>(t0 + t) * E + (j - E)];
      }
    }
    feat[t * D + P + j] = v;
  }
  if (kStage) cp_async_wait_all();
  __syncthreads();

  const float* cur = feat;
  int cur_stride = D;
  float* bufs[2] = {h1, h2};
  for (int j = 0; j < net.n_blocks; ++j) {
    float* o = bufs[j & 1];
    affine_tokens<TOK>(base + net.o_w[j], base + net.o_b[j], net.dims[j + 1], net.dims[j], cur, cur_stride, o, maxh, nt,
                  true);
    __syncthreads();
    cur = o;
    cur_stride = maxh;
  }
  if (net.n_res > 0) {
    // u = residual blocks(x); g = sigmoid(gate_w . pca + gate_b); x = u*g + x.
    const float* uin = cur;
    float* ubuf[2] = {h3, (cur == h1) ? h2 : h1};
    float* u = nullptr;
    for (int j = 0; j < net.n_res; ++j) {
      u = ubuf[j & 1];
      affine_tokens<TOK>(base + net.o_rw[j], base + net.o_rb[j], Wd, Wd, uin, maxh, u, maxh, nt, true);
      __syncthreads();
      uin = u;
    }
    __shared__ float s_gate[TOK];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float* gw = base + net.o_gate;
    for (int t = warp; t < nt; t += blockDim.x >> 5) {
      float d = 0.f;
      for (int i = lane; i < P; i += 32) d += gw[i] * feat[t * D + i];
      d = warp_sum(d);
      if (lane == 0) s_gate[t] = 1.0f / (1.0f + expf(-(d + net.gate_b)));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nt * Wd; i += blockDim.x) {
      const int t = i / Wd, c = i % Wd;
      u[t * maxh + c] = u[t * maxh + c] * s_gate[t] + cur[t * maxh + c];
    }
    __syncthreads();
    cur = u;
  }
  affine_tokens<TOK>(base + net.o_ow, base + net.o_ob, E, Wd, cur, maxh, lg, E, nt, false);
  __syncthreads();
  if (logits_out)
    for (int i = threadIdx.x; i < nt * E; i += blockDim.x) logits_out[static_cast<size_t>(t0) * E + i] = lg[i];

  // Top-k on logits (ties -> lower index) + predicted histogram; one warp per token.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = warp; t < nt; t += blockDim.x >> 5) {
    float v[kMaxE / 32];
#pragma unroll
    for (int i = 0; i < kMaxE / 32; ++i) v[i] = lane + 32 * i < E ? lg[t * E + lane + 32 * i] : -INFINITY;
    for (int r = 0; r < k; ++r) {
      float bv = -INFINITY;
      int bi = 0x7fffffff;
#pragma unroll
      for (int i = 0; i < kMaxE / 32; ++i) {
        const int e = lane + 32 * i;
        if (e < E && (v[i] > bv || (v[i] == bv && e < bi))) { bv = v[i]; bi = e; }
      }
      warp_argmax(bv, bi);
      if (lane == 0) {
        if (ids_out) ids_out[static_cast<size_t>(t0 + t) * k + r] = bi;
        if (pred_counts) atomicAdd(pred_counts + bi, 1);
      }
#pragma unroll
      for (int i = 0; i < kMaxE / 32; ++i)
        if (lane + 32 * i == bi) v[i] = -INFINITY;
    }
  }
}

// ------------------------------------------------------------------ host side

// Shape checks of a trained net (the GPU kernels' limits) and its NetDev dimensions.
NetDev net_dims(const ps_llapor_s& m, const HostNet& hn) {
  NetDev d{};
  d.P = hn.p_rows;
  d.E = hn.E;
  d.n_blocks = static_cast<int>(hn.blocks.size());
  d.n_res = static_cast<int>(hn.res.size());
  require(d.n_blocks >= 1 && d.n_blocks <= kMaxBlocks && d.n_res <= kMaxBlocks, "LLaPor: unsupported block count");
  require(hn.E == m.spec.experts_per_layer && hn.E <= kMaxE, "LLaPor: expert count mismatch");
  require(hn.p_cols == m.spec.hidden_dim || hn.p_rows == 0, "LLaPor: PCA width != hidden_dim");
  require(static_cast<int>(hn.mean.size()) == hn.p_cols, "LLaPor: PCA mean size != hidden_dim");
  d.in_dim = d.P + 2 * d.E;
  d.dims[0] = hn.blocks[0].cols;
  require(d.dims[0] == d.in_dim, "LLaPor: first block input dim != pca + 2E");
  for (int j = 0; j < d.n_blocks; ++j) {
    require(hn.blocks[j].cols == d.dims[j], "LLaPor: block dims do not chain");
    d.dims[j + 1] = hn.blocks[j].rows;
  }
  d.width = d.dims[d.n_blocks];
  for (const HostBlk& r : hn.res) require(r.rows == d.width && r.cols == d.width, "LLaPor: residual block shape");
  require(hn.res.empty() || static_cast<int>(hn.gate_w.size()) == d.P, "LLaPor: gate size != pca dim");
  require(hn.out.cols == d.width && hn.out.rows == d.E, "LLaPor: output block shape");
  return d;
}

// Host nets -> kernel-side bookkeeping (no device work): validates every trained net and
// marks it for upload before its first forward.
void adopt(ps_llapor_s& m) {
  const int n = static_cast<int>(m.host.nets.size());
  m.nets.assign(std::max(n, 1), NetDev{});
  m.stale.assign(std::max(n, 1), 0);
  for (int l = 0; l < n; ++l) {
    const HostNet& hn = m.host.nets[l];
    if (hn.blocks.empty()) continue;  // untrained (nets[0])
    NetDev d = net_dims(m, hn);
    d.valid = 1;
    m.nets[l] = d;
    m.stale[l] = 1;
    m.max_p = std::max(m.max_p, d.P);
    m.max_in = std::max(m.max_in, d.in_dim);
    m.max_width = std::max(m.max_width, d.width);
  }
}

// One contiguous f32 device copy of net `layer` (arrays 16-byte aligned). Earlier copies
// stay allocated until ps_llapor_free: kernels already enqueued may still read them.
void upload(ps_llapor_s& m, int layer) {
  const HostNet& hn = m.host.nets[layer];
  NetDev d = net_dims(m, hn);
  std::vector<float> buf;
  auto put = [&](const std::vector<double>& v) {
    size_t o = buf.size();
    for (double x : v) buf.push_back(static_cast<float>(x));
    while (buf.size() % 4) buf.push_back(0.f);
    return o;
  };
  size_t o_mean = put(hn.mean), o_comp = put(hn.comp);
  std::vector<size_t> o_w, o_b, o_rw, o_rb;
  for (auto& b : hn.blocks) { o_w.push_back(put(b.w)); o_b.push_back(put(b.b)); }
  for (auto& b : hn.res) { o_rw.push_back(put(b.w)); o_rb.push_back(put(b.b)); }
  size_t o_gate = put(hn.gate_w.empty() ? std::vector<double>{0.0} : hn.gate_w);
  size_t o_ow = put(hn.out.w), o_ob = put(hn.out.b);
  // A re-upload (after fine_tune: same shapes) reuses the net's buffer once every kernel
  // that may still read it has finished; a first upload allocates it.
  if (m.net_buf.size() < m.nets.size()) m.net_buf.resize(m.nets.size(), {nullptr, 0});
  float*& dev = m.net_buf[layer].first;
  if (dev && m.net_buf[layer].second == buf.size()) {
    PS_CUDA(cudaDeviceSynchronize());
  } else {
    PS_CUDA(cudaMalloc(&dev, buf.size() * sizeof(float)));
    m.allocs.push_back(dev);
    m.net_buf[layer].second = buf.size();
  }
  PS_CUDA(cudaMemcpy(dev, buf.data(), buf.size() * sizeof(float), cudaMemcpyHostToDevice));
  d.mean = dev + o_mean;
  d.comp = dev + o_comp;
  for (int j = 0; j < d.n_blocks; ++j) { d.w[j] = dev + o_w[j]; d.b[j] = dev + o_b[j]; }
  for (int j = 0; j < d.n_res; ++j) { d.rw[j] = dev + o_rw[j]; d.rb[j] = dev + o_rb[j]; }
  d.gate_w = dev + o_gate;
  d.gate_b = static_cast<float>(hn.gate_b);
  d.out_w = dev + o_ow;
  d.out_b = dev + o_ob;
  d.mlp_floats = static_cast<int>(o_ob + ((hn.out.b.size() + 3) / 4) * 4 - o_w[0]);
  auto rel = [&](size_t o) { return static_cast<int>(o - o_w[0]); };
  for (int j = 0; j < d.n_blocks; ++j) { d.o_w[j] = rel(o_w[j]); d.o_b[j] = rel(o_b[j]); }
  for (int j = 0; j < d.n_res; ++j) { d.o_rw[j] = rel(o_rw[j]); d.o_rb[j] = rel(o_rb[j]); }
  d.o_gate = rel(o_gate);
  d.o_ow = rel(o_ow);
  d.o_ob = rel(o_ob);
  d.valid = 1;
  m.nets[layer] = d;
  m.stale[layer] = 0;
  ++m.generation;
}

}  // namespace
}  // namespace ps

using namespace ps;

// Engine helpers (C++ linkage): make net `layer`'s device copy current (outside any stream
// capture), and the upload generation a CUDA graph of ps_llapor_forward was captured at.
namespace ps {
void llapor_prepare(ps_llapor m, int layer) {
  if (m && layer >= 1 && layer < static_cast<int>(m->nets.size()) && m->nets[layer].valid && m->stale[layer])
    upload(*m, layer);
}
uint64_t llapor_generation(ps_llapor m) { return m ? m->generation : 0; }
}  // namespace ps

extern "C" {

ps_status ps_llapor_load(const char* path, ps_llapor* out, ps_model_spec* spec_out) {
  return guarded([&] {
    require(path && out, "ps_llapor_load: null argument");
    auto m = std::make_unique<ps_llapor_s>();
    m->host = read_llpc(path);
    m->spec = m->host.spec;
    adopt(*m);
    if (spec_out) *spec_out = m->spec;
    *out = m.release();
  });
}

ps_status ps_llapor_random(const ps_model_spec* spec, int pca_in, int pca_mid, int width_in, int width_mid,
                           uint64_t seed, ps_llapor* out) {
  return guarded([&] {
    auto m = std::make_unique<ps_llapor_s>();
    m->spec = *spec;
    m->host.spec = *spec;
    const int L = spec->num_layers, E = spec->experts_per_layer, H = spec->hidden_dim;
    m->host.nets.resize(L);
    m->host.nets[0].E = E;
    m->host.nets[0].group = 0;
    for (int l = 1; l < L; ++l) {
      const int g = l < spec->group_begin_middle ? 0 : l < spec->group_begin_output ? 1 : 2;
      const int P = std::min(g == 1 ? pca_mid : pca_in, H);
      const int width = g == 1 ? width_mid : width_in;
      const int nblocks = g == 1 ? 3 : 2;  // TrainConfig defaults (predictor.hpp:97-100)
      std::mt19937_64 rng(seed ^ (0x9e3779b97f4a7c15ull * (l + 1)));
      HostNet& hn = m->host.nets[l];
      hn.target = l;
      hn.group = g;
      hn.E = E;
      hn.dropout = m->host.cfg.dropout;
      hn.p_rows = P;
      hn.p_cols = H;
      hn.req_dim = hn.eff_dim = P;
      hn.mean.assign(H, 0.0);
      hn.eigen.assign(P, 1.0);
      std::normal_distribution<double> gauss(0.0, 1.0 / std::sqrt(static_cast<double>(H)));
      hn.comp.resize(static_cast<size_t>(P) * H);
      for (double& v : hn.comp) v = gauss(rng);
      auto init = [&](int o, int i) {  // Xavier-uniform (predictor.cpp:486-494)
        HostBlk b{o, i, std::vector<double>(static_cast<size_t>(o) * i), std::vector<double>(o, 0.0)};
        std::uniform_real_distribution<double> u(-std::sqrt(6.0 / (i + o)), std::sqrt(6.0 / (i + o)));
        for (double& v : b.w) v = u(rng);
        return b;
      };
      int d = P + 2 * E;
      for (int j = 0; j < nblocks; ++j) { hn.blocks.push_back(init(width, d)); d = width; }
      if (g == 1) {
        for (int j = 0; j < 2; ++j) hn.res.push_back(init(width, width));
        std::uniform_real_distribution<double> u(-0.1, 0.1);
        hn.gate_w.resize(P);
        for (double& v : hn.gate_w) v = u(rng);
      }
      hn.out = init(E, width);
    }
    adopt(*m);
    *out = m.release();
  });
}

ps_status ps_llapor_free(ps_llapor m) {
  return guarded([&] {
    if (!m) return;
    for (void* p : m->allocs) cudaFree(p);
    delete m;
  });
}

ps_status ps_llapor_save(ps_llapor m, const char* path) {
  return guarded([&] {
    require(m && path, "ps_llapor_save: null argument");
    write_llpc(m->host, path);
  });
}

ps_status ps_llapor_fine_tune(ps_llapor m, int layer, int n, const double* hidden_prev, const int32_t* active_prev,
                              int k_prev, const double* gate_prev, const int32_t* active, int k, int steps, double lr) {
  return guarded([&] {
    require(m && (n == 0 || (hidden_prev && active_prev && gate_prev && active)), "ps_llapor_fine_tune: null argument");
    if (layer < 1 || layer >= static_cast<int>(m->host.nets.size()) || m->host.nets[layer].blocks.empty())
      fail(PS_ERANGE, "llapor net for layer " + std::to_string(layer) + " is untrained/out of range");
    require(n >= 1 && steps >= 0 && k >= 1 && k_prev >= 1, "ps_llapor_fine_tune: bad n/k/steps");
    HostNet& net = m->host.nets[layer];
    const int H = m->spec.hidden_dim, E = net.E;
    std::vector<HostSample> samples(n);
    for (int t = 0; t < n; ++t) {  // build_samples (predictor.cpp:596-613) on the caller's observations
      HostSample& s = samples[t];
      s.reduced = host_pca_apply(net, hidden_prev + static_cast<size_t>(t) * H);
      s.onehot.assign(E, 0.0);
      s.labels.assign(E, 0.0);
      for (int j = 0; j < k_prev; ++j) {
        const int e = active_prev[static_cast<size_t>(t) * k_prev + j];
        if (e < 0 || e >= E) fail(PS_ERANGE, "ps_llapor_fine_tune: expert id out of range");
        s.onehot[e] = 1.0;
      }
      for (int j = 0; j < k; ++j) {
        const int e = active[static_cast<size_t>(t) * k + j];
        if (e < 0 || e >= E) fail(PS_ERANGE, "ps_llapor_fine_tune: expert id out of range");
        s.labels[e] = 1.0;
      }
      s.gate.assign(gate_prev + static_cast<size_t>(t) * E, gate_prev + static_cast<size_t>(t + 1) * E);
    }
    host_fine_tune(net, samples, steps, lr, m->host.cfg);
    m->stale[layer] = 1;  // re-uploaded before the next forward of this net
  });
}

size_t ps_llapor_scratch_bytes(ps_llapor m, int B) {
  if (!m) return 0;
  const size_t splits = (static_cast<size_t>(m->spec.hidden_dim) + kPcaChunk - 1) / kPcaChunk;
  return splits * static_cast<size_t>(B) * std::max(m->max_p, 1) * sizeof(float) + 256;
}

ps_status ps_llapor_forward(ps_llapor m, int layer, const float* hidden, const int32_t* prev_ids, int k_prev,
                            const float* prev_weights, int B, int k, float* logits, int32_t* ids,
                            int32_t* pred_counts, void* scratch, void* stream) {
  return guarded([&] {
    require(m != nullptr, "ps_llapor_forward: null model");
    if (layer < 1 || layer >= static_cast<int>(m->nets.size()) || !m->nets[layer].valid)
      fail(PS_ERANGE, "llapor net for layer " + std::to_string(layer) + " is untrained/out of range");
    if (m->stale[layer]) upload(*m, layer);  // first use, or fine-tuned since the last upload
    const NetDev& net = m->nets[layer];
    require(k >= 1 && k <= net.E && k_prev >= 1 && k_prev <= 32 && B >= 0, "ps_llapor_forward: bad k/B");
    require(m->spec.hidden_dim <= 16 * kPcaChunk, "ps_llapor_forward: hidden_dim > 8192 unsupported");
    cudaStream_t s = as_stream(stream);
    if (pred_counts) PS_CUDA(cudaMemsetAsync(pred_counts, 0, sizeof(int32_t) * net.E, s));
    if (B == 0) return;
    float* part = static_cast<float*>(scratch);
    const int H = m->spec.hidden_dim;
    const int n_part = (H + kPcaChunk - 1) / kPcaChunk;
    dim3 grid((net.P + 2 * kPcaWarps - 1) / (2 * kPcaWarps), n_part);
    pca_partial_kernel<<<grid, kPcaWarps * 32, 0, s>>>(net.comp, net.mean, hidden, B, H, net.P, part);
    PS_LAUNCH_CHECK("pca_partial_kernel");
    int maxh = net.width;
    for (int j = 1; j <= net.n_blocks; ++j) maxh = std::max(maxh, net.dims[j]);
    static const bool force_big = [] {  // PS_LLAPOR_TOK=16: the one-CTA-per-16-tokens kernel (A/B)
      const char* v = std::getenv("PS_LLAPOR_TOK");
      return v && v[0] == '1' && v[1] == '6';
    }();
    const bool small = B <= 64 && !force_big;  // decode batches: 4 tokens per CTA (B = 32: 8 CTAs, not 2)
    const int tok = small ? kMlpTokSmall : kMlpTokBig;
    const size_t act = sizeof(float) * tok * (net.in_dim + 3 * maxh + net.E);
    const size_t staged = act + sizeof(float) * ((net.mlp_floats + 3) / 4 * 4);
    const bool stage_w = staged <= 200 * 1024;
    const size_t smem = stage_w ? staged : act;
    require(smem <= 227 * 1024, "ps_llapor_forward: predictor too wide for one CTA's shared memory");
    using Kfn = void (*)(NetDev, const float*, int, const int32_t*, int, const float*, int, int, float*, int32_t*,
                         int32_t*);
    const Kfn fn = small ? (stage_w ? mlp_kernel<kMlpTokSmall, true> : mlp_kernel<kMlpTokSmall, false>)
                         : (stage_w ? mlp_kernel<kMlpTokBig, true> : mlp_kernel<kMlpTokBig, false>);
    {  // opt in to the dynamic shared memory this net needs (per kernel variant, once)
      static std::mutex mu;
      static size_t smem_set[2][2] = {{0, 0}, {0, 0}};
      std::lock_guard<std::mutex> g(mu);
      if (smem > smem_set[small][stage_w]) {
        PS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(smem)));
        smem_set[small][stage_w] = smem;
      }
    }
    const int grid_m = (B + tok - 1) / tok;
    fn<<<grid_m, kMlpThreads, smem, s>>>(net, part, n_part, prev_ids, k_prev, prev_weights, B, k, logits, ids,
                                         pred_counts);
    PS_LAUNCH_CHECK("mlp_kernel");
  });
}

}  // extern "C"
