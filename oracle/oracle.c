/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the PreScope reference's hot
 * path, used as the CPU checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg. See oracle.h. Built with -ffp-contract=off so doubles follow the
 * reference's evaluation order bit-for-bit.
 *
 * Pinning (tests/test_oracle.py): every function here is checked against the real
 * reference compiled in oracle/_ref (ref_shim.cpp) and against the reference's own
 * golden vectors / KATs committed in tests/golden/.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ bf16 helpers */
float or_bf16_to_f32(uint16_t v) {
  uint32_t u = (uint32_t)v << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

uint16_t or_f32_to_bf16(float f) { /* round-to-nearest-even, NaN kept quiet */
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

/* ------------------------------------------------------------------ routing */

/* workload.cpp:110-119 — stable sort by weight desc, ties lower index, truncate to k.
 * Restated as k rounds of "largest value, lowest index among the remaining". */
int or_topk(const double* w, int n, int k, int32_t* out) {
  if (k > n) k = n;
  if (k < 0) k = 0;
  unsigned char* used = (unsigned char*)calloc((size_t)(n > 0 ? n : 1), 1);
  for (int r = 0; r < k; ++r) {
    int best = -1;
    for (int i = 0; i < n; ++i) {
      if (used[i]) continue;
      if (best < 0 || w[i] > w[best]) best = i; /* strict: ties keep the lower index */
    }
    used[best] = 1;
    out[r] = best;
  }
  free(used);
  return k;
}

/* workload.cpp:176-201. logits[e] = sqrt(H) * sum_d G[e,d] a[d] - zipf*ln(e+1);
 * follow -> logits[(prev_top1+1) % E] = max + 1 (workload.cpp:183-188, 106-108);
 * softmax in f64 (190-195); top-k ranks the softmax WEIGHTS (201). */
void or_route(const double* gate, const double* a, int E, int H, double zipf, int follow,
              int prev_top1, int k, double* logits, double* weights, int32_t* ids) {
  for (int e = 0; e < E; ++e) {
    double s = 0.0;
    const double* row = gate + (size_t)e * H;
    for (int d = 0; d < H; ++d) s += row[d] * a[d];
    logits[e] = s * sqrt((double)H) - zipf * log(e + 1.0);
  }
  if (follow && prev_top1 >= 0) {
    int target = (prev_top1 + 1) % E;
    double mx = logits[0];
    for (int e = 1; e < E; ++e) if (logits[e] > mx) mx = logits[e];
    logits[target] = mx + 1.0;
  }
  double mx = logits[0];
  for (int e = 1; e < E; ++e) if (logits[e] > mx) mx = logits[e];
  double z = 0.0;
  for (int e = 0; e < E; ++e) z += (weights[e] = exp(logits[e] - mx));
  for (int e = 0; e < E; ++e) weights[e] /= z;
  or_topk(weights, E, k, ids);
}

/* The router of generate_trace (workload.cpp:176-202) over a whole batch: token t walks
 * its layers in order (the kappa-follow input is its own previous top-1, workload.cpp:
 * 184-188), tokens are independent (OpenMP over tokens; threads = 1 for the 1-core
 * leg). gate [L,E,H], hidden [B,L,H], follow [B,L], zipf [L] -> weights [B,L,E],
 * ids [B,L,k]. */
void or_route_batch(const double* gate, const double* hidden, const uint8_t* follow, const double* zipf,
                    int B, int L, int E, int H, int k, double* weights, int32_t* ids, int threads) {
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
  for (int t = 0; t < B; ++t) {
    double* lg = (double*)malloc(sizeof(double) * E);
    int prev = -1;
    for (int l = 0; l < L; ++l) {
      const size_t tl = (size_t)t * L + l;
      or_route(gate + (size_t)l * E * H, hidden + tl * H, E, H, zipf[l], follow[tl], prev, k, lg,
               weights + tl * E, ids + tl * k);
      prev = ids[tl * k];
    }
    free(lg);
  }
}

/* simulator.cpp:45-57 over the histogram of workload.cpp:283-288. */
int or_sorted_loads(const int32_t* counts, int E, int layer, const uint8_t* exclude,
                    or_load* out) {
  int n = 0;
  for (int e = 0; e < E; ++e) {
    if (counts[e] < 1 || (exclude && exclude[e])) continue;
    or_load l = {e, layer, counts[e]};
    int j = n++;
    while (j > 0 && (out[j - 1].tokens > l.tokens ||
                     (out[j - 1].tokens == l.tokens && out[j - 1].expert > l.expert))) {
      out[j] = out[j - 1];
      --j;
    }
    out[j] = l;
  }
  return n;
}

/* ------------------------------------------------------------------ cost model */

/* cost_model.cpp:11 */
static int64_t to_ticks(double x) { return (int64_t)floor(x + 0.5); }

/* cost_model.cpp:34-37 */
static int64_t cpu_cost(int tokens, const or_params* p) {
  return to_ticks(p->beta * tokens) + p->startup;
}

/* cost_model.cpp:39-43 */
static int64_t cpu_cost_prefix(const or_load* l, int n, const or_params* p) {
  int64_t t = 0;
  for (int i = 0; i < n; ++i) t += cpu_cost(l[i].tokens, p);
  return t;
}

/* cost_model.cpp:13-18, 20-26; scheduler.cpp:11-24 */
static int validate_inputs(const or_load* lists[3], const int ns[3], const or_params* p,
                           const or_stats* s) {
  if (p->t_io < 0 || p->t_g < 0 || p->t_attn < 0 || p->beta < 0 || p->startup < 0 || p->alpha < 0)
    return OR_EINVAL;
  if (!(p->t_g < p->t_io)) return OR_EINVAL;
  if (s->r_hit < 0 || s->r_hit > 1 || s->r_miss < 0 || s->r_miss > 1) return OR_EINVAL;
  if (fabs(s->r_hit + s->r_miss - 1.0) > 1e-9) return OR_EINVAL;
  if (s->window < 1) return OR_EINVAL;
  for (int li = 0; li < 3; ++li)
    for (int i = 0; i < ns[li]; ++i) {
      if (lists[li][i].tokens < 1) return OR_EINVAL;
      if (i > 0 && lists[li][i - 1].tokens > lists[li][i].tokens) return OR_EINVAL;
    }
  return OR_OK;
}

/* ------------------------------------------------------------------ PreSched */

typedef struct { or_load load; int current; int index_in_list; } merged_t;

/* scheduler.cpp:54-69: stable sort of [cur..., next...] by (tokens asc, current
 * first, expert asc). Insertion sort is stable. */
static int merge_cross_layer(const or_load* cur, int n, const or_load* nxt, int m,
                             merged_t* out) {
  int cnt = 0;
  for (int pass = 0; pass < 2; ++pass) {
    const or_load* src = pass == 0 ? cur : nxt;
    int len = pass == 0 ? n : m;
    for (int i = 0; i < len; ++i) {
      merged_t v = {src[i], pass == 0, i};
      int j = cnt++;
      while (j > 0) {
        const merged_t* a = &out[j - 1];
        int a_after_v;
        if (a->load.tokens != v.load.tokens) a_after_v = a->load.tokens > v.load.tokens;
        else if (a->current != v.current) a_after_v = v.current; /* current first */
        else a_after_v = a->load.expert > v.load.expert;
        if (!a_after_v) break;
        out[j] = out[j - 1];
        --j;
      }
      out[j] = v;
    }
  }
  return cnt;
}

/* scheduler.cpp:80-95 with cross_layer_costs (cost_model.cpp:74-82): keep merged
 * element k iff T_G_all(k) = alpha + (|E_all|-k) t_io + t_g  <  T_C_all(k) =
 * sum_{j<=k} cpu + t_attn. */
static int queue_for(const or_load* cur, int n, const or_load* nxt, int m, const or_params* p,
                     merged_t* merged, merged_t* gpu_q, int64_t* sweep_gpu, int64_t* sweep_cpu) {
  int total = merge_cross_layer(cur, n, nxt, m, merged);
  int q = 0;
  int64_t cpu_prefix = 0;
  for (int k = 0; k < total; ++k) {
    cpu_prefix += cpu_cost(merged[k].load.tokens, p);
    int64_t g = p->alpha + (int64_t)(total - k) * p->t_io + p->t_g;
    int64_t c = cpu_prefix + p->t_attn;
    if (sweep_gpu) sweep_gpu[k] = g;
    if (sweep_cpu) sweep_cpu[k] = c;
    if (g < c) gpu_q[q++] = merged[k];
  }
  return q;
}

/* cost_model.cpp:84-92 */
static void current_layer_costs(int ip, const or_load* cur, int n, const or_params* p,
                                int64_t* g, int64_t* c) {
  *g = p->alpha + (int64_t)(n - ip) * p->t_io + p->t_g;
  *c = cpu_cost_prefix(cur, ip, p);
}

/* scheduler.cpp:99-106 */
static int64_t split_estimate(int s, const or_load* cur, int n, const or_params* p) {
  int64_t tc = cpu_cost_prefix(cur, s, p);
  if (s == n) return tc;
  int64_t tg = p->alpha + (int64_t)(n - s) * p->t_io + p->t_g;
  return tc > tg ? tc : tg;
}

/* scheduler.cpp:108-112: last c elements, reversed (hottest first). */
static int hottest_first(const or_load* list, int len, int c, or_load* out) {
  for (int i = 0; i < c; ++i) out[i] = list[len - 1 - i];
  return c;
}

static void fill_sets(const or_load* cur, int n, int ip, or_plan_info* info, or_load* cpu,
                      or_load* od) {
  info->split_index = ip;
  info->n_cpu = ip;
  info->n_od = n - ip;
  for (int i = 0; i < ip; ++i) cpu[i] = cur[i];
  for (int i = ip; i < n; ++i) od[i - ip] = cur[i];
}

/* scheduler.cpp:188-213 (schedule_layer) with 127-145 (ondemand_split) and
 * 147-186 (prefetch_decision). */
static int schedule_layer(const or_load* cur, int n, const or_load* nxt, int m,
                          const or_load* nxt2, int m2, const or_params* p, const or_stats* s,
                          or_plan_info* info, or_load* cpu, or_load* od, or_load* pf,
                          int64_t* sweep_gpu, int64_t* sweep_cpu) {
  int cap = n + (m > m2 ? m : m2) + 1;
  merged_t* merged = (merged_t*)malloc(sizeof(merged_t) * cap);
  merged_t* gpu_q = (merged_t*)malloc(sizeof(merged_t) * cap);
  int q = queue_for(cur, n, nxt, m, p, merged, gpu_q, sweep_gpu, sweep_cpu);
  info->n_sweep = n + m;

  int chosen = n; /* sentinel "i' = n+1" */
  for (int i = 0; i < q; ++i) {
    if (!gpu_q[i].current) continue;
    int64_t g, c;
    current_layer_costs(gpu_q[i].index_in_list, cur, n, p, &g, &c);
    if (g < c) { chosen = gpu_q[i].index_in_list; break; }
  }
  current_layer_costs(chosen, cur, n, p, &info->t_g_at_split, &info->t_c_at_split);

  /* scheduler.cpp:197-205: all-GPU fallback. */
  if (n > 0 && split_estimate(0, cur, n, p) < split_estimate(chosen, cur, n, p)) {
    chosen = 0;
    info->all_gpu_fallback = 1;
    current_layer_costs(0, cur, n, p, &info->t_g_at_split, &info->t_c_at_split);
  }
  fill_sets(cur, n, chosen, info, cpu, od);

  /* prefetch_decision */
  int has_next = 0;
  for (int i = 0; i < q; ++i) if (!gpu_q[i].current) has_next = 1;
  const or_load* target = nxt;
  int target_len = m;
  int widened = 0, count = 0, done = 0;
  if (!has_next) {
    widened = 1;
    info->widened_window = 1;
    if (m2 == 0) {
      done = 1;
    } else {
      int q2 = queue_for(cur, n, nxt2, m2, p, merged, gpu_q, NULL, NULL);
      int has2 = 0;
      for (int i = 0; i < q2; ++i) if (!gpu_q[i].current) has2 = 1;
      if (!has2) done = 1;
      target = nxt2;
      target_len = m2;
    }
  }
  if (!done) {
    int64_t loads = (int64_t)n - chosen;
    int64_t t_gap = cpu_cost_prefix(cur, chosen, p) - p->alpha - loads * p->t_io;
    double f = (double)(t_gap + p->t_attn) / (double)p->t_io; /* cost_model.cpp:94-100 */
    int f_int = (int)to_ticks(f > 0.0 ? f : 0.0);
    double t_e = (double)p->t_io;                             /* cost_model.cpp:102-106 */
    double xi = s->r_hit * (f - f_int + 1.0) * t_e - s->r_miss * (f_int - f) * t_e;
    int c = xi > 0 ? f_int : (f_int - 1 > 0 ? f_int - 1 : 0);
    if (c > target_len) c = target_len;
    info->t_gap = t_gap;
    info->f = f;
    info->f_int = f_int;
    info->xi = xi;
    count = c;
    hottest_first(target, target_len, c, pf);
  }
  info->issued_prefetches = count;
  info->n_pf = count;
  info->prefetch_from_widened = widened && count > 0;
  free(merged);
  free(gpu_q);
  return OR_OK;
}

/* scheduler.cpp:215-250 */
static void greedy_layer(const or_load* cur, int n, const or_load* nxt, int m,
                         const or_params* p, or_plan_info* info, or_load* cpu, or_load* od,
                         or_load* pf) {
  int best = n;
  int64_t best_cost = split_estimate(n, cur, n, p);
  for (int s = n - 1; s >= 0; --s) {
    int64_t cost = split_estimate(s, cur, n, p);
    if (cost < best_cost) { best_cost = cost; best = s; }
  }
  fill_sets(cur, n, best, info, cpu, od);
  current_layer_costs(best, cur, n, p, &info->t_g_at_split, &info->t_c_at_split);
  int64_t t_free = p->alpha + (int64_t)(n - best) * p->t_io;
  int64_t window_end = best_cost + p->t_attn;
  int cnt = 0;
  if (t_free < window_end) {
    cnt = (int)((window_end - t_free + p->t_io - 1) / p->t_io);
    if (cnt > m) cnt = m;
  }
  info->issued_prefetches = cnt;
  info->n_pf = hottest_first(nxt, m, cnt, pf);
  info->t_gap = info->t_c_at_split - t_free;
  info->f_int = cnt;
}

int or_plan_layer(int policy, int fixed_c, const or_load* cur, int n_cur, const or_load* nxt,
                  int n_next, const or_load* nxt2, int n_next2, const or_params* p,
                  const or_stats* s, or_plan_info* info, or_load* cpu, or_load* od,
                  or_load* pf, int64_t* sweep_gpu, int64_t* sweep_cpu) {
  memset(info, 0, sizeof(*info));
  if (policy == OR_ORACLE) return OR_EINVAL; /* scheduler.cpp:277-278 */
  const or_load* lists[3] = {cur, nxt, nxt2};
  int ns[3] = {n_cur, n_next, n_next2};
  int rc = validate_inputs(lists, ns, p, s);
  if (rc) return rc;
  switch (policy) {
    case OR_PRESCHED:
      return schedule_layer(cur, n_cur, nxt, n_next, nxt2, n_next2, p, s, info, cpu, od, pf,
                            sweep_gpu, sweep_cpu);
    case OR_GREEDY:
      greedy_layer(cur, n_cur, nxt, n_next, p, info, cpu, od, pf);
      return OR_OK;
    case OR_ONDEMAND: /* scheduler.cpp:252-260 */
      fill_sets(cur, n_cur, 0, info, cpu, od);
      current_layer_costs(0, cur, n_cur, p, &info->t_g_at_split, &info->t_c_at_split);
      return OR_OK;
    case OR_FIXED: { /* scheduler.cpp:262-269 */
      greedy_layer(cur, n_cur, nxt, n_next, p, info, cpu, od, pf);
      int cnt = fixed_c < n_next ? fixed_c : n_next;
      info->issued_prefetches = cnt;
      info->n_pf = hottest_first(nxt, n_next, cnt, pf);
      info->f_int = cnt;
      return OR_OK;
    }
  }
  return OR_EINVAL;
}

/* ------------------------------------------------------------------ residency */

typedef struct { int64_t f; int32_t l, e; } rank_t;
static int rank_cmp(const void* a, const void* b) {
  const rank_t* x = (const rank_t*)a;
  const rank_t* y = (const rank_t*)b;
  if (x->f != y->f) return x->f > y->f ? -1 : 1;
  if (x->l != y->l) return x->l < y->l ? -1 : 1;
  return x->e < y->e ? -1 : (x->e > y->e);
}

/* predictor.cpp:405-433 */
int or_plan_residency(const int64_t* freq, int L, int E, uint64_t budget,
                      uint64_t expert_bytes, int32_t* pairs_out) {
  if (expert_bytes == 0) return -1;
  rank_t* r = (rank_t*)malloc(sizeof(rank_t) * (size_t)L * E);
  for (int l = 0; l < L; ++l)
    for (int e = 0; e < E; ++e) r[l * E + e] = (rank_t){freq[l * E + e], l, e};
  qsort(r, (size_t)L * E, sizeof(rank_t), rank_cmp);
  uint64_t count = budget / expert_bytes;
  if (count > (uint64_t)L * E) count = (uint64_t)L * E;
  for (uint64_t i = 0; i < count; ++i) {
    pairs_out[2 * i] = r[i].l;
    pairs_out[2 * i + 1] = r[i].e;
  }
  free(r);
  return (int)count;
}

/* ------------------------------------------------------------------ LLaPor */

/* predictor.cpp:31 */
static double gelu(double x) { return 0.5 * x * (1.0 + erf(x / sqrt(2.0))); }
/* predictor.cpp:39 */
static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

/* predictor.cpp:19-29 */
static void matvec(const double* w, int rows, int cols, const double* x, double* out) {
  for (int r = 0; r < rows; ++r) {
    double s = 0.0;
    const double* row = w + (size_t)r * cols;
    for (int c = 0; c < cols; ++c) s += row[c] * x[c];
    out[r] = s;
  }
}

/* predictor.cpp:166-183 (eval mode: no dropout) */
static void block_forward(const double* w, const double* b, int out_dim, int in_dim,
                          const double* x, double* y) {
  matvec(w, out_dim, in_dim, x, y);
  for (int i = 0; i < out_dim; ++i) y[i] = gelu(y[i] + b[i]);
}

int or_llapor_forward(const or_llapor_net* net, const double* hidden_prev,
                      const int32_t* active_prev, int k_prev, const double* gate_prev, int k,
                      double* reduced_out, double* logits_out, int32_t* topk_out) {
  const int H = net->H, P = net->P, E = net->E;
  const int in_dim = P + 2 * E; /* predictor.cpp:141-143 */
  if (net->n_blocks < 1 || net->dims[0] != in_dim) return OR_EINVAL;
  int maxw = in_dim;
  for (int j = 0; j <= net->n_blocks; ++j) if (net->dims[j] > maxw) maxw = net->dims[j];
  double* centered = (double*)malloc(sizeof(double) * H);
  double* x = (double*)malloc(sizeof(double) * maxw);
  double* y = (double*)malloc(sizeof(double) * maxw);
  double* u = (double*)malloc(sizeof(double) * maxw);
  double* logits = (double*)malloc(sizeof(double) * E);

  /* pca_apply: predictor.cpp:116-124 */
  for (int i = 0; i < H; ++i) centered[i] = hidden_prev[i] - net->pca_mean[i];
  matvec(net->pca_comp, P, H, centered, x);
  if (reduced_out) memcpy(reduced_out, x, sizeof(double) * P);

  /* features: experiment.cpp:85-98; concatenation predictor.cpp:214-220 */
  for (int e = 0; e < E; ++e) x[P + e] = 0.0;
  for (int j = 0; j < k_prev; ++j) x[P + active_prev[j]] = 1.0;
  for (int e = 0; e < E; ++e) x[P + E + e] = gate_prev[e];
  double* reduced = (double*)malloc(sizeof(double) * (P > 0 ? P : 1));
  memcpy(reduced, x, sizeof(double) * P);

  /* blocks: predictor.cpp:222-227 */
  for (int j = 0; j < net->n_blocks; ++j) {
    block_forward(net->w[j], net->b[j], net->dims[j + 1], net->dims[j], x, y);
    memcpy(x, y, sizeof(double) * net->dims[j + 1]);
  }
  const int width = net->dims[net->n_blocks];

  /* gated residual (middle group): predictor.cpp:229-240 */
  if (net->n_res > 0) {
    memcpy(u, x, sizeof(double) * width);
    for (int j = 0; j < net->n_res; ++j) {
      block_forward(net->rw[j], net->rb[j], width, width, u, y);
      memcpy(u, y, sizeof(double) * width);
    }
    double d = 0.0;
    for (int i = 0; i < P; ++i) d += net->gate_w[i] * reduced[i];
    double g = sigmoid(d + net->gate_b);
    for (int i = 0; i < width; ++i) x[i] = u[i] * g + x[i];
  }

  /* output affine map: predictor.cpp:242-245 */
  matvec(net->out_w, E, width, x, logits);
  for (int e = 0; e < E; ++e) logits[e] += net->out_b[e];
  if (logits_out) memcpy(logits_out, logits, sizeof(double) * E);
  /* predict_topk ranks LOGITS: predictor.cpp:669-672 */
  if (topk_out) or_topk(logits, E, k, topk_out);

  free(centered); free(x); free(y); free(u); free(logits); free(reduced);
  return OR_OK;
}

/* ------------------------------------------------------------------ MoE layer
 * No reference code: restated from PAPER.md:162-168, 606. */

void or_permute(const int32_t* ids, int B, int k, int E, int32_t* offsets, int32_t* perm_src,
                int32_t* inv) {
  for (int e = 0; e <= E; ++e) offsets[e] = 0;
  for (int i = 0; i < B * k; ++i) offsets[ids[i] + 1]++;
  for (int e = 0; e < E; ++e) offsets[e + 1] += offsets[e];
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (E > 0 ? E : 1));
  for (int e = 0; e < E; ++e) fill[e] = offsets[e];
  for (int i = 0; i < B * k; ++i) { /* i = token*k + slot ascending => stable order */
    int pos = fill[ids[i]]++;
    perm_src[pos] = i;
    inv[i] = pos;
  }
  free(fill);
}

static double silu(double g) { return g / (1.0 + exp(-g)); }

void or_expert_ffn(const uint16_t* slab, int H, int F, int m, const uint16_t* x, float* y,
                   int round_h) {
  const uint16_t* wg = slab;
  const uint16_t* wu = slab + (size_t)F * H;
  const uint16_t* wd = slab + (size_t)2 * F * H;
  double* h = (double*)malloc(sizeof(double) * F);
  float* xf = (float*)malloc(sizeof(float) * H);
  for (int t = 0; t < m; ++t) {
    for (int d = 0; d < H; ++d) xf[d] = or_bf16_to_f32(x[(size_t)t * H + d]);
    for (int f = 0; f < F; ++f) {
      double g = 0.0, u = 0.0;
      const uint16_t* rg = wg + (size_t)f * H;
      const uint16_t* ru = wu + (size_t)f * H;
      for (int d = 0; d < H; ++d) {
        g += (double)or_bf16_to_f32(rg[d]) * xf[d];
        u += (double)or_bf16_to_f32(ru[d]) * xf[d];
      }
      double hv = silu(g) * u;
      h[f] = round_h ? (double)or_bf16_to_f32(or_f32_to_bf16((float)hv)) : hv;
    }
    for (int r = 0; r < H; ++r) {
      double acc = 0.0;
      const uint16_t* rd = wd + (size_t)r * F;
      for (int f = 0; f < F; ++f) acc += (double)or_bf16_to_f32(rd[f]) * h[f];
      y[(size_t)t * H + r] = (float)acc;
    }
  }
  free(h);
  free(xf);
}

void or_moe_layer(const uint16_t* const* slab, int H, int F, int B, int k, int E,
                  const uint16_t* x, const int32_t* ids, const float* gate, float* y,
                  int round_h, int threads) {
  float* ye = (float*)malloc(sizeof(float) * (size_t)B * k * H);
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : 1)
  for (int i = 0; i < B * k; ++i) {
    int t = i / k;
    or_expert_ffn(slab[ids[i]], H, F, 1, x + (size_t)t * H, ye + (size_t)i * H, round_h);
  }
  for (int t = 0; t < B; ++t)
    for (int d = 0; d < H; ++d) {
      double acc = 0.0;
      for (int j = 0; j < k; ++j) {
        int e = ids[t * k + j];
        acc += (double)gate[(size_t)t * E + e] * ye[((size_t)t * k + j) * H + d];
      }
      y[(size_t)t * H + d] = (float)acc;
    }
  free(ye);
}

/* ------------------------------------------------------------------ weights
 * Restatement of the synthetic-weight definition (DESIGN.md §Synthetic weights; the
 * product implements it in paper_2509_23638_b200/csrc/weights.cu): bf16 of
 * (u0+u1+u2+u3 - 2*65535) * c, ui = 16-bit lanes of splitmix64(base + i). */
static uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

void or_init_slab(uint16_t* slab, int H, int F, uint64_t seed, int layer, int expert) {
  const double sigma = 37837.226631;
  const float c_in = (float)(1.0 / (sigma * sqrt((double)H)));
  const float c_down = (float)(1.0 / (sigma * sqrt((double)F)));
  const uint64_t base = mix64(seed ^ mix64(((uint64_t)(uint32_t)layer << 32) | (uint32_t)expert));
  const uint64_t n = 3ull * H * F, n_in = 2ull * H * F;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t r = mix64(base + i);
    int s = (int)(r & 0xffff) + (int)((r >> 16) & 0xffff) + (int)((r >> 32) & 0xffff) +
            (int)((r >> 48) & 0xffff) - 2 * 65535;
    slab[i] = or_f32_to_bf16((float)s * (i < n_in ? c_in : c_down));
  }
}
