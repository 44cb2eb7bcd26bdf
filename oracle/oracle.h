/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the thing measured or shipped.
 *
 * Plain-C restatement of the PreScope reference's hot-path algorithms
 * (/root/reference/proj, cited file:line per function), plus CPU restatements of
 * the pieces the reference does not contain (SwiGLU expert FFN, permute, combine:
 * "parity unpinned" by the reference's tests).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load this.
 */
#ifndef PRESCOPE_ORACLE_H
#define PRESCOPE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_EINVAL = 1, OR_ERANGE = 2, OR_ERUNTIME = 3 };
enum { OR_PRESCHED = 0, OR_GREEDY = 1, OR_ONDEMAND = 2, OR_FIXED = 3, OR_ORACLE = 4 };

typedef struct { int32_t expert, layer, tokens; } or_load;
typedef struct { int64_t t_io, t_g, t_attn; double beta; int64_t startup, alpha; } or_params;
typedef struct { double r_hit, r_miss; int32_t window; } or_stats;
typedef struct {
  int32_t split_index, issued_prefetches, prefetch_from_widened;
  int32_t n_cpu, n_od, n_pf, n_sweep;
  int64_t t_g_at_split, t_c_at_split, t_gap;
  double f;
  int32_t f_int;
  double xi;
  int32_t widened_window, all_gpu_fallback;
} or_plan_info;

/* workload.cpp:110-119 */
int or_topk(const double* w, int n, int k, int32_t* out);

/* workload.cpp:176-201: one (token, layer) routing decision in f64. */
void or_route(const double* gate /*E*H*/, const double* a /*H*/, int E, int H, double zipf,
              int follow, int prev_top1, int k, double* logits, double* weights, int32_t* ids);

/* workload.cpp:283-288 + simulator.cpp:45-57: histogram then (tokens, expert) order. */
void or_route_batch(const double* gate, const double* hidden, const uint8_t* follow, const double* zipf,
                    int B, int L, int E, int H, int k, double* weights, int32_t* ids, int threads);
int or_sorted_loads(const int32_t* counts /*E*/, int E, int layer, const uint8_t* exclude,
                    or_load* out);

/* scheduler.cpp:402-413 (+ the policies it dispatches to). */
int or_plan_layer(int policy, int fixed_c, const or_load* cur, int n_cur, const or_load* nxt,
                  int n_next, const or_load* nxt2, int n_next2, const or_params* p,
                  const or_stats* s, or_plan_info* info, or_load* cpu, or_load* od,
                  or_load* pf, int64_t* sweep_gpu, int64_t* sweep_cpu);

/* predictor.cpp:405-433: rank (layer, expert) by frequency desc, ties (layer, expert)
 * asc; residents = first floor(budget/expert_bytes). Returns the resident count. */
int or_plan_residency(const int64_t* freq /*L*E*/, int L, int E, uint64_t budget,
                      uint64_t expert_bytes, int32_t* pairs_out);

/* LLaPor inference net (predictor.hpp:58-83), flattened. Block j of `blocks` maps
 * dims[j] -> dims[j+1]; residual blocks are width -> width. */
#define OR_MAX_BLOCKS 8
typedef struct {
  int H, P, E, width;
  const double* pca_mean;  /* [H] */
  const double* pca_comp;  /* [P*H] */
  int n_blocks;
  int dims[OR_MAX_BLOCKS + 1];
  const double* w[OR_MAX_BLOCKS];
  const double* b[OR_MAX_BLOCKS];
  int n_res;
  const double* rw[OR_MAX_BLOCKS];
  const double* rb[OR_MAX_BLOCKS];
  const double* gate_w; /* [P] (n_res > 0) */
  double gate_b;
  const double* out_w;  /* [E*width] */
  const double* out_b;  /* [E] */
} or_llapor_net;

/* predictor.cpp:116-124 + 166-247 + 344-352 + 669-672 (eval mode). */
int or_llapor_forward(const or_llapor_net* net, const double* hidden_prev,
                      const int32_t* active_prev, int k_prev, const double* gate_prev, int k,
                      double* reduced_out, double* logits_out, int32_t* topk_out);

/* --- Parity-unpinned pieces (no reference code) --------- */

/* Counting-sort permutation: rows ordered (expert asc, token asc, slot asc).
 * offsets [E+1]; perm_src [B*k] = token*k+slot at each permuted row; inv [B*k]. */
void or_permute(const int32_t* ids, int B, int k, int E, int32_t* offsets, int32_t* perm_src,
                int32_t* inv);

/* One MoE layer on bf16 weights, f64 accumulation.
 * slab[e] -> [Wg (F*H) | Wu (F*H) | Wd (H*F)] bf16 row-major (expert_bytes = 6*H*F).
 * x bf16 [B*H]; ids [B*k]; gate f32 [B*E] (full-softmax weights, workload.cpp:190-195);
 * y f32 [B*H] = sum_j gate[t, ids[t,j]] * FFN_{ids[t,j]}(x_t).
 * round_h: round the SwiGLU activation to bf16 before the down projection. */
void or_moe_layer(const uint16_t* const* slab, int H, int F, int B, int k, int E,
                  const uint16_t* x, const int32_t* ids, const float* gate, float* y,
                  int round_h, int threads);

/* Single expert on m rows: y [m*H] f32 (f64 accumulation). */
void or_expert_ffn(const uint16_t* slab, int H, int F, int m, const uint16_t* x, float* y,
                   int round_h);

/* Synthetic expert weights (see oracle.c). */
void or_init_slab(uint16_t* slab, int H, int F, uint64_t seed, int layer, int expert);

float or_bf16_to_f32(uint16_t v);
uint16_t or_f32_to_bf16(float v);

#ifdef __cplusplus
}
#endif
#endif
