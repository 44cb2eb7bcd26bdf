/* ps_api.h — C ABI of the B200-native PreScope MoE-inference hot path.
 *
 * Drop-in boundary for the reference's C++ operator API (namespace prescope,
 * /root/reference/proj/include/prescope/ *.hpp). Every entry point below names the
 * reference interface it replaces (file:line). Plain C: integers, doubles, caller-
 * owned buffers, opaque handles, cudaStream_t as void*. No exception crosses this
 * boundary; errors are status codes plus a thread-local message (ps_last_error), and
 * include/prescope_b200.hpp re-throws them as the reference's exception types
 * (invalid_argument / out_of_range / runtime_error, tools/prescope_main.cpp:427-434).
 *
 * Threading: host planning/simulation entry points are pure and reentrant. A ps_engine
 * is single-owner (one host thread per engine). GPU entry points enqueue
 * on the given stream and never synchronise the device unless stated.
 */
#ifndef PS_API_H
#define PS_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------------- status */
typedef enum {
  PS_OK = 0,
  PS_EINVAL = 1,   /* std::invalid_argument */
  PS_ERANGE = 2,   /* std::out_of_range */
  PS_ERUNTIME = 3, /* std::runtime_error (I/O, overflow, checksum) */
  PS_ECUDA = 4,    /* CUDA runtime / driver failure */
  PS_ENCCL = 5     /* NCCL failure */
} ps_status;

const char* ps_last_error(void);
const char* ps_version(void);

/* ---------------------------------------------------------------------- model spec
 * prescope::ModelSpec (workload.hpp:18-31) and presets (workload.cpp:43-79). */
typedef struct {
  int32_t num_layers;
  int32_t experts_per_layer;
  int32_t top_k;
  int32_t hidden_dim;
  uint64_t expert_bytes; /* 3*H*F*2 (bf16 gate/up/down) */
  int32_t group_begin_middle;
  int32_t group_begin_output;
} ps_model_spec;

typedef enum { PS_GROUP_INPUT = 0, PS_GROUP_MIDDLE = 1, PS_GROUP_OUTPUT = 2 } ps_layer_group;

ps_status ps_spec_validate(const ps_model_spec* spec);                      /* workload.cpp:24-32 */
ps_status ps_spec_group_of(const ps_model_spec* spec, int layer, int* group); /* workload.cpp:34-40 */
ps_status ps_spec_preset(const char* name, ps_model_spec* out);             /* workload.cpp:65-71 */
ps_status ps_desk_scale(const ps_model_spec* full, int num_layers, int experts, int hidden,
                        ps_model_spec* out);                               /* workload.cpp:73-79 */
/* F = expert_bytes / (6*H); PS_EINVAL when expert_bytes is not 6*H*F. */
ps_status ps_spec_ffn_dim(const ps_model_spec* spec, int* ffn_dim);

/* ------------------------------------------------------------------ routing (host) */
/* topk_indices (workload.cpp:110-119): weight desc, ties lower index. Returns count. */
int ps_topk_indices(const double* weights, int n, int k, int32_t* out);
/* routing_map (workload.cpp:106-108). */
int ps_routing_map(const ps_model_spec* spec, int expert);

/* Synthetic routing inputs of generate_trace (workload.cpp:139-219) WITHOUT the
 * routing: the gate matrices, the per-(token, layer) hidden state a and the kappa
 * follow flag are routing-independent, so the GPU router consumes
 * them and recomputes the trace's routing. Same RNG stream as the reference.
 *   gate   [L*E*H] f64 (nullable), hidden [B*L*H] f64 (nullable), follow [B*L] u8,
 *   index (token*L + layer). zipf per layer: [L] f64 (nullable). */
typedef struct {
  double rho, kappa, zipf_s;
} ps_group_gen;
typedef struct {
  ps_group_gen input, middle, output;
  double noise_scale;
} ps_trace_gen_config;
ps_status ps_trace_inputs(const ps_trace_gen_config* cfg, const ps_model_spec* spec, int batch,
                          uint64_t seed, double* gate, double* hidden, uint8_t* follow,
                          double* zipf_per_layer);

/* ------------------------------------------------------------------- trace files
 * write_trace / read_trace (workload.cpp:290-436), format v1: one JSON header line
 * {"batch_size","checksum" (FNV-1a 64 of the body),"format_version":1,"seed","spec"},
 * then one TSV line per (token, layer) step in (token, layer) order:
 *   layer \t hidden[H] \t gate_weights[E] \t active[k] \t e:m e:m ...  (doubles %.17g).
 * Errors: PS_ERUNTIME "TraceFormatError: ..." / "TraceChecksumError: ..."
 * (workload.hpp:106-111) or I/O failure; PS_EINVAL for an invalid spec. */
typedef struct ps_trace_s* ps_trace;
uint64_t ps_fnv1a64(const void* data, size_t n);                 /* workload.cpp:290-297 */
ps_status ps_trace_read(const char* path, ps_trace* out);        /* read_trace, workload.cpp:409-436 */
ps_status ps_trace_shape(ps_trace t, ps_model_spec* spec, int32_t* batch, uint64_t* seed,
                         uint64_t* checksum);
/* Dense copies, index (token*L + layer): hidden [B*L*H] f64, gate_weights [B*L*E] f64,
 * active [B*L*k] i32 (weight-desc), tokens [B*L*E] i32 (tokens_per_expert, 0 = absent).
 * Each output nullable. */
ps_status ps_trace_arrays(ps_trace t, double* hidden, double* gate_weights, int32_t* active,
                          int32_t* tokens);
ps_status ps_trace_free(ps_trace t);
/* write_trace (workload.cpp:391-407): byte-identical to the reference for the same trace. */
ps_status ps_trace_write(const char* path, const ps_model_spec* spec, int batch, uint64_t seed,
                         const double* hidden, const double* gate_weights, const int32_t* active,
                         const int32_t* tokens);

/* --------------------------------------------------------------------- cost model
 * prescope::CostParams / ExpertLoad / HitStats (cost_model.hpp:13-62). Ticks = us. */
typedef struct {
  int64_t t_io, t_g, t_attn;
  double beta;
  int64_t startup;
  int64_t alpha;
} ps_cost_params;

typedef enum { PS_LOC_RESIDENT = 0, PS_LOC_INFLIGHT = 1, PS_LOC_HOST = 2 } ps_expert_location;

typedef struct {
  int32_t expert, layer, tokens, location;
} ps_expert_load;

typedef struct {
  double r_hit, r_miss;
  int32_t window;
} ps_hit_stats;

int64_t ps_to_ticks(double x);                                        /* cost_model.cpp:11 */
ps_status ps_cost_params_validate(const ps_cost_params* p);           /* cost_model.cpp:13-18 */
ps_status ps_hit_stats_record(ps_hit_stats* s, int hit);              /* cost_model.cpp:28-32 */
ps_status ps_cpu_cost(int tokens, const ps_cost_params* p, int64_t* out); /* cost_model.cpp:34-37 */
/* overlap_prefetch_count (cost_model.cpp:94-100) and prefetch_gain (102-106). */
ps_status ps_overlap_prefetch_count(int64_t t_gap, const ps_cost_params* p, double* f, int* f_int);
double ps_prefetch_gain(const ps_hit_stats* s, double f, int f_int, const ps_cost_params* p);
/* fit_cost_params (cost_model.cpp:45-72): OLS over (tokens, ticks). */
ps_status ps_fit_cost_params(const int32_t* tokens, const int64_t* ticks, int n, double* beta,
                             double* startup, double* r_squared);

/* ----------------------------------------------------------------------- PreSched
 * LayerInputs / LayerPlan / SchedulerPolicy (scheduler.hpp:13-65). */
typedef struct {
  const ps_expert_load* e_cur;   int32_t n_cur;   /* gating truth, ascending tokens */
  const ps_expert_load* e_next;  int32_t n_next;  /* predicted l+1 */
  const ps_expert_load* e_next2; int32_t n_next2; /* predicted l+2 (widened window) */
  ps_cost_params params;
  ps_hit_stats stats;
} ps_layer_inputs;

typedef struct {
  int64_t* sweep_gpu; /* nullable, capacity >= n_cur + n_next */
  int64_t* sweep_cpu; /* nullable */
  int32_t n_sweep;
  int64_t t_g_at_split, t_c_at_split, t_gap;
  double f;
  int32_t f_int;
  double xi;
  int32_t widened_window, all_gpu_fallback;
} ps_decision_trace;

typedef struct {
  /* caller-owned outputs; capacities: cpu_set/ondemand_seq >= n_cur,
   * prefetch_seq >= max(n_next, n_next2) */
  ps_expert_load* cpu_set;      int32_t n_cpu;
  ps_expert_load* ondemand_seq; int32_t n_ondemand;
  ps_expert_load* prefetch_seq; int32_t n_prefetch;
  int32_t prefetch_from_widened;
  int32_t split_index;
  int32_t issued_prefetches;
  ps_decision_trace trace;
} ps_layer_plan;

typedef enum {
  PS_POLICY_PRESCHED = 0,
  PS_POLICY_GREEDY = 1,
  PS_POLICY_ONDEMAND = 2,
  PS_POLICY_FIXED = 3,
  PS_POLICY_ORACLE = 4
} ps_policy_kind;

typedef struct {
  int32_t kind;
  int32_t fixed_prefetch;
} ps_policy;

ps_status ps_policy_parse(const char* text, ps_policy* out);           /* scheduler.cpp:23-41 */
ps_status ps_policy_name(ps_policy p, char* buf, int cap);             /* scheduler.cpp:43-52 */
ps_status ps_layer_inputs_validate(const ps_layer_inputs* in);         /* scheduler.cpp:8-21 */
/* plan_layer (scheduler.cpp:271-282) dispatching to schedule_layer (188-213),
 * greedy_layer_baseline (215-250), ondemand_only_plan (252-260), fixed_prefetch_plan
 * (262-269). O(n log n) (stable merge + prefix sums) instead of the reference's
 * O((n+n')^2), bit-identical results. Host, pure, reentrant. */
ps_status ps_presched_plan(const ps_layer_inputs* in, ps_policy policy, ps_layer_plan* out);

/* ------------------------------------------------------- AsyncIO model-clock pipeline
 * PipelineInstance / Timeline / SimOptions / simulate_pipeline (simulator.hpp:14-96).
 * Dense layout: truth/predicted [L*E] token counts (0 = absent), resident [L*E] u8,
 * groups [L] (nullable => all middle). */
typedef struct {
  int32_t num_layers, experts;
  const int32_t* truth;
  const int32_t* predicted;
  const uint8_t* resident;
  const int32_t* groups;
} ps_pipeline_instance;

typedef enum { PS_RES_GPU = 0, PS_RES_CPU = 1, PS_RES_IO = 2 } ps_resource;
typedef enum {
  PS_EV_ATTENTION = 0, PS_EV_GPU_EXPERT = 1, PS_EV_CPU_EXPERT = 2,
  PS_EV_LOAD = 3, PS_EV_PREFETCH = 4, PS_EV_IDLE = 5
} ps_event_kind;

typedef struct {
  int64_t t_start, t_end;
  int32_t resource, kind, layer, expert, tokens;
} ps_timeline_event;

typedef struct {
  ps_timeline_event* events; int32_t cap_events; int32_t n_events;
  int64_t* layer_start; /* [L] */
  int64_t* layer_end;   /* [L] */
  int64_t makespan;
  int32_t* plan_summary; /* nullable [4*L]: split, issued, from_widened, n_ondemand */
} ps_timeline;

typedef struct {
  int32_t cpu_slots;        /* default 1 */
  int32_t prefetch_slots;   /* default 8 per target layer */
  double initial_hit_rate;  /* default 1.0 */
  int32_t hit_window;       /* default 32 */
} ps_sim_options;

/* PlanFn plugin seam (simulator.hpp:66): called once per layer. */
typedef ps_status (*ps_plan_fn)(void* user, const ps_layer_inputs* in, int layer,
                                ps_layer_plan* out);

/* simulate_pipeline (simulator.cpp:61-242). plan_fn NULL => plan with `policy`. */
ps_status ps_simulate_pipeline(const ps_pipeline_instance* inst, ps_policy policy,
                               ps_plan_fn plan_fn, void* user, const ps_cost_params* params,
                               const ps_sim_options* opts, ps_timeline* out);
/* verify_timeline (simulator.cpp:323-394): number of violations in *n_violations;
 * messages (nullable) newline-joined into msg_buf. */
ps_status ps_verify_timeline(const ps_timeline_event* events, int n_events,
                             const ps_pipeline_instance* inst, const ps_cost_params* params,
                             int* n_violations, char* msg_buf, int msg_cap);
/* Same checks; measured != 0 for timelines recorded on the GPU (ps_engine_last_timeline):
 * transfer durations are measured, so "atomic t_io interval" becomes "one interval". */
ps_status ps_verify_timeline_ex(const ps_timeline_event* events, int n_events,
                                const ps_pipeline_instance* inst, const ps_cost_params* params,
                                int measured, int* n_violations, char* msg_buf, int msg_cap);
/* export_timeline (simulator.cpp:428-436): "# tick_unit=us makespan=M" then one
 * "t_start t_end resource kind layer expert tokens" line per event (same text as the
 * reference). *needed = bytes incl. NUL; buf (nullable) receives at most cap-1 chars. */
ps_status ps_export_timeline(const ps_timeline_event* events, int n, int64_t makespan, char* buf,
                             int cap, int* needed);
/* compute_metrics (simulator.cpp:396-426) of a Timeline {events, layer_start/end [L],
 * makespan}: makespan is the timeline's own field, as the reference reads it
 * (simulate_pipeline sets it to max t_end, simulator.cpp:239-240). per_layer arrays
 * nullable [L]. An event layer outside [0, L) -> PS_ERANGE (out_of_range). */
typedef struct {
  int64_t makespan, decode_latency;
  double throughput_tokens_per_s, io_busy_fraction, gpu_idle_fraction;
} ps_metrics;
ps_status ps_compute_metrics(const ps_timeline_event* events, int n_events,
                             const int64_t* layer_start, const int64_t* layer_end, int L,
                             int64_t makespan, int output_tokens, ps_metrics* out,
                             int64_t* per_layer_latency, int64_t* cpu_gpu_gap);

/* ------------------------------------------------------------------ hot table / HBM budget
 * build_hot_table + plan_residency (predictor.cpp:405-433). freq [L*E]. */
ps_status ps_plan_residency(const int64_t* freq, int L, int E, uint64_t budget_bytes,
                            uint64_t expert_bytes, int32_t* pairs_out, int* n_out);

/* -------------------------------------------------------------------------- GPU ops
 * All device pointers; `stream` is a cudaStream_t. Shapes: B tokens, H hidden,
 * E experts, k top-k, F ffn dim. bf16 = uint16_t storage. */

/* K1 — fused router: fp32 gate GEMV + zipf bias + kappa-follow override + softmax +
 * top-k (ranking the softmax weights, ties lower index) + per-expert histogram, one
 * launch. Replaces the router loop of generate_trace (workload.cpp:176-202) and
 * aggregate_layer_loads (workload.cpp:283-288).
 *   x [B,H] f32; gate [E,H] f32; bias [E] f32 (= -zipf*ln(e+1), nullable);
 *   follow [B] u8 (nullable); prev_ids [B,prev_k] i32 (nullable: layer 0).
 * Outputs: logits/weights [B,E] f32 (nullable), ids [B,k] i32, counts [E] i32
 * (overwritten), x_bf16 [B,H] (nullable; fused cast for the expert FFN). */
ps_status ps_route_topk(const float* x, const float* gate, const float* bias,
                        const uint8_t* follow, const int32_t* prev_ids, int prev_k, int B,
                        int H, int E, int k, float* logits, float* weights, int32_t* ids,
                        int32_t* counts, uint16_t* x_bf16, void* stream);

/* K1 + K2 index pass in ONE launch for decode batches (1 <= B <= 64): the route CTAs as
 * in ps_route_topk (no histogram: counts = diff of offsets), then the last CTA to finish
 * runs the counting-sort permute of ps_permute over all B*k ids (bit-identical outputs).
 * workspace: 65 int32 on the device (a launch ticket + per-token tickets of the E >= 64
 * split), zero before the first call (the kernel leaves them zero); one per stream. */
ps_status ps_route_permute(const float* x, const float* gate, const float* bias,
                           const uint8_t* follow, const int32_t* prev_ids, int prev_k, int B,
                           int H, int E, int k, float* weights, int32_t* ids, uint16_t* x_bf16,
                           int32_t* offsets, int32_t* perm_src, int32_t* inv, int32_t* workspace,
                           void* stream);

/* K2 — counting-sort permute: rows ordered (expert asc, token asc, slot asc).
 *   offsets [E+1], perm_src [B*k] (= token*k+slot), inv [B*k].
 *   x [B,H] bf16 + x_perm [B*k,H] bf16: optional gather (both nullable). */
ps_status ps_permute(const int32_t* ids, int B, int k, int E, int32_t* offsets,
                     int32_t* perm_src, int32_t* inv, const uint16_t* x, int H,
                     uint16_t* x_perm, void* stream);

/* K2 — row gather: out[i, :] = x[idx[i] / div, :] (bf16 rows, H % 8 == 0). */
ps_status ps_gather_rows(const uint16_t* x, const int32_t* idx, int n, int div, int H, uint16_t* out,
                         void* stream);

/* K2 — weighted combine: y[t] = sum_j weights[t, ids[t,j]] * sum_s y_part[s][inv[t*k+j]]
 * (full-softmax gate weights, workload.cpp:190-195; no top-k renormalisation).
 *   y_part [n_split, B*k, H] f32; y [B,H] f32. */
ps_status ps_combine(const float* y_part, int n_split, const int32_t* inv, const int32_t* ids,
                     const float* weights, int B, int k, int E, int H, float* y, void* stream);

/* x [n] f32 -> bf16 (round to nearest even), the FFN input cast K1 otherwise fuses. */
ps_status ps_cast_bf16(const float* x, int64_t n, uint16_t* out, void* stream);
/* dst[0, n) = host_src[0, n) read by the SMs from mapped pinned host memory (no copy
 * engine), and dst[z*zero_stride, +n) = 0 for z = 1..zero_copies. n, zero_stride % 4 == 0. */
ps_status ps_rows_from_host(const float* host_src, int64_t n, float* dst, int zero_copies, int64_t zero_stride,
                            void* stream);
/* The same for several row ranges of one mapped pinned buffer in one launch: rows
 * [row0[i], row0[i] + m[i]) of host_base (f32, row length H) -> the same rows of dst, and
 * zero_copies zero-filled copies at zero_stride (floats; >= the largest row end * H).
 * n_ranges <= 128, H % 4 == 0. */
ps_status ps_rows_from_host_ranges(const float* host_base, const int32_t* row0, const int32_t* m, int n_ranges,
                                   int H, float* dst, int zero_copies, int64_t zero_stride, void* stream);

/* Shared experts (BASELINE config 3, DeepSeek-V2-Lite: 2 always-active experts with gate
 * weight 1; a north_star extension — the reference's ModelSpec has none): appends
 * virtual experts E..E+S-1 to every token so K2/K3/combine run them with the routed ones.
 *   ids [B,k] -> ids_ext [B,k+S]; weights [B,E] -> weights_ext [B,E+S] (1.0 for shared);
 *   counts [E+S] (nullable): entries E..E+S-1 set to B (K1 wrote 0..E-1). */
ps_status ps_append_shared(const int32_t* ids, const float* weights, int B, int k, int E, int S,
                           int32_t* ids_ext, float* weights_ext, int32_t* counts, void* stream);

/* K3 — grouped SwiGLU expert FFN over a set of experts whose slabs are on device.
 * Slab layout [Wg (F*H) | Wu (F*H) | Wd (H*F)] bf16 row-major = expert_bytes.
 * Rows of expert experts[i] are permuted rows [offsets[e], offsets[e+1]) (K2), token
 * = perm_src[row]/k; x [B,H] bf16.
 * Decode path (HBM-bound GEMV): h [B*k,F] bf16 scratch, y_part [n_split,total_rows,H]
 * f32 with total_rows = B*k (all permuted rows). counts_host [E]: host copy of the
 * histogram (grid sizing only; the kernels read offsets on the device). */
#define PS_MAX_GROUP 256
typedef struct {
  int32_t n;
  int32_t experts[PS_MAX_GROUP];
  const uint16_t* slabs[PS_MAX_GROUP];
} ps_expert_group;

ps_status ps_expert_ffn(const ps_expert_group* group, const int32_t* counts_host,
                        const int32_t* offsets, const int32_t* perm_src, int k,
                        const uint16_t* x, int H, int F, uint16_t* h, float* y_part,
                        int n_split, int total_rows, void* stream);
/* K3 decode path reading the experts' weights as z-slabs (device copies of
 * ps_zslab_encode_tiled output for [H, F] experts, e.g. a prefetch or on-demand copy that
 * just landed): the consumer warps decode their MMA fragments from the z bytes in
 * registers, so the expert's HBM traffic is its z bytes (~70 % of bf16) instead of a
 * decode pass (z read + bf16 write) and the bf16 read. Results are bitwise equal to
 * ps_zslab_decode + ps_expert_ffn. group->slabs is ignored; zslabs[i] is entry i's z-slab.
 * Requires <= 8 tokens per expert, H % 64 == 0, F % 64 == 0, 3*H*F < 2^32 and a down split
 * width (ps_ffn_down_splits) that is a multiple of 64; a slab whose header does not
 * describe a tiled [H, F] expert fails the launch (device trap). */
ps_status ps_expert_ffn_zslab(const ps_expert_group* group, const void* const* zslabs,
                              const int32_t* counts_host, const int32_t* offsets,
                              const int32_t* perm_src, int k, const uint16_t* x, int H, int F,
                              uint16_t* h, float* y_part, int n_split, int total_rows, void* stream);
/* K3 prefill path (tensor-bound): tcgen05/TMEM/TMA grouped GEMM over contiguous
 * permuted rows. x_perm [total_rows, H] bf16 (K2 gather); offsets_host [E+1] / counts_host
 * [E] are host copies of K2's offsets / K1's histogram. Outputs h_perm [total_rows, F]
 * bf16 (SwiGLU activations) and y_perm [total_rows, H] f32 (per-row expert output;
 * combine with ps_combine, n_split = 1). Requires H % 256 == 0, F % 128 == 0. */
ps_status ps_expert_ffn_prefill(const ps_expert_group* group, const int32_t* counts_host,
                                const int32_t* offsets_host, const uint16_t* x_perm, int total_rows,
                                int H, int F, uint16_t* h_perm, float* y_perm, void* stream);
/* Same FFN with the counts on the DEVICE: offsets_dev [E+1] (K2's offsets on the stream);
 * the tile schedule is built by a one-CTA kernel in stream order, so a caller can launch
 * the resident group before it has read the routing back (token-N kernel; experts with
 * no routed rows cost nothing). */
ps_status ps_expert_ffn_prefill_dev(const ps_expert_group* group, const int32_t* offsets_dev,
                                    const uint16_t* x_perm, int total_rows, int H, int F, uint16_t* h_perm,
                                    float* y_perm, void* stream);
/* Prefill kernel choice (process-wide): 0 = single-CTA M=128 token tiles, 1 = CTA pairs
 * (cta_group::2, M=256 token tiles), 3 = token-N CTA pairs (weights as M=256, an
 * expert's tokens as N <= 256 in steps of 16; gate_up and down in one launch),
 * 2 = auto (default) = 3. */
ps_status ps_set_prefill_kernel(int mode);
/* Split-K factor ps_expert_ffn expects for the down projection at this shape. */
int ps_ffn_down_splits(int H, int F);

/* Deterministic synthetic expert weights: counter-hash of (seed, layer, expert, index)
 * -> bf16 ~ N(0, 1/sqrt(fan_in)) by Irwin-Hall sum of 4 uniforms (exact integer
 * arithmetic, identical on host and device). Gate/up rows have fan_in H, down rows F. */
ps_status ps_init_expert_slab(uint16_t* slab, int H, int F, uint64_t seed, int layer,
                              int expert, void* stream);
ps_status ps_init_expert_slab_host(uint16_t* slab, int H, int F, uint64_t seed, int layer,
                                   int expert);

/* Host expert lane (Resource::Cpu of the reference, simulator.cpp:139-146; cpu_cost
 * cost_model.cpp:34-37): SwiGLU expert FFN on the host cores (AVX512-BF16 GEMV, a thread
 * pool, fp32 accumulation, h rounded to bf16 like K3) reading the expert's slab where it
 * lies in (pinned) host DRAM. Opt-in lane of the engine (ps_engine_config.host_threads);
 * PS_ERUNTIME if the CPU lacks AVX512_BF16. A lane is single-owner.
 *   slab [Wg|Wu|Wd] bf16 (host), x [m,H] bf16 (host), y [m,H] f32 (host). H,F % 32 == 0. */
typedef struct ps_host_lane_s* ps_host_lane;
ps_status ps_host_lane_create(int threads, ps_host_lane* out);
ps_status ps_host_lane_destroy(ps_host_lane lane);
int ps_host_lane_threads(ps_host_lane lane);
int ps_host_lane_isa(ps_host_lane lane); /* 2 = AMX-BF16 tiles, 1 = AVX512-BF16 GEMV */
/* 1 if ps_host_expert_ffn_batch_z runs on this host (AMX-BF16 + AVX-512 VBMI2) */
int ps_host_lane_reads_z(ps_host_lane lane);
/* Pin the calling thread (the one that will call ps_host_expert_ffn*: pool worker 0) to
 * the lane's first CPU. The pool's workers are pinned to the last `threads` CPUs of the
 * process affinity set unless PS_HOST_LANE_PIN=0. */
ps_status ps_host_lane_bind_caller(ps_host_lane lane);
ps_status ps_host_expert_ffn(ps_host_lane lane, const uint16_t* slab, int H, int F, const uint16_t* x,
                             int m, float* y);
/* Same, weights read from z-slabs (ps_zslab_encode of the slabs): 1.5 instead of 2 bytes
 * of host DRAM per weight, decoded tile by tile in registers/L1 (AMX-BF16 lanes only,
 * PS_ERUNTIME otherwise). Bitwise the results of the raw-slab call. */
ps_status ps_host_expert_ffn_batch_z(ps_host_lane lane, int n, const uint8_t* const* zslabs,
                                     const int32_t* m, const int32_t* row0, int H, int F,
                                     const uint16_t* x, float* y);
/* A layer's cpu_set in one call: expert j reads x rows [row0[j], row0[j] + m[j]) and
 * writes the same rows of y (both [*, H], host). Same numerics per expert. */
ps_status ps_host_expert_ffn_batch(ps_host_lane lane, int n, const uint16_t* const* slabs,
                                   const int32_t* m, const int32_t* row0, int H, int F,
                                   const uint16_t* x, float* y);
/* The lane's tile layout: ps_host_slab_tile re-lays a slab in place so that every 16-row
 * block of W_gate/W_up [F][H] and W_down [H][F] is a run of 16x32 tiles of 1 KiB (the
 * block keeps its byte range); ps_host_expert_ffn_batch_tiled reads slabs in that layout
 * (AMX-BF16 lanes only) with two sequential streams per block instead of 32 row streams.
 * Bitwise the results of ps_host_expert_ffn_batch on the row-major slabs. */
ps_status ps_host_slab_tile(uint16_t* slab, int H, int F);
ps_status ps_host_slab_untile(uint16_t* slab, int H, int F); /* inverse of ps_host_slab_tile */
ps_status ps_host_expert_ffn_batch_tiled(ps_host_lane lane, int n, const uint16_t* const* slabs,
                                         const int32_t* m, const int32_t* row0, int H, int F,
                                         const uint16_t* x, float* y);

/* z-slabs: lossless transfer format of a host-resident expert slab (csrc/zexpert.cu):
 * verbatim sign+mantissa bytes, 4-bit exponent codes relative to a per-slab base, escapes
 * for the rest (~12 bits per bf16 value), so PCIe moves ~75 % of the bytes. Decoding is
 * bit-exact. Encode on the host (at engine create), decode on the GPU after the copy. */
uint64_t ps_zslab_bound(uint64_t n);  /* worst-case z-slab bytes for n bf16 values */
ps_status ps_zslab_encode(const uint16_t* slab, uint64_t n, uint8_t* out, uint64_t cap,
                          uint64_t* out_bytes, int threads);
ps_status ps_zslab_info(const uint8_t* z_host, uint64_t* n, uint64_t* bytes, uint64_t* n_escapes);
/* z-slab of a slab in the lane's tile layout (after ps_host_slab_tile): header marked
 * tiled, so ps_zslab_decode still writes the row-major slab and the lane's z path reads
 * every 16-row block as two sequential streams. */
ps_status ps_zslab_encode_tiled(const uint16_t* slab_tiled, int H, int F, uint8_t* out, uint64_t cap,
                                uint64_t* out_bytes, int threads);
/* z_dev: device copy of the z-slab; z_host_header: the host z-slab (header read on the host). */
ps_status ps_zslab_decode(const uint8_t* z_dev, const uint8_t* z_host_header, uint16_t* out,
                          void* stream);

/* K4 — LLaPor predictor (predictor.cpp:116-124, 166-247, 344-352, 669-672). */
typedef struct ps_llapor_s* ps_llapor;
/* load_checkpoint (predictor.cpp:866-929): LLPC v1 file -> device-resident nets. */
ps_status ps_llapor_load(const char* path, ps_llapor* out, ps_model_spec* spec_out);
/* Random-init nets at full shapes (pca_dim/width per group, predictor.hpp:97-100). */
ps_status ps_llapor_random(const ps_model_spec* spec, int pca_in, int pca_mid, int width_in,
                           int width_mid, uint64_t seed, ps_llapor* out);
ps_status ps_llapor_free(ps_llapor m);
/* save_checkpoint (predictor.cpp:833-875): LLPC v1, every field of the loaded/fine-tuned
 * model (byte-identical to the reference's file for the same model). Host only. */
ps_status ps_llapor_save(ps_llapor m, const char* path);
/* Online fine_tune (predictor.cpp:654-663) of net `layer` on n observed samples — the
 * reference's build_samples pairs (predictor.cpp:596-613): features of layer-1 (hidden
 * [n,H] f64, active experts [n,k_prev], full-softmax gate weights [n,E] f64) and the
 * labels of layer `layer` (active experts [n,k] -> multi-hot). `steps` AdamW passes at
 * learning rate lr with the model's TrainConfig (batch_size, lambda, gamma, weight decay
 * of the net's group, seed); host f64, bit-identical to the reference. The net's GPU
 * copy is refreshed before its next ps_llapor_forward. Host buffers; no GPU needed. */
ps_status ps_llapor_fine_tune(ps_llapor m, int layer, int n, const double* hidden_prev,
                              const int32_t* active_prev, int k_prev, const double* gate_prev,
                              const int32_t* active, int k, int steps, double lr);
/* Net for target layer `layer` (>=1) on features of layer-1 for B tokens:
 *   hidden [B,H] f32, prev_ids [B,k_prev] i32, prev_weights [B,E] f32.
 * Outputs: logits [B,E] f32 (nullable), ids [B,k] i32 (top-k on LOGITS),
 * pred_counts [E] i32 (overwritten; predicted per-expert histogram, predict_loads
 * experiment.cpp:104-112). scratch: ps_llapor_scratch_bytes. */
size_t ps_llapor_scratch_bytes(ps_llapor m, int B);
ps_status ps_llapor_forward(ps_llapor m, int layer, const float* hidden,
                            const int32_t* prev_ids, int k_prev, const float* prev_weights,
                            int B, int k, float* logits, int32_t* ids, int32_t* pred_counts,
                            void* scratch, void* stream);

/* ---------------------------------------------------------- expert parallelism (EP)
 * SURVEY.md §8e (a north_star extension; the reference has no multi-GPU code,
 * SPEC.md:17): expert e of every layer is owned by rank e % world. Each rank routes its
 * own tokens, permutes them owner-major (virtual id v = (e % G)*ceil(E/G) + e/G, so
 * ps_permute over v yields destination-rank segments), exchanges per-(source, local
 * expert) counts and then the rows (all-to-all dispatch), runs its local experts, and
 * returns the per-row outputs (all-to-all combine) for the weighted sum at home. */
typedef struct ps_ep_comm_s* ps_ep_comm;
int ps_ep_local_experts(int E, int world, int rank);
ps_status ps_ep_remap_ids(const int32_t* ids, int n, int E, int world, int32_t* vids, void* stream);
/* Per-destination counts message [world][2*E_loc]: rows for each of the destination's
 * local experts (from ps_permute offsets over virtual ids, [world*E_loc+1]) followed by
 * this rank's predicted tokens for them (pred [E], nullable). */
ps_status ps_ep_pack_counts(const int32_t* offsets_v, const int32_t* pred, int E, int world,
                            int32_t* out, void* stream);
/* Receiver plan from recv_counts [G][E_loc] (rows from source s for local expert j):
 * offsets [E_loc+1] of the local expert-major order, perm_src [total] (permuted local
 * row -> received row, nullable), recv_seg [G+1] row offsets of each source segment. */
ps_status ps_ep_recv_plan(const int32_t* recv_counts, int world, int E_loc, int32_t* offsets,
                          int32_t* perm_src, int32_t* recv_seg);
/* NCCL transport (grouped ncclSend/ncclRecv over NVLink; NCCL loaded at run time). */
ps_status ps_ep_unique_id(char* out, int cap); /* 128 bytes, broadcast by the caller */
ps_status ps_ep_comm_create(const char* unique_id, int rank, int world, int device, ps_ep_comm* out);
ps_status ps_ep_comm_destroy(ps_ep_comm c);
/* In-process transport with the same all-to-all contract: `world` communicators for
 * `world` host threads of ONE process (one engine per thread, any devices). Lets the
 * expert-parallel engine run at G > 1 on a single GPU (tests). No reference
 * counterpart (the reference has no multi-GPU code). */
ps_status ps_ep_loopback_create(int world, int device, ps_ep_comm* comms_out /* [world] */);
int ps_ep_comm_rank(ps_ep_comm c);
int ps_ep_comm_world(ps_ep_comm c);
/* Segmented all-to-all: segment p of `send` (send_bytes[p]) goes to rank p, segment p
 * of `recv` (recv_bytes[p]) comes from rank p; segments are contiguous and in rank order. */
ps_status ps_ep_all_to_all(ps_ep_comm c, const void* send, const uint64_t* send_bytes, void* recv,
                           const uint64_t* recv_bytes, void* stream);

/* -------------------------------------------------------------------- decode engine
 * K5: the AsyncIO expert loader + HBM expert cache + per-layer decode driver.
 * Resident experts (plan_residency under budget_bytes) live in HBM; the others in
 * pinned host DRAM and are loaded by PreSched plans as cudaMemcpyAsync on a dedicated
 * copy stream (serial I/O channel) into dual on-demand slots (simulator.cpp:181-197)
 * or per-target-layer prefetch slots (simulator.cpp:206-227), event-ordered against
 * the compute stream. */
typedef struct ps_engine_s* ps_engine;

/* The reference's predictor menu (PredictorChoice, experiment.cpp:60-99) for the
 * next-layer load prediction PreSched consumes (predict_loads, experiment.cpp:104-112):
 *   LLAPOR   ps_llapor_forward on the GPU (K4);
 *   GATE     gate_reuse_predict (predictor.cpp:688-690): top-k of layer l's gate weights,
 *            i.e. layer l's own routing histogram;
 *   STATS    stats_predict (predictor.cpp:674-686): the hot table's top-k of layer l+1
 *            for every token;
 *   PERFECT  the true routing of layer l+1 (K1 run one layer early on its inputs);
 *   NONE     no prediction (no prefetch candidates). */
typedef enum {
  PS_PRED_AUTO = 0, PS_PRED_LLAPOR = 1, PS_PRED_GATE = 2, PS_PRED_STATS = 3,
  PS_PRED_PERFECT = 4, PS_PRED_NONE = 5
} ps_predictor_kind;

typedef struct {
  ps_model_spec spec;
  ps_trace_gen_config gen;  /* zipf per group for the router bias */
  uint64_t weight_seed;     /* expert + router weights */
  uint64_t budget_bytes;    /* HBM resident-expert budget */
  const int32_t* resident;  /* nullable [2*n_resident] (layer, expert); else hot table */
  int32_t n_resident;
  int32_t max_batch;
  int32_t prefetch_slots;   /* per target layer, default 8 */
  ps_policy policy;
  ps_cost_params cost;      /* t_io/t_g/t_attn in us; 0 => calibrate at create */
  ps_llapor predictor;      /* nullable => perfect-prediction off; uses gate weights */
  int32_t device;
  int32_t host_pinned;      /* 1: non-resident experts in pinned host DRAM */
  ps_ep_comm ep;            /* nullable: expert-parallel over this communicator; the
                               engine then owns experts e % world == rank only, and
                               `resident`/`budget_bytes` are this rank's */
  int32_t n_shared;         /* always-active shared experts per layer (DeepSeek: 2),
                               HBM-resident outside the routed-expert budget; 0 = none */
  int32_t host_threads;     /* > 0: host expert lane (ps_host_expert_ffn) with this many
                               threads runs PreSched's cpu_set from pinned host DRAM,
                               concurrently with the PCIe loads; beta/startup are then
                               measured at create (unless cost.t_io > 0). 0 = GPU only. */
  int32_t compress_host;    /* 1: host slabs also kept as z-slabs (ps_zslab_encode at create);
                               loads move the z-slab over PCIe and decode it on the GPU */
  int32_t predictor_kind;   /* ps_predictor_kind: which PredictFn (experiment.cpp:60-99)
                               feeds PreSched's e_next (0 = LLaPor when `predictor` is set) */
  const int32_t* stats_ranking; /* PS_PRED_STATS: [L*E] experts of each layer in hot-table
                               order (build_hot_table ranking, predictor.cpp:405-424) */
  const uint16_t* const* expert_weights; /* nullable: the caller's expert slabs, host memory,
                               [L*(E+n_shared)] pointers (index l*(E+n_shared)+e) to bf16
                               [W_gate F*H | W_up F*H | W_down H*F] (expert_bytes each),
                               copied at create (resident -> HBM, others -> the pinned
                               host arena); null = hash-initialised from weight_seed.
                               Under EP only owned experts are read. */
  int32_t lookahead;        /* 0: PreSched's plan only (the reference's executor semantics).
                               d in {1, 2}: a labelled extension — behind PreSched's batch,
                               queue the other predicted non-resident experts of layers
                               l+1..l+d (hottest first, slot cap per target layer); those not
                               started by the next scheduling point are cancelled (R2).
                               3: layer l+2 only, at most two top-up copies per layer. */
  int32_t steal_late;       /* host lane only, 1: a committed prefetch whose copy has not
                               landed when the lane finishes its cpu_set is computed by the
                               lane if the copy needs longer than cpu_cost(m) (the copy's
                               bytes are then unused); 0: the GPU waits for it (R6). */
} ps_engine_config;

ps_status ps_engine_create(const ps_engine_config* cfg, ps_engine* out);
ps_status ps_engine_destroy(ps_engine e);
/* Gate matrices [L,E,H] f32 host (from ps_trace_inputs) -> device. */
ps_status ps_engine_set_router(ps_engine e, const float* gate_host);
/* One decode step over all L layers for B tokens, device buffers:
 *   hidden [L,B,H] f32 (layer-major gating inputs), follow [L,B] u8,
 *   y [L,B,H] f32 out (MoE output per layer), ids [L,B,k] i32 out (routing).
 * Blocks the host until the step's GPU work is complete. */
ps_status ps_engine_decode_step(ps_engine e, const float* hidden, const uint8_t* follow, int B,
                                float* y, int32_t* ids);
/* One decode step with the routing GIVEN instead of computed by K1 — the gating truth of
 * a prescope::Trace (active experts [L,B,k] i32 and full-softmax gate_weights [L,B,E] f32,
 * device buffers, e.g. from ps_trace_read) replayed through the real executor (K2 ->
 * loader/PreSched -> K3 -> combine) with x = hidden [L,B,H] f32. */
ps_status ps_engine_decode_step_routed(ps_engine e, const float* hidden, const int32_t* ids,
                                       const float* weights, int B, float* y);
/* Same, from HOST buffers (pinned or pageable): copies in, step, copies out. */
ps_status ps_engine_decode_step_host(ps_engine e, const float* hidden_host,
                                     const uint8_t* follow_host, int B, float* y_host,
                                     int32_t* ids_host);

/* Stand-alone K5 expert cache: the AsyncIO channel of simulate_pipeline
 * (simulator.cpp:61-242) for a caller that runs its own layer loop and FFN kernels.
 * Resident pairs live in one HBM arena (<= budget); other experts are copied from the
 * caller's host slabs into n_slots HBM staging slots by one serial copy channel (FIFO,
 * queued prefetches cancellable, started copies non-interruptible). A slot keeps its
 * expert after release. prefetch queues at the tail, ondemand ahead of queued prefetches
 * (promoting a queued prefetch of the same expert); acquire makes `stream` wait for the
 * copy and pins the slot; release records when `stream` is done with it (the next copy
 * into that slot waits — R7's dual buffer generalised). No free slot -> PS_ERUNTIME (the
 * simulator's prefetch-buffer overflow, simulator.cpp:209-212). Host slabs should be
 * pinned for asynchronous copies. */
typedef struct ps_cache_s* ps_cache;
typedef struct {
  int32_t num_layers, experts;
  uint64_t expert_bytes;
  const void* const* host_slabs;  /* [L*E] host pointers (caller-owned, outlive the cache) */
  const int32_t* resident;        /* nullable [2*n_resident] (layer, expert) kept in HBM */
  int32_t n_resident;
  uint64_t budget_bytes;          /* n_resident * expert_bytes must fit */
  int32_t n_slots;                /* staging slots for non-resident experts, >= 2 */
  int32_t device;
} ps_cache_config;
typedef struct {
  int64_t prefetches, ondemand_loads, prefetches_cancelled, slot_hits, resident_hits;
} ps_cache_stats;
ps_status ps_cache_create(const ps_cache_config* cfg, ps_cache* out);
ps_status ps_cache_destroy(ps_cache c);
ps_status ps_cache_prefetch(ps_cache c, int layer, int expert);
ps_status ps_cache_ondemand(ps_cache c, int layer, int expert);
ps_status ps_cache_acquire(ps_cache c, int layer, int expert, void* stream, const void** dev_slab);
ps_status ps_cache_release(ps_cache c, int layer, int expert, void* stream);
ps_status ps_cache_cancel_prefetches(ps_cache c, int* n_cancelled);  /* R2 at a scheduling point */
ps_status ps_cache_sync(ps_cache c);  /* host: until every issued copy completed */
ps_status ps_cache_get_stats(ps_cache c, ps_cache_stats* out);

/* Per-layer K5 ABI — the reference's per-layer seam (plan_fn(inputs, l), simulator.cpp:136)
 * for a host model that runs its own attention between MoE layers:
 *
 *   ps_engine_step_begin(e, B);                  // a new decode pass (R1-R3 state)
 *   for (l = 0; l < L; ++l) {
 *     attention(l, ..., stream);                 // caller's kernels -> x_l
 *     ps_engine_layer_forward(e, l, x_l, follow_l, y_l, ids_l, stream);
 *   }
 *   ps_engine_step_end(e);                       // drain, measurement, timeline
 *
 * x_l [B,H] f32 device (router input = FFN input of layer l), follow_l [B] u8 device
 * (kappa-follow flags, nullable), y_l [B,H] f32 device out, ids_l [B,k] i32 device out
 * (nullable). `stream` (nullable): the caller's stream — the engine's compute stream
 * waits for the caller's prior work on it, and it waits for y_l (CUDA events). Layers
 * run in order 0..L-1; the host returns after the layer's work is enqueued (one host
 * sync per layer on the routing, as in a whole step). Same kernels, plans and loads as
 * ps_engine_decode_step: the outputs are bit-identical (tests/test_gpu_layer_api.py).
 * PS_PRED_PERFECT is rejected (it needs layer l+1's input). */
ps_status ps_engine_step_begin(ps_engine e, int B);
ps_status ps_engine_layer_forward(ps_engine e, int layer, const float* x, const uint8_t* follow,
                                  float* y, int32_t* ids, void* stream);
ps_status ps_engine_step_end(ps_engine e);

typedef struct {
  int64_t steps, layers;
  int64_t ondemand_loads, prefetches_committed, prefetches_cancelled, prefetch_hits;
  int64_t resident_hits;
  double h2d_bytes, h2d_busy_ms, compute_wait_ms, step_ms_total;
  double ffn_ms_total;      /* device time of K3 launches (events) */
  double ffn_bytes_total;   /* algorithmic bytes of those launches: 3*H*F*2 per routed expert */
  double route_phase_ms_total; /* K1 + K4 + K2-index + counts D2H per layer (the scheduling point) */
  double combine_ms_total;     /* K2 combine */
  double ffn_flops_total;      /* 6*m_e*H*F summed over FFN launches */
  int64_t tc_launches;         /* K3 launches that took the tcgen05 (prefill) path */
  int64_t ffn_launches, kernel_launches;
  ps_cost_params cost;      /* calibrated costs in use */
  int64_t cpu_experts;      /* experts run on the host lane */
  double cpu_ms_total;      /* host-lane busy time (wall clock) */
  double cpu_bytes_total;   /* expert bytes the host lane streamed */
  int64_t z_decodes;        /* z-slab decodes (compressed loads landed) */
  double h2d_expert_bytes;  /* expert bytes the issued copies delivered (= h2d_bytes
                               without compression) */
  int64_t lookahead_prefetches; /* prefetch jobs queued by the lookahead top-up */
  int64_t stolen_prefetches;    /* late prefetched experts the host lane computed (steal_late) */
  int64_t calibration_fit;      /* 1: the last ps_engine_calibrate took beta/C from fit_cost_params */
  int64_t prefetches_used;      /* committed prefetches whose target layer routed tokens to them */
  double cpu_read_bytes;        /* host-DRAM bytes the lane read (z-slab or raw bytes) */
  double host_head_ms_total;    /* host time of each step's prologue (before its first GPU mark) */
  double host_tail_ms_total;    /* host time after each step's GPU work: channel drain + measurement */
} ps_engine_stats;
ps_status ps_engine_get_stats(ps_engine e, ps_engine_stats* out);
ps_status ps_engine_reset_stats(ps_engine e);
/* Measured timeline of the last step, from the CUDA events the engine records (us from
 * the step start): per layer an ATTENTION event for the scheduling-point phase
 * (K1+K4+K2+counts D2H), GPU_EXPERT events for every routed expert's FFN launch, LOAD /
 * PREFETCH events for every copy on the serial channel. truth_out [L*E] (nullable)
 * receives the step's per-layer routed token counts and resident_out [L*E] (nullable)
 * the resident flags, i.e. the PipelineInstance to check it against
 * (ps_verify_timeline_ex, measured = 1). */
ps_status ps_engine_last_timeline(ps_engine e, ps_timeline* out, int32_t* truth_out,
                                  uint8_t* resident_out);
/* Predicted per-expert token counts of the last step, [L*E] (row l = the prediction
 * made at layer l-1 for layer l; row 0 = 0). */
ps_status ps_engine_last_predictions(ps_engine e, int32_t* out);
/* Routing of the last completed step, host buffers (nullable): ids [L,B,k] i32 and the
 * full-softmax gate weights [L,B,E] f32 — with the step's hidden states, the observed
 * (features of l-1, labels of l) pairs an online ps_llapor_fine_tune consumes. */
ps_status ps_engine_last_routing(ps_engine e, int32_t* ids_out, float* weights_out);
/* Replace the cost parameters PreSched plans with (e.g. beta = 1e9 disables the host
 * lane's cpu_set for a GPU-only comparison on the same engine). */
ps_status ps_engine_set_cost(ps_engine e, const ps_cost_params* cost);
/* Switch the executor extensions between steps (ps_engine_config.lookahead / steal_late;
 * an engine created with lookahead >= 2 pre-allocates slots for three live layers). */
ps_status ps_engine_set_lookahead(ps_engine e, int lookahead, int steal_late);
/* Calibration (cost_model.cpp:45-72 fit + simulator cost semantics): replace the
 * engine's PreSched costs with the means measured since the last stats reset —
 * t_io = mean copy time per expert, t_g = mean FFN time per routed expert, t_attn =
 * mean scheduling-point phase per layer (us). */
ps_status ps_engine_calibrate(ps_engine e, ps_cost_params* out);

#ifdef __cplusplus
}
#endif
#endif /* PS_API_H */
