// K5 — AsyncIO expert loader + HBM expert cache + per-layer decode driver.
//
// Real-hardware counterpart of the reference's simulated executor
// (simulate_pipeline, simulator.cpp:61-242; rules R1-R8 in SURVEY.md §8a):
//   * resident experts (plan_residency under the HBM budget, predictor.cpp:426-433)
//     live in one HBM arena; every other expert lives in pinned host DRAM;
//   * the serial I/O channel (R7/R8) is one copy stream owned by an I/O thread that
//     keeps at most two expert copies in flight and services a FIFO, so prefetches
//     that have not started by the next layer's scheduling point can still be
//     cancelled (R2) while started ones run to completion (non-interruptible);
//   * on-demand loads go through two alternating HBM slots (dual buffer, R7): a copy
//     into a slot waits (cudaStreamWaitEvent) for the FFN that last read it;
//   * prefetches land in a slot pool per target layer (cap = prefetch_slots, R8),
//     released once the target layer's FFNs are done (R3);
//   * PreSched (ps_presched_plan) runs on the host per layer on the GPU-computed
//     histogram (K1) and the LLaPor-predicted histogram of layer l+1 (K4);
//   * resident experts start computing right after routing, before the host plan
//     (kernels read per-expert row counts on the device), hiding the host round trip.
// GPU-only executor: the plan's cpu_set (empty under the default beta = 1e9 costs,
// SURVEY.md §7 hard part 1) is loaded on demand after ondemand_seq.
#include <algorithm>
#include <atomic>
#include <functional>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <tuple>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>
#include <sys/mman.h>

#include "cuda_host.hpp"
#include "io_channel.hpp"
#include "zslab_format.hpp"

namespace ps {
int prefill_launches_per_call();                  // k3_ffn_prefill.cu
void llapor_prepare(ps_llapor m, int layer);      // k4_llapor.cu
uint64_t llapor_generation(ps_llapor m);
}  // namespace ps

namespace ps {
void plan_layer(const ps_layer_inputs& in, ps_policy pol, ps_layer_plan& out);
}

namespace ps {
namespace {

using Clock = std::chrono::steady_clock;
constexpr int kDecodeMaxBatch = 64;  // larger batches (prefill chunks) take the tcgen05 path

double now_us() {
  return std::chrono::duration<double, std::micro>(Clock::now().time_since_epoch()).count();
}

// Pinned host arena on transparent 2 MiB pages: the host lane streams whole experts with
// 12 threads and 4 KiB pages cost it a TLB miss every 4 KiB per stream (measured +5-12 %
// lane bandwidth, scripts/probes/thp_lane_probe.py). Anonymous mmap + MADV_HUGEPAGE,
// pages faulted in parallel, then cudaHostRegister; cudaHostAlloc if any step fails.
struct PinnedArena {
  void* ptr = nullptr;
  size_t bytes = 0;
  bool registered = false;  // mmap + cudaHostRegister (else cudaHostAlloc)
  void alloc(size_t n) {
    bytes = n;
    void* p = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p != MAP_FAILED) {
      madvise(p, n, MADV_HUGEPAGE);
      const size_t page = 2u << 20;
      const size_t pages = (n + page - 1) / page;
      const int T = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
      std::vector<std::thread> ts;
      for (int t = 0; t < T; ++t)
        ts.emplace_back([&, t] {
          for (size_t i = pages * t / T; i < pages * (t + 1) / T; ++i) static_cast<volatile char*>(p)[i * page] = 0;
        });
      for (auto& th : ts) th.join();
      if (cudaHostRegister(p, n, cudaHostRegisterPortable) == cudaSuccess) {
        ptr = p;
        registered = true;
        return;
      }
      cudaGetLastError();
      munmap(p, n);
    }
    PS_CUDA(cudaHostAlloc(&ptr, n, cudaHostAllocPortable));
  }
  void release() {
    if (!ptr) return;
    if (registered) {
      cudaHostUnregister(ptr);
      munmap(ptr, bytes);
    } else {
      cudaFreeHost(ptr);
    }
    ptr = nullptr;
  }
};

struct LayerDev {  // per-layer device outputs kept for the step
  float* weights;  // [B,E]
  int32_t* ids;    // [B,k]
};

// Host expert lane (Resource::Cpu, simulator.cpp:139-146; R5): one driver thread runs a
// layer's cpu_set sequentially on the lane's pool (the driver is pool worker 0) while
// the engine thread keeps issuing the layer's PCIe loads and GPU FFNs. The engine
// submits after the scheduling point and waits before the layer's combine.
struct CpuJob {
  int layer, expert, m, row0;
  const uint16_t* slab;
  const uint8_t* z = nullptr;   // z-slab of the expert (lane reads 1.5 B/weight), null = raw
  double t0_us = 0, t1_us = 0;  // host clock, filled by the driver
};

// The lane reads the z-slabs (1.41 instead of 2 B of host DRAM per weight, 3- or 4-bit
// codes) when every slab of its batch has one: in the engine the lane shares host DRAM
// with the PCIe DMA of the loads, so the 30 % fewer bytes win over the decode cost —
// 96-100 vs 70-87 tok/s, lane 208-234 vs 153-180 GB/s of bf16 weights in alternating
// runs (profiles/r02_bench_lane_z_ab.jsonl). (Round 1 measured no gain only because a
// 3-bit slab disabled the z path for its whole batch.) PS_HOST_LANE_Z=0 opts out.
bool lane_tiles_enabled() {  // PS_HOST_LANE_TILED=0 keeps the row-major host slabs
  static const bool on = [] {
    const char* v = std::getenv("PS_HOST_LANE_TILED");
    return !(v && v[0] == '0');
  }();
  return on;
}

bool lane_z_enabled() {  // PS_HOST_LANE_Z=0 keeps the lane on raw bf16 slabs
  static const bool on = [] {
    const char* v = std::getenv("PS_HOST_LANE_Z");
    return !(v && v[0] == '0');
  }();
  return on;
}

class LaneDriver {
 public:
  LaneDriver(ps_host_lane lane, int H, int F) : lane_(lane), H_(H), F_(F), thread_([this] { loop(); }) {}
  std::atomic<bool> tiled{false};  // raw host slabs are in the lane's tile layout (set before any submit)
  ~LaneDriver() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    thread_.join();
  }
  // xrows / yrows: [rows, H] bf16 / f32, job j reads/writes rows [row0, row0 + m).
  void submit(std::vector<CpuJob>* jobs, const uint16_t* xrows, float* yrows) {
    std::lock_guard<std::mutex> g(mu_);
    jobs_ = jobs;
    x_ = xrows;
    y_ = yrows;
    done_ = false;
    cv_.notify_all();
  }
  // Blocks until no batch is running, dropping any error (used at step entry so a step
  // that failed mid-layer cannot leave the driver reading the next step's job list).
  void drain() {
    std::unique_lock<std::mutex> g(mu_);
    cv_.wait(g, [&] { return done_; });
    err_.clear();
  }
  void wait() {
    std::unique_lock<std::mutex> g(mu_);
    cv_.wait(g, [&] { return done_; });
    if (!err_.empty()) {
      std::string m = err_;
      err_.clear();
      fail(PS_ERUNTIME, "host lane: " + m);
    }
  }

 private:
  void loop() {
    ps_host_lane_bind_caller(lane_);  // the driver is the lane pool's worker 0
    std::unique_lock<std::mutex> g(mu_);
    while (true) {
      cv_.wait(g, [&] { return stop_ || jobs_ != nullptr; });
      if (stop_) return;
      std::vector<CpuJob>* jobs = jobs_;
      g.unlock();
      // One batch call per layer (both pool passes span all experts of the set); every
      // expert of the set is reported with the batch's interval.
      std::string err;
      slabs_.clear();
      zs_.clear();
      m_.clear();
      row0_.clear();
      bool all_z = lane_z_enabled() && ps_host_lane_reads_z(lane_);
      for (const CpuJob& j : *jobs) {
        slabs_.push_back(j.slab);
        zs_.push_back(j.z);
        all_z = all_z && j.z;
        m_.push_back(j.m);
        row0_.push_back(j.row0);
      }
      const double t0 = now_us();
      const int n = static_cast<int>(jobs->size());
      const ps_status st = all_z ? ps_host_expert_ffn_batch_z(lane_, n, zs_.data(), m_.data(), row0_.data(), H_, F_,
                                                              x_, y_)
                                 : (tiled.load() ? ps_host_expert_ffn_batch_tiled : ps_host_expert_ffn_batch)(
                                       lane_, n, slabs_.data(), m_.data(), row0_.data(), H_, F_, x_, y_);
      if (st != PS_OK) err = ps_last_error();
      const double t1 = now_us();
      for (CpuJob& j : *jobs) {
        j.t0_us = t0;
        j.t1_us = t1;
      }
      g.lock();
      jobs_ = nullptr;
      err_ = err;
      done_ = true;
      cv_.notify_all();
    }
  }
  ps_host_lane lane_;
  int H_, F_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<CpuJob>* jobs_ = nullptr;
  const uint16_t* x_ = nullptr;
  float* y_ = nullptr;
  bool stop_ = false, done_ = true;
  std::string err_;
  std::vector<const uint16_t*> slabs_;
  std::vector<const uint8_t*> zs_;
  std::vector<int32_t> m_, row0_;
  std::thread thread_;  // last: starts after the members it uses
};

struct FfnTiming {
  cudaEvent_t a, b;
  double bytes;
  int layer;
  std::vector<int> experts, tokens;  // routed experts of the launch (timeline export)
};

struct StallProbe {
  cudaEvent_t before, after;
};

struct PhaseTiming {  // scheduling-point phase (K1+K4+K2+D2H) and combine, per layer
  cudaEvent_t route0, route1, comb0, comb1;
};

}  // namespace
}  // namespace ps

struct ps_engine_s {
  ps_engine_config cfg{};
  int L = 0, E = 0, K = 0, H = 0, F = 0, maxB = 0, n_split = 1, step_split = 1;
  // Shared experts (cfg.n_shared): virtual experts E..E+S-1 of every token; Et/Kt are the
  // expert count / assignments per token that K2, K3 and the combine see.
  int S = 0, Et = 0, Kt = 0;
  void* shared_arena = nullptr;               // [L*S] slabs, HBM, outside the routed budget
  std::vector<const uint16_t*> shared_slab;   // [L*S]
  int32_t* ids_ext = nullptr;                 // [maxB, Kt]
  float* w_ext = nullptr;                     // [maxB, Et]

  // host expert lane (cfg.host_threads > 0)
  ps_host_lane lane = nullptr;
  std::unique_ptr<ps::LaneDriver> lane_drv;
  uint16_t* lane_x = nullptr;    // pinned: [maxB, H] bf16 x (D2H at the scheduling point)
  uint16_t* lane_recv = nullptr;   // pinned (EP): [rows_max, H] bf16 rows received by this rank
  cudaEvent_t ev_lane_rows = nullptr;  // (EP) received rows are on the host
  uint16_t* lane_xrows = nullptr;  // pinned: [maxB*Kt, H] bf16 gathered rows of CPU experts
  float* lane_yrows = nullptr;     // pinned: [maxB*Kt, H] f32 their outputs
  std::vector<ps::CpuJob> cpu_jobs;      // current layer
  std::vector<ps::CpuJob> cpu_done;      // this step (timeline)
  double cpu_ms_cal = 0, cpu_tokens_cal = 0;  // calibration samples
  std::vector<int32_t> probe_m;               // create-time lane probe (tokens, us)
  std::vector<int64_t> probe_us;
  int last_fit_used = 0;                      // last calibrate used fit_cost_params
  std::vector<int32_t> cal_m;
  std::vector<int64_t> cal_us;
  uint64_t slab_elems = 0;
  cudaStream_t sc = nullptr;  // compute stream
  cudaStream_t s_d2h = nullptr;  // scheduling-point D2H (off the compute stream's critical path)
  cudaStream_t s_pred[2] = {nullptr, nullptr};  // K4 for l+1 / l+2 (off the compute stream)
  cudaEvent_t ev_k1 = nullptr, ev_pred[2] = {nullptr, nullptr};
  void* llapor_scratch2 = nullptr;
  cudaEvent_t last_ffn_end = nullptr;  // end event of the last FFN enqueued (reused as a start mark)
  std::unique_ptr<ps::IoChannel> io;

  // expert placement
  std::vector<const uint16_t*> dev_slab;  // [L*E] resident pointer or null
  std::vector<const uint16_t*> host_slab; // [L*E] pinned host pointer or null
  std::vector<uint8_t> resident;          // [L*E]
  std::vector<uint8_t> has_host;          // [L]: layer has an owned non-resident expert
  size_t host_slab_count = 0;             // owned non-resident experts (0 = fully resident)
  int pred_kind = PS_PRED_NONE;           // resolved ps_predictor_kind
  std::vector<int32_t> stats_rank;        // [L*E] PS_PRED_STATS ranking
  std::vector<int32_t> last_pred;         // [L*E] predictions of the last step
  int32_t* pp_ids = nullptr;              // PS_PRED_PERFECT scratch: [maxB, k] ids
  float* pp_w = nullptr;                  //                          [maxB, E] weights
  void* arena = nullptr;                  // resident HBM arena
  void* host_arena = nullptr;             // pinned host arena
  ps::PinnedArena host_pin, z_pin;        // their allocations (THP + register, or cudaHostAlloc)
  // z-slabs (cfg.compress_host): lossless ~12-bit copies of the host slabs that PCIe
  // carries instead (decoded on the GPU); the raw arena stays for the host lane.
  void* z_arena = nullptr;
  size_t z_cap = 0;                        // bytes per z-slab slot
  std::vector<const uint8_t*> host_z;      // [L*E] or empty
  std::vector<uint64_t> host_z_bytes;      // [L*E]
  bool host_tiled = false;                 // host_slab in the lane's tile layout (lane-only; PCIe reads host_z)
  bool zfuse = false;                      // PS_ZFUSE=1: landed z-slabs feed K3 directly (ps_expert_ffn_zslab)
  ps::Slot od_slot[2];
  std::vector<std::unique_ptr<ps::Slot>> pf_pool;

  // router
  float* gate = nullptr;   // [L,E,H]
  float* bias = nullptr;   // [L,E]

  // step buffers
  std::vector<ps::LayerDev> layer;
  int32_t* counts_dev = nullptr;     // [Et]
  int32_t* pred_dev = nullptr;       // [E] predicted tokens per expert of layer l+1
  int32_t* pred2_dev = nullptr;      // [E] ... of layer l+2 (e_next2, lookahead)
  // Scheduling-point block, one device allocation mirrored in pinned host memory so the
  // per-layer D2H is ONE copy: counts [Et] | pred [Et] | pred2 [Et] | offsets [Et+1] |
  // perm_src [maxB*Kt]
  int32_t* sched_dev = nullptr;
  int32_t* route_ws = nullptr;       // ticket counter of the fused route+permute launch
  // Decode scheduling point as a CUDA graph per (layer, B, variant): K1 (+ fused K2 index
  // pass) and the two K4 predictions on their forked side streams, replayed from staged
  // inputs (x_stage / fol_stage) — one launch instead of ~13 stream operations.
  float* x_stage = nullptr;
  uint8_t* fol_stage = nullptr;
  std::map<std::tuple<int, int, int, uint64_t>, cudaGraphExec_t> sched_graphs;
  bool use_graphs = true;
  int32_t* pinned_counts = nullptr;  // host mirror of sched_dev
  uint16_t* x_bf16 = nullptr;
  uint16_t* x_perm = nullptr;        // [maxB*k, H] bf16 (prefill gather)
  bool prefill_mode = false;         // B > kDecodeMaxBatch: tcgen05 path, exact-count launches
  int32_t *offsets = nullptr, *perm_src = nullptr, *inv = nullptr;
  uint16_t* hbuf = nullptr;
  float* y_part = nullptr;
  void* llapor_scratch = nullptr;
  float* in_hidden = nullptr;   // device staging for the host-buffer entry point
  uint8_t* in_follow = nullptr;
  float* out_y = nullptr;
  int32_t* out_ids = nullptr;
  cudaEvent_t ev_routed = nullptr, ev_step0 = nullptr, ev_step1 = nullptr;

  // Where the FFN of the current layer reads its rows from (set per layer): the local
  // routing (x_bf16 with k slots per token) or, under EP, the rows received from all
  // ranks (k = 1). Offsets are indexed by GLOBAL expert id (zero-length for experts
  // this rank does not own).
  struct FfnSrc {
    const int32_t* offsets_dev;
    const int32_t* perm_dev;
    int k;
    const uint16_t* x;
    int rows;
    const int32_t* offsets_host;  // prefill tile scheduling
  } src{};
  int rows_max = 0;  // capacity of the per-row FFN buffers (G * maxB * k under EP)

  // expert parallelism
  ps_ep_comm ep = nullptr;
  int G = 1, rank = 0, E_loc = 0;
  int32_t* ep_vids = nullptr;      // [maxB*k] owner-major virtual ids
  int32_t* ep_off_v = nullptr;     // [G*E_loc+1]
  int32_t* ep_perm_v = nullptr;    // [maxB*k]
  int32_t* ep_inv_v = nullptr;     // [maxB*k]
  uint16_t* ep_send_x = nullptr;   // [maxB*k, H]
  uint16_t* ep_recv_x = nullptr;   // [G*maxB*k, H]
  float* ep_y_recv = nullptr;      // [G*maxB*k, H]
  float* ep_y_back = nullptr;      // [maxB*k, H]
  int32_t* ep_cnt_send = nullptr;  // [G][2*E_loc]
  int32_t* ep_cnt_recv = nullptr;  // [G][2*E_loc]
  int32_t* ep_plan_dev = nullptr;  // [E+1 | rows | rows]: offsets_glob, perm_loc, inv_loc
  int32_t* ep_plan_host = nullptr; // pinned staging of the same
  int32_t* ep_host = nullptr;      // pinned [G*E_loc+1 | G*2*E_loc]: own offsets_v, recv counts
  float* ep_ones = nullptr;        // [rows_max] combine weights for the unpermute
  int32_t* ep_zeros = nullptr;     // [rows_max]
  std::vector<int32_t> ep_seg, ep_send_rows;  // per-layer receive segments / send rows
  int ep_rows_recv = 0;

  // step in progress (step_begin / layer_forward / step_end)
  bool in_step = false;
  int step_B = 0, next_layer = 0;
  double host_t0_us = 0;
  std::vector<ps_expert_load> cur, nxt, nxt2, cpu_b, od_b, pf_b;  // per-layer scheduler scratch
  std::vector<int32_t> counts_l, pred_l, pred2_l;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;  // caller stream <-> compute stream (per-layer ABI)

  // measured timeline of the last step (row f2 of SURVEY.md §8f)
  int cur_layer = 0;
  std::vector<int32_t> step_truth;             // [L*E] routed tokens per (layer, expert)
  std::vector<ps_timeline_event> last_events;
  std::vector<int64_t> last_layer_start, last_layer_end;
  std::vector<int32_t> last_truth;
  double copy_ms_total = 0, copies = 0, route_ms_total_cal = 0, ffn_expert_ms_total = 0, ffn_experts = 0;

  // scheduler state across layers
  ps_hit_stats stats[3];
  std::vector<std::unique_ptr<ps::IoJob>> jobs;  // owned for the step
  struct Ready { int layer, expert; ps::Slot* slot; ps::IoJob* job; };
  std::vector<Ready> ready;                       // committed prefetches
  std::vector<ps::IoJob*> pending_pf;             // issued/queued prefetches of the previous layer
  struct HitCheck { int layer, expert, group; };
  std::vector<HitCheck> hit_checks;
  double io_free_us = 0.0;
  // Two event pools: compute-stream probes (recorded by this thread) and copy events
  // (recorded only by the I/O thread), so a recycled event is never recorded by one
  // thread while the other still waits on its previous record.
  std::vector<cudaEvent_t> event_pool, job_event_pool;
  size_t event_next = 0, job_event_next = 0;
  std::vector<ps::FfnTiming> ffn_t;
  std::vector<ps::StallProbe> stall_t;
  std::vector<ps::PhaseTiming> phase_t;
  ps_engine_stats st{};
};

namespace ps {
namespace {

cudaEvent_t take_event(ps_engine_s& e) {
  if (e.event_next == e.event_pool.size()) {
    cudaEvent_t ev;
    PS_CUDA(cudaEventCreate(&ev));
    e.event_pool.push_back(ev);
  }
  return e.event_pool[e.event_next++];
}

cudaEvent_t take_job_event(ps_engine_s& e) {
  if (e.job_event_next == e.job_event_pool.size()) {
    cudaEvent_t ev;
    // The I/O thread waits milliseconds on these (one expert copy): blocking sync, so it
    // sleeps instead of spinning on a core the host expert lane could use.
    PS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventBlockingSync));
    e.job_event_pool.push_back(ev);
  }
  return e.job_event_pool[e.job_event_next++];
}

int group_of_layer(const ps_model_spec& s, int l) {
  return l < s.group_begin_middle ? PS_GROUP_INPUT : l < s.group_begin_output ? PS_GROUP_MIDDLE : PS_GROUP_OUTPUT;
}

// Timing events with timestamps serialise the stream front end (~3 us per record between
// two kernels on B200, scripts/engine_timeline.py): callers pass the event that already
// marks the launch point (`start`) instead of recording a new one, and the last FFN's end
// event is reused as the combine's start.
void ffn(ps_engine_s& e, const ps_expert_group& g, const int32_t* counts_host, int B, bool timed,
         bool exact_counts = true, cudaEvent_t start = nullptr, const void* const* zslabs = nullptr) {
  if (g.n == 0) return;
  cudaEvent_t a = nullptr, b = nullptr;
  if (timed) {
    a = start;
    if (!a) {
      a = take_event(e);
      PS_CUDA(cudaEventRecord(a, e.sc));
    }
  }
  // Path choice per launch: the tcgen05 grouped GEMM once an expert has a full 128-row
  // M tile of tokens (prefill), the HBM-streaming GEMV otherwise (decode).
  int max_m = 0;
  double rows = 0;
  for (int i = 0; i < g.n; ++i) {
    max_m = std::max(max_m, counts_host[g.experts[i]]);
    rows += counts_host[g.experts[i]];
  }
  ps_status s;
  (void)B;
  const auto& src = e.src;
  if (e.prefill_mode && !exact_counts && e.H % 256 == 0 && e.F % 128 == 0) {
    // early resident-group launch of a prefill chunk: the tile schedule is built on the
    // device from K2's offsets (no host round trip before the FFN)
    s = ps_expert_ffn_prefill_dev(&g, src.offsets_dev, e.x_perm, src.rows, e.H, e.F, e.hbuf, e.y_part, e.sc);
    e.st.tc_launches += 1;
    e.st.ffn_launches += 1;
    e.st.kernel_launches += 2;  // schedule + FFN
  } else if (e.prefill_mode && max_m >= 128 && e.H % 256 == 0 && e.F % 128 == 0) {
    s = ps_expert_ffn_prefill(&g, counts_host, src.offsets_host, e.x_perm, src.rows, e.H, e.F, e.hbuf, e.y_part,
                              e.sc);
    const int n_launch = prefill_launches_per_call();  // gate_up + down: one launch (token-N) or two
    e.st.tc_launches += n_launch;
    e.st.ffn_launches += n_launch;
    e.st.kernel_launches += n_launch;
  } else if (zslabs) {  // landed z-slabs decoded inside K3 (<= 8 tokens per expert)
    s = ps_expert_ffn_zslab(&g, zslabs, counts_host, src.offsets_dev, src.perm_dev, src.k, src.x, e.H, e.F, e.hbuf,
                            e.y_part, e.step_split, src.rows, e.sc);
    e.st.ffn_launches += 1;
    e.st.kernel_launches += 1;
  } else {
    s = ps_expert_ffn(&g, counts_host, src.offsets_dev, src.perm_dev, src.k, src.x, e.H, e.F, e.hbuf, e.y_part,
                      e.step_split, src.rows, e.sc);
    // One persistent kernel per pass of <= 64 tokens per expert and <= 64 experts.
    int launches = 0;
    for (int base = 0; base < max_m; base += 64) {
      int n = 0;
      for (int i = 0; i < g.n; ++i) n += counts_host[g.experts[i]] > base;
      launches += (n + 63) / 64;
    }
    e.st.ffn_launches += launches;
    e.st.kernel_launches += launches;
  }
  if (s != PS_OK) fail(s, ps_last_error());
  if (exact_counts) e.st.ffn_flops_total += 6.0 * rows * e.H * e.F;
  if (timed) {
    b = take_event(e);
    PS_CUDA(cudaEventRecord(b, e.sc));
    e.last_ffn_end = b;
    FfnTiming t{a, b, 0.0, e.cur_layer, {}, {}};
    for (int i = 0; i < g.n; ++i)
      if (counts_host[g.experts[i]] > 0) {
        t.bytes += static_cast<double>(e.cfg.spec.expert_bytes);
        t.experts.push_back(g.experts[i]);
        t.tokens.push_back(counts_host[g.experts[i]]);
      }
    e.ffn_t.push_back(std::move(t));
  }
}

Slot* take_prefetch_slot(ps_engine_s& e, int target) {
  int used = 0;
  for (auto& s : e.pf_pool) used += s->in_use && s->target_layer == target;
  if (used >= e.cfg.prefetch_slots) fail(PS_ERUNTIME, "engine: prefetch buffer overflow for layer " + std::to_string(target));
  for (auto& s : e.pf_pool)
    if (!s->in_use) {
      s->in_use = true;
      s->target_layer = target;
      return s.get();
    }
  auto s = std::make_unique<Slot>();
  PS_CUDA(cudaMalloc(&s->dev, e.cfg.spec.expert_bytes));
  if (e.z_cap) PS_CUDA(cudaMalloc(&s->zdev, e.z_cap));
  PS_CUDA(cudaEventCreateWithFlags(&s->free_ev, cudaEventDisableTiming));
  s->in_use = true;
  s->target_layer = target;
  e.pf_pool.push_back(std::move(s));
  return e.pf_pool.back().get();
}

// Marks slot reusable after all compute-stream work enqueued so far.
void release_slot_after_compute(ps_engine_s& e, Slot* s) {
  PS_CUDA(cudaEventRecord(s->free_ev, e.sc));
  s->next_gen += 1;
  s->recorded_gen.store(s->next_gen);
  e.io->notify();
}

IoJob* new_job(ps_engine_s& e, int kind, int layer, int expert, int tokens, Slot* slot) {
  auto j = std::make_unique<IoJob>();
  j->kind = kind;
  j->layer = layer;
  j->expert = expert;
  j->tokens = tokens;
  j->slot = slot;
  const size_t idx = static_cast<size_t>(layer) * e.E + expert;
  j->dst = slot->dev;
  j->src = e.host_slab[idx];
  if (!j->src) fail(PS_ERUNTIME, "engine: expert has no host copy");
  j->bytes = e.cfg.spec.expert_bytes;
  if (!e.host_z.empty() && e.host_z[idx]) {  // z-slab: PCIe moves ~75 %, decoded on the GPU
    j->zhost = e.host_z[idx];
    j->src = e.host_z[idx];
    j->dst = slot->zdev;
    j->bytes = e.host_z_bytes[idx];
  }
  j->wait_gen = slot->next_gen;  // the slot's latest reader must be done
  j->t_io_us = static_cast<double>(e.cfg.cost.t_io);
  j->start_ev = take_job_event(e);
  j->done_ev = take_job_event(e);
  e.jobs.push_back(std::move(j));
  return e.jobs.back().get();
}

// Make a landed copy usable by the FFN: after the copy event, decode a z-slab into the
// slot's bf16 buffer (no-op for raw copies). Compute stream.
// fused: the FFN reads the landed z-slab itself (ps_expert_ffn_zslab), no decode here.
// Only 4-bit-code slabs: with 3-bit codes (~3 % escapes) the in-register patching makes the
// fused kernel slower than z_decode + K3 (profiles/README.md).
bool fuse_z(const ps_engine_s& e, const IoJob* j, int tokens) {
  return e.zfuse && j->zhost && tokens <= 8 && reinterpret_cast<const ZHeader*>(j->zhost)->code_bits == 4;
}

void land(ps_engine_s& e, IoJob* j, bool fused = false) {
  PS_CUDA(cudaStreamWaitEvent(e.sc, j->done_ev, 0));
  if (j->zhost && !fused) {
    if (ps_zslab_decode(static_cast<const uint8_t*>(j->dst), j->zhost, static_cast<uint16_t*>(j->slot->dev), e.sc) !=
        PS_OK)
      fail(PS_ECUDA, ps_last_error());
    e.st.kernel_launches += 1;
    e.st.z_decodes += 1;
  }
}

// Host-DRAM bytes the lane reads for one expert: its z-slab when the lane takes the z
// path (every host slab has one and this host can decode them), else the raw slab.
double lane_read_bytes(const ps_engine_s& e, const CpuJob& j) {
  if (j.z && lane_z_enabled() && ps_host_lane_reads_z(e.lane))
    return static_cast<double>(reinterpret_cast<const ZHeader*>(j.z)->bytes);
  return static_cast<double>(e.cfg.spec.expert_bytes);
}

double push_modelled(ps_engine_s& e) {  // channel busy-until model for alpha (R4)
  const double now = now_us();
  e.io_free_us = std::max(e.io_free_us, now) + static_cast<double>(e.cfg.cost.t_io);
  return e.io_free_us;
}

// EP dispatch, part 2 (after the counts exchange landed on the host): the receive plan
// (local expert-major order over the received rows), the per-layer counts the loader
// schedules with, and the row payload all-to-all.

void ep_dispatch_rows(ps_engine_s& e, int B, std::vector<int32_t>& counts_l, std::vector<int32_t>& pred_l) {
  const int G = e.G, El = e.E_loc, Ev = G * El, E = e.E, H = e.H;
  const int32_t* off_v = e.ep_host;
  const int32_t* rc = e.ep_host + Ev + 1;
  std::vector<int32_t> rcnt(static_cast<size_t>(G) * El), off_loc(El + 1);
  e.ep_seg.assign(G + 1, 0);
  for (int s = 0; s < G; ++s)
    for (int j = 0; j < El; ++j) rcnt[s * El + j] = rc[s * 2 * El + j];
  int32_t* og = e.ep_plan_host;
  int32_t* perm = og + (E + 1);
  int32_t* inv = perm + e.rows_max;
  ps_status st = ps_ep_recv_plan(rcnt.data(), G, El, off_loc.data(), nullptr, e.ep_seg.data());
  if (st != PS_OK) fail(st, ps_last_error());
  const int rows = e.ep_seg[G];
  require(rows <= e.rows_max, "EP: received rows exceed capacity");
  st = ps_ep_recv_plan(rcnt.data(), G, El, off_loc.data(), perm, e.ep_seg.data());
  if (st != PS_OK) fail(st, ps_last_error());
  for (int r = 0; r < rows; ++r) inv[perm[r]] = r;
  int running = 0;
  for (int ex = 0; ex < E; ++ex) {
    og[ex] = running;
    counts_l[ex] = pred_l[ex] = 0;
    if (ex % G != e.rank) continue;
    const int j = ex / G;
    counts_l[ex] = off_loc[j + 1] - off_loc[j];
    for (int s = 0; s < G; ++s) pred_l[ex] += rc[s * 2 * El + El + j];
    running += counts_l[ex];
  }
  og[E] = running;
  PS_CUDA(cudaMemcpyAsync(e.ep_plan_dev, e.ep_plan_host, sizeof(int32_t) * (E + 1 + 2 * static_cast<size_t>(e.rows_max)),
                          cudaMemcpyHostToDevice, e.sc));
  std::vector<uint64_t> sb(G), rb(G);
  e.ep_send_rows.assign(G, 0);
  for (int d = 0; d < G; ++d) {
    e.ep_send_rows[d] = off_v[(d + 1) * El] - off_v[d * El];
    sb[d] = static_cast<uint64_t>(e.ep_send_rows[d]) * H * sizeof(uint16_t);
    rb[d] = static_cast<uint64_t>(e.ep_seg[d + 1] - e.ep_seg[d]) * H * sizeof(uint16_t);
  }
  st = ps_ep_all_to_all(e.ep, e.ep_send_x, sb.data(), e.ep_recv_x, rb.data(), e.sc);
  if (st != PS_OK) fail(st, ps_last_error());
  if (e.lane && rows > 0) {  // the host lane computes its cpu_set from the received rows
    PS_CUDA(cudaMemcpyAsync(e.lane_recv, e.ep_recv_x, sizeof(uint16_t) * rows * H, cudaMemcpyDeviceToHost, e.sc));
    PS_CUDA(cudaEventRecord(e.ev_lane_rows, e.sc));
  }
  e.ep_rows_recv = rows;
  const int32_t* plan = e.ep_plan_dev;
  e.src = {plan, plan + (E + 1), 1, e.ep_recv_x, rows, og};
  if (e.prefill_mode && rows > 0) {
    st = ps_gather_rows(e.ep_recv_x, plan + (E + 1), rows, 1, H, e.x_perm, e.sc);
    if (st != PS_OK) fail(st, ps_last_error());
    e.st.kernel_launches += 1;
  }
  (void)B;
}

// EP combine: per-row outputs back to receive order, all-to-all back to the token
// owners, weighted sum at home.
ps_status ep_combine_rows(ps_engine_s& e, int B, const LayerDev& ld, float* y_l) {
  const int G = e.G, H = e.H, E = e.E, K = e.K;
  const int rows = e.ep_rows_recv;
  ps_status st = PS_OK;
  if (rows > 0)
    st = ps_combine(e.y_part, e.step_split, e.ep_plan_dev + (E + 1) + e.rows_max, e.ep_zeros, e.ep_ones, rows, 1, 1, H,
                    e.ep_y_recv, e.sc);
  if (st != PS_OK) return st;
  std::vector<uint64_t> sb(G), rb(G);
  for (int p = 0; p < G; ++p) {
    sb[p] = static_cast<uint64_t>(e.ep_seg[p + 1] - e.ep_seg[p]) * H * sizeof(float);
    rb[p] = static_cast<uint64_t>(e.ep_send_rows[p]) * H * sizeof(float);
  }
  st = ps_ep_all_to_all(e.ep, e.ep_y_recv, sb.data(), e.ep_y_back, rb.data(), e.sc);
  if (st != PS_OK) return st;
  e.st.kernel_launches += 2;
  return ps_combine(e.ep_y_back, 1, e.ep_inv_v, ld.ids, ld.weights, B, K, E, H, y_l, e.sc);
}

// routed_ids / routed_w (nullable, device, [L,B,k] / [L,B,E]): the routing is given (a
// reference trace's gating truth) and replaces K1; everything downstream is unchanged.
// NVTX ranges (header-only nvtx3; no-ops unless a profiler is attached): the step and,
// per layer, the scheduling point, the host plan, the loads and the combine.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Step prologue (R1-R3 state of a new pass): settles anything a failed step left behind,
// resets the per-step bookkeeping and marks the step start on the compute stream.
void step_begin(ps_engine_s& e, int B) {
  require(B >= 1 && B <= e.maxB, "decode_step: batch out of range");
  const double t_head0 = now_us();
  e.step_B = B;
  e.prefill_mode = B > kDecodeMaxBatch;
  // A step that threw mid-layer may have left jobs queued / a lane batch running: settle
  // both before this step recycles the job list (no-ops after a normal step).
  e.io->abandon_queued();
  e.io->drain();
  for (auto& sl : e.pf_pool) sl->in_use = false;
  // Down-projection split-K of the decode GEMV (more CTAs for single-expert on-demand
  // launches); the tcgen05 prefill path writes one split, so prefill steps use 1.
  e.step_split = e.prefill_mode ? 1 : e.n_split;
  e.jobs.clear();
  e.event_next = 0;
  e.job_event_next = 0;
  e.ffn_t.clear();
  e.stall_t.clear();
  e.phase_t.clear();
  e.ready.clear();
  e.pending_pf.clear();
  PS_CUDA(cudaEventRecord(e.ev_step0, e.sc));
  e.host_t0_us = now_us();
  e.cpu_done.clear();
  if (e.lane_drv) e.lane_drv->drain();
  e.cpu_b.assign(e.E, {});
  e.od_b.assign(e.E, {});
  e.pf_b.assign(e.E, {});
  e.counts_l.assign(e.Et, 0);
  e.pred_l.assign(e.E, 0);
  e.pred2_l.assign(e.E, 0);
  e.step_truth.assign(static_cast<size_t>(e.L) * e.E, 0);
  e.last_pred.assign(static_cast<size_t>(e.L) * e.E, 0);
  e.next_layer = 0;
  e.in_step = true;
  e.st.host_head_ms_total += (now_us() - t_head0) / 1e3;
}

// One MoE layer of the current step (rules R1-R8 for layer l): x [B,H] f32 gating input
// (= FFN input), follow [B] u8 (nullable), y [B,H] f32 out. routed_ids / routed_w
// (nullable, [B,k] / [B,E]): the routing is given (a reference trace's gating truth) and
// replaces K1. x_next / follow_next: layer l+1's inputs (PS_PRED_PERFECT only).
// The host lane's output rows of e.cpu_jobs -> y_part (split 0; the other splits' rows
// zeroed), one launch for all of them.
void rows_to_device(ps_engine_s& e, size_t total_rows) {
  std::vector<int32_t> row0, m;
  for (const CpuJob& j : e.cpu_jobs) {
    row0.push_back(j.row0);
    m.push_back(j.m);
  }
  for (size_t i = 0; i < row0.size(); i += 128) {
    const int n = static_cast<int>(std::min<size_t>(128, row0.size() - i));
    const ps_status cs = ps_rows_from_host_ranges(e.lane_yrows, row0.data() + i, m.data() + i, n, e.H, e.y_part,
                                                  e.step_split - 1, static_cast<int64_t>(total_rows) * e.H, e.sc);
    if (cs != PS_OK) fail(cs, ps_last_error());
    e.st.kernel_launches += 1;
  }
}

void layer_forward(ps_engine_s& e, int l, const float* x, const uint8_t* follow, float* y_l,
                   const int32_t* routed_ids, const float* routed_w, const float* x_next, const uint8_t* follow_next) {
  const int L = e.L, E = e.E, K = e.K, H = e.H, B = e.step_B;
  require(e.in_step && l == e.next_layer, "layer_forward: layers must run in order 0..L-1 inside a step");
  e.next_layer = l + 1;
  std::vector<ps_expert_load>& cur = e.cur;
  std::vector<ps_expert_load>& nxt = e.nxt;
  std::vector<ps_expert_load>& cpu_b = e.cpu_b;
  std::vector<ps_expert_load>& od_b = e.od_b;
  std::vector<ps_expert_load>& pf_b = e.pf_b;
  const int Et = e.Et, Kt = e.Kt;
  std::vector<int32_t>& counts_l = e.counts_l;
  std::vector<int32_t>& pred_l = e.pred_l;
  const double host_t0_us = e.host_t0_us;
  {
    e.cur_layer = l;
    LayerDev& ld = e.layer[l];
    // Layer start: a fresh mark (the previous combine's end would also count the host's
    // inter-layer latency, which must not leak into the calibrated t_attn) — except on a
    // fully resident engine, where nothing is planned or calibrated from it and the
    // previous layer's combine end marks the same stream position one record earlier.
    const bool reuse_mark = l > 0 && e.host_slab_count == 0 && !e.ep;
    PhaseTiming ph{reuse_mark ? e.phase_t.back().comb1 : take_event(e), nullptr, nullptr, nullptr};
    if (!reuse_mark) PS_CUDA(cudaEventRecord(ph.route0, e.sc));
    e.last_ffn_end = nullptr;
    nvtxRangePushA("ps.layer.route");
    // --- K1 route (+fused bf16 cast) ------------------------------------------------
    // Decode without shared experts / EP: K1 and K2's index pass in one launch (the last
    // route CTA permutes). Otherwise K1 here and K2 below. Histogram: diff of K2 offsets.
    const bool fused_perm = !e.ep && e.S == 0 && !e.prefill_mode && !routed_ids;
    ps_status s = PS_OK;
    // --- K4 LLaPor: predicted histogram of layer l+1 -------------------------
    // Prefill chunks (B > 64 and >= 16 routed rows per expert on average) activate every
    // expert of the next layer with near certainty: the prediction is then the dense
    // histogram B*k/E per expert and the LLaPor launch is skipped (decode always runs it).
    // The prediction only feeds e_next (non-resident experts of l+1): a fully resident
    // next layer has no prefetch candidates whatever LLaPor says, so K4 is skipped there.
    const bool dense_next = e.prefill_mode && B * K >= 16 * E && l + 1 < L;
    const bool want_pred = l + 1 < L && !dense_next && e.has_host[l + 1];
    const bool predict = want_pred && (e.pred_kind == PS_PRED_LLAPOR || e.pred_kind == PS_PRED_PERFECT);
    // --- K4 for layer l+2: e_next2 of the widened window (simulator.cpp:128-131) and the
    // lookahead top-up. The reference predicts l+2 from the true layer-(l+1) features,
    // which do not exist yet at layer l: nets[l+2] is applied to layer-l features instead.
    const bool want_pred2 = !e.ep && l + 2 < L && !e.prefill_mode && e.has_host[l + 2];
    const bool predict2 = want_pred2 && e.pred_kind == PS_PRED_LLAPOR;
    // K1 (+ K2's index pass when fused) and the K4 predictions, on x / fol.
    auto sched_kernels = [&](const float* xk, const uint8_t* fk) {
      // --- K1 route (+fused bf16 cast) ----------------------------------------------
      // Decode without shared experts / EP: K1 and K2's index pass in one launch (the last
      // route CTA permutes). Otherwise K1 here and K2 below. Histogram: diff of K2 offsets.
      if (routed_ids) {
        PS_CUDA(cudaMemcpyAsync(ld.ids, routed_ids, sizeof(int32_t) * B * K, cudaMemcpyDeviceToDevice, e.sc));
        PS_CUDA(cudaMemcpyAsync(ld.weights, routed_w, sizeof(float) * B * E, cudaMemcpyDeviceToDevice, e.sc));
        s = ps_cast_bf16(xk, static_cast<int64_t>(B) * H, e.x_bf16, e.sc);
      } else if (fused_perm)
        s = ps_route_permute(xk, e.gate + static_cast<size_t>(l) * E * H, e.bias + static_cast<size_t>(l) * E,
                             fk, l > 0 ? e.layer[l - 1].ids : nullptr, K, B, H, E, K, ld.weights, ld.ids, e.x_bf16,
                             e.offsets, e.perm_src, e.inv, e.route_ws, e.sc);
      else
        s = ps_route_topk(xk, e.gate + static_cast<size_t>(l) * E * H, e.bias + static_cast<size_t>(l) * E,
                          fk, l > 0 ? e.layer[l - 1].ids : nullptr, K, B, H, E, K, nullptr, ld.weights, ld.ids, nullptr,
                          e.x_bf16, e.sc);
      if (s != PS_OK) fail(s, ps_last_error());
      // The two predictions run concurrently on two side streams forked after K1 and
      // joined back into Sc before K2 / the resident FFN. (Left unjoined they would queue
      // behind the persistent FFN kernel, which holds every SM, and delay the host's plan:
      // layer-start-to-lane-start 370 vs 220 us, profiles/timelines/r02_hybrid_k4_unjoined.json.)
      if (predict || predict2) PS_CUDA(cudaEventRecord(e.ev_k1, e.sc));
      if (predict && e.pred_kind == PS_PRED_LLAPOR) {
        PS_CUDA(cudaStreamWaitEvent(e.s_pred[0], e.ev_k1, 0));
        s = ps_llapor_forward(e.cfg.predictor, l + 1, xk, ld.ids, K, ld.weights, B, K, nullptr, nullptr, e.pred_dev,
                              e.llapor_scratch, e.s_pred[0]);
        if (s != PS_OK) fail(s, ps_last_error());
      } else if (predict) {  // PERFECT: layer l+1's true routing, K1 one layer early
        require(x_next != nullptr, "PS_PRED_PERFECT needs layer l+1's inputs (not available per layer)");
        PS_CUDA(cudaStreamWaitEvent(e.s_pred[0], e.ev_k1, 0));
        s = ps_route_topk(x_next, e.gate + static_cast<size_t>(l + 1) * E * H,
                          e.bias + static_cast<size_t>(l + 1) * E, follow_next, ld.ids, K, B, H, E, K, nullptr,
                          e.pp_w, e.pp_ids, e.pred_dev, nullptr, e.s_pred[0]);
        if (s != PS_OK) fail(s, ps_last_error());
      }
      if (predict) PS_CUDA(cudaEventRecord(e.ev_pred[0], e.s_pred[0]));
      if (predict2) {
        PS_CUDA(cudaStreamWaitEvent(e.s_pred[1], e.ev_k1, 0));
        s = ps_llapor_forward(e.cfg.predictor, l + 2, xk, ld.ids, K, ld.weights, B, K, nullptr, nullptr, e.pred2_dev,
                              e.llapor_scratch2, e.s_pred[1]);
        if (s != PS_OK) fail(s, ps_last_error());
        PS_CUDA(cudaEventRecord(e.ev_pred[1], e.s_pred[1]));
      }
      if (predict) PS_CUDA(cudaStreamWaitEvent(e.sc, e.ev_pred[0], 0));  // join
      if (predict2) PS_CUDA(cudaStreamWaitEvent(e.sc, e.ev_pred[1], 0));
      // --- K2 permute indices (non-EP; EP permutes owner-major below) ----------------
      // Prefill-sized batches gather x into contiguous permuted rows (TMA operand of the
      // tcgen05 path).
      if (!e.ep) {
        if (e.S) {
          s = ps_append_shared(ld.ids, ld.weights, B, K, E, e.S, e.ids_ext, e.w_ext, nullptr, e.sc);
          if (s != PS_OK) fail(s, ps_last_error());
        }
        if (!fused_perm) {
          s = ps_permute(e.S ? e.ids_ext : ld.ids, B, Kt, Et, e.offsets, e.perm_src, e.inv,
                         e.prefill_mode ? e.x_bf16 : nullptr, H, e.prefill_mode ? e.x_perm : nullptr, e.sc);
          if (s != PS_OK) fail(s, ps_last_error());
        }
      }
    };
    e.st.kernel_launches += 1 + (predict ? (e.pred_kind == PS_PRED_LLAPOR ? 2 : 1) : 0) + (predict2 ? 2 : 0) +
                            (!e.ep && e.S ? 1 : 0) + (!e.ep && !fused_perm ? (e.prefill_mode ? 2 : 1) : 0);
    // Graph replay: decode (fused or separate route + permute, shared experts) with the
    // LLaPor (or no) prediction; EP, prefill chunks and trace replay stay eager.
    const bool graph_ok = e.use_graphs && !e.ep && !e.prefill_mode && !routed_ids &&
                          !(predict && e.pred_kind == PS_PRED_PERFECT) && B <= e.maxB && e.x_stage;
    if (graph_ok) {
      if (predict) llapor_prepare(e.cfg.predictor, l + 1);  // device copies current before a capture/replay
      if (predict2) llapor_prepare(e.cfg.predictor, l + 2);
      PS_CUDA(cudaMemcpyAsync(e.x_stage, x, sizeof(float) * B * H, cudaMemcpyDeviceToDevice, e.sc));
      if (follow) PS_CUDA(cudaMemcpyAsync(e.fol_stage, follow, B, cudaMemcpyDeviceToDevice, e.sc));
      const int variant = (follow ? 1 : 0) | (predict ? 2 : 0) | (predict2 ? 4 : 0);
      const auto key = std::make_tuple(l, B, variant, (predict || predict2) ? llapor_generation(e.cfg.predictor) : 0);
      auto it = e.sched_graphs.find(key);
      if (it == e.sched_graphs.end()) {
        for (auto jt = e.sched_graphs.begin(); jt != e.sched_graphs.end();) {  // older predictor uploads
          if (std::get<0>(jt->first) == l && std::get<1>(jt->first) == B && std::get<2>(jt->first) == variant) {
            cudaGraphExecDestroy(jt->second);
            jt = e.sched_graphs.erase(jt);
          } else {
            ++jt;
          }
        }
        cudaGraph_t graph = nullptr;
        PS_CUDA(cudaStreamBeginCapture(e.sc, cudaStreamCaptureModeThreadLocal));
        try {
          sched_kernels(e.x_stage, follow ? e.fol_stage : nullptr);
        } catch (...) {
          cudaGraph_t dead = nullptr;
          cudaStreamEndCapture(e.sc, &dead);
          if (dead) cudaGraphDestroy(dead);
          throw;
        }
        PS_CUDA(cudaStreamEndCapture(e.sc, &graph));
        cudaGraphExec_t exec = nullptr;
        const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ie != cudaSuccess) fail(PS_ECUDA, std::string("scheduling-point graph: ") + cudaGetErrorString(ie));
        it = e.sched_graphs.emplace(key, exec).first;
      }
      PS_CUDA(cudaGraphLaunch(it->second, e.sc));
    } else {
      sched_kernels(x, follow);
    }
    // --- K2 permute indices ------------------------------------------------------
    // Prefill-sized batches gather x into contiguous permuted rows (TMA operand of the
    // tcgen05 path) and need the offsets on the host for tile scheduling.
    const int Ev = e.G * e.E_loc;  // owner-major virtual expert count under EP
    if (!e.ep) {
      // counts | pred | offsets (| perm_src for the host lane) in one copy, on the side
      // stream: the compute stream goes straight on to the resident FFN while the copy
      // engine brings the scheduling inputs to the host.
      const size_t n_sched = 4 * static_cast<size_t>(Et) + 1 + (e.lane ? static_cast<size_t>(B) * Kt : 0);
      ph.route1 = take_event(e);  // end of the scheduling-point kernels = start of the early FFN
      PS_CUDA(cudaEventRecord(ph.route1, e.sc));
      PS_CUDA(cudaStreamWaitEvent(e.s_d2h, ph.route1, 0));
      PS_CUDA(cudaMemcpyAsync(e.pinned_counts, e.sched_dev, sizeof(int32_t) * n_sched, cudaMemcpyDeviceToHost,
                              e.s_d2h));
      e.src = {e.offsets, e.perm_src, Kt, e.x_bf16, B * Kt, e.pinned_counts + 3 * Et};
      if (e.lane)  // the host lane gathers its rows from x
        PS_CUDA(cudaMemcpyAsync(e.lane_x, e.x_bf16, sizeof(uint16_t) * B * H, cudaMemcpyDeviceToHost, e.s_d2h));
      PS_CUDA(cudaEventRecord(e.ev_routed, e.s_d2h));
    } else {
      // EP dispatch, part 1: owner-major permute + gather of this rank's routed rows,
      // then the (rows, predicted tokens) counts exchange with every owner.
      s = ps_ep_remap_ids(ld.ids, B * K, E, e.G, e.ep_vids, e.sc);
      if (s == PS_OK)
        s = ps_permute(e.ep_vids, B, K, Ev, e.ep_off_v, e.ep_perm_v, e.ep_inv_v, e.x_bf16, H, e.ep_send_x, e.sc);
      if (s == PS_OK) s = ps_ep_pack_counts(e.ep_off_v, predict ? e.pred_dev : nullptr, E, e.G, e.ep_cnt_send, e.sc);
      if (s != PS_OK) fail(s, ps_last_error());
      e.st.kernel_launches += 4;
      std::vector<uint64_t> cb(e.G, sizeof(int32_t) * 2 * e.E_loc);
      s = ps_ep_all_to_all(e.ep, e.ep_cnt_send, cb.data(), e.ep_cnt_recv, cb.data(), e.sc);
      if (s != PS_OK) fail(s, ps_last_error());
      PS_CUDA(cudaMemcpyAsync(e.ep_host, e.ep_off_v, sizeof(int32_t) * (Ev + 1), cudaMemcpyDeviceToHost, e.sc));
      PS_CUDA(cudaMemcpyAsync(e.ep_host + Ev + 1, e.ep_cnt_recv, sizeof(int32_t) * e.G * 2 * e.E_loc,
                              cudaMemcpyDeviceToHost, e.sc));
    }
    if (e.ep) PS_CUDA(cudaEventRecord(e.ev_routed, e.sc));
    if (!ph.route1) {
      ph.route1 = take_event(e);
      PS_CUDA(cudaEventRecord(ph.route1, e.sc));
    }

    // --- resident experts (R6). Decode: start now, before the host knows the counts —
    // the kernels read per-expert row counts from the device offsets, the grid is sized
    // for the worst case m_e = B and warps of unrouted experts exit immediately.
    // Prefill: the same, the token-N kernel scheduling its tiles on the device.
    ps_expert_group grp{};
    std::vector<int32_t> worst(Et, B);
    for (int ex = 0; ex < E; ++ex)
      if (e.resident[static_cast<size_t>(l) * E + ex]) {
        grp.experts[grp.n] = ex;
        grp.slabs[grp.n] = e.dev_slab[static_cast<size_t>(l) * E + ex];
        ++grp.n;
      }
    for (int j = 0; j < e.S; ++j) {  // shared experts run with the resident group
      grp.experts[grp.n] = E + j;
      grp.slabs[grp.n] = e.shared_slab[static_cast<size_t>(l) * e.S + j];
      ++grp.n;
    }
    const size_t resident_timing = e.ffn_t.size();
    const bool early = !e.ep && (!e.prefill_mode || (e.H % 256 == 0 && e.F % 128 == 0));
    if (early) ffn(e, grp, worst.data(), B, true, false, ph.route1);

    // --- R2: resolve the previous layer's prefetch batch at this scheduling point
    {
      std::vector<IoJob*> cancelled = e.io->cancel_queued_prefetches();
      for (IoJob* j : cancelled) {
        j->slot->in_use = false;
        e.st.prefetches_cancelled++;
        e.io_free_us -= static_cast<double>(e.cfg.cost.t_io);
      }
      for (IoJob* j : e.pending_pf) {
        if (j->state.load() != 1) continue;
        e.ready.push_back({j->layer, j->expert, j->slot, j});
        e.st.prefetches_committed++;
        if (j->critical) e.hit_checks.push_back({j->layer, j->expert, j->issue_group});
      }
      e.pending_pf.clear();
    }

    nvtxRangePop();
    nvtxRangePushA("ps.layer.plan");
    // Wait for the routing result on the host (the only per-layer host sync).
    PS_CUDA(cudaEventSynchronize(e.ev_routed));
    if (!e.ep) {
      const int32_t* off_h = e.pinned_counts + 3 * Et;  // aggregate_layer_loads = diff of K2's offsets
      for (int ex = 0; ex < Et; ++ex) counts_l[ex] = off_h[ex + 1] - off_h[ex];
      if (predict) {
        std::memcpy(pred_l.data(), e.pinned_counts + Et, sizeof(int32_t) * E);
      } else if (want_pred && e.pred_kind == PS_PRED_GATE) {  // top-k of layer l's gate weights
        std::copy(counts_l.begin(), counts_l.begin() + E, pred_l.begin());
      } else if (want_pred && e.pred_kind == PS_PRED_STATS) {  // hot table's top-k of l+1, every token
        std::fill(pred_l.begin(), pred_l.end(), 0);
        for (int j = 0; j < K; ++j) pred_l[e.stats_rank[static_cast<size_t>(l + 1) * E + j]] = B;
      } else {
        std::fill(pred_l.begin(), pred_l.end(), dense_next ? (B * K) / E : 0);
      }
      std::fill(e.pred2_l.begin(), e.pred2_l.end(), 0);
      if (predict2) {
        std::memcpy(e.pred2_l.data(), e.pinned_counts + 2 * Et, sizeof(int32_t) * E);
      } else if (want_pred2 && e.pred_kind == PS_PRED_GATE) {
        std::copy(counts_l.begin(), counts_l.begin() + E, e.pred2_l.begin());
      } else if (want_pred2 && e.pred_kind == PS_PRED_STATS) {
        for (int j = 0; j < K; ++j) e.pred2_l[e.stats_rank[static_cast<size_t>(l + 2) * E + j]] = B;
      }
    } else {
      ep_dispatch_rows(e, B, counts_l, pred_l);
      std::fill(e.pred2_l.begin(), e.pred2_l.end(), 0);
    }
    if (!early) {
      ffn(e, grp, counts_l.data(), B, true, true);
    } else if (resident_timing < e.ffn_t.size()) {  // algorithmic bytes/flops: routed experts only
      FfnTiming& t = e.ffn_t[resident_timing];
      double rows = 0;
      t.bytes = 0;
      t.experts.clear();
      t.tokens.clear();
      for (int i = 0; i < grp.n; ++i) {
        const int m = counts_l[grp.experts[i]];
        if (m > 0) {
          t.bytes += static_cast<double>(e.cfg.spec.expert_bytes);
          t.experts.push_back(grp.experts[i]);
          t.tokens.push_back(m);
        }
        rows += m;
      }
      e.st.ffn_flops_total += 6.0 * rows * e.H * e.F;
    }
    std::copy(counts_l.begin(), counts_l.begin() + E, e.step_truth.begin() + static_cast<size_t>(l) * E);
    if (l + 1 < L) std::copy(pred_l.begin(), pred_l.end(), e.last_pred.begin() + static_cast<size_t>(l + 1) * E);
    for (int i = 0; i < grp.n; ++i) e.st.resident_hits += grp.experts[i] < E && counts_l[grp.experts[i]] > 0;

    // Deferred HitStats for critical prefetches that targeted this layer (R2).
    for (auto it = e.hit_checks.begin(); it != e.hit_checks.end();) {
      if (it->layer == l) {
        ps_hit_stats_record(&e.stats[it->group], counts_l[it->expert] > 0);
        e.st.prefetch_hits += counts_l[it->expert] > 0;
        it = e.hit_checks.erase(it);
      } else {
        ++it;
      }
    }

    // Prefetched experts of this layer (committed) compute once their copy lands.
    auto is_ready = [&](int layer, int ex) {
      for (auto& r : e.ready)
        if (r.layer == layer && r.expert == ex) return true;
      return false;
    };
    // With the host lane, a committed prefetch whose copy has not landed yet is deferred:
    // once the lane's batch is done it either lands (GPU) or, if its copy still needs more
    // than the lane's cost for it, the lane computes it instead (steal_late).
    std::vector<const ps_engine_s::Ready*> late;
    auto gpu_ready = [&](const ps_engine_s::Ready& r) {
      const bool fz = fuse_z(e, r.job, counts_l[r.expert]);
      land(e, r.job, fz);
      ps_expert_group one{};
      one.n = 1;
      one.experts[0] = r.expert;
      one.slabs[0] = static_cast<const uint16_t*>(r.slot->dev);
      const void* zp[1] = {r.job->dst};
      ffn(e, one, counts_l.data(), B, true, true, nullptr, fz ? zp : nullptr);
    };
    // Prefetches whose copies have already landed share ONE FFN launch (a single-expert
    // decode launch streams at ~65 % of HBM, a group at ~90 %); the others each wait for
    // their copy in their own launch (or, with steal_late, are deferred).
    // (landed ones first: a later wait on an in-flight copy would hold the group back)
    ps_expert_group landed{}, landed_z{};
    const void* landed_zp[PS_MAX_GROUP];
    std::vector<const ps_engine_s::Ready*> in_flight;
    for (auto& r : e.ready) {
      if (r.layer != l || counts_l[r.expert] == 0) continue;
      e.st.prefetches_used++;  // a committed prefetch its target layer routed tokens to
      if (cudaEventQuery(r.job->done_ev) == cudaSuccess && landed.n + landed_z.n < PS_MAX_GROUP) {
        const bool fz = fuse_z(e, r.job, counts_l[r.expert]);
        land(e, r.job, fz);
        ps_expert_group& g = fz ? landed_z : landed;
        if (fz) landed_zp[landed_z.n] = r.job->dst;
        g.experts[g.n] = r.expert;
        g.slabs[g.n] = static_cast<const uint16_t*>(r.slot->dev);
        ++g.n;
      } else {
        in_flight.push_back(&r);
      }
    }
    if (landed.n > 0) ffn(e, landed, counts_l.data(), B, true);
    if (landed_z.n > 0) ffn(e, landed_z, counts_l.data(), B, true, true, nullptr, landed_zp);
    for (const ps_engine_s::Ready* r : in_flight) {
      if (e.lane && e.cfg.steal_late) late.push_back(r);
      else gpu_ready(*r);
    }

    // --- R4: scheduler inputs ------------------------------------------------------
    cur.clear();
    nxt.clear();
    e.nxt2.clear();
    for (int ex = 0; ex < E; ++ex) {
      if (counts_l[ex] > 0 && !e.resident[static_cast<size_t>(l) * E + ex] && !is_ready(l, ex))
        cur.push_back({ex, l, counts_l[ex], PS_LOC_HOST});
      if (l + 1 < L && pred_l[ex] > 0 && !e.resident[static_cast<size_t>(l + 1) * E + ex] && !is_ready(l + 1, ex))
        nxt.push_back({ex, l + 1, pred_l[ex], PS_LOC_HOST});
      if (l + 2 < L && e.pred2_l[ex] > 0 && !e.resident[static_cast<size_t>(l + 2) * E + ex] && !is_ready(l + 2, ex))
        e.nxt2.push_back({ex, l + 2, e.pred2_l[ex], PS_LOC_HOST});
    }
    auto by_tokens = [](const ps_expert_load& a, const ps_expert_load& b) {
      return a.tokens != b.tokens ? a.tokens < b.tokens : a.expert < b.expert;
    };
    std::sort(cur.begin(), cur.end(), by_tokens);
    std::sort(nxt.begin(), nxt.end(), by_tokens);
    std::sort(e.nxt2.begin(), e.nxt2.end(), by_tokens);
    ps_layer_inputs in{};
    in.e_cur = cur.data();
    in.n_cur = static_cast<int32_t>(cur.size());
    in.e_next = nxt.data();
    in.n_next = static_cast<int32_t>(nxt.size());
    in.e_next2 = e.nxt2.empty() ? nullptr : e.nxt2.data();
    in.n_next2 = static_cast<int32_t>(e.nxt2.size());
    in.params = e.cfg.cost;
    in.params.alpha = static_cast<int64_t>(std::max(0.0, e.io_free_us - now_us()));
    in.stats = e.stats[group_of_layer(e.cfg.spec, l)];
    ps_layer_plan plan{};
    plan.cpu_set = cpu_b.data();
    plan.ondemand_seq = od_b.data();
    plan.prefetch_seq = pf_b.data();
    plan_layer(in, e.cfg.policy, plan);

    nvtxRangePop();
    NvtxRange loads_range("ps.layer.loads_ffn_combine");
    // --- R7: on-demand loads through the dual buffer, FFN per landed expert --------
    std::vector<ps_expert_load> loads(plan.ondemand_seq, plan.ondemand_seq + plan.n_ondemand);
    // R5: cpu_set on the host lane (concurrent with the loads below); without a lane the
    // GPU-only executor loads them after ondemand_seq.
    e.cpu_jobs.clear();
    // Host-lane jobs read their rows from the FFN source on the host: the local routing
    // (x of the B tokens, k slots per token) or, under EP, the rows received from all
    // ranks (copied to the host after the dispatch, one row per permuted row).
    auto lane_job = [&](int ex) {
      const uint16_t* slab = e.host_slab[static_cast<size_t>(l) * E + ex];
      require(slab != nullptr, "host lane: expert has no host copy");
      const int32_t* off = e.ep ? e.ep_plan_host : e.pinned_counts + 3 * Et;
      const int32_t* perm = e.ep ? e.ep_plan_host + (E + 1) : e.pinned_counts + 4 * Et + 1;
      CpuJob j{l, ex, off[ex + 1] - off[ex], off[ex], slab};
      if (!e.host_z.empty()) j.z = e.host_z[static_cast<size_t>(l) * E + ex];  // 3- or 4-bit codes
      for (int r = j.row0; r < j.row0 + j.m; ++r) {
        const uint16_t* src = e.ep ? e.lane_recv + static_cast<size_t>(perm[r]) * H
                                   : e.lane_x + static_cast<size_t>(perm[r] / Kt) * H;
        std::memcpy(e.lane_xrows + static_cast<size_t>(r) * H, src, sizeof(uint16_t) * H);
      }
      return j;
    };
    if (e.lane && plan.n_cpu > 0) {
      if (e.ep) PS_CUDA(cudaEventSynchronize(e.ev_lane_rows));  // received rows on the host
      for (int i = 0; i < plan.n_cpu; ++i) e.cpu_jobs.push_back(lane_job(plan.cpu_set[i].expert));
      e.lane_drv->submit(&e.cpu_jobs, e.lane_xrows, e.lane_yrows);
    } else {
      loads.insert(loads.end(), plan.cpu_set, plan.cpu_set + plan.n_cpu);
    }
    std::vector<IoJob*> od_jobs;
    for (size_t j = 0; j < loads.size(); ++j) {
      Slot* slot = &e.od_slot[j % 2];
      IoJob* job = new_job(e, kOnDemand, l, loads[j].expert, loads[j].tokens, slot);
      // the copy may only overwrite the slot after the FFN of load j-2 (or of the
      // slot's previous user) has been enqueued and completed
      job->wait_gen = slot->next_gen + static_cast<int64_t>(j / 2);
      od_jobs.push_back(job);
      push_modelled(e);
      e.io->push(job);
    }
    for (size_t j = 0; j < loads.size(); ++j) {
      IoJob* job = od_jobs[j];
      e.io->wait_issued(job);
      StallProbe p{take_event(e), take_event(e)};
      PS_CUDA(cudaEventRecord(p.before, e.sc));
      PS_CUDA(cudaStreamWaitEvent(e.sc, job->done_ev, 0));
      PS_CUDA(cudaEventRecord(p.after, e.sc));
      const bool fz = fuse_z(e, job, counts_l[job->expert]);
      land(e, job, fz);
      e.stall_t.push_back(p);
      ps_expert_group one{};
      one.n = 1;
      one.experts[0] = job->expert;
      one.slabs[0] = static_cast<const uint16_t*>(job->slot->dev);
      const void* zp[1] = {job->dst};
      ffn(e, one, counts_l.data(), B, true, true, job->zhost && !fz ? nullptr : p.after, fz ? zp : nullptr);
      release_slot_after_compute(e, job->slot);
      e.st.ondemand_loads++;
    }

    // Host-lane results (R5) -> y_part rows (split 0; other splits zero), then combine.
    if (!e.cpu_jobs.empty()) {
      e.lane_drv->wait();
      e.last_ffn_end = nullptr;  // copies follow the last FFN
      const size_t total_rows = static_cast<size_t>(e.src.rows);
      {  // one batch per layer: T = beta*sum(m) + n*C, so (mean tokens, mean time) per
         // expert is one sample of cpu_cost(m) = beta*m + C for fit_cost_params
        const double us = e.cpu_jobs[0].t1_us - e.cpu_jobs[0].t0_us;
        const double n = static_cast<double>(e.cpu_jobs.size());
        double tok = 0;
        for (const CpuJob& j : e.cpu_jobs) tok += j.m;
        e.st.cpu_ms_total += us / 1e3;
        e.cal_m.push_back(static_cast<int32_t>(std::lround(tok / n)));
        e.cal_us.push_back(ps_to_ticks(us / n));
      }
      // SM-driven read of the mapped pinned rows (a copy-engine H2D here would queue behind
      // an in-flight expert load on the same engine, up to ~4.5 ms), every expert's rows in
      // one launch
      rows_to_device(e, total_rows);
      for (CpuJob& j : e.cpu_jobs) {
        e.st.cpu_experts += 1;
        e.st.cpu_bytes_total += static_cast<double>(e.cfg.spec.expert_bytes);
        e.st.cpu_read_bytes += lane_read_bytes(e, j);
        j.t0_us -= host_t0_us;
        j.t1_us -= host_t0_us;
        e.cpu_done.push_back(j);
      }
      e.cpu_jobs.clear();
    }

    // Deferred prefetches (see `late` above): land on the GPU if the copy is done or ends
    // sooner than the lane would take; otherwise the lane computes the expert (the copy's
    // bytes are then unused, like a mispredicted prefetch's).
    if (!late.empty()) {
      e.cpu_jobs.clear();
      if (e.ep) PS_CUDA(cudaEventSynchronize(e.ev_lane_rows));
      for (const ps_engine_s::Ready* r : late) {
        const int m = counts_l[r->expert];
        const double cost = e.cfg.cost.beta * m + static_cast<double>(e.cfg.cost.startup);
        const bool landed = cudaEventQuery(r->job->done_ev) != cudaErrorNotReady;
        if (landed || r->job->est_done_us.load() - now_us() <= cost) {
          gpu_ready(*r);
          continue;
        }
        e.cpu_jobs.push_back(lane_job(r->expert));
        e.st.stolen_prefetches++;
      }
      if (!e.cpu_jobs.empty()) {
        e.lane_drv->submit(&e.cpu_jobs, e.lane_xrows, e.lane_yrows);
        e.lane_drv->wait();
        e.last_ffn_end = nullptr;
        const size_t total_rows = static_cast<size_t>(e.src.rows);
        rows_to_device(e, total_rows);
        for (CpuJob& j : e.cpu_jobs) {
          e.st.cpu_experts += 1;
          e.st.cpu_bytes_total += static_cast<double>(e.cfg.spec.expert_bytes);
          e.st.cpu_read_bytes += lane_read_bytes(e, j);
          e.st.cpu_ms_total += (j.t1_us - j.t0_us) / 1e3 / static_cast<double>(e.cpu_jobs.size());
          j.t0_us -= host_t0_us;
          j.t1_us -= host_t0_us;
          e.cpu_done.push_back(j);
        }
        e.cpu_jobs.clear();
      }
    }

    // --- combine -> y_l ------------------------------------------------------------
    ph.comb0 = e.last_ffn_end;  // nothing enqueued since the last FFN ended (else a new mark)
    if (!ph.comb0) {
      ph.comb0 = take_event(e);
      PS_CUDA(cudaEventRecord(ph.comb0, e.sc));
    }
    if (!e.ep) {
      s = ps_combine(e.y_part, e.step_split, e.inv, e.S ? e.ids_ext : ld.ids, e.S ? e.w_ext : ld.weights, B, Kt, Et, H,
                     y_l, e.sc);
    } else {
      s = ep_combine_rows(e, B, ld, y_l);
    }
    if (s != PS_OK) fail(s, ps_last_error());
    ph.comb1 = take_event(e);
    PS_CUDA(cudaEventRecord(ph.comb1, e.sc));
    e.phase_t.push_back(ph);
    e.st.kernel_launches += 1;

    // R3: prefetch slots that targeted this layer are free once its FFNs are done.
    for (auto it = e.ready.begin(); it != e.ready.end();) {
      if (it->layer <= l) {
        it->slot->in_use = false;
        release_slot_after_compute(e, it->slot);
        it = e.ready.erase(it);
      } else {
        ++it;
      }
    }

    // --- R8: prefetch dispatch behind the loads on the same channel ---------------
    if (plan.n_prefetch > 0) {
      const int target = plan.prefetch_from_widened ? l + 2 : l + 1;
      // The reference simulator throws when a batch overflows the target layer's slots
      // (simulator.cpp:209-212); the executor instead truncates the batch to the free
      // slots (hottest first survive) and counts the truncation.
      int used = 0;
      for (auto& sl : e.pf_pool) used += sl->in_use && sl->target_layer == target;
      const int room = std::max(0, e.cfg.prefetch_slots - used);
      if (plan.n_prefetch > room) {
        e.st.prefetches_cancelled += plan.n_prefetch - room;
        plan.n_prefetch = room;
      }
      for (int j = 0; j < plan.n_prefetch; ++j) {
        const ps_expert_load& pe = plan.prefetch_seq[j];
        Slot* slot = take_prefetch_slot(e, target);
        IoJob* job = new_job(e, kPrefetch, target, pe.expert, pe.tokens, slot);
        job->critical = j + 1 == plan.n_prefetch;
        job->issue_group = group_of_layer(e.cfg.spec, l);
        e.pending_pf.push_back(job);
        push_modelled(e);
        e.io->push(job);
      }
    }
    // --- lookahead top-up (cfg.lookahead = d > 0; a labelled extension of PreSched, off
    // in the reference configuration): behind PreSched's own batch, queue the remaining
    // predicted non-resident experts of layers l+1 .. l+d (d <= 2), hottest first, up to
    // each target layer's slot cap. Whatever has not started by the next scheduling
    // point is cancelled there (R2), so the channel never idles while a predicted expert
    // is still missing; the host lane takes whatever did not arrive in time.
    if (e.cfg.lookahead > 0 && !e.ep) {
      auto pending = [&](int layer, int ex) {
        for (IoJob* j : e.pending_pf)
          if (j->layer == layer && j->expert == ex) return true;
        return is_ready(layer, ex);
      };
      // lookahead 3 = layer l+2 only, at most two copies per layer: a copy issued now for
      // l+1 lands after l+1's scheduling point and stalls its GPU work, one for l+2 has a
      // whole layer to land (measured: profiles/r02_bench_lookahead_ab*.jsonl).
      const int d0 = e.cfg.lookahead == 3 ? 2 : 1, d1 = std::min(2, e.cfg.lookahead);
      const int per_layer_cap = e.cfg.lookahead == 3 ? 2 : e.cfg.prefetch_slots;
      int queued = 0;
      for (int d = d0; d <= d1 && l + d < L; ++d) {
        const std::vector<ps_expert_load>& cand = d == 1 ? nxt : e.nxt2;
        int used = 0;
        for (auto& sl : e.pf_pool) used += sl->in_use && sl->target_layer == l + d;
        for (auto it = cand.rbegin(); it != cand.rend() && used < e.cfg.prefetch_slots && queued < per_layer_cap;
             ++it) {
          if (pending(l + d, it->expert)) continue;
          Slot* slot = take_prefetch_slot(e, l + d);
          IoJob* job = new_job(e, kPrefetch, l + d, it->expert, it->tokens, slot);
          job->issue_group = group_of_layer(e.cfg.spec, l);
          e.pending_pf.push_back(job);
          push_modelled(e);
          e.io->push(job);
          ++used;
          ++queued;
          e.st.lookahead_prefetches++;
        }
      }
    }
  }
}

// Step epilogue: end mark, drain of the serial channel (pending prefetches cancelled or
// completed), and the step's measurement / measured timeline from its CUDA events.
void step_end(ps_engine_s& e, int32_t* ids_out) {
  require(e.in_step && e.next_layer == e.L, "step_end: not every layer of the step ran");
  e.in_step = false;
  const int L = e.L, E = e.E, K = e.K, B = e.step_B;
  if (ids_out)
    for (int l = 0; l < L; ++l)
      PS_CUDA(cudaMemcpyAsync(ids_out + static_cast<size_t>(l) * B * K, e.layer[l].ids, sizeof(int32_t) * B * K,
                              cudaMemcpyDeviceToDevice, e.sc));
  PS_CUDA(cudaEventRecord(e.ev_step1, e.sc));
  PS_CUDA(cudaEventSynchronize(e.ev_step1));
  const double t_tail0 = now_us();  // host time after the step's GPU work (drain + measurement)
  // Prefetches still pending at the end of the pass are cancelled or drained.
  for (IoJob* j : e.io->cancel_queued_prefetches()) j->slot->in_use = false;
  e.io->drain();
  for (auto& sl : e.pf_pool) sl->in_use = false;
  e.io->check();

  // --- measurement (CUDA events; no extra sync) ------------------------------------
  float ms = 0;
  // Measured timeline (us from the step start) built from the same events.
  auto at_us = [&](cudaEvent_t ev) {
    float t = 0;
    PS_CUDA(cudaEventElapsedTime(&t, e.ev_step0, ev));
    return static_cast<int64_t>(std::llround(static_cast<double>(t) * 1000.0));
  };
  e.last_events.clear();
  e.last_layer_start.assign(L, 0);
  e.last_layer_end.assign(L, 0);
  e.last_truth = e.step_truth;
  for (auto& t : e.ffn_t) {
    PS_CUDA(cudaEventElapsedTime(&ms, t.a, t.b));
    e.st.ffn_ms_total += ms;
    e.st.ffn_bytes_total += t.bytes;
    if (!t.experts.empty()) {
      e.ffn_expert_ms_total += ms;
      e.ffn_experts += static_cast<double>(t.experts.size());
    }
    const int64_t a = at_us(t.a), b = at_us(t.b);
    for (size_t i = 0; i < t.experts.size(); ++i)  // shared experts are not part of the routed timeline
      if (t.experts[i] < E)
        e.last_events.push_back({a, b, PS_RES_GPU, PS_EV_GPU_EXPERT, t.layer, t.experts[i], t.tokens[i]});
  }
  for (size_t l = 0; l < e.phase_t.size(); ++l) {
    auto& p = e.phase_t[l];
    PS_CUDA(cudaEventElapsedTime(&ms, p.route0, p.route1));
    e.st.route_phase_ms_total += ms;
    e.route_ms_total_cal += ms;
    PS_CUDA(cudaEventElapsedTime(&ms, p.comb0, p.comb1));
    e.st.combine_ms_total += ms;
    e.last_layer_start[l] = at_us(p.route0);
    e.last_layer_end[l] = at_us(p.comb1);
    e.last_events.push_back({e.last_layer_start[l], at_us(p.route1), PS_RES_GPU, PS_EV_ATTENTION,
                             static_cast<int32_t>(l), -1, 0});
  }
  for (const CpuJob& j : e.cpu_done)  // host clock from the step start (~ev_step0)
    e.last_events.push_back({static_cast<int64_t>(std::llround(j.t0_us)), static_cast<int64_t>(std::llround(j.t1_us)),
                             PS_RES_CPU, PS_EV_CPU_EXPERT, j.layer, j.expert, j.m});
  for (auto& p : e.stall_t) {
    PS_CUDA(cudaEventElapsedTime(&ms, p.before, p.after));
    e.st.compute_wait_ms += ms;
  }
  for (auto& j : e.jobs) {
    if (j->state.load() != 1) continue;
    PS_CUDA(cudaEventElapsedTime(&ms, j->start_ev, j->done_ev));
    e.st.h2d_busy_ms += ms;
    e.st.h2d_bytes += static_cast<double>(j->bytes);  // issued copies only (cancelled prefetches moved nothing)
    e.st.h2d_expert_bytes += static_cast<double>(e.cfg.spec.expert_bytes);
    e.copy_ms_total += ms;
    e.copies += 1;
    e.last_events.push_back({at_us(j->start_ev), at_us(j->done_ev), PS_RES_IO,
                             j->kind == kOnDemand ? PS_EV_LOAD : PS_EV_PREFETCH, j->layer, j->expert, j->tokens});
  }
  std::stable_sort(e.last_events.begin(), e.last_events.end(),
                   [](const ps_timeline_event& a, const ps_timeline_event& b) {
                     if (a.resource != b.resource) return a.resource < b.resource;
                     if (a.t_start != b.t_start) return a.t_start < b.t_start;
                     return a.t_end < b.t_end;
                   });
  PS_CUDA(cudaEventElapsedTime(&ms, e.ev_step0, e.ev_step1));
  e.st.step_ms_total += ms;
  e.st.steps += 1;
  e.st.layers += L;
  e.st.host_tail_ms_total += (now_us() - t_tail0) / 1e3;
}

void decode_step(ps_engine_s& e, const float* hidden, const uint8_t* follow, int B, float* y, int32_t* ids_out,
                 const int32_t* routed_ids = nullptr, const float* routed_w = nullptr) {
  NvtxRange step_range("ps.decode_step");
  step_begin(e, B);
  const int L = e.L, E = e.E, K = e.K, H = e.H;
  for (int l = 0; l < L; ++l) {
    const size_t xl = static_cast<size_t>(l) * B * H;
    const bool nx = l + 1 < L;
    layer_forward(e, l, hidden + xl, follow ? follow + static_cast<size_t>(l) * B : nullptr, y + xl,
                  routed_ids ? routed_ids + static_cast<size_t>(l) * B * K : nullptr,
                  routed_w ? routed_w + static_cast<size_t>(l) * B * E : nullptr,
                  nx ? hidden + xl + static_cast<size_t>(B) * H : nullptr,
                  nx && follow ? follow + static_cast<size_t>(l + 1) * B : nullptr);
  }
  step_end(e, ids_out);
}

void create_engine(const ps_engine_config& cfg, ps_engine_s& e) {
  e.cfg = cfg;
  const ps_model_spec& sp = cfg.spec;
  PS_CUDA(cudaSetDevice(cfg.device));
  if (ps_spec_validate(&sp) != PS_OK) fail(PS_EINVAL, ps_last_error());
  if (ps_spec_ffn_dim(&sp, &e.F) != PS_OK) fail(PS_EINVAL, ps_last_error());
  e.L = sp.num_layers;
  e.E = sp.experts_per_layer;
  e.K = sp.top_k;
  e.H = sp.hidden_dim;
  e.maxB = cfg.max_batch;
  e.S = cfg.n_shared;
  e.Et = e.E + e.S;
  e.Kt = e.K + e.S;
  require(e.maxB >= 1 && e.Et <= 256 && e.H % 8 == 0 && e.F % 8 == 0, "engine: unsupported shape");
  require(e.S >= 0 && e.S <= 32, "engine: n_shared out of range [0, 32]");
  require(e.S == 0 || !cfg.ep, "engine: shared experts are not supported with expert parallelism");
  if (e.cfg.prefetch_slots <= 0) e.cfg.prefetch_slots = 8;
  require(e.cfg.lookahead >= 0 && e.cfg.lookahead <= 3, "engine: lookahead must be 0..3");
  e.n_split = ps_ffn_down_splits(e.H, e.F);
  e.slab_elems = sp.expert_bytes / 2;
  for (auto& h : e.stats) h = {1.0, 0.0, 32};
  const bool auto_cost = e.cfg.cost.t_io <= 0;
  if (auto_cost) {  // provisional costs: PCIe Gen5 ~55 GB/s, HBM ~6.5 TB/s
    e.cfg.cost.t_io = std::max<int64_t>(2, static_cast<int64_t>(sp.expert_bytes / 55e3));
    e.cfg.cost.t_g = std::max<int64_t>(1, std::min<int64_t>(e.cfg.cost.t_io - 1,
                                                             static_cast<int64_t>(sp.expert_bytes / 6.5e6) + 5));
    e.cfg.cost.t_attn = 30;
    e.cfg.cost.beta = 1e9;  // GPU-only executor: no CPU lane (SURVEY.md §7 hard part 1)
    e.cfg.cost.startup = 0;
  }
  if (ps_cost_params_validate(&e.cfg.cost) != PS_OK) fail(PS_EINVAL, ps_last_error());

  PS_CUDA(cudaStreamCreateWithFlags(&e.sc, cudaStreamNonBlocking));
  PS_CUDA(cudaStreamCreateWithFlags(&e.s_d2h, cudaStreamNonBlocking));
  for (auto& st : e.s_pred) PS_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  PS_CUDA(cudaEventCreateWithFlags(&e.ev_k1, cudaEventDisableTiming));
  for (auto& ev : e.ev_pred) PS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  // Copies the channel keeps enqueued on the copy stream: with 1, "issued" = "started"
  // (the reference's R2: prefetches that started before the next scheduling point commit,
  // the rest are cancelled); with 2, a second copy is enqueued behind the running one and
  // commits although it has not started — the layer then waits ~9 ms for two serial
  // copies while the lane idles (profiles/timelines/r02_hybrid_k4_joined.json, layers
  // 1/3/16/18). Depth 1: +2.3 % tok/s in 4 alternating pairs
  // (profiles/r02_bench_io_depth_ab.jsonl). PS_IO_DEPTH=2 restores the old behaviour.
  static const int io_depth = [] {
    const char* v = std::getenv("PS_IO_DEPTH");
    return v && v[0] == '2' ? 2 : 1;
  }();
  e.io = std::make_unique<IoChannel>(cfg.device, io_depth);

  // Expert parallelism: this rank owns experts e % G == rank of every layer.
  e.ep = cfg.ep;
  if (e.ep) {
    e.G = ps_ep_comm_world(e.ep);
    e.rank = ps_ep_comm_rank(e.ep);
    require(e.G >= 1 && e.rank >= 0 && e.rank < e.G && e.G <= e.E, "engine: bad EP communicator");
  }
  e.E_loc = (e.E + e.G - 1) / e.G;
  auto owned = [&](int ex) { return ex % e.G == e.rank; };

  // Residency: explicit list or nothing (callers plan it with ps_plan_residency).
  const size_t LE = static_cast<size_t>(e.L) * e.E;
  e.resident.assign(LE, 0);
  for (int i = 0; i < cfg.n_resident; ++i) {
    int l = cfg.resident[2 * i], ex = cfg.resident[2 * i + 1];
    require(l >= 0 && l < e.L && ex >= 0 && ex < e.E, "engine: resident pair out of range");
    require(owned(ex), "engine: resident expert not owned by this EP rank");
    e.resident[static_cast<size_t>(l) * e.E + ex] = 1;
  }
  size_t n_res = 0, n_owned = 0;
  for (uint8_t r : e.resident) n_res += r;
  for (int ex = 0; ex < e.E; ++ex) n_owned += owned(ex) ? e.L : 0;
  require(n_res * sp.expert_bytes <= cfg.budget_bytes, "engine: resident set exceeds the HBM budget");
  const size_t n_host = n_owned - n_res;
  e.host_slab_count = n_host;
  e.pred_kind = cfg.predictor_kind == PS_PRED_AUTO ? (cfg.predictor ? PS_PRED_LLAPOR : PS_PRED_NONE)
                                                   : cfg.predictor_kind;
  require(e.pred_kind >= PS_PRED_LLAPOR && e.pred_kind <= PS_PRED_NONE, "engine: bad predictor_kind");
  require(e.pred_kind != PS_PRED_LLAPOR || cfg.predictor, "engine: PS_PRED_LLAPOR needs a predictor");
  require(!(cfg.ep && (e.pred_kind == PS_PRED_GATE || e.pred_kind == PS_PRED_STATS)),
          "engine: host-side predictors (gate, stats) are not supported with expert parallelism");
  if (e.pred_kind == PS_PRED_STATS) {
    require(cfg.stats_ranking != nullptr, "engine: PS_PRED_STATS needs stats_ranking [L*E]");
    e.stats_rank.assign(cfg.stats_ranking, cfg.stats_ranking + static_cast<size_t>(e.L) * e.E);
  }
  e.has_host.assign(e.L, 0);
  for (int l = 0; l < e.L; ++l)
    for (int ex = 0; ex < e.E; ++ex)
      // under EP every rank's prediction feeds every owner's plan (counts exchange)
      if (e.ep || (owned(ex) && !e.resident[static_cast<size_t>(l) * e.E + ex])) e.has_host[l] = 1;

  e.dev_slab.assign(LE, nullptr);
  e.host_slab.assign(LE, nullptr);
  if (n_res) PS_CUDA(cudaMalloc(&e.arena, n_res * sp.expert_bytes));
  if (n_host) {
    e.host_pin.alloc(n_host * sp.expert_bytes);
    e.host_arena = e.host_pin.ptr;
  }
  // Materialise weights: resident on device directly; host ones via a device staging
  // slab and a D2H copy (the hash is identical on both sides, see weights.cu).
  void* stage = nullptr;
  if (n_host) PS_CUDA(cudaMalloc(&stage, 2 * sp.expert_bytes));
  size_t ri = 0, hi = 0, si = 0;
  for (int l = 0; l < e.L; ++l)
    for (int ex = 0; ex < e.E; ++ex) {
      const size_t idx = static_cast<size_t>(l) * e.E + ex;
      if (!owned(ex)) continue;
      // caller-supplied weights (cfg.expert_weights) or the hash-initialised synthetic ones
      const uint16_t* given = cfg.expert_weights ? cfg.expert_weights[static_cast<size_t>(l) * e.Et + ex] : nullptr;
      require(!cfg.expert_weights || given, "engine: expert_weights has a null slab for an owned expert");
      if (e.resident[idx]) {
        uint16_t* p = reinterpret_cast<uint16_t*>(static_cast<char*>(e.arena) + ri++ * sp.expert_bytes);
        if (given)
          PS_CUDA(cudaMemcpyAsync(p, given, sp.expert_bytes, cudaMemcpyHostToDevice, e.sc));
        else if (ps_init_expert_slab(p, e.H, e.F, cfg.weight_seed, l, ex, e.sc) != PS_OK)
          fail(PS_ECUDA, ps_last_error());
        e.dev_slab[idx] = p;
      } else {
        uint16_t* hp = reinterpret_cast<uint16_t*>(static_cast<char*>(e.host_arena) + hi++ * sp.expert_bytes);
        if (given) {
          std::memcpy(hp, given, sp.expert_bytes);
        } else {
          uint16_t* st = reinterpret_cast<uint16_t*>(static_cast<char*>(stage) + (si++ % 2) * sp.expert_bytes);
          if (ps_init_expert_slab(st, e.H, e.F, cfg.weight_seed, l, ex, e.sc) != PS_OK)
            fail(PS_ECUDA, ps_last_error());
          PS_CUDA(cudaMemcpyAsync(hp, st, sp.expert_bytes, cudaMemcpyDeviceToHost, e.sc));
        }
        e.host_slab[idx] = hp;
      }
    }
  // Shared experts: dense weights of every layer, always in HBM (not part of the routed
  // budget PreScope manages); hash-keyed as experts E..E+S-1.
  e.shared_slab.assign(static_cast<size_t>(e.L) * e.S, nullptr);
  if (e.S) {
    PS_CUDA(cudaMalloc(&e.shared_arena, static_cast<size_t>(e.L) * e.S * sp.expert_bytes));
    for (int l = 0; l < e.L; ++l)
      for (int j = 0; j < e.S; ++j) {
        const size_t idx = static_cast<size_t>(l) * e.S + j;
        uint16_t* p = reinterpret_cast<uint16_t*>(static_cast<char*>(e.shared_arena) + idx * sp.expert_bytes);
        const uint16_t* given = cfg.expert_weights ? cfg.expert_weights[static_cast<size_t>(l) * e.Et + e.E + j] : nullptr;
        require(!cfg.expert_weights || given, "engine: expert_weights has a null shared-expert slab");
        if (given)
          PS_CUDA(cudaMemcpyAsync(p, given, sp.expert_bytes, cudaMemcpyHostToDevice, e.sc));
        else if (ps_init_expert_slab(p, e.H, e.F, cfg.weight_seed, l, e.E + j, e.sc) != PS_OK)
          fail(PS_ECUDA, ps_last_error());
        e.shared_slab[idx] = p;
      }
  }
  PS_CUDA(cudaStreamSynchronize(e.sc));
  if (stage) cudaFree(stage);

  // z-slabs: encode every host slab once (all host cores), keep raw ones that do not fit.
  if (cfg.compress_host && n_host) {
    const uint64_t n = sp.expert_bytes / 2, nb = (n + 1023) / 1024, n_pad = nb * 1024;
    e.z_cap = ((64 + n_pad + n_pad / 2 + 4 * (nb + 1) + n / 64) + 4095) / 4096 * 4096;
    e.z_pin.alloc(n_host * e.z_cap);
    e.z_arena = e.z_pin.ptr;
    e.host_z.assign(LE, nullptr);
    e.host_z_bytes.assign(LE, 0);
    // With an AMX host lane, the raw slabs only feed the lane (PCIe reads the z-slabs):
    // re-lay them into the lane's tile layout first and encode the tiled values, so both
    // the lane's raw and z paths read sequential streams (ps_zslab_decode un-tiles on the
    // GPU). If any slab does not fit a z-slab, everything goes back to row-major.
    bool tiled = false;
    if (cfg.host_threads > 0 && lane_tiles_enabled()) {
      ps_host_lane probe_lane = nullptr;
      if (ps_host_lane_create(1, &probe_lane) == PS_OK) {
        tiled = ps_host_lane_isa(probe_lane) == 2;
        ps_host_lane_destroy(probe_lane);
      }
    }
    std::vector<uint16_t*> hosts;
    for (size_t idx = 0; idx < LE; ++idx)
      if (e.host_slab[idx]) hosts.push_back(const_cast<uint16_t*>(e.host_slab[idx]));
    auto parallel_slabs = [&](const std::function<bool(uint16_t*)>& fn) {
      std::atomic<size_t> next{0};
      std::atomic<bool> ok{true};
      std::vector<std::thread> th;
      const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 32));
      for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&] {
          for (size_t i; (i = next.fetch_add(1)) < hosts.size();)
            if (!fn(hosts[i])) ok = false;
        });
      for (auto& t : th) t.join();
      return ok.load();
    };
    if (tiled && !parallel_slabs([&](uint16_t* p) { return ps_host_slab_tile(p, e.H, e.F) == PS_OK; }))
      fail(PS_ERUNTIME, "engine: host slab re-layout failed");
    for (int pass = 0; pass < 2; ++pass) {
      size_t zi = 0;
      bool all = true;
      for (size_t idx = 0; idx < LE; ++idx) {
        if (!e.host_slab[idx]) continue;
        uint8_t* z = static_cast<uint8_t*>(e.z_arena) + zi++ * e.z_cap;
        uint64_t bytes = 0;
        const ps_status st = tiled ? ps_zslab_encode_tiled(e.host_slab[idx], e.H, e.F, z, e.z_cap, &bytes, 0)
                                   : ps_zslab_encode(e.host_slab[idx], n, z, e.z_cap, &bytes, 0);
        e.host_z[idx] = st == PS_OK ? z : nullptr;
        e.host_z_bytes[idx] = st == PS_OK ? bytes : 0;
        all = all && st == PS_OK;
      }
      if (all || !tiled) break;
      if (!parallel_slabs([&](uint16_t* p) { return ps_host_slab_untile(p, e.H, e.F) == PS_OK; }))
        fail(PS_ERUNTIME, "engine: host slab re-layout failed");
      tiled = false;
    }
    e.host_tiled = tiled;
    {  // opt-in: K3 decodes landed tiled z-slabs itself (no z_decode pass, no bf16 copy)
      const char* zf = std::getenv("PS_ZFUSE");
      const int kch = ((e.F + e.n_split - 1) / e.n_split + 31) / 32 * 32;
      e.zfuse = zf && zf[0] == '1' && tiled && e.H % 64 == 0 && e.F % 64 == 0 && kch % 64 == 0 &&
                3ull * e.H * e.F < (1ull << 32);
    }
  }
  if (auto_cost && e.z_cap) {  // provisional t_io from the mean z-slab size
    double zb = 0, cnt = 0;
    for (uint64_t b : e.host_z_bytes)
      if (b) {
        zb += static_cast<double>(b);
        cnt += 1;
      }
    if (cnt > 0) e.cfg.cost.t_io = std::max<int64_t>(e.cfg.cost.t_g + 1, static_cast<int64_t>(zb / cnt / 55e3));
  }
  for (auto& s : e.od_slot) {
    PS_CUDA(cudaMalloc(&s.dev, sp.expert_bytes));
    if (e.z_cap) PS_CUDA(cudaMalloc(&s.zdev, e.z_cap));
    PS_CUDA(cudaEventCreateWithFlags(&s.free_ev, cudaEventDisableTiming));
  }
  // Prefetch slots for two live target layers (R8 cap per layer) up front: a cudaMalloc
  // of an expert-sized buffer inside a step costs milliseconds of host time.
  // (lookahead 2 keeps a third target layer live: l+1 and l+2 queued while l's land)
  const size_t live_layers = e.cfg.lookahead >= 2 ? 3 : 2;  // (3: l+2 only, also three live layers)
  for (size_t i = 0; i < std::min<size_t>(live_layers * static_cast<size_t>(e.cfg.prefetch_slots), n_host); ++i) {
    auto s = std::make_unique<Slot>();
    PS_CUDA(cudaMalloc(&s->dev, sp.expert_bytes));
    if (e.z_cap) PS_CUDA(cudaMalloc(&s->zdev, e.z_cap));
    PS_CUDA(cudaEventCreateWithFlags(&s->free_ev, cudaEventDisableTiming));
    e.pf_pool.push_back(std::move(s));
  }

  // Router bias: -zipf_g * ln(e+1) per layer (workload.cpp:180-181).
  PS_CUDA(cudaMalloc(&e.gate, sizeof(float) * e.L * e.E * e.H));
  PS_CUDA(cudaMemset(e.gate, 0, sizeof(float) * e.L * e.E * e.H));
  std::vector<float> bias(static_cast<size_t>(e.L) * e.E);
  for (int l = 0; l < e.L; ++l) {
    const int g = group_of_layer(sp, l);
    const double z = g == PS_GROUP_INPUT ? cfg.gen.input.zipf_s : g == PS_GROUP_OUTPUT ? cfg.gen.output.zipf_s
                                                                                          : cfg.gen.middle.zipf_s;
    for (int ex = 0; ex < e.E; ++ex) bias[static_cast<size_t>(l) * e.E + ex] = static_cast<float>(-z * std::log(ex + 1.0));
  }
  PS_CUDA(cudaMalloc(&e.bias, sizeof(float) * bias.size()));
  PS_CUDA(cudaMemcpy(e.bias, bias.data(), sizeof(float) * bias.size(), cudaMemcpyHostToDevice));

  const size_t B = e.maxB, rows = B * e.K, rows_t = B * e.Kt;
  e.rows_max = static_cast<int>(e.G * rows_t);  // FFN rows: everything routed here by all ranks
  const size_t frows = static_cast<size_t>(e.rows_max);
  e.layer.resize(e.L);
  for (auto& ld : e.layer) {
    PS_CUDA(cudaMalloc(&ld.weights, sizeof(float) * B * e.E));
    PS_CUDA(cudaMalloc(&ld.ids, sizeof(int32_t) * rows));
  }
  const size_t n_sched = 4 * static_cast<size_t>(e.Et) + 1 + rows_t;
  PS_CUDA(cudaMalloc(&e.sched_dev, sizeof(int32_t) * n_sched));
  PS_CUDA(cudaMemsetAsync(e.sched_dev, 0, sizeof(int32_t) * n_sched, e.sc));
  PS_CUDA(cudaHostAlloc(&e.pinned_counts, sizeof(int32_t) * n_sched, cudaHostAllocDefault));
  e.counts_dev = e.sched_dev;
  PS_CUDA(cudaMalloc(&e.route_ws, sizeof(int32_t) * 65));
  if (e.use_graphs) {
    const char* g = std::getenv("PS_SCHED_GRAPH");  // 0: eager scheduling point (A/B)
    e.use_graphs = !(g && g[0] == '0');
  }
  PS_CUDA(cudaMalloc(&e.x_stage, sizeof(float) * static_cast<size_t>(e.maxB) * e.H));
  PS_CUDA(cudaMalloc(&e.fol_stage, static_cast<size_t>(e.maxB)));
  PS_CUDA(cudaMemsetAsync(e.route_ws, 0, sizeof(int32_t) * 65, e.sc));
  e.pred_dev = e.sched_dev + e.Et;
  e.pred2_dev = e.sched_dev + 2 * e.Et;
  e.offsets = e.sched_dev + 3 * e.Et;
  e.perm_src = e.sched_dev + 4 * e.Et + 1;
  if (e.S) {
    PS_CUDA(cudaMalloc(&e.ids_ext, sizeof(int32_t) * rows_t));
    PS_CUDA(cudaMalloc(&e.w_ext, sizeof(float) * B * e.Et));
  }
  PS_CUDA(cudaMalloc(&e.x_bf16, sizeof(uint16_t) * B * e.H));
  PS_CUDA(cudaMalloc(&e.x_perm, sizeof(uint16_t) * frows * e.H));
  PS_CUDA(cudaMalloc(&e.inv, sizeof(int32_t) * rows_t));
  PS_CUDA(cudaMalloc(&e.hbuf, sizeof(uint16_t) * frows * e.F));
  PS_CUDA(cudaMalloc(&e.y_part, sizeof(float) * e.n_split * frows * e.H));
  if (e.ep) {
    const size_t Ev = static_cast<size_t>(e.G) * e.E_loc;
    PS_CUDA(cudaMalloc(&e.ep_vids, sizeof(int32_t) * rows));
    PS_CUDA(cudaMalloc(&e.ep_off_v, sizeof(int32_t) * (Ev + 1)));
    PS_CUDA(cudaMalloc(&e.ep_perm_v, sizeof(int32_t) * rows));
    PS_CUDA(cudaMalloc(&e.ep_inv_v, sizeof(int32_t) * rows));
    PS_CUDA(cudaMalloc(&e.ep_send_x, sizeof(uint16_t) * rows * e.H));
    PS_CUDA(cudaMalloc(&e.ep_recv_x, sizeof(uint16_t) * frows * e.H));
    PS_CUDA(cudaMalloc(&e.ep_y_recv, sizeof(float) * frows * e.H));
    PS_CUDA(cudaMalloc(&e.ep_y_back, sizeof(float) * rows * e.H));
    PS_CUDA(cudaMalloc(&e.ep_cnt_send, sizeof(int32_t) * 2 * Ev));
    PS_CUDA(cudaMalloc(&e.ep_cnt_recv, sizeof(int32_t) * 2 * Ev));
    PS_CUDA(cudaMalloc(&e.ep_plan_dev, sizeof(int32_t) * (e.E + 1 + 2 * frows)));
    PS_CUDA(cudaHostAlloc(&e.ep_plan_host, sizeof(int32_t) * (e.E + 1 + 2 * frows), cudaHostAllocDefault));
    PS_CUDA(cudaHostAlloc(&e.ep_host, sizeof(int32_t) * (Ev + 1 + 2 * Ev), cudaHostAllocDefault));
    PS_CUDA(cudaMalloc(&e.ep_ones, sizeof(float) * frows));
    PS_CUDA(cudaMalloc(&e.ep_zeros, sizeof(int32_t) * frows));
    std::vector<float> ones(frows, 1.0f);
    PS_CUDA(cudaMemcpy(e.ep_ones, ones.data(), sizeof(float) * frows, cudaMemcpyHostToDevice));
    PS_CUDA(cudaMemset(e.ep_zeros, 0, sizeof(int32_t) * frows));
  }
  if (cfg.predictor) {
    PS_CUDA(cudaMalloc(&e.llapor_scratch, ps_llapor_scratch_bytes(cfg.predictor, e.maxB)));
    PS_CUDA(cudaMalloc(&e.llapor_scratch2, ps_llapor_scratch_bytes(cfg.predictor, e.maxB)));
  }
  if (e.pred_kind == PS_PRED_PERFECT) {
    PS_CUDA(cudaMalloc(&e.pp_ids, sizeof(int32_t) * B * e.K));
    PS_CUDA(cudaMalloc(&e.pp_w, sizeof(float) * B * e.E));
  }
  PS_CUDA(cudaMalloc(&e.in_hidden, sizeof(float) * e.L * B * e.H));
  PS_CUDA(cudaMalloc(&e.in_follow, e.L * B));
  PS_CUDA(cudaMalloc(&e.out_y, sizeof(float) * e.L * B * e.H));
  PS_CUDA(cudaMalloc(&e.out_ids, sizeof(int32_t) * e.L * rows));
  PS_CUDA(cudaEventCreateWithFlags(&e.ev_routed, cudaEventDisableTiming));
  PS_CUDA(cudaEventCreateWithFlags(&e.ev_in, cudaEventDisableTiming));
  PS_CUDA(cudaEventCreateWithFlags(&e.ev_out, cudaEventDisableTiming));
  PS_CUDA(cudaEventCreate(&e.ev_step0));
  PS_CUDA(cudaEventCreate(&e.ev_step1));

  if (cfg.host_threads > 0) {
    if (ps_host_lane_create(cfg.host_threads, &e.lane) != PS_OK) fail(PS_ERUNTIME, ps_last_error());
    PS_CUDA(cudaHostAlloc(&e.lane_x, sizeof(uint16_t) * B * e.H, cudaHostAllocDefault));
    // lane rows: this rank's routed rows, or under EP every row routed here by all ranks
    PS_CUDA(cudaHostAlloc(&e.lane_xrows, sizeof(uint16_t) * frows * e.H, cudaHostAllocDefault));
    PS_CUDA(cudaHostAlloc(&e.lane_yrows, sizeof(float) * frows * e.H, cudaHostAllocMapped));
    if (e.ep) {
      PS_CUDA(cudaHostAlloc(&e.lane_recv, sizeof(uint16_t) * frows * e.H, cudaHostAllocDefault));
      PS_CUDA(cudaEventCreateWithFlags(&e.ev_lane_rows, cudaEventDisableTiming | cudaEventBlockingSync));
    }
    e.lane_drv = std::make_unique<LaneDriver>(e.lane, e.H, e.F);
    e.lane_drv->tiled = e.host_tiled;
    // cpu_cost = beta*m + C (cost_model.cpp:34-37) measured on this host: the lane on a
    // host-resident expert slab at two token counts (below), best of 3 each.
    const uint16_t* probe = nullptr;
    const uint8_t* probe_z = nullptr;  // the lane reads z-slabs when they exist (AMX)
    for (size_t i = 0; i < e.host_slab.size(); ++i)
      if (e.host_slab[i]) {
        probe = e.host_slab[i];
        if (!e.host_z.empty() && lane_z_enabled() && ps_host_lane_reads_z(e.lane) && e.host_z[i])
          probe_z = e.host_z[i];
        break;
      }
    if (auto_cost && probe) {
      std::memset(e.lane_xrows, 0, sizeof(uint16_t) * rows_t * e.H);
      auto best = [&](int m) {
        double t = 1e30;
        for (int r = 0; r < 3; ++r) {
          const double a = now_us();
          const int32_t row0 = 0;
          const ps_status st = probe_z ? ps_host_expert_ffn_batch_z(e.lane, 1, &probe_z, &m, &row0, e.H, e.F,
                                                                    e.lane_xrows, e.lane_yrows)
                                       : (e.host_tiled ? ps_host_expert_ffn_batch_tiled : ps_host_expert_ffn_batch)(
                                             e.lane, 1, &probe, &m, &row0, e.H, e.F, e.lane_xrows, e.lane_yrows);
          if (st != PS_OK) fail(PS_ERUNTIME, ps_last_error());
          t = std::min(t, now_us() - a);
        }
        return t;
      };
      // Decode engines (maxB <= 64): the line through m = 1 and m = min(16, maxB), the
      // DRAM-bound regime decode experts live in. Prefill-capable engines: the line
      // through m = 16 and 128, where the AMX lane is compute-bound (cost grows with
      // ceil(m/16)), so 100+-token experts are not under-priced against PCIe.
      const bool prefill = e.maxB > 64;
      const int m1 = prefill ? 16 : 1;
      const int m2 = std::min<int>(prefill ? 128 : std::max(1, std::min(16, e.maxB)), static_cast<int>(rows_t));
      const double t1 = best(m1), t2 = m2 > m1 ? best(m2) : t1;
      e.probe_m = {m1, m2};
      e.probe_us = {ps_to_ticks(t1), ps_to_ticks(t2)};
      const double beta = m2 > m1 ? std::max(0.0, (t2 - t1) / (m2 - m1)) : 0.0;
      e.cfg.cost.beta = std::max(beta, 1e-3);
      e.cfg.cost.startup = std::max<int64_t>(0, ps_to_ticks(t1 - beta * m1));
    }
  }
  e.st.cost = e.cfg.cost;
}

void destroy_engine(ps_engine_s& e) {
  // A step that failed mid-layer can leave on-demand jobs queued behind a slot
  // generation that will never be recorded: forget them before draining the channel.
  if (e.io) {
    e.io->abandon_queued();
    e.io->drain();
  }
  e.io.reset();
  e.lane_drv.reset();
  if (e.lane) ps_host_lane_destroy(e.lane);
  for (void* p : {(void*)e.lane_x, (void*)e.lane_xrows, (void*)e.lane_yrows, (void*)e.lane_recv})
    if (p) cudaFreeHost(p);
  if (e.sc) cudaStreamSynchronize(e.sc);
  if (e.s_d2h) cudaStreamSynchronize(e.s_d2h);
  for (auto& kv : e.sched_graphs) cudaGraphExecDestroy(kv.second);
  e.sched_graphs.clear();
  if (e.x_stage) cudaFree(e.x_stage);
  if (e.fol_stage) cudaFree(e.fol_stage);
  for (auto& ld : e.layer) {
    cudaFree(ld.weights);
    cudaFree(ld.ids);
  }
  for (void* p : {(void*)e.arena, (void*)e.gate, (void*)e.bias, (void*)e.sched_dev, (void*)e.route_ws, (void*)e.pp_ids, (void*)e.pp_w,
                  (void*)e.x_bf16, (void*)e.x_perm, (void*)e.inv, (void*)e.hbuf,
                  (void*)e.y_part, e.llapor_scratch, e.llapor_scratch2, (void*)e.in_hidden, (void*)e.in_follow, (void*)e.out_y,
                  (void*)e.out_ids, (void*)e.ep_vids, (void*)e.ep_off_v, (void*)e.ep_perm_v, (void*)e.ep_inv_v,
                  (void*)e.ep_send_x, (void*)e.ep_recv_x, (void*)e.ep_y_recv, (void*)e.ep_y_back,
                  (void*)e.ep_cnt_send, (void*)e.ep_cnt_recv, (void*)e.ep_plan_dev, (void*)e.ep_ones,
                  (void*)e.ep_zeros, e.shared_arena, (void*)e.ids_ext, (void*)e.w_ext})
    if (p) cudaFree(p);
  if (e.ep_plan_host) cudaFreeHost(e.ep_plan_host);
  if (e.ep_host) cudaFreeHost(e.ep_host);
  e.host_pin.release();
  e.z_pin.release();
  if (e.pinned_counts) cudaFreeHost(e.pinned_counts);
  for (auto& s : e.od_slot) {
    if (s.dev) cudaFree(s.dev);
    if (s.zdev) cudaFree(s.zdev);
    if (s.free_ev) cudaEventDestroy(s.free_ev);
  }
  for (auto& s : e.pf_pool) {
    cudaFree(s->dev);
    if (s->zdev) cudaFree(s->zdev);
    cudaEventDestroy(s->free_ev);
  }
  for (cudaEvent_t ev : e.event_pool) cudaEventDestroy(ev);
  for (cudaEvent_t ev : e.job_event_pool) cudaEventDestroy(ev);
  for (cudaEvent_t ev : {e.ev_routed, e.ev_step0, e.ev_step1, e.ev_in, e.ev_out, e.ev_lane_rows, e.ev_k1, e.ev_pred[0],
                         e.ev_pred[1]})
    if (ev) cudaEventDestroy(ev);
  for (cudaStream_t st : e.s_pred)
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  if (e.sc) cudaStreamDestroy(e.sc);
  if (e.s_d2h) cudaStreamDestroy(e.s_d2h);
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

ps_status ps_engine_create(const ps_engine_config* cfg, ps_engine* out) {
  auto e = std::make_unique<ps_engine_s>();
  ps_status s = guarded([&] { create_engine(*cfg, *e); });
  if (s != PS_OK) {
    destroy_engine(*e);
    return s;
  }
  *out = e.release();
  return PS_OK;
}

ps_status ps_engine_destroy(ps_engine e) {
  return guarded([&] {
    if (!e) return;
    destroy_engine(*e);
    delete e;
  });
}

ps_status ps_engine_set_router(ps_engine e, const float* gate_host) {
  return guarded([&] {
    PS_CUDA(cudaMemcpy(e->gate, gate_host, sizeof(float) * e->L * e->E * e->H, cudaMemcpyHostToDevice));
  });
}

ps_status ps_engine_decode_step(ps_engine e, const float* hidden, const uint8_t* follow, int B, float* y,
                                int32_t* ids) {
  return guarded([&] { decode_step(*e, hidden, follow, B, y, ids); });
}

ps_status ps_engine_decode_step_routed(ps_engine e, const float* hidden, const int32_t* ids, const float* weights, int B,
                                       float* y) {
  return guarded([&] {
    require(e && hidden && ids && weights && y, "decode_step_routed: null argument");
    require(e->pred_kind != PS_PRED_PERFECT, "decode_step_routed: PS_PRED_PERFECT routes from the trace inputs");
    decode_step(*e, hidden, nullptr, B, y, nullptr, ids, weights);
  });
}

ps_status ps_engine_decode_step_host(ps_engine e, const float* hidden_host, const uint8_t* follow_host, int B,
                                     float* y_host, int32_t* ids_host) {
  return guarded([&] {
    require(B >= 1 && B <= e->maxB, "decode_step_host: batch out of range");
    const size_t nh = static_cast<size_t>(e->L) * B * e->H;
    PS_CUDA(cudaMemcpyAsync(e->in_hidden, hidden_host, sizeof(float) * nh, cudaMemcpyHostToDevice, e->sc));
    if (follow_host)
      PS_CUDA(cudaMemcpyAsync(e->in_follow, follow_host, static_cast<size_t>(e->L) * B, cudaMemcpyHostToDevice, e->sc));
    decode_step(*e, e->in_hidden, follow_host ? e->in_follow : nullptr, B, e->out_y, ids_host ? e->out_ids : nullptr);
    PS_CUDA(cudaMemcpyAsync(y_host, e->out_y, sizeof(float) * nh, cudaMemcpyDeviceToHost, e->sc));
    if (ids_host)
      PS_CUDA(cudaMemcpyAsync(ids_host, e->out_ids, sizeof(int32_t) * e->L * B * e->K, cudaMemcpyDeviceToHost, e->sc));
    PS_CUDA(cudaStreamSynchronize(e->sc));
  });
}

ps_status ps_engine_step_begin(ps_engine e, int B) {
  return guarded([&] {
    require(e != nullptr, "ps_engine_step_begin: null engine");
    step_begin(*e, B);
  });
}

ps_status ps_engine_layer_forward(ps_engine e, int layer, const float* x, const uint8_t* follow, float* y,
                                  int32_t* ids, void* stream) {
  return guarded([&] {
    require(e && x && y, "ps_engine_layer_forward: null argument");
    require(e->in_step, "ps_engine_layer_forward: no step in progress (ps_engine_step_begin)");
    require(layer >= 0 && layer < e->L, "ps_engine_layer_forward: layer out of range");
    require(e->pred_kind != PS_PRED_PERFECT, "ps_engine_layer_forward: PS_PRED_PERFECT needs the whole step's inputs");
    cudaStream_t cs = as_stream(stream);
    const bool foreign = stream != nullptr && cs != e->sc;
    if (foreign) {  // the layer's inputs were produced on the caller's stream
      PS_CUDA(cudaEventRecord(e->ev_in, cs));
      PS_CUDA(cudaStreamWaitEvent(e->sc, e->ev_in, 0));
    }
    layer_forward(*e, layer, x, follow, y, nullptr, nullptr, nullptr, nullptr);
    if (ids)
      PS_CUDA(cudaMemcpyAsync(ids, e->layer[layer].ids, sizeof(int32_t) * e->step_B * e->K, cudaMemcpyDeviceToDevice,
                              e->sc));
    if (foreign) {  // the caller's next kernels (attention of layer+1) read y
      PS_CUDA(cudaEventRecord(e->ev_out, e->sc));
      PS_CUDA(cudaStreamWaitEvent(cs, e->ev_out, 0));
    }
  });
}

ps_status ps_engine_step_end(ps_engine e) {
  return guarded([&] {
    require(e != nullptr, "ps_engine_step_end: null engine");
    step_end(*e, nullptr);
  });
}

ps_status ps_engine_get_stats(ps_engine e, ps_engine_stats* out) {
  return guarded([&] {
    *out = e->st;
    out->cost = e->cfg.cost;
    out->calibration_fit = e->last_fit_used;
  });
}

ps_status ps_engine_reset_stats(ps_engine e) {
  return guarded([&] {
    e->st = ps_engine_stats{};
    e->st.cost = e->cfg.cost;
    // calibration samples are "since the last stats reset" (ps_engine_calibrate)
    e->copy_ms_total = e->copies = e->route_ms_total_cal = e->ffn_expert_ms_total = e->ffn_experts = 0;
    e->cal_m.clear();
    e->cal_us.clear();
  });
}

ps_status ps_engine_last_timeline(ps_engine e, ps_timeline* out, int32_t* truth_out, uint8_t* resident_out) {
  return guarded([&] {
    require(e && out, "ps_engine_last_timeline: null argument");
    const int n = static_cast<int>(e->last_events.size());
    if (n > out->cap_events) fail(PS_ERANGE, "ps_engine_last_timeline: event buffer too small (" + std::to_string(n) + ")");
    std::copy(e->last_events.begin(), e->last_events.end(), out->events);
    out->n_events = n;
    out->makespan = 0;
    for (const auto& ev : e->last_events) out->makespan = std::max(out->makespan, ev.t_end);
    if (out->layer_start) std::copy(e->last_layer_start.begin(), e->last_layer_start.end(), out->layer_start);
    if (out->layer_end) std::copy(e->last_layer_end.begin(), e->last_layer_end.end(), out->layer_end);
    if (truth_out) std::copy(e->last_truth.begin(), e->last_truth.end(), truth_out);
    if (resident_out) std::copy(e->resident.begin(), e->resident.end(), resident_out);
  });
}

ps_status ps_engine_last_routing(ps_engine e, int32_t* ids_out, float* weights_out) {
  return guarded([&] {
    require(e != nullptr, "ps_engine_last_routing: null engine");
    require(!e->in_step && e->step_B > 0, "ps_engine_last_routing: no completed step");
    const size_t B = static_cast<size_t>(e->step_B);
    for (int l = 0; l < e->L; ++l) {
      if (ids_out)
        PS_CUDA(cudaMemcpy(ids_out + l * B * e->K, e->layer[l].ids, sizeof(int32_t) * B * e->K, cudaMemcpyDeviceToHost));
      if (weights_out)
        PS_CUDA(cudaMemcpy(weights_out + l * B * e->E, e->layer[l].weights, sizeof(float) * B * e->E,
                           cudaMemcpyDeviceToHost));
    }
  });
}

ps_status ps_engine_last_predictions(ps_engine e, int32_t* out) {
  return guarded([&] {
    require(e && out, "ps_engine_last_predictions: null argument");
    std::copy(e->last_pred.begin(), e->last_pred.end(), out);
  });
}

ps_status ps_engine_set_lookahead(ps_engine e, int lookahead, int steal_late) {
  return guarded([&] {
    require(e != nullptr, "ps_engine_set_lookahead: null engine");
    require(lookahead >= 0 && lookahead <= 3 && (steal_late == 0 || steal_late == 1),
            "ps_engine_set_lookahead: lookahead in 0..3, steal_late in {0, 1}");
    require(!e->in_step, "ps_engine_set_lookahead: a step is in progress");
    e->cfg.lookahead = lookahead;
    e->cfg.steal_late = steal_late;
  });
}

ps_status ps_engine_set_cost(ps_engine e, const ps_cost_params* cost) {
  return guarded([&] {
    require(e && cost, "ps_engine_set_cost: null argument");
    if (ps_cost_params_validate(cost) != PS_OK) fail(PS_EINVAL, ps_last_error());
    e->cfg.cost = *cost;
    e->st.cost = *cost;
  });
}

ps_status ps_engine_calibrate(ps_engine e, ps_cost_params* out) {
  return guarded([&] {
    ps_cost_params c = e->cfg.cost;
    if (e->copies > 0) c.t_io = std::max<int64_t>(1, std::llround(1000.0 * e->copy_ms_total / e->copies));
    if (e->ffn_experts > 0) c.t_g = std::max<int64_t>(0, std::llround(1000.0 * e->ffn_expert_ms_total / e->ffn_experts));
    if (e->st.layers > 0) c.t_attn = std::llround(1000.0 * e->route_ms_total_cal / static_cast<double>(e->st.layers));
    if (c.t_g >= c.t_io) c.t_g = c.t_io - 1;  // CostParams invariant t_g < t_io (cost_model.cpp:16)
    // Host lane: cpu_cost = beta*m + C, refit with fit_cost_params (OLS, cost_model.cpp:
    // 45-72) over the in-step samples (one per layer batch: mean tokens vs mean time per
    // expert, measured under PCIe contention) plus the create-time probe points (m1, m2
    // in isolation), which anchor the slope when the steps' token counts barely vary.
    // The fit is used when it is physical (beta > 0, C >= 0, R^2 >= 0.3); otherwise beta
    // stays the probe's and C is the median residual of the in-step samples.
    e->last_fit_used = 0;
    if (!e->cal_m.empty()) {
      std::vector<int32_t> m(e->cal_m.begin(), e->cal_m.end());
      std::vector<int64_t> us(e->cal_us.begin(), e->cal_us.end());
      m.insert(m.end(), e->probe_m.begin(), e->probe_m.end());
      us.insert(us.end(), e->probe_us.begin(), e->probe_us.end());
      double beta = 0, startup = 0, r2 = 0;
      const bool fit_ok = ps_fit_cost_params(m.data(), us.data(), static_cast<int>(m.size()), &beta, &startup, &r2) ==
                              PS_OK && beta > 0 && startup >= 0 && r2 >= 0.3;
      if (fit_ok) {
        c.beta = beta;
        c.startup = ps_to_ticks(startup);
        e->last_fit_used = 1;
      } else {
        std::vector<double> res;
        for (size_t i = 0; i < e->cal_m.size(); ++i) res.push_back(e->cal_us[i] - c.beta * e->cal_m[i]);
        std::nth_element(res.begin(), res.begin() + res.size() / 2, res.end());
        c.startup = std::max<int64_t>(0, ps_to_ticks(res[res.size() / 2]));
      }
    }
    if (ps_cost_params_validate(&c) != PS_OK) fail(PS_EINVAL, ps_last_error());
    e->cfg.cost = c;
    e->st.cost = c;
    if (out) *out = c;
  });
}

}  // extern "C"
