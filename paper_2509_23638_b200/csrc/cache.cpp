// K5 as a stand-alone HBM expert cache (ps_cache_create / prefetch /
// ondemand / acquire / release): the AsyncIO channel of simulate_pipeline
// (simulator.cpp:61-242) for a caller that runs its own layer loop and FFN kernels.
//
//   * resident (layer, expert) pairs are copied to one HBM arena at create (the budget);
//   * every other expert is served from `n_slots` HBM staging slots, loaded from the
//     caller's host slab by the serial I/O channel (io_channel.hpp: one copy stream, FIFO,
//     queued prefetches cancellable, started copies non-interruptible);
//   * prefetch(l, e) queues a copy at the tail, ondemand(l, e) ahead of the queued
//     prefetches; a slot keeps its expert after release (a later request for it is a hit);
//   * acquire(l, e, stream) makes `stream` wait for the copy (event) and pins the slot;
//     release(l, e, stream) records when `stream` is done with it — the slot's next copy
//     waits for that (the dual-buffer rule R7 generalised to n slots).
// A request needing a slot when every slot is pinned or still loading fails with
// PS_ERUNTIME, like the simulator's prefetch-buffer overflow (simulator.cpp:209-212).
#include <cstring>
#include <memory>
#include <unordered_map>
#include <vector>

#include "io_channel.hpp"

struct ps_cache_s {
  ps_cache_config cfg{};
  std::vector<const void*> host;                // [L*E] caller's host slabs
  void* arena = nullptr;                         // resident slabs
  std::vector<const void*> resident;             // [L*E] device pointer or null
  struct Entry {
    ps::Slot slot;
    int key = -1;                                // l*E + e held (or being loaded), -1 = empty
    ps::IoJob* job = nullptr;                    // the copy that filled it
    int pins = 0;
    uint64_t last_use = 0;
  };
  std::vector<std::unique_ptr<Entry>> entries;
  std::vector<std::unique_ptr<ps::IoJob>> jobs;  // owned (a job lives as long as its entry)
  std::unordered_map<int, Entry*> by_key;
  std::unique_ptr<ps::IoChannel> io;
  std::vector<cudaEvent_t> events;
  uint64_t tick = 0;
  ps_cache_stats st{};
};

namespace ps {
namespace {

int key_of(const ps_cache_s& c, int layer, int expert) {
  if (layer < 0 || layer >= c.cfg.num_layers || expert < 0 || expert >= c.cfg.experts)
    fail(PS_ERANGE, "ps_cache: (layer, expert) out of range");
  return layer * c.cfg.experts + expert;
}

// A free slot: unpinned and not loading, least recently used first; empty slots first.
ps_cache_s::Entry* take_slot(ps_cache_s& c) {
  ps_cache_s::Entry* best = nullptr;
  for (auto& e : c.entries) {
    if (e->pins > 0) continue;
    if (e->job && e->job->state.load() == 0) continue;  // queued copy not issued yet
    if (e->key < 0) {
      best = e.get();
      break;
    }
    if (!best || e->last_use < best->last_use) best = e.get();
  }
  if (!best) fail(PS_ERUNTIME, "ps_cache: no free staging slot (all pinned or loading)");
  if (best->key >= 0) c.by_key.erase(best->key);
  return best;
}

cudaEvent_t new_event(ps_cache_s& c) {
  cudaEvent_t ev;
  PS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventBlockingSync));
  c.events.push_back(ev);
  return ev;
}

void request(ps_cache_s& c, int layer, int expert, bool ondemand) {
  const int key = key_of(c, layer, expert);
  if (c.resident[key]) {
    c.st.resident_hits++;
    return;
  }
  auto it = c.by_key.find(key);
  if (it != c.by_key.end()) {  // already present or on its way
    ps_cache_s::Entry* e = it->second;
    if (ondemand && e->job && e->job->kind == kPrefetch && e->job->state.load() == 0) {  // promote a queued prefetch
      for (IoJob* j : c.io->cancel_queued_prefetches()) {  // the others go back in their order
        j->state = 0;
        if (j != e->job) c.io->push(j);
      }
      e->job->kind = kOnDemand;
      c.io->push_front(e->job);
    }
    c.st.slot_hits++;
    return;
  }
  require(c.host[key] != nullptr, "ps_cache: expert has no host slab");
  ps_cache_s::Entry* e = take_slot(c);
  auto j = std::make_unique<IoJob>();
  j->kind = ondemand ? kOnDemand : kPrefetch;
  j->layer = layer;
  j->expert = expert;
  j->slot = &e->slot;
  j->dst = e->slot.dev;
  j->src = c.host[key];
  j->bytes = c.cfg.expert_bytes;
  j->wait_gen = e->slot.next_gen;  // after the slot's last release
  j->start_ev = new_event(c);
  j->done_ev = new_event(c);
  e->key = key;
  e->job = j.get();
  e->last_use = ++c.tick;
  c.by_key[key] = e;
  IoJob* raw = j.get();
  c.jobs.push_back(std::move(j));
  if (ondemand) {
    c.io->push_front(raw);
    c.st.ondemand_loads++;
  } else {
    c.io->push(raw);
    c.st.prefetches++;
  }
}

void destroy(ps_cache_s& c) {
  if (c.io) {
    c.io->abandon_queued();
    c.io->drain();
  }
  c.io.reset();
  for (auto& e : c.entries) {
    if (e->slot.dev) cudaFree(e->slot.dev);
    if (e->slot.free_ev) cudaEventDestroy(e->slot.free_ev);
  }
  if (c.arena) cudaFree(c.arena);
  for (cudaEvent_t ev : c.events) cudaEventDestroy(ev);
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

ps_status ps_cache_create(const ps_cache_config* cfg, ps_cache* out) {
  auto c = std::make_unique<ps_cache_s>();
  ps_status s = guarded([&] {
    require(cfg && out && cfg->host_slabs, "ps_cache_create: null argument");
    require(cfg->num_layers >= 1 && cfg->experts >= 1 && cfg->expert_bytes > 0 && cfg->n_slots >= 2,
            "ps_cache_create: bad shape (n_slots >= 2)");
    c->cfg = *cfg;
    PS_CUDA(cudaSetDevice(cfg->device));
    const size_t LE = static_cast<size_t>(cfg->num_layers) * cfg->experts;
    c->host.assign(cfg->host_slabs, cfg->host_slabs + LE);
    c->resident.assign(LE, nullptr);
    require(static_cast<uint64_t>(cfg->n_resident) * cfg->expert_bytes <= cfg->budget_bytes,
            "ps_cache_create: resident set exceeds the HBM budget");
    if (cfg->n_resident > 0) PS_CUDA(cudaMalloc(&c->arena, static_cast<size_t>(cfg->n_resident) * cfg->expert_bytes));
    for (int i = 0; i < cfg->n_resident; ++i) {
      const int key = key_of(*c, cfg->resident[2 * i], cfg->resident[2 * i + 1]);
      require(c->host[key] != nullptr, "ps_cache_create: resident expert has no host slab");
      char* dst = static_cast<char*>(c->arena) + static_cast<size_t>(i) * cfg->expert_bytes;
      PS_CUDA(cudaMemcpy(dst, c->host[key], cfg->expert_bytes, cudaMemcpyHostToDevice));
      c->resident[key] = dst;
    }
    for (int i = 0; i < cfg->n_slots; ++i) {
      auto e = std::make_unique<ps_cache_s::Entry>();
      PS_CUDA(cudaMalloc(&e->slot.dev, cfg->expert_bytes));
      PS_CUDA(cudaEventCreateWithFlags(&e->slot.free_ev, cudaEventDisableTiming));
      c->entries.push_back(std::move(e));
    }
    c->io = std::make_unique<IoChannel>(cfg->device, 2);
  });
  if (s != PS_OK) {
    destroy(*c);
    return s;
  }
  *out = c.release();
  return PS_OK;
}

ps_status ps_cache_destroy(ps_cache c) {
  return guarded([&] {
    if (!c) return;
    destroy(*c);
    delete c;
  });
}

ps_status ps_cache_prefetch(ps_cache c, int layer, int expert) {
  return guarded([&] {
    require(c != nullptr, "ps_cache_prefetch: null cache");
    request(*c, layer, expert, false);
  });
}

ps_status ps_cache_ondemand(ps_cache c, int layer, int expert) {
  return guarded([&] {
    require(c != nullptr, "ps_cache_ondemand: null cache");
    request(*c, layer, expert, true);
  });
}

ps_status ps_cache_acquire(ps_cache c, int layer, int expert, void* stream, const void** dev_slab) {
  return guarded([&] {
    require(c && dev_slab, "ps_cache_acquire: null argument");
    const int key = key_of(*c, layer, expert);
    if (c->resident[key]) {
      *dev_slab = c->resident[key];
      return;
    }
    auto it = c->by_key.find(key);
    if (it == c->by_key.end()) fail(PS_EINVAL, "ps_cache_acquire: expert was neither prefetched nor requested");
    ps_cache_s::Entry* e = it->second;
    c->io->wait_issued(e->job);  // host: until the copy is on the copy stream
    if (e->job->state.load() == 2) fail(PS_ERUNTIME, "ps_cache_acquire: the expert's prefetch was cancelled");
    PS_CUDA(cudaStreamWaitEvent(as_stream(stream), e->job->done_ev, 0));
    e->pins++;
    e->last_use = ++c->tick;
    *dev_slab = e->slot.dev;
  });
}

ps_status ps_cache_release(ps_cache c, int layer, int expert, void* stream) {
  return guarded([&] {
    require(c != nullptr, "ps_cache_release: null cache");
    const int key = key_of(*c, layer, expert);
    if (c->resident[key]) return;
    auto it = c->by_key.find(key);
    if (it == c->by_key.end() || it->second->pins == 0) fail(PS_EINVAL, "ps_cache_release: expert is not acquired");
    ps_cache_s::Entry* e = it->second;
    PS_CUDA(cudaEventRecord(e->slot.free_ev, as_stream(stream)));  // the slot's next copy waits for this
    e->slot.next_gen += 1;
    e->slot.recorded_gen.store(e->slot.next_gen);
    e->pins--;
    c->io->notify();
  });
}

ps_status ps_cache_cancel_prefetches(ps_cache c, int* n_cancelled) {
  return guarded([&] {
    require(c != nullptr, "ps_cache_cancel_prefetches: null cache");
    int n = 0;
    for (IoJob* j : c->io->cancel_queued_prefetches()) {  // R2: not started -> dropped
      for (auto& e : c->entries)
        if (e->job == j) {
          c->by_key.erase(e->key);
          e->key = -1;
          e->job = nullptr;
        }
      ++n;
    }
    c->st.prefetches_cancelled += n;
    if (n_cancelled) *n_cancelled = n;
  });
}

ps_status ps_cache_get_stats(ps_cache c, ps_cache_stats* out) {
  return guarded([&] {
    require(c && out, "ps_cache_get_stats: null argument");
    *out = c->st;
  });
}

ps_status ps_cache_sync(ps_cache c) {
  return guarded([&] {
    require(c != nullptr, "ps_cache_sync: null cache");
    c->io->drain();
    c->io->check();
  });
}

}  // extern "C"
