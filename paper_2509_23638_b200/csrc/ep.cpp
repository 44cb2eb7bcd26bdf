// Expert parallelism: experts of every layer are owned by rank
// e % world; each rank routes its own tokens (data parallel), sends the routed rows to
// the owners (all-to-all dispatch), runs its local experts through its own HBM cache /
// loader, and gets the expert outputs back (all-to-all combine) for the weighted sum at
// the token's home rank.
//
// This file holds the host-side pieces: the receive plan (which permuted local row is
// which received row) and the NCCL transport (grouped ncclSend/ncclRecv per peer over
// NVLink/NVSwitch). NCCL is resolved at run time (dlopen "libnccl.so.2" — the copy
// torch already loaded, or the system one), so the library has no link-time NCCL
// dependency and EP fails loudly (PS_ENCCL) where NCCL is absent.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "cuda_host.hpp"

namespace ps {
namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.handle) break;
    }
    if (!api.handle) return;
    auto sym = [](const char* n) { return dlsym(api.handle, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!api.handle || !api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.GroupStart ||
      !api.GroupEnd)
    fail(PS_ENCCL, "NCCL (libnccl.so.2) is not available");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* msg = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    fail(PS_ENCCL, std::string(what) + ": " + msg);
  }
}

// In-process transport: `world` ranks of one process, one host thread per rank (each
// driving its own engine and streams, on any devices). Same contract as the NCCL
// grouped send/recv all-to-all — stream-ordered on every rank's stream, per-peer byte
// counts, source/destination-major segments — built from CUDA events and peer copies:
//   1. each rank records `ready` on its stream (its send buffer is written) and posts
//      its buffers; host barrier;
//   2. each rank waits on every peer's `ready`, copies the peer's segment for it into
//      its own receive buffer on its own stream, records `done`; host barrier;
//   3. each rank's stream waits on every peer's `done`, so nothing later on a rank's
//      stream (the next write of its send buffer) overtakes a peer still reading it.
// One process can thus run the real EP engine at G = 2/4/8 on one GPU (tests), with
// exactly the engine code that runs over NCCL across GPUs.
struct LoopGroup {
  explicit LoopGroup(int w) : world(w), posts(w) {}
  struct Post {
    const char* send = nullptr;
    char* recv = nullptr;
    std::vector<uint64_t> sb, rb;
    cudaStream_t stream = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
    int device = 0;
  };
  int world;
  std::vector<Post> posts;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  void barrier() {
    std::unique_lock<std::mutex> g(mu);
    const uint64_t my = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    // A rank that failed outside the collective never arrives: time out instead of
    // hanging every peer (NCCL would block the same way; tests want an error).
    if (!cv.wait_for(g, std::chrono::seconds(300), [&] { return gen != my || broken; })) {
      broken = true;
      cv.notify_all();
    }
    if (broken) fail(PS_ENCCL, "loopback all-to-all: a peer rank failed or never arrived");
  }
  void abort() {
    std::lock_guard<std::mutex> g(mu);
    broken = true;
    cv.notify_all();
  }
};

}  // namespace
}  // namespace ps

struct ps_ep_comm_s {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  std::shared_ptr<ps::LoopGroup> loop;  // in-process transport (ps_ep_loopback_create)
  cudaEvent_t ready = nullptr, done = nullptr;
};

namespace ps {
namespace {

void loop_all_to_all(ps_ep_comm_s* c, const void* send, const uint64_t* send_bytes, void* recv,
                     const uint64_t* recv_bytes, cudaStream_t s) {
  LoopGroup& g = *c->loop;
  const int W = g.world, r = c->rank;
  int dev = 0;
  PS_CUDA(cudaGetDevice(&dev));
  try {
    PS_CUDA(cudaEventRecord(c->ready, s));
    LoopGroup::Post& me = g.posts[r];
    me.send = static_cast<const char*>(send);
    me.recv = static_cast<char*>(recv);
    me.sb.assign(send_bytes, send_bytes + W);
    me.rb.assign(recv_bytes, recv_bytes + W);
    me.stream = s;
    me.ready = c->ready;
    me.done = c->done;
    me.device = dev;
    g.barrier();  // every rank posted
    uint64_t ro = 0;
    for (int p = 0; p < W; ++p) {
      const LoopGroup::Post& peer = g.posts[p];
      uint64_t so = 0;
      for (int q = 0; q < r; ++q) so += peer.sb[q];
      require(peer.sb[r] == me.rb[p], "loopback all-to-all: send/recv byte counts disagree");
      if (me.rb[p]) {
        if (p != r) PS_CUDA(cudaStreamWaitEvent(s, peer.ready, 0));
        if (peer.device == dev)
          PS_CUDA(cudaMemcpyAsync(me.recv + ro, peer.send + so, me.rb[p], cudaMemcpyDeviceToDevice, s));
        else
          PS_CUDA(cudaMemcpyPeerAsync(me.recv + ro, dev, peer.send + so, peer.device, me.rb[p], s));
      }
      ro += me.rb[p];
    }
    PS_CUDA(cudaEventRecord(c->done, s));
    g.barrier();  // every rank's copies are enqueued
    for (int p = 0; p < W; ++p)
      if (p != r) PS_CUDA(cudaStreamWaitEvent(s, g.posts[p].done, 0));
    g.barrier();  // nobody re-posts (overwrites its entry) before every peer read it
  } catch (...) {
    g.abort();
    throw;
  }
}

}  // namespace
}  // namespace ps

using namespace ps;

extern "C" {

ps_status ps_ep_recv_plan(const int32_t* recv_counts, int G, int E_loc, int32_t* offsets, int32_t* perm_src,
                          int32_t* recv_seg) {
  return guarded([&] {
    require(G >= 1 && E_loc >= 1 && recv_counts && offsets && recv_seg, "ps_ep_recv_plan: bad arguments");
    // Received buffer = source-major segments; within a segment, rows are ordered by
    // local expert (the sender permuted by owner-major virtual id), then token, slot.
    recv_seg[0] = 0;
    for (int s = 0; s < G; ++s) {
      int seg = 0;
      for (int j = 0; j < E_loc; ++j) {
        require(recv_counts[s * E_loc + j] >= 0, "ps_ep_recv_plan: negative count");
        seg += recv_counts[s * E_loc + j];
      }
      recv_seg[s + 1] = recv_seg[s] + seg;
    }
    // Local expert-major order: expert j's rows are source 0's block, then source 1's...
    offsets[0] = 0;
    for (int j = 0; j < E_loc; ++j) {
      int tot = 0;
      for (int s = 0; s < G; ++s) tot += recv_counts[s * E_loc + j];
      offsets[j + 1] = offsets[j] + tot;
    }
    if (!perm_src) return;
    for (int s = 0; s < G; ++s) {
      int in_seg = recv_seg[s];
      for (int j = 0; j < E_loc; ++j) {
        int before = 0;  // rows of expert j from sources < s
        for (int s2 = 0; s2 < s; ++s2) before += recv_counts[s2 * E_loc + j];
        const int c = recv_counts[s * E_loc + j];
        for (int r = 0; r < c; ++r) perm_src[offsets[j] + before + r] = in_seg + r;
        in_seg += c;
      }
    }
  });
}

int ps_ep_local_experts(int E, int G, int rank) {
  return rank < E % G || E % G == 0 ? (E + G - 1) / G : E / G;
}

ps_status ps_ep_unique_id(char* out, int cap) {
  return guarded([&] {
    require(cap >= NCCL_UNIQUE_ID_BYTES, "ps_ep_unique_id: buffer < 128 bytes");
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

ps_status ps_ep_comm_create(const char* unique_id, int rank, int world, int device, ps_ep_comm* out) {
  return guarded([&] {
    require(world >= 1 && rank >= 0 && rank < world, "ps_ep_comm_create: bad rank/world");
    PS_CUDA(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(id.internal, unique_id, NCCL_UNIQUE_ID_BYTES);
    auto c = std::make_unique<ps_ep_comm_s>();
    c->rank = rank;
    c->world = world;
    nccl_check(nccl().CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
    *out = c.release();
  });
}

ps_status ps_ep_loopback_create(int world, int device, ps_ep_comm* comms) {
  return guarded([&] {
    require(world >= 1 && world <= 64 && comms, "ps_ep_loopback_create: bad world");
    PS_CUDA(cudaSetDevice(device));
    auto group = std::make_shared<LoopGroup>(world);
    std::vector<std::unique_ptr<ps_ep_comm_s>> out;
    for (int r = 0; r < world; ++r) {
      auto c = std::make_unique<ps_ep_comm_s>();
      c->rank = r;
      c->world = world;
      c->loop = group;
      PS_CUDA(cudaEventCreateWithFlags(&c->ready, cudaEventDisableTiming));
      PS_CUDA(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
      out.push_back(std::move(c));
    }
    for (int r = 0; r < world; ++r) comms[r] = out[r].release();
  });
}

ps_status ps_ep_comm_destroy(ps_ep_comm c) {
  return guarded([&] {
    if (!c) return;
    if (c->comm) nccl().CommDestroy(c->comm);
    if (c->ready) cudaEventDestroy(c->ready);
    if (c->done) cudaEventDestroy(c->done);
    delete c;
  });
}

// All-to-all with per-peer byte counts (grouped send/recv; displacements are the
// prefix sums, i.e. source/destination-major contiguous segments).
ps_status ps_ep_all_to_all(ps_ep_comm c, const void* send, const uint64_t* send_bytes, void* recv,
                           const uint64_t* recv_bytes, void* stream) {
  return guarded([&] {
    require(c != nullptr, "ps_ep_all_to_all: null communicator");
    cudaStream_t s = as_stream(stream);
    if (c->loop) {
      loop_all_to_all(c, send, send_bytes, recv, recv_bytes, s);
      return;
    }
    const NcclApi& api = nccl();
    uint64_t so = 0, ro = 0;
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < c->world; ++p) {
      if (send_bytes[p])
        nccl_check(api.Send(static_cast<const char*>(send) + so, send_bytes[p], ncclUint8, p, c->comm, s), "ncclSend");
      if (recv_bytes[p])
        nccl_check(api.Recv(static_cast<char*>(recv) + ro, recv_bytes[p], ncclUint8, p, c->comm, s), "ncclRecv");
      so += send_bytes[p];
      ro += recv_bytes[p];
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
  });
}

int ps_ep_comm_rank(ps_ep_comm c) { return c ? c->rank : -1; }
int ps_ep_comm_world(ps_ep_comm c) { return c ? c->world : 0; }

}  // extern "C"
