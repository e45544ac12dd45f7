// Exchange layer of the sharded solver.
//
// K is split into P row blocks (K x, CSR) and P column blocks (K^T y, CSC).
// Every vector lives in a PADDED index space: block b's entries occupy
// [b * slice, b * slice + size_b), so one in-place all-gather of `slice`
// doubles per rank rebuilds the full vector on every rank, and a column
// index of K (already remapped into that space at setup) addresses the
// gathered buffer directly -- no unpacking, no extra copy.
//
// Implementations:
//   LocalComm  every shard lives in this process and writes straight into the
//              shared full buffers: exchanges are no-ops (P = 1, and the
//              in-process multi-shard mode the parity tests drive on one GPU);
//   NcclComm   one shard per process/GPU; ncclAllGather in place over
//              NVLink/NVSwitch, ncclAllReduce for the check pack. NCCL is
//              dlopen'ed on first use (whichever libnccl.so.2 the process
//              already holds -- torch's -- or the system one), so the library
//              has no link-time NCCL dependency. Calls are stream-ordered and
//              graph-capturable, so they sit inside the captured PDHG block.
#pragma once

#include <dlfcn.h>

#include <cstdio>

#include <cstdlib>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "darray.cuh"

namespace pdhg {

// Ghost-only exchange of one gather pattern: instead of the
// whole vector, each rank receives just the entries its matrix block reads
// from other blocks (the staircase's one boundary stage), and sends the
// entries of its own slice that other blocks read. Index lists are padded
// positions; per-peer ranges in send/recv are [off[p], off[p + 1]).
struct GhostPlan {
  bool use = false;   // ghost exchange (all ranks agree) instead of all-gather
  int64_t slice = 0;  // padded slice of the pattern's vector
  int32_t* send_idx = nullptr;
  int32_t* recv_idx = nullptr;
  double* send_buf = nullptr;
  double* recv_buf = nullptr;
  std::vector<int64_t> send_off, recv_off;  // world + 1 each
};

static __global__ void k_ghost_pack(const double* __restrict__ buf, const int32_t* __restrict__ idx, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = buf[idx[i]];
}
static __global__ void k_ghost_unpack(double* __restrict__ buf, const int32_t* __restrict__ idx, const double* in, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[idx[i]] = in[i];
}

class Comm {
 public:
  virtual ~Comm() = default;
  virtual bool local() const = 0;
  // Collectives may be captured into CUDA graphs (false: the loopback
  // transport, whose event barriers cannot cross captures).
  virtual bool graphs() const { return true; }
  // In place: this rank's slice is buf[rank * slice, (rank + 1) * slice).
  virtual void AllGather(double* buf, int64_t slice, cudaStream_t st) = 0;
  // The entries this rank's block reads (ghost plan), or the full vector.
  virtual void Exchange(double* buf, const GhostPlan& plan, cudaStream_t st) { AllGather(buf, plan.slice, st); }
  virtual void AllReduceSum(double* buf, int64_t n, cudaStream_t st) = 0;
  virtual void AllReduceMax(double* buf, int64_t n, cudaStream_t st) = 0;
};

class LocalComm final : public Comm {
 public:
  bool local() const override { return true; }
  void AllGather(double*, int64_t, cudaStream_t) override {}
  void Exchange(double*, const GhostPlan&, cudaStream_t) override {}
  void AllReduceSum(double*, int64_t, cudaStream_t) override {}
  void AllReduceMax(double*, int64_t, cudaStream_t) override {}
};

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  static const NcclApi& Get() {
    static NcclApi api = Load();
    if (!api.AllGather) throw Error(4, "NCCL unavailable: libnccl.so.2 could not be loaded");
    return api;
  }

 private:
  static NcclApi Load() {
    NcclApi a;
    // Already in the process (e.g. PyTorch's) -> that one; else the library
    // PDHG_NCCL_LIB names (the Python layer points it at the NCCL PyTorch
    // ships, so a later `import torch` resolves against the same build);
    // else the system's.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    const char* path = std::getenv("PDHG_NCCL_LIB");
    if (!h && path && path[0]) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.Send = reinterpret_cast<decltype(a.Send)>(dlsym(h, "ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(dlsym(h, "ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    if (!a.GetUniqueId || !a.CommInitRank || !a.CommDestroy || !a.AllReduce || !a.GetErrorString || !a.Send ||
        !a.Recv || !a.GroupStart || !a.GroupEnd)
      a.AllGather = nullptr;
    return a;
  }
};

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(4, std::string(what) + ": " + NcclApi::Get().GetErrorString(r));
}

class NcclComm final : public Comm {
 public:
  NcclComm(const void* id, int world, int rank) : rank_(rank) {
    const NcclApi& api = NcclApi::Get();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    nccl_check(api.CommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) NcclApi::Get().CommDestroy(comm_);
  }
  bool local() const override { return false; }
  void AllGather(double* buf, int64_t slice, cudaStream_t st) override {
    if (slice <= 0) return;
    nccl_check(NcclApi::Get().AllGather(buf + rank_ * slice, buf, static_cast<size_t>(slice), ncclFloat64, comm_, st),
               "ncclAllGather");
  }
  // Pack the entries peers read from this slice, one grouped send/recv per
  // peer pair (only pairs with a non-empty list), unpack into the gathered
  // positions. Stream-ordered and graph-capturable like the collectives.
  void Exchange(double* buf, const GhostPlan& plan, cudaStream_t st) override {
    if (!plan.use) return AllGather(buf, plan.slice, st);
    const NcclApi& api = NcclApi::Get();
    const int world = static_cast<int>(plan.send_off.size()) - 1;
    const int64_t ns = plan.send_off[world], nr = plan.recv_off[world];
    if (ns) k_ghost_pack<<<static_cast<int>(std::min<int64_t>((ns + 255) / 256, 1184)), 256, 0, st>>>(
        buf, plan.send_idx, plan.send_buf, ns);
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int p = 0; p < world; ++p) {
      if (p == rank_) continue;
      const int64_t sc = plan.send_off[p + 1] - plan.send_off[p], rc = plan.recv_off[p + 1] - plan.recv_off[p];
      if (sc) nccl_check(api.Send(plan.send_buf + plan.send_off[p], sc, ncclFloat64, p, comm_, st), "ncclSend");
      if (rc) nccl_check(api.Recv(plan.recv_buf + plan.recv_off[p], rc, ncclFloat64, p, comm_, st), "ncclRecv");
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    if (nr) k_ghost_unpack<<<static_cast<int>(std::min<int64_t>((nr + 255) / 256, 1184)), 256, 0, st>>>(
        buf, plan.recv_idx, plan.recv_buf, nr);
  }
  void AllReduceSum(double* buf, int64_t n, cudaStream_t st) override {
    nccl_check(NcclApi::Get().AllReduce(buf, buf, static_cast<size_t>(n), ncclFloat64, ncclSum, comm_, st),
               "ncclAllReduce");
  }
  void AllReduceMax(double* buf, int64_t n, cudaStream_t st) override {
    nccl_check(NcclApi::Get().AllReduce(buf, buf, static_cast<size_t>(n), ncclFloat64, ncclMax, comm_, st),
               "ncclAllReduce");
  }

 private:
  ncclComm_t comm_ = nullptr;
  int rank_ = 0;
};

// ---------------------------------------------------------------- loopback
// In-process loopback transport (tests, one GPU): P one-shard sessions in ONE
// process on ONE device, each driven by its own host thread, run the session's
// multi-rank code path -- padded slices, ghost pack / send / recv / unpack,
// per-rank check packs summed over ranks, rank 0's clock, the observer-abort
// reduction -- with this transport in place of NCCL. It replaces only NCCL's
// data movement:
//  * a host rendezvous per collective call: every rank posts its argument
//    (buffer or ghost plan) and receives every peer's;
//  * device ordering by CUDA events, never by spinning kernels: a device
//    barrier records an event on this rank's stream, exchanges the events
//    through a host rendezvous and makes the stream wait on every peer's.
//    Two barriers per collective: "ready" before reading peers' buffers,
//    "done" after, so no rank overwrites data a peer is still reading. (Ranks
//    that spin on each other's flags from different streams of one device
//    have no forward-progress guarantee -- a spinning kernel can hold the
//    hardware queue its peer's kernel waits in -- and deadlocked here.)
//    An event wait cannot cross stream captures, so sessions over this
//    transport run their blocks eagerly instead of as CUDA graphs
//    (Comm::graphs); the kernels and their order are the same;
//  * data: kernels on the rank's stream (all-gather, ghost segments) or a
//    fixed-order kernel (all-reduce: sum over ranks 0..P-1, the order the
//    in-process shard mode uses -- so results are bitwise comparable with it).
constexpr int kLoopMaxRanks = 16;
constexpr int64_t kLoopScratch = 1 << 16;  // doubles: the largest all-reduce
constexpr int kLoopEvents = 4;             // event ring per rank (a rank runs at most one barrier ahead)

struct LoopGroup {
  int P = 0;
  int device = 0;
  std::mutex mu;
  std::condition_variable cv;
  struct Slot {
    std::vector<const void*> arg;
    int posted = 0, taken = 0;
  };
  std::map<uint64_t, Slot> slots;

  std::vector<const void*> Rendezvous(uint64_t seq, int rank, const void* arg, const char* what) {
    static const bool trace = [] {
      const char* e = std::getenv("PDHG_LOOP_TRACE");
      return e && e[0] == '1';
    }();
    if (trace) std::fprintf(stderr, "[loop] rank %d call %llu %s\n", rank, (unsigned long long)seq, what);
    std::unique_lock<std::mutex> lk(mu);
    Slot& s = slots[seq];
    if (s.arg.empty()) s.arg.assign(static_cast<size_t>(P), nullptr);
    s.arg[rank] = arg;
    ++s.posted;
    cv.notify_all();
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return s.posted == P; })) {
      std::string who;
      for (int r = 0; r < P; ++r)
        if (!s.arg[r]) who += " " + std::to_string(r);
      throw Error(4, "loopback rendezvous timed out at call " + std::to_string(seq) + " (" + what +
                         "), missing ranks" + who);
    }
    std::vector<const void*> out = s.arg;
    if (++s.taken == P) slots.erase(seq);
    return out;
  }

  static std::shared_ptr<LoopGroup> Join(uint64_t key, int P, int device) {
    static std::mutex reg_mu;
    static std::map<uint64_t, std::weak_ptr<LoopGroup>> reg;
    std::lock_guard<std::mutex> g(reg_mu);
    std::shared_ptr<LoopGroup> grp = reg[key].lock();
    if (!grp) {
      grp = std::make_shared<LoopGroup>();
      grp->P = P;
      grp->device = device;
      reg[key] = grp;
    }
    if (grp->P != P || grp->device != device) throw Error(1, "loopback group: world / device mismatch");
    return grp;
  }
};

struct LoopPtrs {
  const double* p[kLoopMaxRanks];
};
// Up to kLoopMaxRanks (src, dst, n) segments copied by one kernel.
struct LoopCopies {
  const double* src[kLoopMaxRanks];
  double* dst[kLoopMaxRanks];
  int64_t n[kLoopMaxRanks];
  int count;
};
static __global__ void k_loop_copy(LoopCopies c) {
  for (int k = 0; k < c.count; ++k) {
    const double* __restrict__ s = c.src[k];
    double* __restrict__ d = c.dst[k];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < c.n[k]; i += (int64_t)gridDim.x * blockDim.x)
      d[i] = s[i];
  }
}
inline void loop_copy(const LoopCopies& c, cudaStream_t st) {
  int64_t mx = 0;
  for (int k = 0; k < c.count; ++k) mx = std::max(mx, c.n[k]);
  if (!mx) return;
  k_loop_copy<<<static_cast<int>(std::min<int64_t>((mx + 255) / 256, 592)), 256, 0, st>>>(c);
}
static __global__ void k_loop_reduce(LoopPtrs src, int P, int64_t n, int mx, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = src.p[0][i];
    for (int r = 1; r < P; ++r) {
      const double w = src.p[r][i];
      v = mx ? ((v < w) ? w : v) : v + w;
    }
    out[i] = v;
  }
}

class LoopbackComm final : public Comm {
 public:
  LoopbackComm(uint64_t key, int world, int rank, int device) : rank_(rank), P_(world) {
    if (world < 1 || world > kLoopMaxRanks) throw Error(1, "loopback world must be 1..16");
    grp_ = LoopGroup::Join(key, world, device);
    scratch_.alloc(kLoopScratch);
    for (cudaEvent_t& e : ev_) PDHG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  ~LoopbackComm() override {
    for (cudaEvent_t e : ev_)
      if (e) cudaEventDestroy(e);
  }
  bool local() const override { return false; }
  bool graphs() const override { return false; }
  void AllGather(double* buf, int64_t slice, cudaStream_t st) override {
    const std::vector<const void*> peers = grp_->Rendezvous(++hseq_, rank_, buf, "allgather");
    if (slice <= 0) return;
    Barrier(st);
    LoopCopies c{};
    for (int p = 0; p < P_; ++p) {
      if (p == rank_) continue;
      c.src[c.count] = static_cast<const double*>(peers[p]) + p * slice;
      c.dst[c.count] = buf + p * slice;
      c.n[c.count++] = slice;
    }
    loop_copy(c, st);
    Barrier(st);
  }
  void Exchange(double* buf, const GhostPlan& plan, cudaStream_t st) override {
    if (!plan.use) return AllGather(buf, plan.slice, st);
    const std::vector<const void*> peers = grp_->Rendezvous(++hseq_, rank_, &plan, "ghost");
    const int64_t ns = plan.send_off[P_], nr = plan.recv_off[P_];
    if (ns) k_ghost_pack<<<static_cast<int>(std::min<int64_t>((ns + 255) / 256, 1184)), 256, 0, st>>>(
        buf, plan.send_idx, plan.send_buf, ns);
    LoopCopies c{};
    for (int p = 0; p < P_; ++p) {
      if (p == rank_) continue;
      const GhostPlan& q = *static_cast<const GhostPlan*>(peers[p]);
      const int64_t rc = plan.recv_off[p + 1] - plan.recv_off[p];
      const int64_t sc = q.send_off[rank_ + 1] - q.send_off[rank_];
      if (rc != sc)
        throw Error(4, "loopback ghost exchange: rank " + std::to_string(rank_) + " expects " + std::to_string(rc) +
                           " entries from rank " + std::to_string(p) + ", which sends " + std::to_string(sc));
      if (rc) {
        c.src[c.count] = q.send_buf + q.send_off[rank_];
        c.dst[c.count] = plan.recv_buf + plan.recv_off[p];
        c.n[c.count++] = rc;
      }
    }
    Barrier(st);
    loop_copy(c, st);
    Barrier(st);
    if (nr) k_ghost_unpack<<<static_cast<int>(std::min<int64_t>((nr + 255) / 256, 1184)), 256, 0, st>>>(
        buf, plan.recv_idx, plan.recv_buf, nr);
  }
  void AllReduceSum(double* buf, int64_t n, cudaStream_t st) override { Reduce(buf, n, false, st); }
  void AllReduceMax(double* buf, int64_t n, cudaStream_t st) override { Reduce(buf, n, true, st); }

 private:
  // Device barrier: every rank's stream passes this point only after every
  // rank's stream has reached it (event record -> host exchange -> waits).
  // The host rendezvous orders each record before the peers' waits, and a
  // rank can be at most one barrier ahead of a peer, so a ring of
  // kLoopEvents events is never re-recorded before the peers waited on it.
  void Barrier(cudaStream_t st) {
    cudaEvent_t e = ev_[nev_++ % kLoopEvents];
    PDHG_CUDA(cudaEventRecord(e, st));
    const std::vector<const void*> evs = grp_->Rendezvous(++hseq_, rank_, e, "barrier");
    for (int p = 0; p < P_; ++p)
      if (p != rank_) PDHG_CUDA(cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(const_cast<void*>(evs[p])), 0));
  }
  void Reduce(double* buf, int64_t n, bool mx, cudaStream_t st) {
    const std::vector<const void*> peers = grp_->Rendezvous(++hseq_, rank_, buf, mx ? "max" : "sum");
    if (n <= 0) return;
    if (n > kLoopScratch) throw Error(4, "loopback all-reduce larger than its scratch");
    LoopPtrs src{};
    for (int p = 0; p < P_; ++p) src.p[p] = static_cast<const double*>(peers[p]);
    Barrier(st);
    k_loop_reduce<<<static_cast<int>(std::min<int64_t>((n + 255) / 256, 256)), 256, 0, st>>>(src, P_, n, mx,
                                                                                          scratch_.p);
    Barrier(st);
    LoopCopies c{};
    c.src[0] = scratch_.p;
    c.dst[0] = buf;
    c.n[0] = n;
    c.count = 1;
    loop_copy(c, st);
  }

  std::shared_ptr<LoopGroup> grp_;
  DArray<double> scratch_;
  cudaEvent_t ev_[kLoopEvents] = {};
  uint64_t nev_ = 0;
  uint64_t hseq_ = 0;
  int rank_ = 0, P_ = 1;
};

// A loopback id: the 8-byte magic, then the group key (128 bytes like an
// ncclUniqueId, so it travels through the same pdhg_shard_spec field).
constexpr char kLoopMagic[8] = {'P', 'D', 'H', 'G', 'L', 'O', 'O', 'P'};
inline bool is_loopback_id(const void* id) { return id && std::memcmp(id, kLoopMagic, 8) == 0; }
inline uint64_t loopback_key(const void* id) {
  uint64_t k;
  std::memcpy(&k, static_cast<const char*>(id) + 8, sizeof(k));
  return k;
}
inline void loopback_id(void* out) {
  static std::atomic<uint64_t> next{1};
  std::memset(out, 0, 128);
  std::memcpy(out, kLoopMagic, 8);
  const uint64_t k = (static_cast<uint64_t>(std::chrono::steady_clock::now().time_since_epoch().count()) << 16) ^
                     next.fetch_add(1);
  std::memcpy(static_cast<char*>(out) + 8, &k, sizeof(k));
}

inline void nccl_unique_id(void* out) {
  ncclUniqueId uid;
  nccl_check(NcclApi::Get().GetUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out, &uid, sizeof(uid));
}

}  // namespace pdhg
