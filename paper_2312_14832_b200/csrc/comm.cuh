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

#include <cstdlib>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>
#include <algorithm>

#include "common.cuh"

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

inline void nccl_unique_id(void* out) {
  ncclUniqueId uid;
  nccl_check(NcclApi::Get().GetUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out, &uid, sizeof(uid));
}

}  // namespace pdhg
