#include <cuda.h>

#include <cstring>
#include <map>
#include <utility>

#include "comm.hpp"
#include "kernels.hpp"

namespace spl {

namespace {

constexpr int kMaxLocal = 16;
struct PtrPack {
  const void* p[kMaxLocal];
};

template <typename T>
__global__ void rs_local_k(PtrPack parts, int nparts, int64_t offset, int64_t n, T* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = to_f(static_cast<const T*>(parts.p[0])[offset + i]);
    for (int r = 1; r < nparts; ++r) acc += to_f(static_cast<const T*>(parts.p[r])[offset + i]);
    out[i] = from_f<T>(acc);
  }
}

inline int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > kNumSMs * 16) g = kNumSMs * 16;
  return (int)(g < 1 ? 1 : g);
}

// ---------------------------------------------------------------- peer address exchange
// A buffer is named to the peers by (IPC handle of its allocation, offset): layer buffers may
// live inside a pooled allocation (stack workspaces), and CUDA IPC exports whole allocations.
struct PeerEntry {
  cudaIpcMemHandle_t handle;
  uint64_t offset;
};
PeerEntry peer_entry(const void* p) {
  using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static RangeFn range = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    SPL_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
    if (f == nullptr || q != cudaDriverEntryPointSuccess) raise(3, "cuMemGetAddressRange unavailable");
    return reinterpret_cast<RangeFn>(f);
  }();
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)p) != CUDA_SUCCESS) raise(3, "cuMemGetAddressRange failed");
  PeerEntry e;
  SPL_CUDA(cudaIpcGetMemHandle(&e.handle, (void*)base));
  e.offset = (uint64_t)((CUdeviceptr)p - base);
  return e;
}
// Opened peer allocations, one mapping per (peer, allocation) for the process's lifetime
// (closed when the transport is destroyed).
class PeerMaps {
 public:
  const void* open(int q, const PeerEntry& e) {
    std::string key(reinterpret_cast<const char*>(&e.handle), sizeof e.handle);
    key += std::to_string(q);
    auto it = maps_.find(key);
    if (it == maps_.end()) {
      void* p = nullptr;
      SPL_CUDA(cudaIpcOpenMemHandle(&p, e.handle, cudaIpcMemLazyEnablePeerAccess));
      it = maps_.emplace(std::move(key), p).first;
    }
    return static_cast<const char*>(it->second) + e.offset;
  }
  ~PeerMaps() {
    for (auto& kv : maps_) cudaIpcCloseMemHandle(kv.second);
  }

 private:
  std::map<std::string, void*> maps_;
};

// ---------------------------------------------------------------- peer-memory protocol kernels
__device__ __forceinline__ uint32_t ld_acq_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// A wait that gives up after 20 s (a peer that never arrives): it records the failure in
// err[0] and traps, so the rank's next synchronisation fails loudly instead of the GPU hanging.
__device__ __forceinline__ void spin_until_ge(const uint32_t* p, uint32_t target, int* err) {
  const uint64_t t0 = gtimer();
  while ((int32_t)(ld_acq_sys(p) - target) < 0) {
    __nanosleep(256);
    if (gtimer() - t0 > 20000000000ull) {
      atomicExch(err, 1);
      __trap();
    }
  }
}

struct PeerPtrs {
  void* p[kMaxLocal];
};

// Fused reduce-scatter back-pressure: source `src` may overwrite its slot in destination q only
// after q consumed the previous landing, i.e. q's generation reached src's arrivals at q.
__global__ void p2p_ready_k(PeerPtrs gen, PeerPtrs arrivals, int n, int* err) {
  const int q = threadIdx.x;
  if (q < n) {
    const uint32_t target = ld_acq_sys(static_cast<const uint32_t*>(arrivals.p[q]));
    spin_until_ge(static_cast<const uint32_t*>(gen.p[q]), target, err);
  }
}

// Barrier of an IPC group: generation g = ++ctrl[kGen]; write g into every rank's arrival slot
// for this rank (release, system scope); wait until every rank's arrival here reached g.
constexpr int kArrive = 0, kGen = 64, kRsFlags = 128, kRsGen = 192, kErr = 224, kCtrlWords = 256;
__global__ void ipc_barrier_k(PeerPtrs ctrl, int t, int rank) {
  uint32_t* mine = static_cast<uint32_t*>(ctrl.p[rank]);
  int* err = reinterpret_cast<int*>(mine + kErr);
  __shared__ uint32_t g;
  if (threadIdx.x == 0) {
    g = mine[kGen] + 1u;
    mine[kGen] = g;
    __threadfence_system();  // this rank's pushes (previous kernels) before the arrival flags
  }
  __syncthreads();
  if ((int)threadIdx.x < t) st_rel_sys(static_cast<uint32_t*>(ctrl.p[threadIdx.x]) + kArrive + rank, g);
  if ((int)threadIdx.x < t) spin_until_ge(mine + kArrive + threadIdx.x, g, err);
  __syncthreads();
}

// push: dst[q] + off_bytes(q) <- src + src_off(q), `bytes` each, q = 0..t-1. The inbox parity
// is the current barrier generation's (read on the device, so graph replays stay in step).
struct PushArgs {
  const char* src;
  int64_t src_stride;  // bytes between the pieces sent to consecutive ranks (0: same piece)
  char* dst[kMaxLocal];
  int64_t dst_off;     // offset of this rank's slot inside a parity half
  int64_t parity_bytes;
  const uint32_t* gen;
  int64_t bytes;
  int t;
};
__global__ void ipc_push_k(PushArgs a) {
  const int64_t par = (int64_t)(*a.gen & 1u) * a.parity_bytes;
  const bool v16 = (a.bytes % 16) == 0 && (a.src_stride % 16) == 0 && (a.dst_off % 16) == 0 &&
                   ((uintptr_t)a.src % 16) == 0;
  const int q = blockIdx.y;
  const char* s = a.src + q * a.src_stride;
  char* d = a.dst[q] + par + a.dst_off;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (v16) {
    const int64_t nv = a.bytes / 16;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride)
      reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(s)[i];
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.bytes; i += stride) d[i] = s[i];
  }
  __threadfence_system();
}

// gather: out[q*bytes ..] <- own inbox slot q of the previous generation's parity
__global__ void ipc_collect_k(const char* inbox, int64_t parity_bytes, int64_t slot_bytes,
                              const uint32_t* gen, char* out, int64_t bytes, int t) {
  const int64_t par = (int64_t)((*gen - 1u) & 1u) * parity_bytes;
  const int q = blockIdx.y;
  const char* s = inbox + par + q * slot_bytes;
  char* d = out + q * bytes;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (bytes % 16 == 0) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < bytes / 16; i += stride)
      reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(s)[i];
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < bytes; i += stride) d[i] = s[i];
  }
}

// out[i] = rank-ordered fp32 sum of the t inbox slots (as rs_local_k), rounded to T
template <typename T>
__global__ void ipc_sum_k(const char* inbox, int64_t parity_bytes, int64_t slot_bytes,
                          const uint32_t* gen, int t, int64_t n, T* out) {
  const int64_t par = (int64_t)((*gen - 1u) & 1u) * parity_bytes;
  const T* base = reinterpret_cast<const T*>(inbox + par);
  const int64_t se = slot_bytes / (int64_t)sizeof(T);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = to_f(base[i]);
    for (int r = 1; r < t; ++r) acc += to_f(base[r * se + i]);
    out[i] = from_f<T>(acc);
  }
}

class LocalComm final : public Comm {
 public:
  explicit LocalComm(int t) {
    require(t >= 1 && t <= kMaxLocal, "local rank group must have 1..16 ranks");
    t_ = t;
    local_ = t;
    rank0_ = 0;
  }
  void all_gather(const void* const* shard, void* const* full, int64_t n, DType dt,
                  cudaStream_t st) override {
    const size_t bytes = (size_t)n * dsize(dt);
    for (int r = 0; r < t_; ++r) {
      bool dup = false;  // ranks may share one gathered buffer in the simulated group
      for (int q = 0; q < r; ++q) dup |= full[q] == full[r];
      if (dup) continue;
      for (int q = 0; q < t_; ++q)
        SPL_CUDA(cudaMemcpyAsync(static_cast<char*>(full[r]) + q * bytes, shard[q], bytes,
                                 cudaMemcpyDeviceToDevice, st));
    }
  }
  void reduce_scatter(const void* const* part, void* const* shard, int64_t n, DType dt,
                      cudaStream_t st) override {
    PtrPack pp{};
    for (int q = 0; q < t_; ++q) pp.p[q] = part[q];
    for (int r = 0; r < t_; ++r) {
      if (dt == DType::F32)
        rs_local_k<float><<<grid_for(n), 256, 0, st>>>(pp, t_, r * n, n, static_cast<float*>(shard[r]));
      else
        rs_local_k<bf16><<<grid_for(n), 256, 0, st>>>(pp, t_, r * n, n, static_cast<bf16*>(shard[r]));
      SPL_CHECK_LAUNCH();
    }
  }
  void all_reduce(void* const* buf, int64_t n, DType dt, cudaStream_t st) override {
    // sum into rank 0's buffer via a scratch-free two-step: out = ordered sum, then broadcast.
    ensure_scratch((size_t)n * dsize(dt), st);
    PtrPack pp{};
    for (int q = 0; q < t_; ++q) pp.p[q] = buf[q];
    if (dt == DType::F32)
      rs_local_k<float><<<grid_for(n), 256, 0, st>>>(pp, t_, 0, n, static_cast<float*>(scratch_));
    else
      rs_local_k<bf16><<<grid_for(n), 256, 0, st>>>(pp, t_, 0, n, static_cast<bf16*>(scratch_));
    SPL_CHECK_LAUNCH();
    for (int r = 0; r < t_; ++r)
      SPL_CUDA(cudaMemcpyAsync(buf[r], scratch_, (size_t)n * dsize(dt), cudaMemcpyDeviceToDevice, st));
  }
  void all_reduce_f32(float* const* buf, int64_t n, cudaStream_t st) override {
    all_reduce(reinterpret_cast<void* const*>(buf), n, DType::F32, st);
  }
  void reserve(size_t bytes) override {
    if (bytes <= scratch_bytes_) return;
    if (scratch_ && own_) SPL_CUDA(cudaFree(scratch_));
    SPL_CUDA(cudaMalloc(&scratch_, bytes));
    scratch_bytes_ = bytes;
    own_ = true;
  }
  void use_scratch(void* p, size_t bytes) override {
    if (scratch_ && own_) SPL_CUDA(cudaFree(scratch_));
    scratch_ = p;
    scratch_bytes_ = bytes;
    own_ = false;
  }
  ~LocalComm() override {
    free_p2p();
    if (scratch_ && own_) cudaFree(scratch_);
  }

  // simulated ranks: every rank's slots and counters are plain buffers on the one device
  bool p2p_setup(size_t slot_bytes) override {
    if (slot_bytes <= slot_bytes_) return true;
    free_p2p();
    slot_bytes_ = slot_bytes;
    for (int q = 0; q < t_; ++q) {
      void *sl = nullptr, *fl = nullptr;
      SPL_CUDA(cudaMalloc(&sl, slot_bytes * t_));
      SPL_CUDA(cudaMalloc(&fl, sizeof(uint32_t) * (t_ + 1)));
      SPL_CUDA(cudaMemset(fl, 0, sizeof(uint32_t) * (t_ + 1)));
      slots_.push_back(sl);
      flags_.push_back(static_cast<uint32_t*>(fl));
    }
    return true;
  }
  void* p2p_slot(int dst, int src) override {
    return static_cast<char*>(slots_[dst]) + (size_t)src * slot_bytes_;
  }
  uint32_t* p2p_flag(int dst, int src) override { return flags_[dst] + src; }
  const void* p2p_slot_local(int dst, int src) override { return p2p_slot(dst, src); }
  uint32_t* p2p_flags_local(int dst) override { return flags_[dst]; }
  uint32_t* p2p_gen(int dst) override { return flags_[dst] + t_; }

 private:
  void free_p2p() {
    for (void* p : slots_) cudaFree(p);
    for (uint32_t* p : flags_) cudaFree(p);
    slots_.clear();
    flags_.clear();
    slot_bytes_ = 0;
  }
  std::vector<void*> slots_;
  std::vector<uint32_t*> flags_;  // per rank: [t arrival counters, generation]
  size_t slot_bytes_ = 0;

  void ensure_scratch(size_t bytes, cudaStream_t st) {
    if (bytes <= scratch_bytes_) return;
    if (scratch_ && own_) {
      SPL_CUDA(cudaStreamSynchronize(st));
      SPL_CUDA(cudaFree(scratch_));
    }
    SPL_CUDA(cudaMalloc(&scratch_, bytes));
    scratch_bytes_ = bytes;
    own_ = true;
  }
  void* scratch_ = nullptr;
  size_t scratch_bytes_ = 0;
  bool own_ = true;
};

#define SPL_NCCL(expr)                                                             \
  do {                                                                             \
    ncclResult_t r_ = (expr);                                                      \
    if (r_ != ncclSuccess)                                                         \
      ::spl::raise(4, std::string(#expr " failed: ") + ncclGetErrorString(r_));    \
  } while (0)

inline ncclDataType_t nccl_type(DType dt) { return dt == DType::F32 ? ncclFloat32 : ncclBfloat16; }

class NcclComm final : public Comm {
 public:
  NcclComm(int t, int rank, const unsigned char id[128]) {
    require(t >= 1 && rank >= 0 && rank < t, "nccl rank out of range");
    t_ = t;
    local_ = 1;
    rank0_ = rank;
    ncclUniqueId uid;
    static_assert(sizeof(uid.internal) == 128, "ncclUniqueId size");
    std::memcpy(uid.internal, id, 128);
    SPL_NCCL(ncclCommInitRank(&comm_, t, uid, rank));
  }
  ~NcclComm() override {
    for (size_t q = 0; q < peer_slots_.size(); ++q)
      if ((int)q != rank0_ && peer_slots_[q]) {
        cudaIpcCloseMemHandle(peer_slots_[q]);
        cudaIpcCloseMemHandle(peer_flags_[q]);
      }
    if (slots_) cudaFree(slots_);
    if (flags_) cudaFree(flags_);
    if (err_) cudaFree(err_);
    if (bar_) cudaFree(bar_);
    if (comm_) ncclCommDestroy(comm_);
  }

  // One process per GPU: this rank's slots and counters are exported with CUDA IPC, the t
  // handle pairs exchanged with one ncclAllGather, and the peers' buffers mapped (NVLink P2P).
  bool p2p_setup(size_t slot_bytes) override {
    if (slot_bytes <= slot_bytes_) return true;
    require(slots_ == nullptr, "fused reduce-scatter slots can only be sized once");
    slot_bytes_ = slot_bytes;
    SPL_CUDA(cudaMalloc(&slots_, slot_bytes * t_));
    SPL_CUDA(cudaMalloc(&flags_, sizeof(uint32_t) * (t_ + 1)));
    SPL_CUDA(cudaMemset(flags_, 0, sizeof(uint32_t) * (t_ + 1)));
    cudaIpcMemHandle_t mine[2];
    SPL_CUDA(cudaIpcGetMemHandle(&mine[0], slots_));
    SPL_CUDA(cudaIpcGetMemHandle(&mine[1], flags_));
    const size_t hb = sizeof(mine);
    char* dev = nullptr;
    SPL_CUDA(cudaMalloc(&dev, hb * (t_ + 1)));
    SPL_CUDA(cudaMemcpy(dev + hb * t_, mine, hb, cudaMemcpyHostToDevice));
    SPL_NCCL(ncclAllGather(dev + hb * t_, dev, hb, ncclUint8, comm_, 0));
    SPL_CUDA(cudaStreamSynchronize(0));
    std::vector<cudaIpcMemHandle_t> all(2 * t_);
    SPL_CUDA(cudaMemcpy(all.data(), dev, hb * t_, cudaMemcpyDeviceToHost));
    SPL_CUDA(cudaFree(dev));
    peer_slots_.assign(t_, nullptr);
    peer_flags_.assign(t_, nullptr);
    for (int q = 0; q < t_; ++q) {
      if (q == rank0_) {
        peer_slots_[q] = slots_;
        peer_flags_[q] = flags_;
        continue;
      }
      SPL_CUDA(cudaIpcOpenMemHandle(&peer_slots_[q], all[2 * q], cudaIpcMemLazyEnablePeerAccess));
      SPL_CUDA(cudaIpcOpenMemHandle(&peer_flags_[q], all[2 * q + 1], cudaIpcMemLazyEnablePeerAccess));
    }
    return true;
  }
  void* p2p_slot(int dst, int src) override {
    return static_cast<char*>(peer_slots_[dst]) + (size_t)src * slot_bytes_;
  }
  uint32_t* p2p_flag(int dst, int src) override {
    return static_cast<uint32_t*>(peer_flags_[dst]) + src;
  }
  const void* p2p_slot_local(int dst, int src) override {
    (void)dst;
    return static_cast<char*>(slots_) + (size_t)src * slot_bytes_;
  }
  uint32_t* p2p_flags_local(int dst) override {
    (void)dst;
    return static_cast<uint32_t*>(flags_);
  }
  uint32_t* p2p_gen(int dst) override {
    (void)dst;
    return static_cast<uint32_t*>(flags_) + t_;
  }
  void p2p_ready_wait(int src, cudaStream_t st) override {
    PeerPtrs g{}, a{};
    for (int q = 0; q < t_; ++q) {
      g.p[q] = static_cast<uint32_t*>(peer_flags_[q]) + t_;
      a.p[q] = static_cast<uint32_t*>(peer_flags_[q]) + src;
    }
    if (err_ == nullptr) SPL_CUDA(cudaMalloc(&err_, sizeof(int)));
    p2p_ready_k<<<1, 32, 0, st>>>(g, a, t_, err_);
    SPL_CHECK_LAUNCH();
  }
  bool p2p_map(const void* mine, std::vector<const void*>& all) override {
    const PeerEntry e = peer_entry(mine);
    char* dev = nullptr;
    SPL_CUDA(cudaMalloc(&dev, sizeof(PeerEntry) * (t_ + 1)));
    SPL_CUDA(cudaMemcpy(dev + sizeof(PeerEntry) * t_, &e, sizeof e, cudaMemcpyHostToDevice));
    SPL_NCCL(ncclAllGather(dev + sizeof(PeerEntry) * t_, dev, sizeof(PeerEntry), ncclUint8, comm_, 0));
    SPL_CUDA(cudaStreamSynchronize(0));
    std::vector<PeerEntry> ents(t_);
    SPL_CUDA(cudaMemcpy(ents.data(), dev, sizeof(PeerEntry) * t_, cudaMemcpyDeviceToHost));
    SPL_CUDA(cudaFree(dev));
    all.assign(t_, nullptr);
    for (int q = 0; q < t_; ++q) all[q] = q == rank0_ ? mine : maps_.open(q, ents[q]);
    return true;
  }
  // NCCL has no barrier; a one-element all-reduce completes only once every rank reached it
  void p2p_barrier(cudaStream_t st) override {
    if (bar_ == nullptr) {
      SPL_CUDA(cudaMalloc(&bar_, sizeof(float)));
      SPL_CUDA(cudaMemset(bar_, 0, sizeof(float)));
    }
    SPL_NCCL(ncclAllReduce(bar_, bar_, 1, ncclFloat32, ncclSum, comm_, st));
  }
  void all_gather(const void* const* shard, void* const* full, int64_t n, DType dt,
                  cudaStream_t st) override {
    SPL_NCCL(ncclAllGather(shard[0], full[0], (size_t)n, nccl_type(dt), comm_, st));
  }
  void reduce_scatter(const void* const* part, void* const* shard, int64_t n, DType dt,
                      cudaStream_t st) override {
    SPL_NCCL(ncclReduceScatter(part[0], shard[0], (size_t)n, nccl_type(dt), ncclSum, comm_, st));
  }
  void all_reduce(void* const* buf, int64_t n, DType dt, cudaStream_t st) override {
    SPL_NCCL(ncclAllReduce(buf[0], buf[0], (size_t)n, nccl_type(dt), ncclSum, comm_, st));
  }
  void all_reduce_f32(float* const* buf, int64_t n, cudaStream_t st) override {
    SPL_NCCL(ncclAllReduce(buf[0], buf[0], (size_t)n, ncclFloat32, ncclSum, comm_, st));
  }

 private:
  ncclComm_t comm_ = nullptr;
  PeerMaps maps_;
  float* bar_ = nullptr;
  int* err_ = nullptr;
  void* slots_ = nullptr;
  void* flags_ = nullptr;
  size_t slot_bytes_ = 0;
  std::vector<void*> peer_slots_, peer_flags_;
};


// ---------------------------------------------------------------- CUDA-IPC transport
// Region of one rank (one cudaMalloc, exported with one IPC handle):
//   [ctrl: 256 u32 — arrivals[64], generation, fused-RS counters[64], fused-RS generation, err]
//   [inbox: 2 parities × t slots × slot_bytes]  (pushed collectives)
//   [fused-RS landing slots: t × slot_bytes]
class IpcRankImpl final : public IpcRank {
 public:
  IpcRankImpl(int device, int t, int rank, size_t slot_bytes)
      : device_(device), t_(t), rank_(rank), slot_(round16(slot_bytes)) {
    require(t >= 1 && t <= kMaxLocal, "IPC group must have 1..16 ranks");
    require(rank >= 0 && rank < t, "IPC rank out of range");
    SPL_CUDA(cudaSetDevice(device));
    bytes_ = ctrl_bytes() + 2 * (size_t)t * slot_ + (size_t)t * slot_;
    SPL_CUDA(cudaMalloc(&base_, bytes_));
    SPL_CUDA(cudaMemset(base_, 0, ctrl_bytes()));
    SPL_CUDA(cudaIpcGetMemHandle(&handle_, base_));
  }
  ~IpcRankImpl() override {
    if (base_) {
      cudaSetDevice(device_);
      cudaFree(base_);
    }
  }
  void export_handle(unsigned char out[kHandleBytes]) const override {
    static_assert(sizeof(cudaIpcMemHandle_t) == kHandleBytes, "IPC handle size");
    std::memcpy(out, &handle_, kHandleBytes);
  }
  static size_t round16(size_t b) { return (b + 15) / 16 * 16; }
  static size_t ctrl_bytes() { return 4096; }

  int device_, t_, rank_;
  size_t slot_, bytes_ = 0;
  void* base_ = nullptr;
  cudaIpcMemHandle_t handle_{};
};

class IpcComm final : public Comm {
 public:
  IpcComm(std::unique_ptr<IpcRankImpl> mine, const unsigned char* handles) : r_(std::move(mine)) {
    t_ = r_->t_;
    local_ = 1;
    rank0_ = r_->rank_;
    dev_ = r_->device_;
    SPL_CUDA(cudaSetDevice(dev_));
    base_.assign(t_, nullptr);
    for (int q = 0; q < t_; ++q) {
      if (q == rank0_) {
        base_[q] = static_cast<char*>(r_->base_);
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + (size_t)q * IpcRank::kHandleBytes, IpcRank::kHandleBytes);
      void* p = nullptr;
      SPL_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      base_[q] = static_cast<char*>(p);
    }
  }
  ~IpcComm() override {
    cudaSetDevice(dev_);
    cudaDeviceSynchronize();
    for (int q = 0; q < t_; ++q)
      if (q != rank0_ && base_[q]) cudaIpcCloseMemHandle(base_[q]);
  }
  bool serial_order() const override { return true; }
  bool p2p_default() const override { return true; }
  bool pull_default() const override { return true; }

  // The (handle, offset) entries travel through each rank's exported control region: write
  // mine, barrier, read the peers' (mapped) regions, barrier (nobody rewrites its entry before
  // every rank read it).
  bool p2p_map(const void* mine, std::vector<const void*>& all) override {
    const PeerEntry e = peer_entry(mine);
    SPL_CUDA(cudaMemcpy(base_[rank0_] + kXchOff, &e, sizeof e, cudaMemcpyHostToDevice));
    barrier(0);
    SPL_CUDA(cudaStreamSynchronize(0));
    all.assign(t_, nullptr);
    for (int q = 0; q < t_; ++q) {
      if (q == rank0_) {
        all[q] = mine;
        continue;
      }
      PeerEntry pe;
      SPL_CUDA(cudaMemcpy(&pe, base_[q] + kXchOff, sizeof pe, cudaMemcpyDeviceToHost));
      all[q] = maps_.open(q, pe);
    }
    barrier(0);
    SPL_CUDA(cudaStreamSynchronize(0));
    return true;
  }
  void p2p_barrier(cudaStream_t st) override { barrier(st); }

  void all_gather(const void* const* shard, void* const* full, int64_t n, DType dt,
                  cudaStream_t st) override {
    const int64_t bytes = n * (int64_t)dsize(dt);
    push(static_cast<const char*>(shard[0]), 0, bytes, st);
    barrier(st);
    ipc_collect_k<<<dim3(grid_for(bytes / 16 + 1), t_), 256, 0, st>>>(
        inbox(rank0_), parity_bytes(), (int64_t)r_->slot_, gen(), static_cast<char*>(full[0]),
        bytes, t_);
    SPL_CHECK_LAUNCH();
  }
  void reduce_scatter(const void* const* part, void* const* shard, int64_t n, DType dt,
                      cudaStream_t st) override {
    const int64_t bytes = n * (int64_t)dsize(dt);
    push(static_cast<const char*>(part[0]), bytes, bytes, st);  // piece q to rank q
    barrier(st);
    sum(shard[0], n, dt, st);
  }
  void all_reduce(void* const* buf, int64_t n, DType dt, cudaStream_t st) override {
    const int64_t bytes = n * (int64_t)dsize(dt);
    push(static_cast<const char*>(buf[0]), 0, bytes, st);
    barrier(st);
    sum(buf[0], n, dt, st);
  }
  void all_reduce_f32(float* const* buf, int64_t n, cudaStream_t st) override {
    all_reduce(reinterpret_cast<void* const*>(buf), n, DType::F32, st);
  }

  // fused reduce-scatter landing slots (the region's last t slots) and their counters
  bool p2p_setup(size_t slot_bytes) override { return slot_bytes <= r_->slot_; }
  void* p2p_slot(int dst, int src) override {
    return base_[dst] + rs_off() + (size_t)src * r_->slot_;
  }
  uint32_t* p2p_flag(int dst, int src) override { return ctrl(dst) + kRsFlags + src; }
  const void* p2p_slot_local(int dst, int src) override {
    (void)dst;
    return base_[rank0_] + rs_off() + (size_t)src * r_->slot_;
  }
  uint32_t* p2p_flags_local(int dst) override { (void)dst; return ctrl(rank0_) + kRsFlags; }
  uint32_t* p2p_gen(int dst) override { (void)dst; return ctrl(rank0_) + kRsGen; }
  void p2p_ready_wait(int src, cudaStream_t st) override {
    PeerPtrs g{}, a{};
    for (int q = 0; q < t_; ++q) {
      g.p[q] = ctrl(q) + kRsGen;
      a.p[q] = ctrl(q) + kRsFlags + src;
    }
    p2p_ready_k<<<1, 32, 0, st>>>(g, a, t_, reinterpret_cast<int*>(ctrl(rank0_) + kErr));
    SPL_CHECK_LAUNCH();
  }

 private:
  uint32_t* ctrl(int q) const { return reinterpret_cast<uint32_t*>(base_[q]); }
  const uint32_t* gen() const { return ctrl(rank0_) + kGen; }
  char* inbox(int q) const { return base_[q] + IpcRankImpl::ctrl_bytes(); }
  int64_t parity_bytes() const { return (int64_t)t_ * (int64_t)r_->slot_; }
  size_t rs_off() const { return IpcRankImpl::ctrl_bytes() + 2 * (size_t)t_ * r_->slot_; }

  // every rank q receives src + q*src_stride (bytes) in its inbox slot for this rank
  void push(const char* src, int64_t src_stride, int64_t bytes, cudaStream_t st) {
    require(bytes <= (int64_t)r_->slot_, "IPC collective larger than the exchange slot");
    PushArgs a{};
    a.src = src;
    a.src_stride = src_stride;
    for (int q = 0; q < t_; ++q) a.dst[q] = inbox(q);
    a.dst_off = (int64_t)rank0_ * (int64_t)r_->slot_;
    a.parity_bytes = parity_bytes();
    a.gen = gen();
    a.bytes = bytes;
    a.t = t_;
    ipc_push_k<<<dim3(grid_for(bytes / 16 + 1), t_), 256, 0, st>>>(a);
    SPL_CHECK_LAUNCH();
  }
  void barrier(cudaStream_t st) {
    PeerPtrs c{};
    for (int q = 0; q < t_; ++q) c.p[q] = base_[q];
    ipc_barrier_k<<<1, 32, 0, st>>>(c, t_, rank0_);
    SPL_CHECK_LAUNCH();
  }
  void sum(void* out, int64_t n, DType dt, cudaStream_t st) {
    if (dt == DType::F32)
      ipc_sum_k<float><<<grid_for(n), 256, 0, st>>>(inbox(rank0_), parity_bytes(), (int64_t)r_->slot_,
                                                    gen(), t_, n, static_cast<float*>(out));
    else
      ipc_sum_k<bf16><<<grid_for(n), 256, 0, st>>>(inbox(rank0_), parity_bytes(), (int64_t)r_->slot_,
                                                   gen(), t_, n, static_cast<bf16*>(out));
    SPL_CHECK_LAUNCH();
  }

  static constexpr size_t kXchOff = 2048;  // address-exchange entry in the control region
  static_assert(kXchOff >= kCtrlWords * 4 && kXchOff + sizeof(PeerEntry) <= 4096, "ctrl layout");
  std::unique_ptr<IpcRankImpl> r_;
  std::vector<char*> base_;
  PeerMaps maps_;  // destroyed before the peers' regions are closed (declared after base_)
  int dev_ = 0;
};
}  // namespace

std::unique_ptr<Comm> make_local_comm(int t) { return std::make_unique<LocalComm>(t); }
std::unique_ptr<Comm> make_nccl_comm(int t, int rank, const unsigned char id[128]) {
  return std::make_unique<NcclComm>(t, rank, id);
}
std::unique_ptr<IpcRank> ipc_open(int device, int t, int rank, size_t slot_bytes) {
  return std::make_unique<IpcRankImpl>(device, t, rank, slot_bytes);
}
std::unique_ptr<Comm> ipc_connect(std::unique_ptr<IpcRank> r, const unsigned char* handles) {
  require(r != nullptr && handles != nullptr, "null IPC rank or handles");
  std::unique_ptr<IpcRankImpl> impl(static_cast<IpcRankImpl*>(r.release()));
  return std::make_unique<IpcComm>(std::move(impl), handles);
}

}  // namespace spl
