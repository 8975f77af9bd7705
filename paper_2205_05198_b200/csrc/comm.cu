#include <cstring>

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
  void* slots_ = nullptr;
  void* flags_ = nullptr;
  size_t slot_bytes_ = 0;
  std::vector<void*> peer_slots_, peer_flags_;
};

}  // namespace

std::unique_ptr<Comm> make_local_comm(int t) { return std::make_unique<LocalComm>(t); }
std::unique_ptr<Comm> make_nccl_comm(int t, int rank, const unsigned char id[128]) {
  return std::make_unique<NcclComm>(t, rank, id);
}

}  // namespace spl
