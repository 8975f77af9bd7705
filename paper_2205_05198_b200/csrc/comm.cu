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
    if (scratch_ && own_) cudaFree(scratch_);
  }

 private:
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
    if (comm_) ncclCommDestroy(comm_);
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
};

}  // namespace

std::unique_ptr<Comm> make_local_comm(int t) { return std::make_unique<LocalComm>(t); }
std::unique_ptr<Comm> make_nccl_comm(int t, int rank, const unsigned char id[128]) {
  return std::make_unique<NcclComm>(t, rank, id);
}

}  // namespace spl
