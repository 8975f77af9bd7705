// SpLayer: one pre-LN GPT layer under tensor + sequence parallelism on B200, with
// none / selective / full activation recomputation. Restates the schedule of the reference's
// seqpar_block_forward / seqpar_block_backward (block.cpp:512-749) as device kernels and
// collectives; see DESIGN.md for the per-regime data layout.
#pragma once
#include <array>
#include <memory>
#include <string>
#include <vector>

#include "../../include/spl.h"
#include "comm.hpp"
#include "kernels.hpp"

namespace spl {

// Saved-tensor categories for the accountant.
enum BufCat : int { kParam = 0, kGrad = 1, kSaved = 2, kSavedUncounted = 3, kWork = 4 };

struct Buffer {
  void* ptr = nullptr;
  size_t bytes = 0;
};

struct LedgerItem {
  std::string name;
  int64_t elements = 0;
  int64_t bytes = 0;      // reference convention (ByteConvention widths)
  int64_t physical = 0;   // bytes actually held on the device
};

class LayerBase {
 public:
  virtual ~LayerBase() = default;
  virtual void load_params(const double* packed) = 0;
  virtual void init_params(uint64_t seed) = 0;
  virtual void forward(const void* const* x, void* const* y) = 0;
  virtual void backward(const void* const* dy, void* const* dx) = 0;
  virtual void step_host(const void* x, const void* dy, void* y, void* dx) = 0;
  virtual void step_host_async(const void* x, const void* dy, void* y, void* dx) = 0;
  virtual void step_host_wait() = 0;
  virtual void get_grads(double* packed) = 0;
  virtual void get_w1_grad_shard(int r, double* out) = 0;
  virtual void get_saved(int r, const std::string& name, double* out, int64_t n) = 0;
  virtual void attention_interior(int r, double* out3) = 0;
  virtual std::vector<LedgerItem> ledger(int r) const = 0;
  virtual void saved_bytes(int r, int64_t* ledger, int64_t* physical, int64_t* uncounted) const = 0;
  virtual Comm& comm() = 0;
  virtual cudaStream_t stream() const = 0;
  virtual void set_profile(bool on) = 0;
  virtual void read_profile(double ms[K_NCLASS], int64_t launches[K_NCLASS],
                            double flops[K_NCLASS], double bytes[K_NCLASS]) = 0;
  virtual int64_t launch_count(bool reset) = 0;
  virtual void comm_paths(int out[2]) const = 0;
  virtual void set_graphs(bool on) = 0;
  virtual int local_ranks() const = 0;
  virtual void set_caller_stream(cudaStream_t s) = 0;
  // Device bytes this layer allocated per BufCat (kWork: only buffers it owns, not a pool's).
  virtual void alloc_bytes(int64_t out[5]) const = 0;
  // MaskKey microbatch field of the dropout masks of the next calls (rng.cpp:39-45).
  virtual void set_microbatch(uint32_t microbatch) = 0;
  // Backward adds its parameter gradients to the held ones instead of overwriting them.
  virtual void set_grad_accumulate(bool on) = 0;
};

// Transient device buffers shared by the layers of a stack. Layers of one stack have identical
// shapes and run one after another on the caller stream, so the i-th workspace request of every
// layer maps to the same buffer: an L-layer stack holds L sets of saved activations but one
// workspace (the unit total_first_stage_bytes / simulate_memory count, activation_memory.cpp
// :112-123, pipeline_sim.cpp:222-275).
struct WorkPool {
  int device = 0;
  std::vector<std::pair<void*, size_t>> bufs;
  int64_t bytes() const {
    int64_t n = 0;
    for (auto& b : bufs) n += (int64_t)b.second;
    return n;
  }
  ~WorkPool() {
    cudaSetDevice(device);
    for (auto& b : bufs) cudaFree(b.first);
  }
};

// `params`: parameters and gradients shared with the other handles built on the same pool (the
// i-th parameter / gradient request maps to the same buffer) — the several activation slots
// of one layer in a microbatch window.
std::unique_ptr<LayerBase> make_layer(const spl_layer_desc& d, int device,
                                      std::unique_ptr<Comm> comm,
                                      std::shared_ptr<WorkPool> pool = nullptr,
                                      std::shared_ptr<WorkPool> params = nullptr);

// Accountant (activation_memory.cpp:54-82) — exact, floor once.
int per_layer_bytes_exact(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                          int sp, int64_t act, int64_t mask, __int128* num, __int128* den);

}  // namespace spl
