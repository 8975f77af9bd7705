// Collectives of the tensor+sequence-parallel layer (the g / ḡ transitions and their duals,
// collectives.hpp:57-62 of the reference), behind one interface with two transports:
//   LocalComm — t simulated ranks on one device (the reference's in-process harness); sums in
//               rank order 0..t-1 with fp32 accumulation (collectives.cpp:40-46).
//   NcclComm  — one rank per process/GPU over NCCL (NVLink 5 / NVSwitch on a B200 node).
// Sequence shards are contiguous axis-0 chunks of {s, b, h}, so every collective is a flat
// buffer operation with no packing.
#pragma once
#include <nccl.h>

#include <memory>
#include <vector>

#include "common.hpp"

namespace spl {

// CommTag of collectives.hpp:28 plus the forward re-run of full recomputation.
enum CommTag : int { kSchedule = 0, kRegather = 1, kGradSync = 2, kRecompute = 3 };

struct CommCounters {
  int64_t all_gathers = 0, reduce_scatters = 0, all_reduces = 0, ring_elements = 0;
};

class Comm {
 public:
  virtual ~Comm() = default;
  int t() const { return t_; }
  int local() const { return local_; }
  int rank0() const { return rank0_; }
  // full[r] (t*n elements) = concat_q shard[q] (n elements each), every local rank r.
  virtual void all_gather(const void* const* shard, void* const* full, int64_t n, DType dt,
                          cudaStream_t st) = 0;
  // shard[r] (n) = sum_q part[q][r*n .. (r+1)*n), for every local rank r.
  virtual void reduce_scatter(const void* const* part, void* const* shard, int64_t n, DType dt,
                              cudaStream_t st) = 0;
  // buf[r] (n) = sum_q buf[q], in place.
  virtual void all_reduce(void* const* buf, int64_t n, DType dt, cudaStream_t st) = 0;
  virtual void all_reduce_f32(float* const* buf, int64_t n, cudaStream_t st) = 0;
  // Pre-allocate any scratch a collective of up to `bytes` may need (so that no allocation
  // happens while a CUDA graph is being captured).
  virtual void reserve(size_t bytes) { (void)bytes; }
  // Use a caller-owned device buffer as that scratch (a layer's workspace, shared in a stack).
  virtual void use_scratch(void* p, size_t bytes) { (void)p; (void)bytes; }

  // ---- landing slots of the reduce-scatter fused into the producing GEMM (peer memory).
  // Destination rank q owns t slots of `slot_bytes` (one per source rank), t arrival counters
  // and a generation counter. A source GEMM writes its rows of shard q straight into
  // slot(q, src); signal() bumps q's counter for src; the consumer on q waits for all t
  // counters to pass its generation, sums the slots in rank order and advances the generation.
  // Counters live on the device, so the protocol survives CUDA-graph replays.
  virtual bool p2p_setup(size_t slot_bytes) { (void)slot_bytes; return false; }
  // writer side (device of `src`): q's slot for src, q's arrival counter for src
  virtual void* p2p_slot(int dst, int src) { (void)dst; (void)src; return nullptr; }
  virtual uint32_t* p2p_flag(int dst, int src) { (void)dst; (void)src; return nullptr; }
  // reader side (device of `dst`): its slot array base, counters and generation
  virtual const void* p2p_slot_local(int dst, int src) { (void)dst; (void)src; return nullptr; }
  virtual uint32_t* p2p_flags_local(int dst) { (void)dst; return nullptr; }
  virtual uint32_t* p2p_gen(int dst) { (void)dst; return nullptr; }
  // Back-pressure of the fused reduce-scatter: before source `src` overwrites its slots in the
  // destination ranks, wait (on `st`) until every destination consumed the previous landing
  // (its generation caught up with src's arrival count there).
  virtual void p2p_ready_wait(int src, cudaStream_t st) { (void)src; (void)st; }
  // Whether the fused reduce-scatter is on by default for this transport.
  virtual bool p2p_default() const { return local_ == t_; }

  // ---- all-gather fused into the consuming GEMM by pulling (peer ranks): the GEMM's TMA
  // reads every rank's shard where it lies (peer memory over NVLink), so the transfer is spread
  // over the GEMM's tiles. p2p_map exchanges the address of a buffer every rank holds in the
  // same role (collective: every rank calls it in the same order) and returns the t ranks'
  // addresses valid in this process; p2p_barrier (on `st`) orders every rank's writes issued
  // before it ahead of every rank's reads issued after it.
  virtual bool p2p_map(const void* mine, std::vector<const void*>& all) {
    (void)mine;
    (void)all;
    return false;
  }
  virtual void p2p_barrier(cudaStream_t st) { (void)st; }
  // Whether the pulled all-gather is on by default for this transport.
  virtual bool pull_default() const { return false; }
  // Whether collectives must be issued on one stream in one order on every rank (device-side
  // sequence-numbered protocols); the layer then keeps them all on its compute stream.
  virtual bool serial_order() const { return false; }

  void log(CommTag tag, int kind, int64_t logical_elems) {
    CommCounters& c = counters[tag];
    if (kind == 0) c.all_gathers++;
    if (kind == 1) c.reduce_scatters++;
    if (kind == 2) c.all_reduces++;
    c.ring_elements += (kind == 2 ? 2 : 1) * (logical_elems / t_) * (t_ - 1);
  }
  CommCounters counters[4];

 protected:
  int t_ = 1, local_ = 1, rank0_ = 0;
};

std::unique_ptr<Comm> make_local_comm(int t);
std::unique_ptr<Comm> make_nccl_comm(int t, int rank, const unsigned char id[128]);

// One rank of a t-way group whose collectives run over CUDA-IPC-mapped peer memory (NVLink P2P
// loads/stores between GPUs; same-device IPC when several processes share one GPU), with no
// NCCL: a device-side barrier of system-scope release/acquire flags sequences them. Two-phase
// setup: open() allocates this rank's exported region and returns its IPC handle; after the
// caller exchanged the t handles (rank order), connect() maps the peers.
class IpcRank {
 public:
  static constexpr int kHandleBytes = 64;
  virtual ~IpcRank() = default;
  virtual void export_handle(unsigned char out[kHandleBytes]) const = 0;
};
std::unique_ptr<IpcRank> ipc_open(int device, int t, int rank, size_t slot_bytes);
std::unique_ptr<Comm> ipc_connect(std::unique_ptr<IpcRank> r, const unsigned char* handles);

}  // namespace spl
