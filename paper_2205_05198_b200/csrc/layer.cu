// SpLayer implementation. The schedule below is the reference's seqpar_block_forward /
// seqpar_block_backward (/root/reference/proj/core/src/seqpar/block.cpp:512-749) with:
//  - per-rank work as device kernels (LN, fused bias-dropout-residual(+LN2), tcgen05 GEMMs
//    with fused bias / bias+GELU / GELU-backward epilogues, flash-style attention),
//  - g / ḡ (and duals) as all-gather / reduce-scatter on contiguous sequence chunks,
//  - the three recompute regimes executed (the reference only accounts for them):
//      none      — stores the attention interior (softmax_out, mask, dropout_out),
//      selective — stores Q/K/V and a per-row LSE; backward recomputes QKᵀ, softmax, dropout,
//      full      — stores only the layer input; backward re-runs the forward first,
//  - SP off (TP baseline): LN/dropout regions replicated, f/f̄ as all-reduces.
// Local ranks r of a handle map to global TP ranks rank0 + r.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <type_traits>

#include "layer.hpp"

namespace spl {

namespace {

using k::Epi;
using k::GemmArgs;
using k::Major;

constexpr int kChunkRows = 64;

struct Alloc {
  void* ptr;
  size_t bytes;
  int cat;
  int rank;
};

struct Graph {
  cudaGraphExec_t exec = nullptr;
  std::vector<const void*> in;
  std::vector<void*> out;
  int64_t launches = 0;
  CommCounters comm[4];  // the CommLog increments the captured body makes, replayed per launch
};

template <typename T>
class Layer final : public LayerBase {
 public:
  Layer(const spl_layer_desc& d, int device, std::unique_ptr<Comm> comm,
        std::shared_ptr<WorkPool> pool, std::shared_ptr<WorkPool> params)
      : d_(d), dev_(device), comm_(std::move(comm)), pool_(std::move(pool)),
        params_(std::move(params)) {
    t_ = comm_->t();
    L_ = comm_->local();
    rank0_ = comm_->rank0();
    s_ = d.seq;
    b_ = d.batch;
    h_ = d.hidden;
    a_ = d.heads;
    validate();
    hd_ = h_ / a_;
    lh_ = a_ / t_;
    lw_ = h_ / t_;
    fw_ = 4 * h_ / t_;
    RF_ = s_ * b_;
    sp_ = d.sequence_parallel != 0;
    RL_ = sp_ ? RF_ / t_ : RF_;
    kind_ = d.recompute;
    scale_ = (float)(1.0 / std::sqrt((double)hd_));
    make_keys();
    SPL_CUDA(cudaSetDevice(dev_));
    SPL_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    SPL_CUDA(cudaStreamCreateWithFlags(&st_rng_, cudaStreamNonBlocking));
    SPL_CUDA(cudaStreamCreateWithFlags(&st_comm_, cudaStreamNonBlocking));
    for (auto* e : {&ev_cfork_, &ev_regather_, &ev_rs_})
      SPL_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    SPL_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    SPL_CUDA(cudaEventCreateWithFlags(&ev_bits_, cudaEventDisableTiming));
    SPL_CUDA(cudaEventCreateWithFlags(&ev_in_, cudaEventDisableTiming));
    SPL_CUDA(cudaEventCreateWithFlags(&ev_out_, cudaEventDisableTiming));
    allocate();
    {  // collective scratch from the workspace (shared by the layers of a stack)
      const size_t scr = std::max<size_t>((size_t)(RF_ * h_) * sizeof(T), (size_t)(6 * h_) * sizeof(float));
      comm_->use_scratch(alloc<uint8_t>((int64_t)scr, kWork, 0), scr);
      comm_->reserve(scr);
    }
    // The keep-bit RNG pass runs on the main stream by default: overlapping it with the GEMMs
    // on a side stream measured no faster (the GEMMs already hold the chip at its power cap).
    {  // reduce-scatter fused into the row-parallel GEMMs: on for simulated ranks and the
       // CUDA-IPC transport; NCCL ranks opt in with SPL_FUSED_RS=1 (IPC peer slots over NVLink)
      const char* f = std::getenv("SPL_FUSED_RS");
      const bool want = f != nullptr ? f[0] == '1' : comm_->p2p_default();
      if (want && std::is_same_v<T, bf16> && sp_ && t_ > 1 && t_ <= k::kMaxScatterRanks &&
          h_ % 8 == 0)
        fused_rs_ = comm_->p2p_setup((size_t)(RL_ * h_) * sizeof(T));
    }
    {  // all-gather fused into the consuming GEMMs (their TMA reads every rank's shard) when
       // every consumer runs on the CTA-pair kernel: simulated ranks read each other's device
       // buffers; peer ranks pull the shards from the peers' memory (mapped once here), on by
       // default for the CUDA-IPC transport, opt-in for NCCL ranks (SPL_FUSED_AG=1 / 0)
      const char* f = std::getenv("SPL_FUSED_AG");
      const bool local = comm_->local() == t_;
      const bool want = f != nullptr ? f[0] == '1' : (local || comm_->pull_default());
      if (want && std::is_same_v<T, bf16> && sp_ && t_ > 1 && t_ <= GemmArgs::kMaxShards &&
          RL_ % 128 == 0) {
        if (local) {
          fused_ag_ = fused_ag_eligible();
        } else {
          pull_ = true;  // shard_of() reads peer_ (the probe only needs shapes: own buffers)
          for (int w = 1; w < 4; ++w)
            for (int q = 0; q < t_; ++q) peer_[w][q] = own_shard((Gath)w);
          if (fused_ag_eligible()) {
            std::vector<const void*> all;
            for (int w = 1; w < 4; ++w) {
              if (!comm_->p2p_map(own_shard((Gath)w), all)) break;
              for (int q = 0; q < t_; ++q) peer_[w][q] = all[q];
              fused_ag_ = w == 3;
            }
          }
          pull_ = fused_ag_;
        }
      }
    }
    const char* e = std::getenv("SPL_KEEPBITS_SIDE");
    bits_serial_ = !(e != nullptr && e[0] == '1');
    const char* c = std::getenv("SPL_SERIAL_COMM");
    // transports whose collectives are sequenced on the device need one issue order per rank
    comm_serial_ = (c != nullptr && c[0] == '1') || comm_->serial_order();
  }

  ~Layer() override {
    cudaSetDevice(dev_);
    cudaStreamSynchronize(st_);
    for (auto* set : {&gfwd_, &gbwd_})
      for (Graph& g : *set)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto& a : allocs_) cudaFree(a.ptr);
    if (pinned_) cudaFreeHost(pinned_);
    for (auto& e : evpool_) cudaEventDestroy(e);
    cudaEventDestroy(ev_in_);
    cudaEventDestroy(ev_out_);
    cudaEventDestroy(ev_fork_);
    cudaEventDestroy(ev_bits_);
    if (st_up_) {
      cudaStreamSynchronize(st_up_);
      cudaStreamSynchronize(st_down_);
      cudaStreamDestroy(st_up_);
      cudaStreamDestroy(st_down_);
      for (int i = 0; i < 2; ++i)
        for (auto e : {ev_x_[i], ev_dy_[i], ev_f_[i], ev_b_[i], ev_free_[i]}) cudaEventDestroy(e);
    }
    cudaStreamSynchronize(st_rng_);
    cudaStreamDestroy(st_rng_);
    cudaStreamSynchronize(st_comm_);
    cudaStreamDestroy(st_comm_);
    for (auto e : {ev_cfork_, ev_regather_, ev_rs_}) cudaEventDestroy(e);
    cudaStreamDestroy(st_);
  }

  int local_ranks() const override { return L_; }
  void comm_paths(int out[2]) const override {
    out[0] = fused_rs_ ? 1 : 0;
    out[1] = fused_ag_ ? (pull_ ? 2 : 1) : 0;
  }
  void set_caller_stream(cudaStream_t s) override { caller_ = s; }

  // Run `body` (which issues work on st_, possibly forking to the side streams and joining
  // back) either eagerly or as a CUDA graph captured on the first call with these pointers.
  // One executable graph per (input, output) pointer set, up to kMaxGraphs per direction
  // (double-buffered callers alternate between two sets).
  static constexpr size_t kMaxGraphs = 4;
  template <typename F>
  void run_graphed(std::vector<Graph>& set, const std::vector<const void*>& in,
                   const std::vector<void*>& out, F&& body) {
    const bool use = graphs_ && !profiling_ && !d_.check_finite;
    if (!use) {
      body();
      return;
    }
    Graph* gp = nullptr;
    for (Graph& c : set)
      if (c.exec != nullptr && c.in == in && c.out == out) gp = &c;
    if (gp == nullptr) {
      if (set.size() >= kMaxGraphs) {
        if (set.front().exec != nullptr) SPL_CUDA(cudaGraphExecDestroy(set.front().exec));
        set.erase(set.begin());
      }
      Graph g;
      const int64_t l0 = launches_;
      CommCounters c0[4];
      std::copy(comm_->counters, comm_->counters + 4, c0);
      cudaGraph_t graph = nullptr;
      SPL_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeThreadLocal));
      try {
        body();
      } catch (...) {
        cudaStreamEndCapture(st_, &graph);  // end the capture, drop the partial graph
        if (graph != nullptr) cudaGraphDestroy(graph);
        launches_ = l0;
        std::copy(c0, c0 + 4, comm_->counters);
        throw;
      }
      SPL_CUDA(cudaStreamEndCapture(st_, &graph));
      const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
      cudaGraphDestroy(graph);
      SPL_CUDA(ie);
      g.in = in;
      g.out = out;
      g.launches = launches_ - l0;
      launches_ = l0;
      for (int k = 0; k < 4; ++k) {  // the capture's CommLog increments, applied per launch
        CommCounters& d = g.comm[k];
        const CommCounters& a = comm_->counters[k];
        d.all_gathers = a.all_gathers - c0[k].all_gathers;
        d.reduce_scatters = a.reduce_scatters - c0[k].reduce_scatters;
        d.all_reduces = a.all_reduces - c0[k].all_reduces;
        d.ring_elements = a.ring_elements - c0[k].ring_elements;
        comm_->counters[k] = c0[k];
      }
      set.push_back(std::move(g));
      gp = &set.back();
    }
    Graph& g = *gp;
    SPL_CUDA(cudaGraphLaunch(g.exec, st_));
    launches_ += g.launches;
    for (int k = 0; k < 4; ++k) {
      CommCounters& c = comm_->counters[k];
      c.all_gathers += g.comm[k].all_gathers;
      c.reduce_scatters += g.comm[k].reduce_scatters;
      c.all_reduces += g.comm[k].all_reduces;
      c.ring_elements += g.comm[k].ring_elements;
    }
  }

  // fork: our stream waits for the caller's prior work; join: the caller waits for ours.
  void enter() {
    SPL_CUDA(cudaSetDevice(dev_));
    SPL_CUDA(cudaEventRecord(ev_in_, caller_));
    SPL_CUDA(cudaStreamWaitEvent(st_, ev_in_, 0));
  }
  void leave() {
    SPL_CUDA(cudaEventRecord(ev_out_, st_));
    SPL_CUDA(cudaStreamWaitEvent(caller_, ev_out_, 0));
  }
  Comm& comm() override { return *comm_; }
  cudaStream_t stream() const override { return st_; }

  // ------------------------------------------------------------------ params
  void load_params(const double* P) override {
    SPL_CUDA(cudaSetDevice(dev_));
    const int64_t h = h_;
    // named_tensors() offsets (block.cpp:293-298)
    const int64_t o_wq = 0, o_wk = h * h, o_wv = 2 * h * h, o_bq = 3 * h * h, o_bk = o_bq + h,
                  o_bv = o_bk + h, o_wo = o_bv + h, o_bo = o_wo + h * h, o_w1 = o_bo + h,
                  o_b1 = o_w1 + 4 * h * h, o_w2 = o_b1 + 4 * h, o_b2 = o_w2 + 4 * h * h,
                  o_g1 = o_b2 + h, o_be1 = o_g1 + h, o_g2 = o_be1 + h, o_be2 = o_g2 + h;
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      const int64_t g = rank0_ + r;
      std::vector<T> w((size_t)(h * 3 * lw_));
      for (int which = 0; which < 3; ++which) {
        const double* src = P + (which == 0 ? o_wq : which == 1 ? o_wk : o_wv);
        for (int64_t i = 0; i < h; ++i)
          for (int64_t j = 0; j < lw_; ++j)
            w[(size_t)(i * 3 * lw_ + which * lw_ + j)] = cvt(src[i * h + g * lw_ + j]);
      }
      up(R.wqkv, w);
      std::vector<float> bq((size_t)(3 * lw_));
      for (int which = 0; which < 3; ++which) {
        const double* src = P + (which == 0 ? o_bq : which == 1 ? o_bk : o_bv);
        for (int64_t j = 0; j < lw_; ++j) bq[(size_t)(which * lw_ + j)] = (float)src[g * lw_ + j];
      }
      up(R.bqkv, bq);
      w.assign((size_t)(lw_ * h), T());
      for (int64_t i = 0; i < lw_; ++i)
        for (int64_t j = 0; j < h; ++j) w[(size_t)(i * h + j)] = cvt(P[o_wo + (g * lw_ + i) * h + j]);
      up(R.wo, w);
      w.assign((size_t)(h * fw_), T());
      for (int64_t i = 0; i < h; ++i)
        for (int64_t j = 0; j < fw_; ++j)
          w[(size_t)(i * fw_ + j)] = cvt(P[o_w1 + i * 4 * h + g * fw_ + j]);
      up(R.w1, w);
      w.assign((size_t)(fw_ * h), T());
      for (int64_t i = 0; i < fw_; ++i)
        for (int64_t j = 0; j < h; ++j) w[(size_t)(i * h + j)] = cvt(P[o_w2 + (g * fw_ + i) * h + j]);
      up(R.w2, w);
      auto upf = [&](float* dst, int64_t off, int64_t n) {
        std::vector<float> v((size_t)n);
        for (int64_t j = 0; j < n; ++j) v[(size_t)j] = (float)P[off + j];
        up(dst, v);
      };
      std::vector<float> b1((size_t)fw_);
      for (int64_t j = 0; j < fw_; ++j) b1[(size_t)j] = (float)P[o_b1 + g * fw_ + j];
      up(R.b1, b1);
      upf(R.bo, o_bo, h);
      upf(R.b2, o_b2, h);
      upf(R.g1, o_g1, h);
      upf(R.be1, o_be1, h);
      upf(R.g2, o_g2, h);
      upf(R.be2, o_be2, h);
    }
    SPL_CUDA(cudaStreamSynchronize(st_));
  }

  void init_params(uint64_t seed) override {
    SPL_CUDA(cudaSetDevice(dev_));
    const int64_t h = h_;
    const double ws = 1.0 / std::sqrt((double)h);
    auto key = [&](int salt) { return hash_counter(seed, (uint64_t)salt); };
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      const int64_t g = rank0_ + r;
      for (int which = 0; which < 3; ++which) {
        k::init_uniform<T>(R.wqkv + which * lw_, h, lw_, 3 * lw_, 0, g * lw_, h, key(1 + which),
                           -ws, ws, 0.0, st_);
        k::init_uniform<float>(R.bqkv + which * lw_, 1, lw_, lw_, 0, g * lw_, h, key(4 + which),
                               -0.1, 0.1, 0.0, st_);
      }
      k::init_uniform<T>(R.wo, lw_, h, h, g * lw_, 0, h, key(7), -ws, ws, 0.0, st_);
      k::init_uniform<float>(R.bo, 1, h, h, 0, 0, h, key(8), -0.1, 0.1, 0.0, st_);
      k::init_uniform<T>(R.w1, h, fw_, fw_, 0, g * fw_, 4 * h, key(9), -ws, ws, 0.0, st_);
      k::init_uniform<float>(R.b1, 1, fw_, fw_, 0, g * fw_, 4 * h, key(10), -0.1, 0.1, 0.0, st_);
      k::init_uniform<T>(R.w2, fw_, h, h, g * fw_, 0, h, key(11), -ws, ws, 0.0, st_);
      k::init_uniform<float>(R.b2, 1, h, h, 0, 0, h, key(12), -0.1, 0.1, 0.0, st_);
      k::init_uniform<float>(R.g1, 1, h, h, 0, 0, h, key(13), -0.1, 0.1, 1.0, st_);
      k::init_uniform<float>(R.be1, 1, h, h, 0, 0, h, key(14), -0.1, 0.1, 0.0, st_);
      k::init_uniform<float>(R.g2, 1, h, h, 0, 0, h, key(15), -0.1, 0.1, 1.0, st_);
      k::init_uniform<float>(R.be2, 1, h, h, 0, 0, h, key(16), -0.1, 0.1, 0.0, st_);
    }
    SPL_CUDA(cudaStreamSynchronize(st_));
  }

  // ------------------------------------------------------------------ forward
  void forward(const void* const* x, void* const* y) override {
    enter();
    for (int r = 0; r < L_; ++r)
      require(x[r] != nullptr && y[r] != nullptr, "expected one input shard per rank");
    std::vector<T*> ys(L_);
    for (int r = 0; r < L_; ++r) ys[r] = static_cast<T*>(y[r]);
    run_graphed(gfwd_, std::vector<const void*>(x, x + L_), std::vector<void*>(y, y + L_), [&] {
      for (int r = 0; r < L_; ++r)
        SPL_CUDA(cudaMemcpyAsync(R_[r].x_s, x[r], (size_t)(RL_ * h_) * sizeof(T),
                                 cudaMemcpyDeviceToDevice, st_));
      if (d_.check_finite) SPL_CUDA(cudaMemsetAsync(nonfinite_, 0, sizeof(int), st_));
      run_forward(ys.data(), kSchedule, d_.check_finite ? nonfinite_ : nullptr);
    });
    if (d_.check_finite) {
      int flag = 0;
      SPL_CUDA(cudaMemcpyAsync(&flag, nonfinite_, sizeof(int), cudaMemcpyDeviceToHost, st_));
      SPL_CUDA(cudaStreamSynchronize(st_));
      if (flag) {
        have_fwd_ = false;
        raise(2, "seqpar_block_forward produced non-finite values");
      }
    }
    have_fwd_ = true;
    leave();
  }

  void backward(const void* const* dy, void* const* dx) override {
    enter();
    if (!have_fwd_) raise(5, "missing saved forward state");
    for (int r = 0; r < L_; ++r) require(dy[r] != nullptr && dx[r] != nullptr, "expected one gradient shard per rank");
    run_graphed(gbwd_, std::vector<const void*>(dy, dy + L_), std::vector<void*>(dx, dx + L_), [&] {
      if (kind_ == SPL_RECOMPUTE_FULL) {
        // Full recomputation: only x_s survived; re-run the forward (with its collectives).
        std::vector<T*> ys(L_);
        for (int r = 0; r < L_; ++r) ys[r] = R_[r].y_re;
        run_forward(ys.data(), kRecompute, nullptr);
      }
      run_backward(dy, dx);
    });
    leave();
  }

  // One training step through host buffers, issued asynchronously: H2D of x and dy on the
  // upload stream, forward / backward on the compute stream, D2H of y and dx on the download
  // stream, each side waiting only for what it needs (x before the forward, dy before the
  // backward, y after the forward, dx after the backward). The device staging buffers are
  // double-buffered, so step k+1's uploads overlap step k's compute and step k's downloads
  // overlap step k+1's compute. step_host_wait() returns when the last issued step's results
  // are in host memory; the host buffers must stay untouched until then.
  void step_host_async(const void* x, const void* dy, void* y, void* dx) override {
    SPL_CUDA(cudaSetDevice(dev_));
    const size_t shard = (size_t)(RL_ * h_) * sizeof(T);
    ensure_staging();
    if (st_up_ == nullptr) {
      SPL_CUDA(cudaStreamCreateWithFlags(&st_up_, cudaStreamNonBlocking));
      SPL_CUDA(cudaStreamCreateWithFlags(&st_down_, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i)
        for (auto* e : {&ev_x_[i], &ev_dy_[i], &ev_f_[i], &ev_b_[i], &ev_free_[i]}) {
          SPL_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
          SPL_CUDA(cudaEventRecord(*e, st_));  // recorded once so that the first waits pass
        }
    }
    const int sl = (int)(host_steps_++ & 1);
    std::vector<const void*> xs(L_), dys(L_);
    std::vector<void*> ysv(L_), dxs(L_);
    for (int r = 0; r < L_; ++r) {
      T* const* b = &stage_[(size_t)(8 * r + 4 * sl)];
      xs[r] = b[0];
      dys[r] = b[1];
      ysv[r] = b[2];
      dxs[r] = b[3];
    }
    // uploads into this slot once its previous user (two steps ago) has been downloaded
    SPL_CUDA(cudaStreamWaitEvent(st_up_, ev_free_[sl], 0));
    for (int r = 0; r < L_; ++r)
      SPL_CUDA(cudaMemcpyAsync(const_cast<void*>(xs[r]), static_cast<const char*>(x) + r * shard,
                               shard, cudaMemcpyHostToDevice, st_up_));
    SPL_CUDA(cudaEventRecord(ev_x_[sl], st_up_));
    for (int r = 0; r < L_; ++r)
      SPL_CUDA(cudaMemcpyAsync(const_cast<void*>(dys[r]), static_cast<const char*>(dy) + r * shard,
                               shard, cudaMemcpyHostToDevice, st_up_));
    SPL_CUDA(cudaEventRecord(ev_dy_[sl], st_up_));
    SPL_CUDA(cudaStreamWaitEvent(st_, ev_x_[sl], 0));
    forward(xs.data(), ysv.data());
    SPL_CUDA(cudaEventRecord(ev_f_[sl], st_));
    SPL_CUDA(cudaStreamWaitEvent(st_, ev_dy_[sl], 0));
    backward(dys.data(), dxs.data());
    SPL_CUDA(cudaEventRecord(ev_b_[sl], st_));
    SPL_CUDA(cudaStreamWaitEvent(st_down_, ev_f_[sl], 0));
    for (int r = 0; r < L_; ++r)
      SPL_CUDA(cudaMemcpyAsync(static_cast<char*>(y) + r * shard, ysv[r], shard,
                               cudaMemcpyDeviceToHost, st_down_));
    SPL_CUDA(cudaStreamWaitEvent(st_down_, ev_b_[sl], 0));
    for (int r = 0; r < L_; ++r)
      SPL_CUDA(cudaMemcpyAsync(static_cast<char*>(dx) + r * shard, dxs[r], shard,
                               cudaMemcpyDeviceToHost, st_down_));
    SPL_CUDA(cudaEventRecord(ev_free_[sl], st_down_));
  }
  void step_host_wait() override {
    SPL_CUDA(cudaSetDevice(dev_));
    if (st_down_) SPL_CUDA(cudaStreamSynchronize(st_down_));
    SPL_CUDA(cudaStreamSynchronize(st_));
  }
  void step_host(const void* x, const void* dy, void* y, void* dx) override {
    step_host_async(x, dy, y, dx);
    step_host_wait();
  }

  // ------------------------------------------------------------------ read-back
  void get_grads(double* P) override {
    SPL_CUDA(cudaSetDevice(dev_));
    SPL_CUDA(cudaStreamSynchronize(st_));
    const int64_t h = h_;
    const int64_t np = 12 * h * h + 13 * h;
    std::memset(P, 0, sizeof(double) * (size_t)np);
    const int64_t o_wq = 0, o_wk = h * h, o_wv = 2 * h * h, o_bq = 3 * h * h, o_bk = o_bq + h,
                  o_bv = o_bk + h, o_wo = o_bv + h, o_bo = o_wo + h * h, o_w1 = o_bo + h,
                  o_b1 = o_w1 + 4 * h * h, o_w2 = o_b1 + 4 * h, o_b2 = o_w2 + 4 * h * h,
                  o_g1 = o_b2 + h, o_be1 = o_g1 + h, o_g2 = o_be1 + h, o_be2 = o_g2 + h;
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      const int64_t g = rank0_ + r;
      auto wqkv = down(R.dwqkv, h * 3 * lw_);
      for (int which = 0; which < 3; ++which) {
        double* dst = P + (which == 0 ? o_wq : which == 1 ? o_wk : o_wv);
        for (int64_t i = 0; i < h; ++i)
          for (int64_t j = 0; j < lw_; ++j)
            dst[i * h + g * lw_ + j] = wqkv[(size_t)(i * 3 * lw_ + which * lw_ + j)];
      }
      auto bqkv = down(R.dbqkv, 3 * lw_);
      for (int which = 0; which < 3; ++which) {
        double* dst = P + (which == 0 ? o_bq : which == 1 ? o_bk : o_bv);
        for (int64_t j = 0; j < lw_; ++j) dst[g * lw_ + j] = bqkv[(size_t)(which * lw_ + j)];
      }
      auto wo = down(R.dwo, lw_ * h);
      for (int64_t i = 0; i < lw_ * h; ++i) P[o_wo + g * lw_ * h + i] = wo[(size_t)i];
      auto w1 = down(R.dw1, h * fw_);
      for (int64_t i = 0; i < h; ++i)
        for (int64_t j = 0; j < fw_; ++j) P[o_w1 + i * 4 * h + g * fw_ + j] = w1[(size_t)(i * fw_ + j)];
      auto b1 = down(R.db1, fw_);
      for (int64_t j = 0; j < fw_; ++j) P[o_b1 + g * fw_ + j] = b1[(size_t)j];
      auto w2 = down(R.dw2, fw_ * h);
      for (int64_t i = 0; i < fw_ * h; ++i) P[o_w2 + g * fw_ * h + i] = w2[(size_t)i];
      if (r == 0) {
        auto repl = down(R.repl, 6 * h);
        const int64_t dst[6] = {o_bo, o_b2, o_g1, o_be1, o_g2, o_be2};
        for (int kx = 0; kx < 6; ++kx)
          for (int64_t j = 0; j < h; ++j) P[dst[kx] + j] = repl[(size_t)(kx * h + j)];
      }
    }
  }

  void get_w1_grad_shard(int r, double* out) override {
    require(r >= 0 && r < L_, "local rank out of range");
    SPL_CUDA(cudaStreamSynchronize(st_));
    auto w1 = down(R_[r].dw1, h_ * fw_);
    for (size_t i = 0; i < w1.size(); ++i) out[i] = w1[i];
  }

  void get_saved(int r, const std::string& name, double* out, int64_t n) override {
    require(r >= 0 && r < L_, "local rank out of range");
    SPL_CUDA(cudaSetDevice(dev_));
    if (!have_fwd_) raise(5, "missing saved forward state");
    Rank& R = R_[r];
    const T* src = nullptr;
    const uint8_t* msrc = nullptr;
    int64_t cnt = 0, col = -1, width = 0, ld = 0;
    if (name == "ln1_input") { src = R.x_s; cnt = RL_ * h_; }
    else if (name == "qkv_input") { src = R.y1_s; cnt = RL_ * h_; }
    else if (name == "query" || name == "key" || name == "value") {
      src = R.qkv; cnt = RF_ * lw_; width = lw_; ld = 3 * lw_;
      col = name == "query" ? 0 : name == "key" ? lw_ : 2 * lw_;
    }
    else if (name == "softmax_out" && R.sm) { src = R.sm; cnt = lh_ * b_ * s_ * s_; }
    else if (name == "softmax_dropout_mask" && R.mask_i) { msrc = R.mask_i; cnt = lh_ * b_ * s_ * s_; }
    else if (name == "softmax_dropout_out" && R.sd) { src = R.sd; cnt = lh_ * b_ * s_ * s_; }
    else if (name == "attn_proj_input") { src = R.api; cnt = RF_ * lw_; }
    else if (name == "attn_dropout_mask") { msrc = R.amask; cnt = RL_ * h_; }
    else if (name == "ln2_input") { src = R.r1; cnt = RL_ * h_; }
    else if (name == "mlp_fc1_input") { src = R.y2; cnt = RL_ * h_; }
    else if (name == "gelu_input") { src = R.gin; cnt = RF_ * fw_; }
    else if (name == "mlp_fc2_input") { src = R.fin; cnt = RF_ * fw_; }
    else if (name == "mlp_dropout_mask") { msrc = R.mmask; cnt = RL_ * h_; }
    else raise(1, "unknown or not-stored saved tensor: " + name);
    require(n == cnt, "saved tensor size mismatch for " + name);
    double* dbuf = nullptr;
    SPL_CUDA(cudaMalloc(&dbuf, sizeof(double) * (size_t)cnt));
    if (msrc) {
      k::u8_to_f64(msrc, dbuf, cnt, st_);
    } else if (col >= 0) {
      T* tmp = nullptr;
      SPL_CUDA(cudaMalloc(&tmp, sizeof(T) * (size_t)cnt));
      SPL_CUDA(cudaMemcpy2DAsync(tmp, width * sizeof(T), src + col, ld * sizeof(T),
                                 width * sizeof(T), RF_, cudaMemcpyDeviceToDevice, st_));
      k::cast_to_f64<T>(tmp, dbuf, cnt, st_);
      SPL_CUDA(cudaStreamSynchronize(st_));
      cudaFree(tmp);
    } else {
      k::cast_to_f64<T>(src, dbuf, cnt, st_);
    }
    SPL_CUDA(cudaMemcpyAsync(out, dbuf, sizeof(double) * (size_t)cnt, cudaMemcpyDeviceToHost, st_));
    SPL_CUDA(cudaStreamSynchronize(st_));
    cudaFree(dbuf);
  }

  void attention_interior(int r, double* out3) override {
    require(r >= 0 && r < L_, "local rank out of range");
    if (!have_fwd_) raise(5, "missing saved forward state");
    SPL_CUDA(cudaSetDevice(dev_));
    const int64_t n = lh_ * b_ * s_ * s_;
    T *sm = nullptr, *sd = nullptr, *o = nullptr;
    uint8_t* mk = nullptr;
    double* dbuf = nullptr;
    SPL_CUDA(cudaMalloc(&sm, sizeof(T) * n));
    SPL_CUDA(cudaMalloc(&sd, sizeof(T) * n));
    SPL_CUDA(cudaMalloc(&mk, n));
    SPL_CUDA(cudaMalloc(&o, sizeof(T) * RF_ * lw_));
    SPL_CUDA(cudaMalloc(&dbuf, sizeof(double) * 3 * n));
    k::AttnArgs a = attn_args(r);
    a.o = o;
    a.ldo = lw_;
    a.lse = nullptr;
    a.sm = sm;
    a.mask = mk;
    a.sd = sd;
    k::attn_keep_bits(a, st_);
    k::attn_fwd<T>(a, st_);
    k::cast_to_f64<T>(sm, dbuf, n, st_);
    k::u8_to_f64(mk, dbuf + n, n, st_);
    k::cast_to_f64<T>(sd, dbuf + 2 * n, n, st_);
    SPL_CUDA(cudaMemcpyAsync(out3, dbuf, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, st_));
    SPL_CUDA(cudaStreamSynchronize(st_));
    cudaFree(sm); cudaFree(sd); cudaFree(mk); cudaFree(o); cudaFree(dbuf);
  }

  // ------------------------------------------------------------------ accounting
  std::vector<LedgerItem> ledger(int r) const override {
    (void)r;
    std::vector<LedgerItem> v;
    const int64_t A = d_.act_bytes, M = d_.mask_bytes, TS = sizeof(T);
    auto add = [&](const char* n, int64_t e, bool mask) {
      v.push_back({n, e, e * (mask ? M : A), e * (mask ? 1 : TS)});
    };
    add("ln1_input", RL_ * h_, false);
    if (kind_ == SPL_RECOMPUTE_FULL) return v;
    add("qkv_input", RL_ * h_, false);
    add("query", RF_ * lw_, false);
    add("key", RF_ * lw_, false);
    add("value", RF_ * lw_, false);
    if (kind_ == SPL_RECOMPUTE_NONE) {
      const int64_t ni = lh_ * b_ * s_ * s_;
      add("softmax_out", ni, false);
      add("softmax_dropout_mask", ni, true);
      add("softmax_dropout_out", ni, false);
    }
    add("attn_proj_input", RF_ * lw_, false);
    add("attn_dropout_mask", RL_ * h_, true);
    add("ln2_input", RL_ * h_, false);
    add("mlp_fc1_input", RL_ * h_, false);
    add("gelu_input", RF_ * fw_, false);
    add("mlp_fc2_input", RF_ * fw_, false);
    add("mlp_dropout_mask", RL_ * h_, true);
    return v;
  }

  void alloc_bytes(int64_t out[5]) const override {
    for (int c = 0; c < 5; ++c) out[c] = 0;
    for (auto& a : allocs_) out[a.cat] += (int64_t)a.bytes;
  }

  void saved_bytes(int r, int64_t* lb, int64_t* pb, int64_t* ub) const override {
    int64_t l = 0, p = 0;
    for (auto& e : ledger(r)) {
      l += e.bytes;
      p += e.physical;
    }
    int64_t u = 0;
    if (kind_ != SPL_RECOMPUTE_FULL) u += 4 * RL_ * (int64_t)sizeof(float);  // LN stats
    if (kind_ == SPL_RECOMPUTE_SELECTIVE) u += lh_ * b_ * s_ * (int64_t)sizeof(float);  // LSE
    *lb = l;
    *pb = p;
    *ub = u;
  }

  // ------------------------------------------------------------------ profiling
  void set_profile(bool on) override {
    SPL_CUDA(cudaStreamSynchronize(st_));
    profiling_ = on;
    pending_.clear();
    for (int c = 0; c < K_NCLASS; ++c) prof_ms_[c] = prof_flops_[c] = prof_bytes_[c] = 0, prof_n_[c] = 0;
    ev_next_ = 0;
  }
  void read_profile(double ms[K_NCLASS], int64_t n[K_NCLASS], double fl[K_NCLASS],
                    double by[K_NCLASS]) override {
    SPL_CUDA(cudaStreamSynchronize(st_));
    for (auto& p : pending_) {
      float e = 0.f;
      SPL_CUDA(cudaEventElapsedTime(&e, p.a, p.b));
      prof_ms_[p.cls] += e;
    }
    pending_.clear();
    ev_next_ = 0;
    for (int c = 0; c < K_NCLASS; ++c) {
      ms[c] = prof_ms_[c];
      n[c] = prof_n_[c];
      fl[c] = prof_flops_[c];
      by[c] = prof_bytes_[c];
    }
  }
  int64_t launch_count(bool reset) override {
    const int64_t v = launches_;
    if (reset) launches_ = 0;
    return v;
  }
  void set_graphs(bool on) override {
    graphs_ = on;
    if (!on) drop_graphs();
  }
  void drop_graphs() {
    for (auto* set : {&gfwd_, &gbwd_}) {
      for (Graph& g : *set)
        if (g.exec) SPL_CUDA(cudaGraphExecDestroy(g.exec));
      set->clear();
    }
  }
  // Captured graphs hold the keys and the epilogue modes by value: re-capture on change.
  void set_microbatch(uint32_t microbatch) override {
    if (microbatch == d_.microbatch) return;
    d_.microbatch = microbatch;
    make_keys();
    drop_graphs();
  }
  void set_grad_accumulate(bool on) override {
    if (on == grad_acc_) return;
    grad_acc_ = on;
    drop_graphs();
  }
  void make_keys() {
    const spl_layer_desc& d = d_;
    k_soft_ = make_drop_key(d.seed, d.layer_index, kSoftmaxDrop, d.microbatch, d.dropout_p);
    k_attn_ = make_drop_key(d.seed, d.layer_index, kAttnOutDrop, d.microbatch, d.dropout_p);
    k_mlp_ = make_drop_key(d.seed, d.layer_index, kMlpDrop, d.microbatch, d.dropout_p);
  }

 private:
  struct Rank {
    T *wqkv = nullptr, *wo = nullptr, *w1 = nullptr, *w2 = nullptr;
    float *bqkv = nullptr, *bo = nullptr, *b1 = nullptr, *b2 = nullptr, *g1 = nullptr,
          *be1 = nullptr, *g2 = nullptr, *be2 = nullptr;
    float *dwqkv = nullptr, *dbqkv = nullptr, *dwo = nullptr, *dw1 = nullptr, *db1 = nullptr,
          *dw2 = nullptr, *repl = nullptr, *repl_new = nullptr;
    T *x_s = nullptr, *y1_s = nullptr, *qkv = nullptr, *sm = nullptr, *sd = nullptr,
      *api = nullptr, *r1 = nullptr, *y2 = nullptr, *gin = nullptr, *fin = nullptr;
    uint8_t *mask_i = nullptr, *amask = nullptr, *mmask = nullptr;
    float *mu1 = nullptr, *rs1 = nullptr, *mu2 = nullptr, *rs2 = nullptr, *lse = nullptr;
    T *yfull = nullptr, *part = nullptr, *rs_out = nullptr, *dfull = nullptr, *dgin = nullptr,
      *dqkv = nullptr, *dproj = nullptr, *d_s = nullptr, *dr1 = nullptr, *y_re = nullptr;
    float *delta = nullptr, *partials = nullptr;
    uint32_t* keepbits = nullptr;
    float *dq_acc = nullptr, *bstat = nullptr;  // fused attention backward workspaces
  };
  bool bits_t_ = false;  // keep bits currently in the transposed (fused backward) layout
  // SPL_KEEPBITS_T=1: the selective backward's keep bits in the transposed layout (the RNG
  // pass stores (key, 32 queries) words; the fused kernel skips its per-tile warp transposes)
  static bool keep_bits_t_env() {
    static const bool on = [] {
      const char* e = std::getenv("SPL_KEEPBITS_T");
      return e != nullptr && e[0] == '1';
    }();
    return on;
  }

  void validate() {
    require(t_ >= 1, "t must be >= 1");
    require(a_ >= 1 && h_ >= 1 && s_ >= 1 && b_ >= 1, "shape fields must be >= 1");
    require(h_ % a_ == 0, "hidden not divisible by heads");
    require(s_ % t_ == 0 && h_ % t_ == 0, "s and h must be divisible by t");
    require(a_ % t_ == 0, "attention heads must be divisible by t");
    require(d_.dropout_p >= 0.0 && d_.dropout_p < 1.0, "dropout probability must lie in [0, 1)");
    require(d_.recompute >= 0 && d_.recompute <= 2, "unknown recompute kind");
    require(d_.act_bytes >= 1 && d_.mask_bytes >= 1, "byte convention widths must be >= 1");
    require(h_ / a_ <= 256, "head_dim > 256 unsupported");
  }

  static T cvt(double v) {
    if constexpr (std::is_same_v<T, float>) return (float)v;
    else return __double2bfloat16(v);
  }

  template <typename U>
  U* alloc(int64_t n, int cat, int r) {
    void* p = nullptr;
    const size_t bytes = (size_t)std::max<int64_t>(n, 1) * sizeof(U);
    if ((cat == kParam || cat == kGrad) && params_) {  // window slot: shared parameters
      const size_t i = param_next_++;
      if (i < params_->bufs.size()) {
        require(params_->bufs[i].second == bytes, "parameter pool: layer shapes differ");
        return static_cast<U*>(params_->bufs[i].first);
      }
      SPL_CUDA(cudaMalloc(&p, bytes));
      SPL_CUDA(cudaMemset(p, 0, bytes));
      params_->bufs.push_back({p, bytes});
      return static_cast<U*>(p);
    }
    if (cat == kWork && pool_) {  // stack member: the i-th workspace request is shared
      const size_t i = work_next_++;
      if (i < pool_->bufs.size()) {
        require(pool_->bufs[i].second == bytes, "workspace pool: layer shapes differ");
        return static_cast<U*>(pool_->bufs[i].first);
      }
      SPL_CUDA(cudaMalloc(&p, bytes));
      SPL_CUDA(cudaMemset(p, 0, bytes));
      pool_->bufs.push_back({p, bytes});
      return static_cast<U*>(p);
    }
    SPL_CUDA(cudaMalloc(&p, bytes));
    SPL_CUDA(cudaMemset(p, 0, bytes));
    allocs_.push_back({p, bytes, cat, r});
    return static_cast<U*>(p);
  }

  template <typename U>
  void up(U* dst, const std::vector<U>& v) {
    SPL_CUDA(cudaMemcpy(dst, v.data(), v.size() * sizeof(U), cudaMemcpyHostToDevice));
  }
  std::vector<double> down(const float* src, int64_t n) {
    std::vector<float> f((size_t)n);
    SPL_CUDA(cudaMemcpy(f.data(), src, sizeof(float) * (size_t)n, cudaMemcpyDeviceToHost));
    return std::vector<double>(f.begin(), f.end());
  }

  void allocate() {
    R_.resize(L_);
    const int64_t ni = lh_ * b_ * s_ * s_;
    const int saved = kind_ == SPL_RECOMPUTE_FULL ? kWork : kSaved;
    const int saved_u = kind_ == SPL_RECOMPUTE_FULL ? kWork : kSavedUncounted;
    const int nch_l = k::num_chunks(RL_, kChunkRows), nch_f = k::num_chunks(RF_, kChunkRows);
    const int64_t npart = std::max<int64_t>(2 * (int64_t)nch_l * h_, nch_f * std::max<int64_t>(3 * lw_, fw_));
    T *yfull = nullptr, *dfull = nullptr, *dgin = nullptr, *dqkv = nullptr, *dproj = nullptr;
    float *delta = nullptr, *partials = nullptr, *dq_acc = nullptr, *bstat = nullptr;
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      R.wqkv = alloc<T>(h_ * 3 * lw_, kParam, r);
      R.bqkv = alloc<float>(3 * lw_, kParam, r);
      R.wo = alloc<T>(lw_ * h_, kParam, r);
      R.bo = alloc<float>(h_, kParam, r);
      R.w1 = alloc<T>(h_ * fw_, kParam, r);
      R.b1 = alloc<float>(fw_, kParam, r);
      R.w2 = alloc<T>(fw_ * h_, kParam, r);
      R.b2 = alloc<float>(h_, kParam, r);
      R.g1 = alloc<float>(h_, kParam, r);
      R.be1 = alloc<float>(h_, kParam, r);
      R.g2 = alloc<float>(h_, kParam, r);
      R.be2 = alloc<float>(h_, kParam, r);
      R.dwqkv = alloc<float>(h_ * 3 * lw_, kGrad, r);
      R.dbqkv = alloc<float>(3 * lw_, kGrad, r);
      R.dwo = alloc<float>(lw_ * h_, kGrad, r);
      R.dw1 = alloc<float>(h_ * fw_, kGrad, r);
      R.db1 = alloc<float>(fw_, kGrad, r);
      R.dw2 = alloc<float>(fw_ * h_, kGrad, r);
      R.repl = alloc<float>(6 * h_, kGrad, r);
      R.repl_new = alloc<float>(6 * h_, kWork, r);
      R.x_s = alloc<T>(RL_ * h_, kSaved, r);
      R.y1_s = alloc<T>(RL_ * h_, saved, r);
      R.qkv = alloc<T>(RF_ * 3 * lw_, saved, r);
      if (kind_ == SPL_RECOMPUTE_NONE) {
        R.sm = alloc<T>(ni, kSaved, r);
        R.mask_i = alloc<uint8_t>(ni, kSaved, r);
        R.sd = alloc<T>(ni, kSaved, r);
      } else {
        R.lse = alloc<float>(lh_ * b_ * s_, saved_u, r);
      }
      R.api = alloc<T>(RF_ * lw_, saved, r);
      R.amask = alloc<uint8_t>(RL_ * h_, saved, r);
      R.r1 = alloc<T>(RL_ * h_, saved, r);
      R.y2 = alloc<T>(RL_ * h_, saved, r);
      R.gin = alloc<T>(RF_ * fw_, saved, r);
      R.fin = alloc<T>(RF_ * fw_, saved, r);
      R.mmask = alloc<uint8_t>(RL_ * h_, saved, r);
      R.mu1 = alloc<float>(RL_, saved_u, r);
      R.rs1 = alloc<float>(RL_, saved_u, r);
      R.mu2 = alloc<float>(RL_, saved_u, r);
      R.rs2 = alloc<float>(RL_, saved_u, r);
      // workspaces (transient, not stored activations)
      if (sp_) {
        if (!yfull || comm_->local() == 1) yfull = alloc<T>(RF_ * h_, kWork, r);
        if (!dfull || comm_->local() == 1) dfull = alloc<T>(RF_ * h_, kWork, r);
        R.yfull = yfull;
        R.dfull = dfull;
        R.rs_out = alloc<T>(RL_ * h_, kWork, r);
      }
      R.part = alloc<T>(RF_ * h_, kWork, r);
      dgin = alloc<T>(RF_ * fw_, kWork, r);
      dqkv = alloc<T>(RF_ * 3 * lw_, kWork, r);
      if (!dproj) {
        dproj = alloc<T>(RF_ * lw_, kWork, r);
        delta = alloc<float>(lh_ * b_ * s_, kWork, r);
        partials = alloc<float>(npart, kWork, r);
      }
      // transient keep bits of the softmax dropout (1 bit / interior element), refilled on the
      // side stream at the start of every forward and backward call
      if (std::is_same_v<T, bf16> && d_.dropout_p > 0.0)
        R.keepbits = alloc<uint32_t>(k::keepbits_words(lh_, b_, s_), kWork, r);
      // fused attention backward (bf16, head_dim 64/96; recompute regimes and the stored
      // interior): fp32 dQ accumulator and per-row statistics
      if (std::is_same_v<T, bf16> && (hd_ == 64 || hd_ == 96) && s_ % 128 == 0) {
        if (!dq_acc) {
          dq_acc = alloc<float>(lh_ * b_ * s_ * hd_, kWork, r);
          bstat = alloc<float>(2 * lh_ * b_ * s_, kWork, r);
        }
        R.dq_acc = dq_acc;
        R.bstat = bstat;
      }
      R.dgin = dgin;
      R.dqkv = dqkv;
      R.dproj = dproj;
      R.delta = delta;
      R.partials = partials;
      R.d_s = alloc<T>(RL_ * h_, kWork, r);
      R.dr1 = alloc<T>(RL_ * h_, kWork, r);
      if (kind_ == SPL_RECOMPUTE_FULL) R.y_re = alloc<T>(RL_ * h_, kWork, r);
    }
    nonfinite_ = alloc<int>(1, kWork, 0);
  }

  void ensure_staging() {  // [rank][slot][x, dy, y, dx]
    if (!stage_.empty()) return;
    for (int r = 0; r < L_; ++r)
      for (int i = 0; i < 8; ++i) stage_.push_back(alloc<T>(RL_ * h_, kWork, r));
  }

  // ---- launch bookkeeping
  template <typename F>
  void launch(KClass cls, int kernels, double flops, double bytes, F&& f) {
    launch_on(st_, cls, kernels, flops, bytes, std::forward<F>(f));
  }
  template <typename F>
  void launch_on(cudaStream_t stream, KClass cls, int kernels, double flops, double bytes, F&& f) {
    launches_ += kernels;
    if (!profiling_) {
      f();
      return;
    }
    if (ev_next_ + 2 > evpool_.size()) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        SPL_CUDA(cudaEventCreate(&e));
        evpool_.push_back(e);
      }
    }
    cudaEvent_t ea = evpool_[ev_next_++], eb = evpool_[ev_next_++];
    SPL_CUDA(cudaEventRecord(ea, stream));
    f();
    SPL_CUDA(cudaEventRecord(eb, stream));
    pending_.push_back({ea, eb, cls});
    prof_n_[cls] += kernels;
    prof_flops_[cls] += flops;
    prof_bytes_[cls] += bytes;
  }

  // Which gathered tensor a GEMM operand is: with the fused all-gather the operand is read
  // from every rank's shard instead of the gathered copy.
  enum Gath : int { kNoGath = 0, kGY1, kGY2, kGD };
  const void* shard_of(Gath w, int q) const {
    if (pull_) return peer_[w][q];  // peer ranks: the shard in rank q's memory
    return w == kGY1 ? (const void*)R_[q].y1_s : w == kGY2 ? (const void*)R_[q].y2
                                                           : (const void*)R_[q].d_s;
  }
  const void* own_shard(Gath w) const {
    return w == kGY1 ? (const void*)R_[0].y1_s : w == kGY2 ? (const void*)R_[0].y2
                                                           : (const void*)R_[0].d_s;
  }
  GemmArgs gemm_args(int64_t M, int64_t N, int64_t K, const T* A, int64_t lda, Major am,
                     const T* B, int64_t ldb, Major bm, void* C, int64_t ldc, Epi epi,
                     Gath ga, Gath gb) const {
    GemmArgs g;
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.lda = lda; g.amaj = am;
    g.B = B; g.ldb = ldb; g.bmaj = bm;
    g.C = C; g.ldc = ldc; g.epi = epi;
    if (ga != kNoGath || gb != kNoGath) {
      g.shard_rows = RL_;
      for (int q = 0; q < t_; ++q) {
        if (ga != kNoGath) g.a_shard[q] = shard_of(ga, q);
        if (gb != kNoGath) g.b_shard[q] = shard_of(gb, q);
      }
      g.a_shards = ga != kNoGath ? t_ : 0;
      g.b_shards = gb != kNoGath ? t_ : 0;
    }
    return g;
  }
  // every GEMM that consumes a gathered tensor must run on the pair kernel (probed with the
  // real buffers of rank 0)
  bool fused_ag_eligible() const {
    if (!(RF_ % 256 == 0)) return false;
    const Rank& R = R_[0];
    const GemmArgs probes[] = {
        gemm_args(RF_, 3 * lw_, h_, nullptr, h_, Major::K, R.wqkv, 3 * lw_, Major::MN, R.qkv,
                  3 * lw_, Epi::Bias, kGY1, kNoGath),
        gemm_args(RF_, fw_, h_, nullptr, h_, Major::K, R.w1, fw_, Major::MN, R.gin, fw_,
                  Epi::BiasGelu, kGY2, kNoGath),
        gemm_args(RF_, fw_, h_, nullptr, h_, Major::K, R.w2, h_, Major::K, R.dgin, fw_,
                  Epi::GeluBwd, kGD, kNoGath),
        gemm_args(fw_, h_, RF_, R.fin, fw_, Major::MN, nullptr, h_, Major::MN, R.dw2, h_,
                  Epi::F32, kNoGath, kGD),
        gemm_args(h_, fw_, RF_, nullptr, h_, Major::MN, R.dgin, fw_, Major::MN, R.dw1, fw_,
                  Epi::F32, kGY2, kNoGath),
        gemm_args(RF_, lw_, h_, nullptr, h_, Major::K, R.wo, h_, Major::K, R.dproj, lw_,
                  Epi::Store, kGD, kNoGath),
        gemm_args(lw_, h_, RF_, R.api, lw_, Major::MN, nullptr, h_, Major::MN, R.dwo, h_,
                  Epi::F32, kNoGath, kGD),
        gemm_args(h_, 3 * lw_, RF_, nullptr, h_, Major::MN, R.dqkv, 3 * lw_, Major::MN,
                  R.dwqkv, 3 * lw_, Epi::F32, kGY1, kNoGath)};
    for (const GemmArgs& g : probes) {
      GemmArgs p = g;
      if (p.epi == Epi::BiasGelu) p.C2 = R.fin;
      if (p.epi == Epi::GeluBwd) {
        p.aux = R.gin;
        p.ldaux = fw_;
      }
      if (!k::gemm_tc_pair_path(p)) return false;
    }
    return true;
  }

  void gemm(int64_t M, int64_t N, int64_t K, const T* A, int64_t lda, Major am, const T* B,
            int64_t ldb, Major bm, void* C, int64_t ldc, Epi epi, const float* bias = nullptr,
            void* C2 = nullptr, const T* aux = nullptr, int64_t ldaux = 0, int scatter_rank = -1,
            Gath ga = kNoGath, Gath gb = kNoGath) {
    if (!fused_ag_) ga = gb = kNoGath;
    GemmArgs g = gemm_args(M, N, K, A, lda, am, B, ldb, bm, C, ldc, epi, ga, gb);
    g.bias = bias; g.C2 = C2; g.aux = aux; g.ldaux = ldaux;
    g.accumulate = epi == Epi::F32 && grad_acc_;
    if (scatter_rank >= 0) {  // the reduce-scatter fused into this row-parallel GEMM
      // back-pressure: the destinations consumed this source's previous landing (peer ranks;
      // simulated ranks are ordered by the one stream)
      if (comm_->local() != t_)
        launch(K_COMM, 1, 0, 0, [&] { comm_->p2p_ready_wait(rank0_ + scatter_rank, st_); });
      for (int q = 0; q < t_; ++q) g.scatter[q] = comm_->p2p_slot(q, rank0_ + scatter_rank);
      g.scatter_n = t_;
      g.scatter_rows = RL_;
    }
    const double es = sizeof(T);
    const double bytes = (M * K + K * N) * es + M * N * (epi == Epi::F32 ? 4.0 : es) *
                         (epi == Epi::BiasGelu ? 2 : 1) + (epi == Epi::GeluBwd ? M * N * es : 0);
    launch(K_GEMM, 1, 2.0 * M * N * K, bytes, [&] { k::gemm<T>(g, st_); });
  }

  k::AttnArgs attn_args(int r) {
    Rank& R = R_[r];
    k::AttnArgs a;
    a.s = s_; a.b = b_; a.lh = lh_; a.hd = hd_;
    a.head_offset = (rank0_ + r) * lh_;
    a.heads_total = a_;
    a.qkv = R.qkv; a.ld = 3 * lw_; a.qoff = 0; a.koff = lw_; a.voff = 2 * lw_;
    a.o = R.api; a.ldo = lw_;
    a.scale = scale_;
    a.causal = d_.causal;
    a.drop = k_soft_;
    a.lse = R.lse;
    a.sm = R.sm; a.mask = R.mask_i; a.sd = R.sd;
    a.keepbits = R.keepbits;
    a.dq_acc = R.dq_acc;
    a.bstat = R.bstat;
    a.keep_t = bits_t_ ? 1 : 0;
    return a;
  }

  double attn_flops(bool bwd) const {
    // QKᵀ and P·V per head: 2·s²·hd each (halved when causal); backward: 5 GEMM-equivalents
    // of which recompute of QKᵀ is one (flash-style backward).
    const double per = 2.0 * (double)s_ * s_ * hd_ * lh_ * b_ * (d_.causal ? 0.5 : 1.0);
    return bwd ? per * 5.0 : per * 2.0;
  }

  // ---- collectives
  std::vector<const void*> cptrs(std::function<const void*(int)> f) {
    std::vector<const void*> v(L_);
    for (int r = 0; r < L_; ++r) v[r] = f(r);
    return v;
  }
  std::vector<void*> mptrs(std::function<void*(int)> f) {
    std::vector<void*> v(L_);
    for (int r = 0; r < L_; ++r) v[r] = f(r);
    return v;
  }
  DType dt() const { return std::is_same_v<T, float> ? DType::F32 : DType::BF16; }

  // g (forward) / ḡ-dual (backward): shards {RL,h} -> full {RF,h}
  void gather(std::function<const void*(int)> shard, std::function<void*(int)> full, CommTag tag) {
    comm_->log(tag, 0, RF_ * h_);
    if (t_ == 1) return;  // identity; callers read the shard itself (see gathered())
    if (fused_ag_) {  // the consuming GEMMs read the shards (GemmArgs::a_shard/b_shard)
      // peer ranks: every rank's shard written before any rank's consumer reads it. The
      // re-gathers (stored Y1 / Y2, gather_async) need none: written in the forward, many
      // barriers ago. Write-after-read is ordered by the schedule: a rank rewrites Y1 / Y2 in
      // its next forward, after the gradient all-reduce every rank enters after its last
      // reader; dY shards (d_s) are rewritten after the reduce-scatter that follows every
      // rank's readers of them.
      if (pull_) launch(K_COMM, 1, 0, 0, [&] { comm_->p2p_barrier(st_); });
      return;
    }
    auto s = cptrs(shard);
    auto f = mptrs(full);
    launch(K_COMM, 1, 0, (double)RF_ * h_ * sizeof(T) * (t_ - 1) / t_,
           [&] { comm_->all_gather(s.data(), f.data(), RL_ * h_, dt(), st_); });
  }
  // ḡ (forward) / g-dual (backward): partials {RF,h} -> shards {RL,h}; without SP an
  // all-reduce in place (f̄ / f), the result left in part.
  void scatter(CommTag tag) {
    if (sp_) {
      comm_->log(tag, 1, RF_ * h_);
      if (t_ == 1) return;  // identity: scattered(r) returns part
      auto p = cptrs([&](int r) { return (const void*)R_[r].part; });
      auto o = mptrs([&](int r) { return (void*)R_[r].rs_out; });
      launch(K_COMM, 1, 0, (double)RF_ * h_ * sizeof(T) * (t_ - 1) / t_,
             [&] { comm_->reduce_scatter(p.data(), o.data(), RL_ * h_, dt(), st_); });
    } else if (t_ > 1) {
      auto p = mptrs([&](int r) { return (void*)R_[r].part; });
      comm_->log(tag, 2, RF_ * h_);
      launch(K_COMM, 1, 0, 2.0 * RF_ * h_ * sizeof(T) * (t_ - 1) / t_,
             [&] { comm_->all_reduce(p.data(), RF_ * h_, dt(), st_); });
    }
  }
  // ---- reduce-scatter fused into the row-parallel GEMMs (GemmArgs::scatter): the producing
  // GEMM of local rank r lands its rows of shard q in q's slot for r (peer memory over
  // NVLink for NCCL ranks, device buffers for simulated ranks), signal() publishes them, the
  // consumer of shard r waits for all t sources and sums the slots in rank order.
  int fused_rank(int r) const { return fused_rs_ ? r : -1; }
  void fused_signal(int r) {
    k::FlagPtrs f;
    for (int q = 0; q < t_; ++q) f.p[q] = comm_->p2p_flag(q, rank0_ + r);
    f.n = t_;
    launch(K_COMM, 1, 0, 0, [&] { k::p2p_signal(f, st_); });
  }
  k::SlotSrc fused_src(int r) {
    k::SlotSrc a;
    for (int q = 0; q < t_; ++q) a.p[q] = comm_->p2p_slot_local(rank0_ + r, q);
    a.n = t_;
    a.flags = comm_->p2p_flags_local(rank0_ + r);
    a.gen = comm_->p2p_gen(rank0_ + r);
    return a;
  }
  void fused_advance(int r) {
    uint32_t* gen = comm_->p2p_gen(rank0_ + r);
    launch(K_COMM, 1, 0, 0, [&] { k::p2p_advance(gen, st_); });
  }
  // the backward's consumers read rs_out: sum the slots into it
  void fused_reduce(int r) {
    const k::SlotSrc a = fused_src(r);
    launch(K_COMM, 1, 0, (double)t_ * RL_ * h_ * sizeof(T), [&] {
      k::reduce_slots<T>(a, R_[r].rs_out, RL_ * h_, st_);
    });
    fused_advance(r);
  }

  // Collective on the comm stream after everything issued so far on the compute stream;
  // returns the event the consumer waits on (nullptr when there is nothing to wait for).
  cudaEvent_t gather_async(std::function<const void*(int)> shard, std::function<void*(int)> full,
                           CommTag tag, cudaEvent_t done) {
    if (!(sp_ && t_ > 1) || fused_ag_) {
      comm_->log(tag, 0, RF_ * h_);
      return nullptr;
    }
    if (comm_serial_) {
      auto s = cptrs(shard);
      auto f = mptrs(full);
      comm_->log(tag, 0, RF_ * h_);
      launch(K_COMM, 1, 0, (double)RF_ * h_ * sizeof(T) * (t_ - 1) / t_,
             [&] { comm_->all_gather(s.data(), f.data(), RL_ * h_, dt(), st_); });
      return nullptr;
    }
    SPL_CUDA(cudaEventRecord(ev_cfork_, st_));
    SPL_CUDA(cudaStreamWaitEvent(st_comm_, ev_cfork_, 0));
    auto s = cptrs(shard);
    auto f = mptrs(full);
    comm_->log(tag, 0, RF_ * h_);
    launch_on(st_comm_, K_COMM, 1, 0, (double)RF_ * h_ * sizeof(T) * (t_ - 1) / t_,
              [&] { comm_->all_gather(s.data(), f.data(), RL_ * h_, dt(), st_comm_); });
    SPL_CUDA(cudaEventRecord(done, st_comm_));
    return done;
  }
  cudaEvent_t scatter_async(CommTag tag, cudaEvent_t done) {
    if (t_ == 1 || comm_serial_) {
      scatter(tag);
      return nullptr;
    }
    SPL_CUDA(cudaEventRecord(ev_cfork_, st_));
    SPL_CUDA(cudaStreamWaitEvent(st_comm_, ev_cfork_, 0));
    cudaStream_t keep = st_;
    st_ = st_comm_;  // scatter() launches on st_
    try {
      scatter(tag);
    } catch (...) {
      st_ = keep;
      throw;
    }
    st_ = keep;
    SPL_CUDA(cudaEventRecord(done, st_comm_));
    return done;
  }
  void wait_on(cudaEvent_t e) {
    if (e != nullptr) SPL_CUDA(cudaStreamWaitEvent(st_, e, 0));
  }

  T* scattered(int r) { return (sp_ && t_ > 1) ? R_[r].rs_out : R_[r].part; }
  // the gathered {s,b,h} view of a sequence-sharded tensor (the shard itself when t == 1)
  const T* gathered(int r, const T* shard) const { return (sp_ && t_ > 1) ? R_[r].yfull : shard; }
  const T* gathered_d(int r, const T* shard) const { return (sp_ && t_ > 1) ? R_[r].dfull : shard; }

  // Fork the data-independent dropout-mask RNG onto the side stream (it overlaps the GEMMs
  // that precede attention); join() makes the main stream wait for it.
  // transposed: the backward's bits for the fused attention backward (k::attn_bwd_uses_fused)
  void fork_keep_bits(bool transposed = false) {
    if (R_.empty() || R_[0].keepbits == nullptr) return;
    bits_t_ = false;
    if (transposed) {
      k::AttnArgs a0 = attn_args(0);
      a0.keep_t = 1;
      bits_t_ = k::attn_bwd_uses_fused(a0);
    }
    if (bits_serial_) {  // on the main stream, right before its consumer
      for (int r = 0; r < L_; ++r) {
        k::AttnArgs a = attn_args(r);
        launch(K_OTHER, 1, 0, (double)lh_ * b_ * s_ * s_ / 8.0, [&] { k::attn_keep_bits(a, st_); });
      }
      return;
    }
    SPL_CUDA(cudaEventRecord(ev_fork_, st_));
    SPL_CUDA(cudaStreamWaitEvent(st_rng_, ev_fork_, 0));
    for (int r = 0; r < L_; ++r) {
      k::AttnArgs a = attn_args(r);
      const double elems = (double)lh_ * b_ * s_ * s_;
      launch_on(st_rng_, K_OTHER, 1, 0, elems / 8.0, [&] { k::attn_keep_bits(a, st_rng_); });
    }
    SPL_CUDA(cudaEventRecord(ev_bits_, st_rng_));
    bits_pending_ = true;
  }
  void join_keep_bits() {
    if (!bits_pending_) return;
    SPL_CUDA(cudaStreamWaitEvent(st_, ev_bits_, 0));
    bits_pending_ = false;
  }

  // ------------------------------------------------------------------ schedules
  void run_forward(T* const* y, CommTag tag, int* nonfinite) {
    fork_keep_bits();
    const int64_t h = h_;
    const float eps = (float)d_.ln_eps;
    const double eb = sizeof(T);
    // LN1 on sequence shards (block.cpp:546-550)
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      launch(K_ELEM, 1, 0, 2.0 * RL_ * h * eb, [&] {
        k::layernorm_fwd<T>(R.x_s, R.g1, R.be1, R.y1_s, R.mu1, R.rs1, RL_, h, eps, st_);
      });
    }
    // g: all-gather Y1 (block.cpp:551)
    if (sp_) gather([&](int r) { return (const void*)R_[r].y1_s; },
                    [&](int r) { return (void*)R_[r].yfull; }, tag);
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      const T* y1 = gathered(r, R.y1_s);
      // fused QKV projection, column-parallel (block.cpp:556-558)
      gemm(RF_, 3 * lw_, h, y1, h, Major::K, R.wqkv, 3 * lw_, Major::MN, R.qkv, 3 * lw_,
           Epi::Bias, R.bqkv, nullptr, nullptr, 0, -1, kGY1);
      // attention interior + attention over values (block.cpp:559-562)
      k::AttnArgs a = attn_args(r);
      join_keep_bits();
      launch(K_ATTN, 1, attn_flops(false), 0, [&] { k::attn_fwd<T>(a, st_); });
      // row-parallel projection partial (block.cpp:563); with the fused reduce-scatter its rows
      // land directly in the slots of the ranks that own them
      gemm(RF_, h, lw_, R.api, lw_, Major::K, R.wo, h, Major::MN, R.part, h, Epi::Store, nullptr,
           nullptr, nullptr, 0, fused_rank(r));
      if (fused_rs_) fused_signal(r);
    }
    if (fused_rs_) comm_->log(tag, 1, RF_ * h_);
    else scatter(tag);  // ḡ (block.cpp:567)
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      const uint64_t base = sp_ ? (uint64_t)((rank0_ + r) * RL_ * h) : 0;
      // bias + dropout + residual, fused with LN2 (block.cpp:568-578)
      if (fused_rs_) {
        const k::SlotSrc a = fused_src(r);
        launch(K_ELEM, 1, 0, (2.0 * t_ + 3.0) * eb * RL_ * h + RL_ * h, [&] {
          k::bias_dropout_residual_slots<T>(a, R.bo, R.x_s, R.r1, R.amask, R.y2, R.g2, R.be2,
                                            R.mu2, R.rs2, RL_, h, k_attn_, base, eps, nullptr, st_);
        });
        fused_advance(r);
        continue;
      }
      launch(K_ELEM, 1, 0, (4.0 * eb + 1.0) * RL_ * h, [&] {
        k::bias_dropout_residual<T>(scattered(r), R.bo, R.x_s, R.r1, R.amask, R.y2, R.g2, R.be2,
                                    R.mu2, R.rs2, RL_, h, k_attn_, base, eps, nullptr, st_);
      });
    }
    if (sp_) gather([&](int r) { return (const void*)R_[r].y2; },
                    [&](int r) { return (void*)R_[r].yfull; }, tag);  // block.cpp:580
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      const T* y2 = gathered(r, R.y2);
      // FC1 + bias + GELU, keeping both pre- and post-activation (block.cpp:584-585)
      gemm(RF_, fw_, h, y2, h, Major::K, R.w1, fw_, Major::MN, R.gin, fw_, Epi::BiasGelu, R.b1,
           R.fin, nullptr, 0, -1, kGY2);
      gemm(RF_, h, fw_, R.fin, fw_, Major::K, R.w2, h, Major::MN, R.part, h, Epi::Store,  // 586
           nullptr, nullptr, nullptr, 0, fused_rank(r));
      if (fused_rs_) fused_signal(r);
    }
    if (fused_rs_) comm_->log(tag, 1, RF_ * h_);
    else scatter(tag);  // block.cpp:588
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      const uint64_t base = sp_ ? (uint64_t)((rank0_ + r) * RL_ * h) : 0;
      if (fused_rs_) {
        const k::SlotSrc a = fused_src(r);
        launch(K_ELEM, 1, 0, (2.0 * t_ + 2.0) * eb * RL_ * h + RL_ * h, [&] {
          k::bias_dropout_residual_slots<T>(a, R.b2, R.r1, y[r], R.mmask, nullptr, nullptr,
                                            nullptr, nullptr, nullptr, RL_, h, k_mlp_, base, eps,
                                            nonfinite, st_);
        });
        fused_advance(r);
        continue;
      }
      launch(K_ELEM, 1, 0, (3.0 * eb + 1.0) * RL_ * h, [&] {
        k::bias_dropout_residual<T>(scattered(r), R.b2, R.r1, y[r], R.mmask, nullptr, nullptr,
                                    nullptr, nullptr, nullptr, RL_, h, k_mlp_, base, eps,
                                    nonfinite, st_);
      });
    }
  }

  void run_backward(const void* const* dyv, void* const* dxv) {
    const int64_t h = h_;
    // recompute regimes regenerate the keep bits (full recomputation just re-ran the forward,
    // whose bits are still in the buffer); the no-recompute regime reads the stored mask
    if (kind_ == SPL_RECOMPUTE_SELECTIVE) fork_keep_bits(keep_bits_t_env());
    const double eb = sizeof(T);
    const int nch_l = k::num_chunks(RL_, kChunkRows), nch_f = k::num_chunks(RF_, kChunkRows);
    const float inv_keep = k_mlp_.inv_keep;
    // ---- MLP branch (block.cpp:642-681)
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      const T* dy = static_cast<const T*>(dyv[r]);
      launch(K_ELEM, 2, 0, (2.0 * eb + 1.0) * RL_ * h, [&] {
        k::dropout_bwd_colsum<T>(dy, R.mmask, inv_keep, R.d_s, R.partials, RL_, h, kChunkRows, st_);
        k::reduce_partials(R.partials, nch_l, h, repl_w(R) + 1 * h, false, st_);  // b2 partial
      });
    }
    if (sp_)
      gather([&](int r) { return (const void*)R_[r].d_s; }, [&](int r) { return (void*)R_[r].dfull; },
             kSchedule);  // block.cpp:653
    // re-gather Y2 (block.cpp:655) on the comm stream, overlapped with the FC2 GEMMs
    cudaEvent_t y2_ready = gather_async([&](int r) { return (const void*)R_[r].y2; },
                                        [&](int r) { return (void*)R_[r].yfull; }, kRegather,
                                        ev_regather_);
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      const T* dmo = gathered_d(r, R.d_s);
      // FC2 dgrad fused with GELU backward (block.cpp:660, 662)
      gemm(RF_, fw_, h, dmo, h, Major::K, R.w2, h, Major::K, R.dgin, fw_, Epi::GeluBwd, nullptr,
           nullptr, R.gin, fw_, -1, kGD);
      // FC2 wgrad (block.cpp:661)
      gemm(fw_, h, RF_, R.fin, fw_, Major::MN, dmo, h, Major::MN, R.dw2, h, Epi::F32, nullptr,
           nullptr, nullptr, 0, -1, kNoGath, kGD);
      // b1 grad (block.cpp:663)
      launch(K_ELEM, 2, 0, eb * RF_ * fw_, [&] {
        k::colsum_partial<T>(R.dgin, RF_, fw_, fw_, R.partials, kChunkRows, st_);
        k::reduce_partials(R.partials, nch_f, fw_, R.db1, grad_acc_, st_);
      });
      // FC1 dgrad (block.cpp:665) first, so its reduce-scatter overlaps the FC1 wgrad
      gemm(RF_, h, fw_, R.dgin, fw_, Major::K, R.w1, fw_, Major::K, R.part, h, Epi::Store,
           nullptr, nullptr, nullptr, 0, fused_rank(r));
      if (fused_rs_) fused_signal(r);
    }
    cudaEvent_t rs_done = nullptr;  // g-dual: block.cpp:668-669
    if (fused_rs_) comm_->log(kSchedule, 1, RF_ * h_);
    else rs_done = scatter_async(kSchedule, ev_rs_);
    wait_on(y2_ready);
    for (int r = 0; r < L_; ++r) {  // FC1 wgrad on the re-gathered Y2 (block.cpp:664)
      Rank& R = R_[r];
      gemm(h, fw_, RF_, gathered(r, R.y2), h, Major::MN, R.dgin, fw_, Major::MN, R.dw1, fw_, Epi::F32,
           nullptr, nullptr, nullptr, 0, -1, kGY2);
    }
    wait_on(rs_done);
    if (fused_rs_)
      for (int r = 0; r < L_; ++r) fused_reduce(r);
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      const T* dy = static_cast<const T*>(dyv[r]);
      launch(K_ELEM, 2, 0, 5.0 * eb * RL_ * h, [&] {
        k::layernorm_bwd<T>(scattered(r), R.r1, R.mu2, R.rs2, R.g2, dy, R.dr1, R.partials,
                            R.partials + (int64_t)nch_l * h, RL_, h, kChunkRows, st_);
      });
      launch(K_ELEM, 2, 0, 0, [&] {
        k::reduce_partials(R.partials, nch_l, h, repl_w(R) + 4 * h, false, st_);
        k::reduce_partials(R.partials + (int64_t)nch_l * h, nch_l, h, repl_w(R) + 5 * h, false, st_);
      });
    }
    // ---- attention branch (block.cpp:683-726)
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      launch(K_ELEM, 2, 0, (2.0 * eb + 1.0) * RL_ * h, [&] {
        k::dropout_bwd_colsum<T>(R.dr1, R.amask, inv_keep, R.d_s, R.partials, RL_, h, kChunkRows, st_);
        k::reduce_partials(R.partials, nch_l, h, repl_w(R) + 0 * h, false, st_);  // bo partial
      });
    }
    if (sp_)
      gather([&](int r) { return (const void*)R_[r].d_s; }, [&](int r) { return (void*)R_[r].dfull; },
             kSchedule);  // block.cpp:691
    // re-gather Y1 (block.cpp:692) on the comm stream, overlapped with proj and attention bwd
    cudaEvent_t y1_ready = gather_async([&](int r) { return (const void*)R_[r].y1_s; },
                                        [&](int r) { return (void*)R_[r].yfull; }, kRegather,
                                        ev_regather_);
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      const T* dao = gathered_d(r, R.d_s);
      gemm(RF_, lw_, h, dao, h, Major::K, R.wo, h, Major::K, R.dproj, lw_, Epi::Store,  // 699
           nullptr, nullptr, nullptr, 0, -1, kGD);
      gemm(lw_, h, RF_, R.api, lw_, Major::MN, dao, h, Major::MN, R.dwo, h, Epi::F32,  // 700
           nullptr, nullptr, nullptr, 0, -1, kNoGath, kGD);
      k::AttnArgs a = attn_args(r);
      join_keep_bits();
      launch(K_ATTN, 3, attn_flops(true), 0,
             [&] { k::attn_bwd<T>(a, R.dproj, R.dqkv, R.delta, st_); });  // 701-702
      launch(K_ELEM, 2, 0, eb * RF_ * 3 * lw_, [&] {
        k::colsum_partial<T>(R.dqkv, RF_, 3 * lw_, 3 * lw_, R.partials, kChunkRows, st_);
        k::reduce_partials(R.partials, nch_f, 3 * lw_, R.dbqkv, grad_acc_, st_);  // 703-705
      });
      // dY1 = dQ·Wqᵀ + dK·Wkᵀ + dV·Wvᵀ as one GEMM over the fused 3h/t weight (709-711)
      gemm(RF_, h, 3 * lw_, R.dqkv, 3 * lw_, Major::K, R.wqkv, 3 * lw_, Major::K, R.part, h,
           Epi::Store, nullptr, nullptr, nullptr, 0, fused_rank(r));
      if (fused_rs_) fused_signal(r);
    }
    rs_done = nullptr;  // block.cpp:714-715, overlaps the QKV wgrad
    if (fused_rs_) comm_->log(kSchedule, 1, RF_ * h_);
    else rs_done = scatter_async(kSchedule, ev_rs_);
    wait_on(y1_ready);
    for (int r = 0; r < L_; ++r) {  // QKV wgrad on the re-gathered Y1 (block.cpp:706-708)
      Rank& R = R_[r];
      gemm(h, 3 * lw_, RF_, gathered(r, R.y1_s), h, Major::MN, R.dqkv, 3 * lw_, Major::MN,
           R.dwqkv, 3 * lw_, Epi::F32, nullptr, nullptr, nullptr, 0, -1, kGY1);
    }
    wait_on(rs_done);
    if (fused_rs_)
      for (int r = 0; r < L_; ++r) fused_reduce(r);
    for (int r = 0; r < L_; ++r) {
      Rank& R = R_[r];
      launch(K_ELEM, 2, 0, 5.0 * eb * RL_ * h, [&] {
        k::layernorm_bwd<T>(scattered(r), R.x_s, R.mu1, R.rs1, R.g1, R.dr1,
                            static_cast<T*>(dxv[r]), R.partials, R.partials + (int64_t)nch_l * h,
                            RL_, h, kChunkRows, st_);
      });
      launch(K_ELEM, 2, 0, 0, [&] {
        k::reduce_partials(R.partials, nch_l, h, repl_w(R) + 2 * h, false, st_);
        k::reduce_partials(R.partials + (int64_t)nch_l * h, nch_l, h, repl_w(R) + 3 * h, false, st_);
      });
    }
    // replicated-parameter gradients: one packed all-reduce (the 6 GradSync ARs, 741-746)
    if (sp_ && t_ > 1) {
      std::vector<float*> bufs(L_);
      for (int r = 0; r < L_; ++r) bufs[r] = repl_w(R_[r]);
      for (int i = 0; i < 6; ++i) comm_->log(kGradSync, 2, h);
      launch(K_COMM, 1, 0, 2.0 * 6 * h * 4 * (t_ - 1) / t_,
             [&] { comm_->all_reduce_f32(bufs.data(), 6 * h, st_); });
    }
    if (grad_acc_)  // replicated-parameter gradients of this microbatch onto the running sum
      for (int r = 0; r < L_; ++r)
        launch(K_ELEM, 1, 0, 12.0 * 6 * h,
               [&] { k::reduce_partials(R_[r].repl_new, 1, 6 * h, R_[r].repl, true, st_); });
  }
  float* repl_w(Rank& R) const { return grad_acc_ ? R.repl_new : R.repl; }

  spl_layer_desc d_;
  int dev_;
  std::unique_ptr<Comm> comm_;
  int t_ = 1, L_ = 1, rank0_ = 0;
  int64_t s_ = 0, b_ = 0, h_ = 0, a_ = 0, hd_ = 0, lh_ = 0, lw_ = 0, fw_ = 0, RF_ = 0, RL_ = 0;
  bool sp_ = true;
  int kind_ = 0;
  float scale_ = 1.f;
  DropKey k_soft_{}, k_attn_{}, k_mlp_{};
  cudaStream_t st_ = nullptr;
  cudaEvent_t ev_in_ = nullptr, ev_out_ = nullptr, ev_fork_ = nullptr, ev_bits_ = nullptr;
  cudaStream_t st_rng_ = nullptr;
  cudaStream_t st_up_ = nullptr, st_down_ = nullptr;  // host-step H2D / D2H copies
  cudaEvent_t ev_x_[2] = {}, ev_dy_[2] = {}, ev_f_[2] = {}, ev_b_[2] = {}, ev_free_[2] = {};
  uint64_t host_steps_ = 0;
  cudaStream_t st_comm_ = nullptr;  // backward collectives overlapped with the GEMMs
  cudaEvent_t ev_cfork_ = nullptr, ev_regather_ = nullptr, ev_rs_ = nullptr;
  cudaStream_t caller_ = 0;  // legacy default stream unless set
  std::vector<Rank> R_;
  std::vector<Alloc> allocs_;
  std::shared_ptr<WorkPool> pool_;  // shared workspace of a stack (nullptr: own buffers)
  size_t work_next_ = 0;
  std::shared_ptr<WorkPool> params_;  // parameters + gradients shared by window slots
  size_t param_next_ = 0;
  bool grad_acc_ = false;
  std::vector<T*> stage_;
  void* pinned_ = nullptr;
  int* nonfinite_ = nullptr;
  bool have_fwd_ = false;
  bool bits_pending_ = false;
  bool bits_serial_ = true;
  bool comm_serial_ = false;  // SPL_SERIAL_COMM=1: backward collectives on the main stream
  bool fused_ag_ = false;     // all-gather fused into the consuming GEMMs
  bool pull_ = false;         // ... reading the peer ranks' shards in their memory
  const void* peer_[4][GemmArgs::kMaxShards] = {};  // [Gath][rank] shard addresses (pull_)
  bool fused_rs_ = false;  // reduce-scatters fused into the row-parallel GEMMs  // SPL_KEEPBITS_SIDE=1: RNG pass on the side stream
  bool graphs_ = false;
  std::vector<Graph> gfwd_, gbwd_;
  // profiling
  struct Pending {
    cudaEvent_t a, b;
    int cls;
  };
  bool profiling_ = false;
  std::vector<cudaEvent_t> evpool_;
  size_t ev_next_ = 0;
  std::vector<Pending> pending_;
  double prof_ms_[K_NCLASS] = {}, prof_flops_[K_NCLASS] = {}, prof_bytes_[K_NCLASS] = {};
  int64_t prof_n_[K_NCLASS] = {};
  int64_t launches_ = 0;
};

}  // namespace

std::unique_ptr<LayerBase> make_layer(const spl_layer_desc& d, int device,
                                      std::unique_ptr<Comm> comm, std::shared_ptr<WorkPool> pool,
                                      std::shared_ptr<WorkPool> params) {
  if (d.dtype == SPL_DTYPE_F32)
    return std::make_unique<Layer<float>>(d, device, std::move(comm), std::move(pool),
                                          std::move(params));
  if (d.dtype == SPL_DTYPE_BF16)
    return std::make_unique<Layer<bf16>>(d, device, std::move(comm), std::move(pool),
                                         std::move(params));
  raise(1, "unknown dtype");
}

// ---------------------------------------------------------------- accountant
// activation_memory.cpp:23-77: per sbh, 4 replicated + 12 tensor-sharded activation
// elements and 2 replicated masks; per a·s²·b, 2 activations + 1 mask (interior). SP divides
// the replicated part by t, selective drops the interior, full keeps A·sbh (not divided by
// t, activation_memory.cpp:59-63). All terms share the denominator t: exact in __int128.
int per_layer_bytes_exact(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                          int sp, int64_t act, int64_t mask, __int128* num, __int128* den) {
  if (a < 1 || h < 1 || s < 1 || b < 1 || t < 1) return 1;
  if (h % a || h % t || s % t) return 1;
  if (act < 1 || mask < 1 || kind < 0 || kind > 2) return 1;
  const __int128 sbh = (__int128)s * b * h;
  if (kind == SPL_RECOMPUTE_FULL) {
    *num = (__int128)act * sbh;
    *den = 1;
    return 0;
  }
  const __int128 rep = ((__int128)4 * act + (__int128)2 * mask) * sbh;
  const __int128 shd = (__int128)12 * act * sbh;
  __int128 n = sp ? rep + shd : rep * t + shd;
  if (kind == SPL_RECOMPUTE_NONE) n += ((__int128)2 * act + mask) * ((__int128)a * s * s * b);
  __int128 d = t, x = n, y = d;
  while (y) {
    __int128 q = x % y;
    x = y;
    y = q;
  }
  *num = n / x;
  *den = d / x;
  return 0;
}

}  // namespace spl
