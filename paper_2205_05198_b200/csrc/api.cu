// extern "C" boundary of libspl (include/spl.h). Maps spl::Error and std exceptions to the
// reference's error classes: std::invalid_argument -> SPL_EINVAL, std::domain_error ->
// SPL_EDOMAIN (block.cpp:518-534, 596-598), plus CUDA / NCCL / state errors.
#include <nccl.h>

#include <cstring>
#include <string>

#include "layer.hpp"
#include "window.hpp"

struct spl_handle {
  std::unique_ptr<spl::LayerBase> layer;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  int device = 0;
};

namespace spl {
thread_local std::string g_last_error;
}

namespace {
template <typename F>
int guard(F&& f) {
  return spl::c_guard(std::forward<F>(f));
}

void check_handle(const spl_handle* h) {
  if (h == nullptr || !h->layer) spl::raise(SPL_EINVAL, "null handle");
}

spl_handle* make_handle(const spl_layer_desc* d, int device, std::unique_ptr<spl::Comm> comm,
                        std::shared_ptr<spl::WorkPool> pool = nullptr,
                        std::shared_ptr<spl::WorkPool> params = nullptr) {
  auto* h = new spl_handle();
  h->device = device;
  try {
    SPL_CUDA(cudaSetDevice(device));
    h->layer = spl::make_layer(*d, device, std::move(comm), std::move(pool), std::move(params));
    SPL_CUDA(cudaEventCreate(&h->t0));
    SPL_CUDA(cudaEventCreate(&h->t1));
  } catch (...) {
    delete h;
    throw;
  }
  return h;
}
}  // namespace

// L layers (layer_index = d.layer_index + l) sharing one workspace pool, plus two ping-pong
// shard buffers per local rank for the activations passed between layers.
struct spl_stack {
  std::vector<spl_handle*> layers;
  std::shared_ptr<spl::WorkPool> pool;
  std::vector<void*> ping[2];
  int64_t ping_bytes = 0;
  int device = 0;
  int local = 0;
};

namespace {
void check_stack(const spl_stack* st) {
  if (st == nullptr || st->layers.empty()) spl::raise(SPL_EINVAL, "null stack");
}
void destroy_stack(spl_stack* st) {
  cudaSetDevice(st->device);
  for (spl_handle* h : st->layers) {
    h->layer.reset();
    if (h->t0) cudaEventDestroy(h->t0);
    if (h->t1) cudaEventDestroy(h->t1);
    delete h;
  }
  st->layers.clear();
  st->pool.reset();
  for (auto& v : st->ping)
    for (void* p : v) cudaFree(p);
  delete st;
}

// ---- accountant helpers (activation_memory.cpp:54-123, rational.hpp:32-49)
__int128 gcd128(__int128 x, __int128 y) {
  if (x < 0) x = -x;
  if (y < 0) y = -y;
  while (y) {
    const __int128 r = x % y;
    x = y;
    y = r;
  }
  return x;
}
void layer_rational(int64_t a, int64_t hh, int64_t s, int64_t b, int64_t t, int kind, int sp,
                    int64_t act, int64_t mask, __int128* n, __int128* d) {
  if (spl::per_layer_bytes_exact(a, hh, s, b, t, kind, sp, act, mask, n, d))
    spl::raise(SPL_EINVAL, "invalid configuration");
}
int64_t fit64(__int128 v) {
  if (v > (__int128)INT64_MAX || v < (__int128)INT64_MIN)
    spl::raise(SPL_EINVAL, "value does not fit in 64-bit integer");
  return (int64_t)v;
}
}  // namespace

extern "C" {

const char* spl_last_error(void) { return spl::g_last_error.c_str(); }

void spl_desc_default(spl_layer_desc* d) {
  std::memset(d, 0, sizeof(*d));
  d->seed = 42;
  d->microbatch = 1;
  d->ln_eps = 1e-5;
  d->recompute = SPL_RECOMPUTE_NONE;
  d->sequence_parallel = 1;
  d->dtype = SPL_DTYPE_BF16;
  d->check_finite = 1;
  d->act_bytes = 2;
  d->mask_bytes = 1;
}

int spl_create_local(const spl_layer_desc* d, int device, int t, spl_handle** out) {
  return guard([&] {
    spl::require(d != nullptr && out != nullptr, "null argument");
    spl::require(t >= 1, "t must be >= 1");
    *out = make_handle(d, device, spl::make_local_comm(t));
  });
}

int spl_create(const spl_layer_desc* d, const int* devices, int t, spl_handle** out) {
  return guard([&] {
    spl::require(d != nullptr && devices != nullptr && out != nullptr, "null argument");
    spl::require(t >= 1, "t must be >= 1");
    for (int r = 1; r < t; ++r)
      spl::require(devices[r] == devices[0],
                   "one handle drives one GPU: use spl_create_nccl, one process per GPU");
    *out = make_handle(d, devices[0], spl::make_local_comm(t));
  });
}

int spl_nccl_unique_id(unsigned char id_out[128]) {
  return guard([&] {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) spl::raise(SPL_ENCCL, "ncclGetUniqueId failed");
    std::memcpy(id_out, id.internal, 128);
  });
}

int spl_create_nccl(const spl_layer_desc* d, int device, int t, int rank,
                    const unsigned char nccl_id[128], spl_handle** out) {
  return guard([&] {
    spl::require(d != nullptr && out != nullptr && nccl_id != nullptr, "null argument");
    SPL_CUDA(cudaSetDevice(device));
    *out = make_handle(d, device, spl::make_nccl_comm(t, rank, nccl_id));
  });
}

struct spl_ipc {
  std::unique_ptr<spl::IpcRank> rank;
  spl_layer_desc desc;
  int device = 0, t = 1;
};

int spl_ipc_open(const spl_layer_desc* d, int device, int t, int rank, spl_ipc** out,
                 unsigned char handle_out[64]) {
  return guard([&] {
    spl::require(d != nullptr && out != nullptr && handle_out != nullptr, "null argument");
    spl::require(t >= 1 && rank >= 0 && rank < t, "IPC rank out of range");
    spl::require(d->seq % t == 0 && d->hidden % t == 0 && d->heads % t == 0,
                 "s, h and the head count must be divisible by t");
    // the largest payload of one collective: a sequence shard (g, ḡ and their duals), the
    // whole activation without SP (f̄ all-reduce), the fp32 replicated-parameter gradients
    const size_t es = d->dtype == SPL_DTYPE_F32 ? 4 : 2;
    const size_t rows = (size_t)(d->seq * d->batch) / (d->sequence_parallel ? (size_t)t : 1);
    const size_t slot = std::max(rows * (size_t)d->hidden * es, (size_t)(6 * d->hidden) * 4);
    auto* o = new spl_ipc();
    try {
      o->rank = spl::ipc_open(device, t, rank, slot);
      o->rank->export_handle(handle_out);
    } catch (...) {
      delete o;
      throw;
    }
    o->desc = *d;
    o->device = device;
    o->t = t;
    *out = o;
  });
}

int spl_create_ipc(const spl_layer_desc* d, spl_ipc* ipc, const unsigned char* handles,
                   spl_handle** out) {
  std::unique_ptr<spl_ipc> own(ipc);  // consumed whatever happens
  return guard([&] {
    spl::require(d != nullptr && own != nullptr && handles != nullptr && out != nullptr,
                 "null argument");
    spl::require(d->seq == own->desc.seq && d->batch == own->desc.batch &&
                     d->hidden == own->desc.hidden && d->dtype == own->desc.dtype &&
                     d->sequence_parallel == own->desc.sequence_parallel,
                 "desc differs from the one the IPC rank was opened with");
    SPL_CUDA(cudaSetDevice(own->device));
    auto comm = spl::ipc_connect(std::move(own->rank), handles);
    *out = make_handle(d, own->device, std::move(comm));
  });
}

int spl_ipc_close(spl_ipc* ipc) {
  delete ipc;
  return SPL_OK;
}

int spl_destroy(spl_handle* h) {
  return guard([&] {
    if (!h) return;
    cudaSetDevice(h->device);
    h->layer.reset();
    if (h->t0) cudaEventDestroy(h->t0);
    if (h->t1) cudaEventDestroy(h->t1);
    delete h;
  });
}

int spl_local_ranks(const spl_handle* h) { return h && h->layer ? h->layer->local_ranks() : 0; }

int spl_set_stream(spl_handle* h, void* stream) {
  return guard([&] {
    check_handle(h);
    h->layer->set_caller_stream(static_cast<cudaStream_t>(stream));
  });
}

int spl_load_params(spl_handle* h, const double* p) {
  return guard([&] {
    check_handle(h);
    spl::require(p != nullptr, "null params");
    h->layer->load_params(p);
  });
}

int spl_init_params(spl_handle* h, uint64_t seed) {
  return guard([&] {
    check_handle(h);
    h->layer->init_params(seed);
  });
}

int spl_forward(spl_handle* h, const void* const* x, void* const* y) {
  return guard([&] {
    check_handle(h);
    spl::require(x != nullptr && y != nullptr, "expected one input shard per rank");
    h->layer->forward(x, y);
  });
}

int spl_backward(spl_handle* h, const void* const* dy, void* const* dx) {
  return guard([&] {
    check_handle(h);
    spl::require(dy != nullptr && dx != nullptr, "expected one gradient shard per rank");
    h->layer->backward(dy, dx);
  });
}

int spl_step_host(spl_handle* h, const void* x, const void* dy, void* y, void* dx) {
  return guard([&] {
    check_handle(h);
    spl::require(x && dy && y && dx, "null host buffer");
    h->layer->step_host(x, dy, y, dx);
  });
}

int spl_step_host_async(spl_handle* h, const void* x, const void* dy, void* y, void* dx) {
  return guard([&] {
    check_handle(h);
    spl::require(x && dy && y && dx, "null host buffer");
    h->layer->step_host_async(x, dy, y, dx);
  });
}

int spl_step_host_wait(spl_handle* h) {
  return guard([&] {
    check_handle(h);
    h->layer->step_host_wait();
  });
}

int spl_get_grads(spl_handle* h, double* out) {
  return guard([&] {
    check_handle(h);
    h->layer->get_grads(out);
  });
}

int spl_get_w1_grad_shard(spl_handle* h, int r, double* out) {
  return guard([&] {
    check_handle(h);
    h->layer->get_w1_grad_shard(r, out);
  });
}

int spl_get_saved(spl_handle* h, int r, const char* name, double* out, int64_t n) {
  return guard([&] {
    check_handle(h);
    spl::require(name != nullptr && out != nullptr, "null argument");
    h->layer->get_saved(r, name, out, n);
  });
}

int spl_attention_interior(spl_handle* h, int r, double* out3) {
  return guard([&] {
    check_handle(h);
    h->layer->attention_interior(r, out3);
  });
}

int spl_ledger(spl_handle* h, int r, spl_ledger_entry* entries, int* n) {
  return guard([&] {
    check_handle(h);
    spl::require(n != nullptr, "null count");
    spl::require(r >= 0 && r < h->layer->local_ranks(), "local rank out of range");
    auto items = h->layer->ledger(r);
    const int cap = *n;
    *n = (int)items.size();
    if (entries == nullptr) return;
    for (int i = 0; i < (int)items.size() && i < cap; ++i) {
      std::memset(entries[i].name, 0, sizeof(entries[i].name));
      std::strncpy(entries[i].name, items[i].name.c_str(), sizeof(entries[i].name) - 1);
      entries[i].elements = items[i].elements;
      entries[i].bytes = items[i].bytes;
      entries[i].physical_bytes = items[i].physical;
    }
  });
}

int spl_saved_bytes(spl_handle* h, int r, int64_t* lb, int64_t* pb, int64_t* ub) {
  return guard([&] {
    check_handle(h);
    spl::require(r >= 0 && r < h->layer->local_ranks(), "local rank out of range");
    h->layer->saved_bytes(r, lb, pb, ub);
  });
}

int spl_comm_log(spl_handle* h, int64_t c[16]) {
  return guard([&] {
    check_handle(h);
    auto& comm = h->layer->comm();
    for (int tag = 0; tag < 4; ++tag) {
      c[tag * 4 + 0] = comm.counters[tag].all_gathers;
      c[tag * 4 + 1] = comm.counters[tag].reduce_scatters;
      c[tag * 4 + 2] = comm.counters[tag].all_reduces;
      c[tag * 4 + 3] = comm.counters[tag].ring_elements;
    }
  });
}

int spl_comm_log_reset(spl_handle* h) {
  return guard([&] {
    check_handle(h);
    auto& comm = h->layer->comm();
    for (auto& c : comm.counters) c = spl::CommCounters{};
  });
}

int spl_per_layer_bytes(int64_t a, int64_t hh, int64_t s, int64_t b, int64_t t, int kind,
                        int sp, int64_t act, int64_t mask, int64_t* out) {
  return guard([&] {
    __int128 n, d;
    if (spl::per_layer_bytes_exact(a, hh, s, b, t, kind, sp, act, mask, &n, &d))
      spl::raise(SPL_EINVAL, "invalid configuration");
    const __int128 q = n / d;
    if (q > (__int128)INT64_MAX) spl::raise(SPL_EINVAL, "value does not fit in 64-bit integer");
    *out = (int64_t)q;
  });
}

int spl_per_layer_bytes_exact(int64_t a, int64_t hh, int64_t s, int64_t b, int64_t t, int kind,
                              int sp, int64_t act, int64_t mask, int64_t* num, int64_t* den) {
  return guard([&] {
    __int128 n, d;
    if (spl::per_layer_bytes_exact(a, hh, s, b, t, kind, sp, act, mask, &n, &d))
      spl::raise(SPL_EINVAL, "invalid configuration");
    if (n > (__int128)INT64_MAX) spl::raise(SPL_EINVAL, "value does not fit in 64-bit integer");
    *num = (int64_t)n;
    *den = (int64_t)d;
  });
}

int spl_layer_component_breakdown(int64_t a, int64_t hh, int64_t s, int64_t b, int64_t act,
                                  int64_t mask, int64_t out[4]) {
  return guard([&] {
    __int128 n, d;
    layer_rational(a, hh, s, b, 1, SPL_RECOMPUTE_NONE, 0, act, mask, &n, &d);  // validation
    const __int128 sbh = (__int128)s * b * hh, interior = (__int128)a * s * s * b;
    const __int128 attn = (__int128)5 * act * sbh + (__int128)mask * sbh + ((__int128)2 * act + mask) * interior;
    const __int128 mlp = (__int128)9 * act * sbh + (__int128)mask * sbh;
    const __int128 lns = (__int128)2 * act * sbh;
    out[0] = fit64(attn);
    out[1] = fit64(mlp);
    out[2] = fit64(lns);
    out[3] = fit64(attn + mlp + lns);
  });
}

int spl_percent_of_baseline(int64_t a, int64_t hh, int64_t s, int64_t b, int64_t t, int kind,
                            int sp, int64_t act, int64_t mask, int64_t* num, int64_t* den) {
  return guard([&] {
    __int128 n1, d1, n0, d0;
    layer_rational(a, hh, s, b, t, kind, sp, act, mask, &n1, &d1);
    layer_rational(a, hh, s, b, t, SPL_RECOMPUTE_NONE, 0, act, mask, &n0, &d0);
    __int128 n = n1 * d0, d = d1 * n0;
    const __int128 g = gcd128(n, d);
    if (g > 1) {
      n /= g;
      d /= g;
    }
    *num = fit64(n);
    *den = fit64(d);
  });
}

int spl_total_first_stage_bytes(int64_t a, int64_t hh, int64_t s, int64_t b, int64_t t,
                                int kind, int sp, int64_t layers, int64_t pipeline,
                                int64_t interleave, int64_t act, int64_t mask, int64_t* out) {
  return guard([&] {
    spl::require(layers >= 1, "L must be >= 1");
    spl::require(pipeline >= 1, "p must be >= 1");
    spl::require(interleave >= 1, "m must be >= 1");
    spl::require(layers % (pipeline * interleave) == 0, "L must be divisible by p*m");
    __int128 n, d;
    layer_rational(a, hh, s, b, t, kind, sp, act, mask, &n, &d);
    n *= layers;
    if (interleave > 1) {  // interleave_factor = 1 + (p-1)/(p*m) (activation_memory.cpp:106-110)
      n *= (__int128)pipeline * interleave + pipeline - 1;
      d *= (__int128)pipeline * interleave;
    }
    *out = fit64(n / d);  // floor once
  });
}

int spl_layer_comm_bytes(int64_t s, int64_t b, int64_t hh, int64_t t, int64_t elem_bytes,
                         int sequence_parallel, int64_t* bytes_out) {
  return guard([&] {
    spl::require(s >= 1 && b >= 1 && hh >= 1 && t >= 1 && elem_bytes >= 1 && bytes_out != nullptr,
                 "shape fields must be >= 1");
    const __int128 tensor = (__int128)s * b * hh * elem_bytes;
    // collectives.cpp:75-87: 4 all-reduces at 2(t-1)/t each, or 4 all-gathers + 4
    // reduce-scatters at (t-1)/t each — the same volume, 8·(N/t)·(t-1)
    const __int128 v = sequence_parallel ? (__int128)8 * (tensor / t) * (t - 1)
                                         : (__int128)4 * 2 * (tensor / t) * (t - 1);
    *bytes_out = fit64(v);
  });
}

}  // extern "C"

namespace {
// L layers on t simulated ranks over one workspace pool (`pool`, created when null); `params`
// (one pool per layer, or empty) shares parameters and gradients with other stacks.
spl_stack* build_stack(const spl_layer_desc* d, int device, int t, int layers,
                       std::shared_ptr<spl::WorkPool> pool,
                       const std::vector<std::shared_ptr<spl::WorkPool>>& params) {
    spl::require(d != nullptr, "null argument");
    spl::require(t >= 1, "t must be >= 1");
    spl::require(layers >= 1, "L must be >= 1");
    SPL_CUDA(cudaSetDevice(device));
    auto* st = new spl_stack();
    st->device = device;
    try {
      st->pool = pool;
      if (!st->pool) {
        st->pool = std::make_shared<spl::WorkPool>();
        st->pool->device = device;
      }
      for (int l = 0; l < layers; ++l) {
        spl_layer_desc dl = *d;
        dl.layer_index = d->layer_index + (uint32_t)l;
        st->layers.push_back(make_handle(&dl, device, spl::make_local_comm(t), st->pool,
                                         params.empty() ? nullptr : params[(size_t)l]));
      }
      st->local = st->layers[0]->layer->local_ranks();
      const int64_t rows = d->sequence_parallel ? d->seq / t : d->seq;
      st->ping_bytes = rows * d->batch * d->hidden * (d->dtype == SPL_DTYPE_F32 ? 4 : 2);
      for (auto& v : st->ping)
        for (int r = 0; r < st->local; ++r) {
          void* p = nullptr;
          SPL_CUDA(cudaMalloc(&p, (size_t)st->ping_bytes));
          v.push_back(p);
        }
    } catch (...) {
      destroy_stack(st);
      throw;
    }
    return st;
}

void stack_forward(spl_stack* st, const void* const* x, void* const* y) {
  spl::require(x != nullptr && y != nullptr, "expected one input shard per rank");
  const int L = (int)st->layers.size();
  std::vector<const void*> in(x, x + st->local);
  std::vector<void*> out(st->local);
  for (int l = 0; l < L; ++l) {
    for (int r = 0; r < st->local; ++r) out[r] = l == L - 1 ? y[r] : st->ping[l & 1][r];
    st->layers[l]->layer->forward(in.data(), out.data());
    for (int r = 0; r < st->local; ++r) in[r] = out[r];
  }
}

void stack_backward(spl_stack* st, const void* const* dy, void* const* dx) {
  spl::require(dy != nullptr && dx != nullptr, "expected one gradient shard per rank");
  const int L = (int)st->layers.size();
  std::vector<const void*> g(dy, dy + st->local);
  std::vector<void*> out(st->local);
  for (int l = L - 1; l >= 0; --l) {
    for (int r = 0; r < st->local; ++r) out[r] = l == 0 ? dx[r] : st->ping[l & 1][r];
    st->layers[l]->layer->backward(g.data(), out.data());
    for (int r = 0; r < st->local; ++r) g[r] = out[r];
  }
}
}  // namespace

// Microbatch window: one pipeline rank's 1F1B program (pipeline_sim.cpp:40-56) over n_mb
// microbatches. Fully stored microbatches run on no-recompute slot stacks, checkpointed ones on
// slot stacks of the inner regime; every slot of layer l shares layer l's parameters and
// gradients (one parameter pool per layer), slots of one regime share one workspace.
struct spl_window {
  std::vector<spl_stack*> slots[2];  // [0] checkpointed, [1] fully stored
  std::vector<std::shared_ptr<spl::WorkPool>> params;
  std::vector<uint8_t> modes;
  std::vector<spl::ProgEvent> prog;
  uint32_t mb_base = 1;
  int device = 0, local = 0;
  int64_t slot_ledger[2] = {0, 0};  // ledger bytes of one slot (rank 0), per mode
  int64_t live_peak = 0;
};

namespace {
void destroy_window(spl_window* w) {
  for (auto& v : w->slots)
    for (spl_stack* st : v) destroy_stack(st);
  w->params.clear();
  delete w;
}
void check_window(const spl_window* w) {
  if (w == nullptr || (w->slots[0].empty() && w->slots[1].empty()))
    spl::raise(SPL_EINVAL, "null window");
}
spl_stack* window_first(spl_window* w) {
  return w->slots[1].empty() ? w->slots[0][0] : w->slots[1][0];
}
}  // namespace

extern "C" {

int spl_stack_create_local(const spl_layer_desc* d, int device, int t, int layers,
                           spl_stack** out) {
  return guard([&] {
    spl::require(out != nullptr, "null argument");
    *out = build_stack(d, device, t, layers, nullptr, {});
  });
}

int spl_stack_destroy(spl_stack* st) {
  return guard([&] {
    if (st) destroy_stack(st);
  });
}

int spl_stack_layers(const spl_stack* st) { return st ? (int)st->layers.size() : 0; }

int spl_stack_layer(spl_stack* st, int l, spl_handle** out) {
  return guard([&] {
    check_stack(st);
    spl::require(l >= 0 && l < (int)st->layers.size() && out != nullptr, "layer index out of range");
    *out = st->layers[l];
  });
}

int spl_stack_set_stream(spl_stack* st, void* stream) {
  return guard([&] {
    check_stack(st);
    for (spl_handle* h : st->layers) h->layer->set_caller_stream(static_cast<cudaStream_t>(stream));
  });
}

int spl_stack_forward(spl_stack* st, const void* const* x, void* const* y) {
  return guard([&] {
    check_stack(st);
    stack_forward(st, x, y);
  });
}

int spl_stack_backward(spl_stack* st, const void* const* dy, void* const* dx) {
  return guard([&] {
    check_stack(st);
    stack_backward(st, dy, dx);
  });
}

int spl_stack_memory(spl_stack* st, int local_rank, int64_t out[7]) {
  return guard([&] {
    check_stack(st);
    spl::require(local_rank >= 0 && local_rank < st->local, "local rank out of range");
    for (int i = 0; i < 7; ++i) out[i] = 0;
    for (spl_handle* h : st->layers) {
      int64_t lb, pb, ub, cat[5];
      h->layer->saved_bytes(local_rank, &lb, &pb, &ub);
      h->layer->alloc_bytes(cat);
      out[0] += lb;
      out[1] += pb;
      out[2] += ub;
      out[4] += cat[spl::kParam];
      out[5] += cat[spl::kGrad];
      out[6] += cat[spl::kWork];
    }
    out[3] = st->pool->bytes() + 2 * st->ping_bytes * st->local;
  });
}

int spl_timer_start(spl_handle* h) {
  return guard([&] {
    check_handle(h);
    SPL_CUDA(cudaEventRecord(h->t0, h->layer->stream()));
  });
}

int spl_timer_stop(spl_handle* h, float* ms) {
  return guard([&] {
    check_handle(h);
    SPL_CUDA(cudaEventRecord(h->t1, h->layer->stream()));
    SPL_CUDA(cudaEventSynchronize(h->t1));
    SPL_CUDA(cudaEventElapsedTime(ms, h->t0, h->t1));
  });
}

int spl_synchronize(spl_handle* h) {
  return guard([&] {
    check_handle(h);
    SPL_CUDA(cudaStreamSynchronize(h->layer->stream()));
  });
}

int spl_profile_enable(spl_handle* h, int on) {
  return guard([&] {
    check_handle(h);
    h->layer->set_profile(on != 0);
  });
}

int spl_profile_read(spl_handle* h, double ms[5], int64_t n[5], double fl[5], double by[5]) {
  return guard([&] {
    check_handle(h);
    h->layer->read_profile(ms, n, fl, by);
  });
}

int spl_launch_count(spl_handle* h, int64_t* count, int reset) {
  return guard([&] {
    check_handle(h);
    *count = h->layer->launch_count(reset != 0);
  });
}

int spl_comm_paths(const spl_handle* h, int out[2]) {
  return guard([&] {
    check_handle(h);
    if (out == nullptr) throw std::invalid_argument("null output");
    h->layer->comm_paths(out);
  });
}

int spl_set_graphs(spl_handle* h, int on) {
  return guard([&] {
    check_handle(h);
    h->layer->set_graphs(on != 0);
  });
}

int spl_gemm_bf16(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int a_mn,
                  const void* B, int64_t ldb, int b_mn, void* C, int64_t ldc, int epi,
                  const float* bias, void* C2, const void* aux, int64_t ldaux, void* stream,
                  int* backend) {
  return guard([&] {
    spl::require(epi >= 0 && epi <= 4, "unknown epilogue");
    spl::k::GemmArgs g;
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.lda = lda; g.amaj = a_mn ? spl::k::Major::MN : spl::k::Major::K;
    g.B = B; g.ldb = ldb; g.bmaj = b_mn ? spl::k::Major::MN : spl::k::Major::K;
    g.C = C; g.ldc = ldc; g.epi = (spl::k::Epi)epi;
    g.bias = bias; g.C2 = C2; g.aux = aux; g.ldaux = ldaux;
    if (backend) *backend = spl::k::gemm_backend<spl::bf16>(g);
    spl::k::gemm<spl::bf16>(g, static_cast<cudaStream_t>(stream));
  });
}

// ---- microbatch-level recompute window (pipeline_sim.cpp:26-56, 192-359)
void spl_model_desc_default(spl_model_desc* m) {
  std::memset(m, 0, sizeof(*m));
  m->tensor = m->pipeline = m->interleave = m->microbatch = m->microbatches = 1;
  m->recompute = SPL_RECOMPUTE_SELECTIVE;
  m->sequence_parallel = 1;
  m->act_bytes = 2;
  m->mask_bytes = 1;
  m->logits_bytes = 4;
}

int spl_microbatch_bytes(const spl_model_desc* m, int64_t stage, int64_t* fully_stored,
                         int64_t* checkpointed) {
  return guard([&] {
    spl::require(m && fully_stored && checkpointed, "null argument");
    const spl::MbBytes b = spl::microbatch_bytes(*m, stage);
    *fully_stored = b.fully_stored;
    *checkpointed = b.checkpointed;
  });
}

int spl_window_plan(const spl_model_desc* m, int64_t budget, uint8_t* modes,
                    int64_t* stage_counts, int64_t* recomputed_num, int64_t* recomputed_den,
                    int64_t* min_feasible_budget) {
  return guard([&] {
    spl::require(m != nullptr, "null model desc");
    const spl::WindowPlanOut plan = spl::window_plan(*m, budget, min_feasible_budget);
    if (modes) std::memcpy(modes, plan.modes.data(), plan.modes.size());
    if (stage_counts)
      std::memcpy(stage_counts, plan.stage_counts.data(), plan.stage_counts.size() * 8);
    if (recomputed_num) *recomputed_num = fit64(plan.rec_num);
    if (recomputed_den) *recomputed_den = fit64(plan.rec_den);
  });
}

int spl_stage_timeline(const spl_model_desc* m, int64_t stage, const uint8_t* modes_row,
                       int dealloc, int64_t* bytes_after, int64_t cap, int64_t* n_events,
                       int64_t* peak) {
  return guard([&] {
    spl::require(m != nullptr, "null model desc");
    std::vector<int64_t> tl;
    const int64_t pk = spl::stage_timeline(*m, stage, modes_row, dealloc != 0, &tl);
    if (n_events) *n_events = (int64_t)tl.size();
    if (peak) *peak = pk;
    if (bytes_after) {
      spl::require(cap >= (int64_t)tl.size(), "bytes_after capacity too small");
      std::memcpy(bytes_after, tl.data(), tl.size() * 8);
    }
  });
}

// ---- microbatch window executor
int spl_window_create_local(const spl_layer_desc* d, int device, int t, int layers, int64_t p,
                            int64_t stage, int64_t n_mb, const uint8_t* modes_row,
                            spl_window** out) {
  return guard([&] {
    spl::require(d != nullptr && modes_row != nullptr && out != nullptr, "null argument");
    spl::require(p >= 1 && stage >= 0 && stage < p, "stage must lie in [0, p)");
    spl::require(n_mb >= p, "n_mb < p (pipeline cannot be filled)");
    spl::require(layers >= 1, "L must be >= 1");
    auto* w = new spl_window();
    w->device = device;
    w->mb_base = d->microbatch;
    w->modes.assign(modes_row, modes_row + n_mb);
    w->prog = spl::rank_program(p, stage, n_mb);
    try {
      // slots per mode = the most microbatches of that mode alive at once in the program
      int live[2] = {0, 0}, need[2] = {0, 0};
      for (const spl::ProgEvent& ev : w->prog) {
        const int m = w->modes[(size_t)ev.microbatch - 1] ? 1 : 0;
        live[m] += ev.forward ? 1 : -1;
        need[m] = std::max(need[m], live[m]);
      }
      spl::require(need[0] == 0 || d->recompute != SPL_RECOMPUTE_NONE,
                   "checkpointed microbatches need a full or selective inner strategy");
      for (int l = 0; l < layers; ++l) {
        w->params.push_back(std::make_shared<spl::WorkPool>());
        w->params.back()->device = device;
      }
      for (int m = 1; m >= 0; --m) {
        spl_layer_desc dm = *d;
        if (m == 1) dm.recompute = SPL_RECOMPUTE_NONE;
        std::shared_ptr<spl::WorkPool> pool;
        for (int i = 0; i < need[m]; ++i) {
          spl_stack* st = build_stack(&dm, device, t, layers, pool, w->params);
          w->slots[m].push_back(st);
          pool = st->pool;
          for (spl_handle* h : st->layers) h->layer->set_graphs(false);
        }
        if (need[m] > 0)
          for (spl_handle* h : w->slots[m][0]->layers) {
            int64_t lb, pb, ub;
            h->layer->saved_bytes(0, &lb, &pb, &ub);
            w->slot_ledger[m] += lb;
          }
      }
      w->local = window_first(w)->local;
    } catch (...) {
      destroy_window(w);
      throw;
    }
    *out = w;
  });
}

int spl_window_destroy(spl_window* w) {
  return guard([&] {
    if (w) destroy_window(w);
  });
}

int spl_window_layer(spl_window* w, int layer, spl_handle** out) {
  return guard([&] {
    check_window(w);
    spl_stack* st = window_first(w);
    spl::require(layer >= 0 && layer < (int)st->layers.size() && out != nullptr,
                 "layer index out of range");
    *out = st->layers[(size_t)layer];
  });
}

int spl_window_set_stream(spl_window* w, void* stream) {
  return guard([&] {
    check_window(w);
    for (auto& v : w->slots)
      for (spl_stack* st : v)
        for (spl_handle* h : st->layers)
          h->layer->set_caller_stream(static_cast<cudaStream_t>(stream));
  });
}

int spl_window_run(spl_window* w, const void* const* x, const void* const* dy, void* const* y,
                   void* const* dx) {
  return guard([&] {
    check_window(w);
    spl::require(x && dy && y && dx, "expected n_mb x local-rank pointer arrays");
    const size_t n_mb = w->modes.size();
    std::vector<int> slot_of(n_mb, -1);
    std::vector<uint8_t> busy[2] = {std::vector<uint8_t>(w->slots[0].size(), 0),
                                    std::vector<uint8_t>(w->slots[1].size(), 0)};
    int64_t live = 0;
    w->live_peak = 0;
    bool first_backward = true;
    for (const spl::ProgEvent& ev : w->prog) {
      const size_t i = (size_t)ev.microbatch - 1;
      const int m = w->modes[i] ? 1 : 0;
      const size_t off = i * (size_t)w->local;
      if (ev.forward) {
        size_t k = 0;
        while (k < busy[m].size() && busy[m][k]) ++k;
        spl::require(k < busy[m].size(), "window: no free activation slot");
        busy[m][k] = 1;
        slot_of[i] = (int)k;
        spl_stack* st = w->slots[m][k];
        for (spl_handle* h : st->layers) h->layer->set_microbatch(w->mb_base + (uint32_t)i);
        stack_forward(st, x + off, y + off);
        live += w->slot_ledger[m];
        w->live_peak = std::max(w->live_peak, live);
      } else {
        spl::require(slot_of[i] >= 0, "window: backward before forward");
        spl_stack* st = w->slots[m][(size_t)slot_of[i]];
        for (spl_handle* h : st->layers) {
          h->layer->set_microbatch(w->mb_base + (uint32_t)i);
          h->layer->set_grad_accumulate(!first_backward);
        }
        stack_backward(st, dy + off, dx + off);
        first_backward = false;
        busy[m][(size_t)slot_of[i]] = 0;
        slot_of[i] = -1;
        live -= w->slot_ledger[m];
      }
    }
  });
}

int spl_window_memory(spl_window* w, int64_t out[6]) {
  return guard([&] {
    check_window(w);
    out[0] = (int64_t)w->slots[1].size();
    out[1] = (int64_t)w->slots[0].size();
    out[2] = out[0] * w->slot_ledger[1] + out[1] * w->slot_ledger[0];
    out[3] = w->live_peak;
    out[4] = 0;
    for (auto& pp : w->params) out[4] += pp->bytes();
    out[5] = 0;
    for (auto& v : w->slots)
      if (!v.empty()) out[5] += v[0]->pool->bytes();
    for (auto& v : w->slots)
      for (spl_stack* st : v) out[5] += 2 * st->ping_bytes * st->local;
  });
}

}  // extern "C"
