/*
 * spl.h — C ABI of the B200 sequence-parallel transformer layer (libspl.so).
 *
 * Drop-in for the hot path of the reference `actplan` library (arXiv 2205.05198):
 * one pre-LN GPT layer, forward + backward, under Megatron tensor + sequence parallelism
 * with none / selective / full activation recomputation, plus the activation-memory
 * accountant. Every entry point below names the reference interface it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types.
 *  - Every function returns an int status: SPL_OK, or a code mapped 1:1 from the
 *    reference's exceptions (std::invalid_argument -> SPL_EINVAL, std::domain_error ->
 *    SPL_EDOMAIN) plus CUDA / NCCL failures. spl_last_error() gives the message
 *    (thread-local).
 *  - Tensors follow the reference layouts: activations {s, b, h} row-major, sequence
 *    shards are contiguous axis-0 chunks {s/t, b, h}; weights [in, out] row-major (y = x·W);
 *    parameters packed in LayerParams::named_tensors() order (block.cpp:293-298).
 *  - A handle owns t "local ranks": t simulated ranks on one device (spl_create_local —
 *    the reference's simulated-rank harness, collectives as device copies/ordered sums)
 *    or exactly one rank of a t-way NCCL group, one process per GPU (spl_create_nccl).
 *    Array arguments indexed by local rank have spl_local_ranks() entries.
 *  - A handle is not re-entrant; distinct handles may be used from distinct threads.
 */
#ifndef SPL_H
#define SPL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SPL_OK = 0,
  SPL_EINVAL = 1,  /* std::invalid_argument (block.cpp:518-534, 626-635; collectives.cpp:21-28) */
  SPL_EDOMAIN = 2, /* std::domain_error: non-finite layer output (block.cpp:454-456, 596-598)  */
  SPL_ECUDA = 3,
  SPL_ENCCL = 4,
  SPL_ESTATE = 5,  /* backward without a matching forward ("missing saved forward state")     */
  SPL_EBUDGET = 6  /* pipeline::InfeasibleBudgetError (pipeline_sim.hpp:98-103)                */
};

/* RecomputeKind order of config.hpp:51 (None, Full, Selective). */
enum { SPL_RECOMPUTE_NONE = 0, SPL_RECOMPUTE_FULL = 1, SPL_RECOMPUTE_SELECTIVE = 2 };
enum { SPL_DTYPE_F32 = 0, SPL_DTYPE_BF16 = 1,
       SPL_DTYPE_F64 = 2 /* collectives only (the reference's own fp64 tensors) */ };

/* BlockConfig (block.hpp:28-42) + RecomputeStrategy (config.hpp:53-70) + ByteConvention
 * (config.hpp:74-80) + execution dtype. */
typedef struct spl_layer_desc {
  int64_t heads, hidden, seq, batch;
  double dropout_p;
  int32_t causal;
  uint64_t seed;
  uint32_t layer_index, microbatch;
  double ln_eps;
  int32_t recompute;         /* SPL_RECOMPUTE_* */
  int32_t sequence_parallel; /* 1: g/ḡ = all-gather/reduce-scatter; 0: f/f̄ = all-reduce */
  int32_t dtype;             /* SPL_DTYPE_*: storage/GEMM type; accumulation always fp32 */
  int32_t check_finite;      /* 1: forward fails with SPL_EDOMAIN on non-finite y (reference) */
  int64_t act_bytes, mask_bytes; /* ByteConvention for the ledger/accountant (2, 1 default) */
} spl_layer_desc;

typedef struct spl_handle spl_handle;

/* Fill a desc with the reference defaults (BlockConfig{} + ByteConvention{}). */
void spl_desc_default(spl_layer_desc* d);

/* t simulated ranks on one CUDA device (the reference's in-process harness,
 * seqpar_block_forward(x_shards, params, t, cfg), block.cpp:512). */
int spl_create_local(const spl_layer_desc* d, int device, int t, spl_handle** out);
/* The SURVEY §8(b) form: t ranks on devices[0..t-1]. A handle drives one device, so every
 * entry must name the same GPU (the t ranks are then simulated on it, = spl_create_local);
 * a t-GPU group is one process per GPU with spl_create_nccl. */
int spl_create(const spl_layer_desc* d, const int* devices, int t, spl_handle** out);
/* One rank of a t-way tensor-parallel group over NCCL (one process per GPU). `nccl_id` is the
 * 128-byte ncclUniqueId from spl_nccl_unique_id() on rank 0, distributed by the caller. */
int spl_nccl_unique_id(unsigned char id_out[128]);
int spl_create_nccl(const spl_layer_desc* d, int device, int t, int rank,
                    const unsigned char nccl_id[128], spl_handle** out);
/* One rank of a t-way group whose collectives run over CUDA-IPC-mapped peer memory instead of
 * NCCL (P2P loads/stores over NVLink between GPUs; the same path lets several processes share
 * one GPU). Two phases: spl_ipc_open allocates this rank's exported exchange region and returns
 * its 64-byte IPC handle; the caller all-gathers the t handles (rank order, any host transport)
 * and passes them to spl_create_ipc, which maps the peers and consumes the spl_ipc (also on
 * failure; spl_ipc_close frees one that is never used). Collectives are sequenced by a device
 * barrier of system-scope release/acquire flags; a peer that does not arrive within 20 s traps
 * the kernel (the call fails, the GPU does not hang). Results are bit-identical to
 * spl_create_local with the same t (rank-ordered fp32 sums). */
typedef struct spl_ipc spl_ipc;
int spl_ipc_open(const spl_layer_desc* d, int device, int t, int rank, spl_ipc** out,
                 unsigned char handle_out[64]);
int spl_create_ipc(const spl_layer_desc* d, spl_ipc* ipc, const unsigned char* handles,
                   spl_handle** out);
int spl_ipc_close(spl_ipc* ipc);
int spl_destroy(spl_handle* h);
int spl_local_ranks(const spl_handle* h);
const char* spl_last_error(void);

/* Stream ordering: every call is asynchronous on an internal stream that first waits for
 * all work previously issued on the caller stream and that the caller stream then waits on
 * (event fork/join), so caller-stream producers/consumers of x, y, dy, dx need no extra
 * synchronisation. Default caller stream: the legacy default stream (0). */
int spl_set_stream(spl_handle* h, void* cuda_stream);

/* Parameters. Replaces passing `const LayerParams&` (block.hpp:47-59) to every call:
 * the full-layout fp64 params are sliced per rank (shard_params, block.cpp:122-135) and
 * cast once. packed_f64 holds 12h²+13h doubles in named_tensors() order. */
int spl_load_params(spl_handle* h, const double* packed_f64);
/* LayerParams::random(cfg, seed) generated on the device, bit-identical to the host
 * values before the cast (block.cpp:234-265, rng.cpp:59-66); each rank makes only its shard. */
int spl_init_params(spl_handle* h, uint64_t seed);

/* Forward: seqpar_block_forward (block.cpp:512-602). x[r], y[r] are DEVICE pointers of the
 * desc dtype, one per local rank: {s/t, b, h} with SP, {s, b, h} (replicated) without. */
int spl_forward(spl_handle* h, const void* const* x, void* const* y);
/* Backward: seqpar_block_backward (block.cpp:622-749). Consumes the state of the last
 * forward. dy[r], dx[r] as above. Parameter gradients stay on the device (fp32). */
int spl_backward(spl_handle* h, const void* const* dy, void* const* dx);
/* One training step through HOST buffers (the end-to-end path): H2D of x and dy, forward,
 * backward, D2H of y and dx. Buffers are the local ranks' shards concatenated in rank
 * order, in the desc dtype; pinned host memory is used directly, pageable is staged. */
int spl_step_host(spl_handle* h, const void* x_host, const void* dy_host, void* y_host,
                  void* dx_host);
/* The same step issued asynchronously (a training loop's overlapped data path): uploads run
 * on an upload stream, downloads on a download stream, and the device staging is double
 * buffered, so step k+1's H2D and step k's D2H overlap the compute. The host buffers of a step
 * must stay valid and untouched until spl_step_host_wait() returns (it waits for every step
 * issued so far); use pinned memory for the copies to be asynchronous. */
int spl_step_host_async(spl_handle* h, const void* x_host, const void* dy_host, void* y_host,
                        void* dx_host);
int spl_step_host_wait(spl_handle* h);

/* Gradients assembled into the full fp64 layout (block.cpp:730-746). For an NCCL rank, only
 * the rank's own shard of column/row-sharded tensors is filled (others left zero) and the
 * replicated tensors hold the all-reduced values. */
int spl_get_grads(spl_handle* h, double* packed_f64_out);
/* One rank's w1 gradient shard [h, 4h/t] (SeqparBackward::w1_grad_shards, block.hpp:169). */
int spl_get_w1_grad_shard(spl_handle* h, int local_rank, double* out);

/* Host read of one saved activation (by ledger name) of a local rank, converted to fp64
 * (masks as 0/1); for tests of the stored state and the recompute property. */
int spl_get_saved(spl_handle* h, int local_rank, const char* name, double* out, int64_t n);
/* Attention interior recomputed from the saved Q/K by the device kernel, full fp64
 * {local_heads, b, s, s} x3 (softmax_out, dropout_mask, dropout_out): the
 * attention_interior() call of the reference's recompute property (verify.cpp:253-283). */
int spl_attention_interior(spl_handle* h, int local_rank, double* out3);

/* ActivationLedger (block.hpp:61-73): one entry per saved tensor of the last forward.
 * bytes = elements × the desc ByteConvention width (the reference's counting);
 * physical_bytes = what the device actually holds for it. */
typedef struct {
  char name[32];
  int64_t elements;
  int64_t bytes;
  int64_t physical_bytes;
} spl_ledger_entry;
int spl_ledger(spl_handle* h, int local_rank, spl_ledger_entry* entries, int* n_inout);
/* Totals per local rank: reference-convention ledger bytes, physical saved bytes, and the
 * saved bytes the reference does not count (LN statistics, softmax LSE). */
int spl_saved_bytes(spl_handle* h, int local_rank, int64_t* ledger_bytes,
                    int64_t* physical_bytes, int64_t* uncounted_bytes);

/* CommLog (collectives.hpp:28-52): counts and modelled ring elements per tag.
 * tag 0 Schedule (g/ḡ), 1 Regather (Y_i^s re-gathers), 2 GradSync, 3 Recompute (the forward
 * re-run of full recomputation). counters[tag*4 + {0 AG, 1 RS, 2 AR, 3 ring_elements}]. */
int spl_comm_log(spl_handle* h, int64_t counters[16]);
int spl_comm_log_reset(spl_handle* h);

/* ---- Free-standing reference functions on device buffers (no handle).
 *
 * attention_interior(q, k, cfg, head_offset, local_heads) (block.hpp:100-101,
 * block.cpp:381-417): q, k {s, b, local_heads·hd} in the desc dtype (f32 or bf16; the desc's
 * recompute / SP fields are ignored); outputs {local_heads, b, s, s}: softmax_out and
 * dropout_out in the desc dtype, dropout_mask as u8 0/1, the mask sliced from the global
 * {a, b, s, s} mask at head_offset (mask_slice, block.cpp:42-68). Requires heads % local_heads
 * == 0 and head_offset a multiple of local_heads (SPL_EINVAL otherwise). Asynchronous on
 * `cuda_stream` (NULL: legacy default stream). */
int spl_attention_interior_qk(const spl_layer_desc* d, int device, const void* q, const void* k,
                              int64_t head_offset, int64_t local_heads, void* softmax_out,
                              uint8_t* dropout_mask, void* dropout_out, void* cuda_stream);
/* all_gather / reduce_scatter / all_reduce(span<const Tensor>, axis, CommLog*, CommTag)
 * (collectives.hpp:57-62, collectives.cpp:21-73) over t simulated rank buffers on the current
 * device: `shards[r]` / `partials[r]` are device pointers of one common `shape` (ndim dims),
 * dtype SPL_DTYPE_F64 / F32 / BF16. Reductions sum in rank order 0..t-1 (fp64: bit-identical to
 * the reference's ordered_sum; bf16: fp32 accumulation, one rounding). all_gather writes the
 * concatenation along `axis`; reduce_scatter writes piece r of the sum along `axis` to out[r]
 * (SPL_EINVAL "split axis not divisible by part count" when shape[axis] % t != 0).
 * `log` (optional, 12 int64 = CommLog schedule/regather/grad_sync × {AG, RS, AR,
 * ring_elements}) is incremented under `tag` (0/1/2) with the ring model of
 * collectives.cpp:30-38. t <= 64. Asynchronous on `cuda_stream`. */
int spl_all_gather(const void* const* shards, int t, const int64_t* shape, int ndim, int axis,
                   int dtype, void* out, int64_t log[12], int tag, void* cuda_stream);
int spl_reduce_scatter(const void* const* partials, int t, const int64_t* shape, int ndim,
                       int axis, int dtype, void* const* out, int64_t log[12], int tag,
                       void* cuda_stream);
int spl_all_reduce(const void* const* partials, int t, const int64_t* shape, int ndim, int dtype,
                   void* out, int64_t log[12], int tag, void* cuda_stream);

/* Activation-memory accountant: per_layer_bytes / _exact (activation_memory.cpp:54-82),
 * kind = SPL_RECOMPUTE_*. Floor-once exact arithmetic. */
int spl_per_layer_bytes(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                        int sequence_parallel, int64_t act_bytes, int64_t mask_bytes,
                        int64_t* bytes_out);
int spl_per_layer_bytes_exact(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                              int sequence_parallel, int64_t act_bytes, int64_t mask_bytes,
                              int64_t* num, int64_t* den);

/* layer_component_breakdown (activation_memory.cpp:84-104): serial-layer bytes of the
 * attention block, the MLP block and the two layer norms, and their total: out[4]. */
int spl_layer_component_breakdown(int64_t a, int64_t h, int64_t s, int64_t b, int64_t act_bytes,
                                  int64_t mask_bytes, int64_t out[4]);
/* percent_of_baseline (activation_memory.cpp:195-200): per-layer bytes of the regime over the
 * tensor-parallel no-recompute baseline, as an exact fraction num/den. */
int spl_percent_of_baseline(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                            int sequence_parallel, int64_t act_bytes, int64_t mask_bytes,
                            int64_t* num, int64_t* den);
/* total_first_stage_bytes (activation_memory.cpp:112-123): per-layer bytes x L x
 * interleave_factor (1 + (p-1)/(p*m) for m > 1), floored once. L % (p*m) == 0. */
int spl_total_first_stage_bytes(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                                int sequence_parallel, int64_t layers, int64_t pipeline,
                                int64_t interleave, int64_t act_bytes, int64_t mask_bytes,
                                int64_t* bytes_out);

/* Per-layer, per-rank communication volume of the tensor-parallel (4 all-reduces) or the
 * tensor+sequence-parallel schedule (4 all-gathers + 4 reduce-scatters): the reference's
 * layer_comm_bytes_tensor_parallel / _tensor_sequence (collectives.cpp:75-87). */
int spl_layer_comm_bytes(int64_t s, int64_t b, int64_t h, int64_t t, int64_t elem_bytes,
                         int sequence_parallel, int64_t* bytes_out);

/* Layer stack: L layers of one desc (layer l uses layer_index = d->layer_index + l, so every
 * layer draws its own dropout masks) on t simulated ranks, sharing ONE transient workspace;
 * each layer keeps only its own saved activations. The p = 1 stage that
 * total_first_stage_bytes and simulate_memory (pipeline_sim.cpp:222-275) account for.
 * spl_stack_forward runs layers 0..L-1 (x -> y), spl_stack_backward L-1..0 (dy -> dx); the
 * inter-layer activations live in two stack-owned ping-pong buffers. Per-layer parameters,
 * gradients, ledgers and profiles go through the borrowed handle of spl_stack_layer (do not
 * spl_destroy it). */
typedef struct spl_stack spl_stack;
int spl_stack_create_local(const spl_layer_desc* d, int device, int t, int layers,
                           spl_stack** out);
int spl_stack_destroy(spl_stack* st);
int spl_stack_layers(const spl_stack* st);
int spl_stack_layer(spl_stack* st, int layer, spl_handle** out);
int spl_stack_set_stream(spl_stack* st, void* cuda_stream);
int spl_stack_forward(spl_stack* st, const void* const* x, void* const* y);
int spl_stack_backward(spl_stack* st, const void* const* dy, void* const* dx);
/* Device bytes of one local rank summed over the layers: out[0] ledger (reference
 * convention), [1] physical saved activations, [2] saved but uncounted (LN stats / LSE),
 * [3] shared workspace (pool + ping-pong), [4] parameters, [5] gradients, [6] per-layer
 * workspace outside the pool (0 for a stack). */
int spl_stack_memory(spl_stack* st, int local_rank, int64_t out[7]);

/* Device timing on the handle's compute stream (CUDA events; synchronizes at stop). */
int spl_timer_start(spl_handle* h);
int spl_timer_stop(spl_handle* h, float* ms);
int spl_synchronize(spl_handle* h);
/* Per-kernel-class device time: when enabled, every launch is bracketed by CUDA events on
 * its own stream. Classes: 0 gemm, 1 attention, 2 layernorm/elementwise, 3 collective,
 * 4 other. ms[c], launches[c], flops[c] (algorithmic FLOPs), bytes[c] (algorithmic bytes). */
int spl_profile_enable(spl_handle* h, int on);
int spl_profile_read(spl_handle* h, double ms[5], int64_t launches[5], double flops[5],
                     double bytes[5]);
/* Number of kernel launches of this library recorded since the last reset. */
int spl_launch_count(spl_handle* h, int64_t* count, int reset);
/* Which collective paths the handle runs: out[0] = 1 when the reduce-scatters
 * are fused into the row-parallel GEMMs (peer landing slots); out[1] = 1 when the all-gathers
 * are fused into the consuming GEMMs reading the simulated ranks' shards, 2 when those GEMMs
 * pull the shards from the peer ranks' memory (CUDA IPC / NVLink), 0 when gathered copies
 * are materialised. */
int spl_comm_paths(const spl_handle* h, int out[2]);

/* Kernel-level entry (tests / microbenchmarks): C[M,N] = A[M,K]·B[K,N] in bf16 with fp32
 * accumulation on the layer's GEMM kernels. A(m,k) = A[m*lda+k] (a_mn=0) or A[k*lda+m]
 * (a_mn=1); B(k,n) = B[n*ldb+k] (b_mn=0) or B[k*ldb+n] (b_mn=1). epi: 0 store, 1 +bias,
 * 2 +bias and GELU (second output C2), 3 ×GELU'(aux), 4 fp32 output. Device pointers;
 * asynchronous on `stream`. Returns the backend used in *backend (1 = tcgen05). */
int spl_gemm_bf16(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int a_mn,
                  const void* B, int64_t ldb, int b_mn, void* C, int64_t ldc, int epi,
                  const float* bias, void* C2, const void* aux, int64_t ldaux, void* stream,
                  int* backend);

/* Capture forward+backward into CUDA graphs after the first call (1) or run eagerly (0). */
int spl_set_graphs(spl_handle* h, int on);

/* ---- Microbatch-level recompute window (pipeline_sim.cpp:26-56,
 * 192-359). ModelShape (config.hpp:27-35) + ParallelLayout (config.hpp:39-48, without d) +
 * the inner RecomputeStrategy + ByteConvention (config.hpp:74-80, logits 4 by default). */
typedef struct spl_model_desc {
  int64_t heads, hidden, layers, seq, vocab;
  int64_t tensor, pipeline, interleave, microbatch, microbatches; /* t, p, m, b, n_mb */
  int32_t recompute, sequence_parallel;                           /* inner strategy */
  int64_t act_bytes, mask_bytes, logits_bytes;
} spl_model_desc;
/* t = p = m = b = n_mb = 1, selective, SP on, bytes {2, 1, 4}; shape fields zero. */
void spl_model_desc_default(spl_model_desc* m);
/* microbatch_bytes (pipeline_sim.cpp:192-220): activation bytes one microbatch pins on
 * pipeline rank `stage` when fully stored / checkpointed under the inner strategy. */
int spl_microbatch_bytes(const spl_model_desc* m, int64_t stage, int64_t* fully_stored,
                         int64_t* checkpointed);
/* microbatch_window_plan (pipeline_sim.cpp:297-359): modes[p*n_mb] (row = rank, 1 = fully
 * stored), stage_counts[2p] (fully stored, checkpointed per rank), the recomputed fraction
 * num/den and the minimum feasible budget. The inner strategy must be full or selective
 * (SPL_EINVAL); a budget below the all-checkpointed peak returns SPL_EBUDGET with
 * *min_feasible_budget set (InfeasibleBudgetError::min_feasible_budget). */
int spl_window_plan(const spl_model_desc* m, int64_t budget, uint8_t* modes,
                    int64_t* stage_counts, int64_t* recomputed_num, int64_t* recomputed_den,
                    int64_t* min_feasible_budget);
/* simulate_memory_with_modes (pipeline_sim.cpp:222-275) for one rank: bytes held after each
 * event of the rank's program (2·n_mb events, plus one recompute event before every
 * checkpointed backward when the strategy recomputes) into bytes_after (capacity `cap`,
 * *n_events set) and the peak. modes_row: n_mb entries, 1 = fully stored. */
int spl_stage_timeline(const spl_model_desc* m, int64_t stage, const uint8_t* modes_row,
                       int dealloc, int64_t* bytes_after, int64_t cap, int64_t* n_events,
                       int64_t* peak);

/* Window executor: rank `stage` of a p-stage pipeline running its 1F1B program
 * (pipeline_sim.cpp:40-56) over n_mb microbatches on one device with `layers` layers and t
 * simulated ranks. modes_row[n_mb] (1 = fully stored, e.g. a row of spl_window_plan) picks per
 * microbatch a no-recompute stack or one of the inner regime d->recompute; the slot count per
 * mode is the most microbatches of that mode alive at once. All slots of a layer share its
 * parameters and gradients; spl_window_run accumulates the gradients over the microbatches
 * (running fp32 sum in microbatch-backward order). Microbatch i (1-based) draws the dropout
 * masks of MaskKey microbatch d->microbatch + i - 1. Runs eagerly (no CUDA graphs). */
typedef struct spl_window spl_window;
int spl_window_create_local(const spl_layer_desc* d, int device, int t, int layers, int64_t p,
                            int64_t stage, int64_t n_mb, const uint8_t* modes_row,
                            spl_window** out);
int spl_window_destroy(spl_window* w);
/* Borrowed handle of layer l (parameters, gradients; do not spl_destroy it). */
int spl_window_layer(spl_window* w, int layer, spl_handle** out);
int spl_window_set_stream(spl_window* w, void* cuda_stream);
/* x, dy, y, dx: n_mb x local-rank device pointers, microbatch-major. */
int spl_window_run(spl_window* w, const void* const* x, const void* const* dy, void* const* y,
                   void* const* dx);
/* out[0] fully-stored slots, [1] checkpointed slots, [2] saved-activation ledger bytes held by
 * all slots (rank 0), [3] peak ledger bytes of live microbatches during the last run, [4]
 * parameter + gradient bytes, [5] workspace bytes. */
int spl_window_memory(spl_window* w, int64_t out[6]);

#ifdef __cplusplus
}
#endif
#endif
