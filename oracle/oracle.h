/*
 * oracle.h — CPU fp64 restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This library is the parity checker for the B200 path. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. The product library
 * (libspl.so) never links or calls it.
 *
 * It restates, in plain C, the algorithm of the reference `actplan` seqpar harness:
 *   rng         /root/reference/proj/core/src/seqpar/rng.cpp:22-66
 *   layer       /root/reference/proj/core/src/seqpar/block.cpp:42-749
 *   GEMM/axis   /root/reference/proj/core/src/seqpar/tensor.cpp:57-225
 *   collectives /root/reference/proj/core/src/seqpar/collectives.cpp:21-87
 *   accountant  /root/reference/proj/core/src/activation_memory.cpp:23-104,195-200
 *   validation  /root/reference/proj/core/src/config.cpp:86-133
 *
 * Pinning: the RNG is checked bit-for-bit against the reference rng.cpp compiled from
 * /root/reference (oracle/Makefile -> oracle/_ref, vectors in tests/golden/rng_kat.json);
 * the accountant against the reference tests' known answers; the layer numerics
 * relationally, by the reference's own verify suites (verify.cpp:74-321) — the reference
 * ships no golden layer vectors and block.cpp needs Eigen3, which is absent here.
 *
 * Layouts follow the reference: tensors {s, b, h} row-major, weights [in, out] row-major
 * (y = x·W), parameters packed in LayerParams::named_tensors() order (block.cpp:293-298).
 */
#ifndef SPL_ORACLE_H
#define SPL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.cpp ---- */
uint64_t orc_mix64(uint64_t x);
uint64_t orc_hash_counter(uint64_t key, uint64_t index);
double orc_uniform01(uint64_t key, uint64_t index);
uint64_t orc_mask_key_fold(uint64_t seed, uint32_t layer, uint32_t op, uint32_t microbatch);
void orc_random_uniform(uint64_t key, int64_t n, double lo, double hi, double* out);
/* dropout_mask(key, shape, p) over a flat index range [0, n); 1.0 keep / 0.0 drop */
int orc_dropout_mask(uint64_t folded_key, int64_t n, double p_drop, double* out);

/* ---- BlockConfig (block.hpp:28-42) ---- */
typedef struct {
  int64_t heads, hidden, seq, batch;
  double dropout_p;
  int32_t causal;
  uint64_t seed;
  uint32_t layer_index, microbatch;
  double ln_eps;
} orc_block_cfg;

/* Packed LayerParams: 16 tensors in named_tensors() order. */
enum {
  ORC_WQ, ORC_WK, ORC_WV, ORC_BQ, ORC_BK, ORC_BV, ORC_WO, ORC_BO, ORC_W1, ORC_B1, ORC_W2, ORC_B2,
  ORC_LN1_GAIN, ORC_LN1_BIAS, ORC_LN2_GAIN, ORC_LN2_BIAS, ORC_NPARAM
};
/* offsets[i] / sizes[i] in doubles for hidden h; returns total. */
int64_t orc_param_layout(int64_t h, int64_t offsets[ORC_NPARAM], int64_t sizes[ORC_NPARAM]);
/* LayerParams::random (block.cpp:234-265) */
void orc_params_random(int64_t h, uint64_t seed, double* packed);
/* LayerParams::zeros (block.cpp:267-291): gains 1, everything else 0 */
void orc_params_zeros(int64_t h, double* packed);

/* ---- primitive ops ---- */
void orc_layer_norm(const double* x, int64_t rows, int64_t h, const double* gain,
                    const double* bias, double eps, double* out, double* mean, double* inv_std);
void orc_layer_norm_backward(const double* dy, const double* x, const double* mean,
                             const double* inv_std, int64_t rows, int64_t h, const double* gain,
                             double* dx, double* dgain, double* dbias);
void orc_gelu(const double* x, int64_t n, double* out);
void orc_gelu_backward(const double* dy, const double* x, int64_t n, double* out);
/* C[M,N] = A[M,K]·B[K,N] (+bias) — tensor.cpp:57-79 */
void orc_matmul(const double* a, const double* b, const double* bias, int64_t m, int64_t k,
                int64_t n, double* c);
/* attention_interior (block.cpp:381-417): q,k {s,b,local_heads*hd}; outputs {lh,b,s,s} */
int orc_attention_interior(const orc_block_cfg* cfg, const double* q, const double* k,
                           int64_t head_offset, int64_t local_heads, double* softmax_out,
                           double* dropout_mask, double* dropout_out);

/* ---- comm log (collectives.hpp:28-52) ---- */
typedef struct {
  int64_t all_gathers, reduce_scatters, all_reduces;
  int64_t ring_elements;
} orc_comm_counters;
typedef struct {
  orc_comm_counters schedule, regather, grad_sync;
} orc_comm_log;

/* ---- ledger (block.cpp:195-219) ---- */
#define ORC_LEDGER_ENTRIES 15
typedef struct {
  int64_t elements[ORC_LEDGER_ENTRIES];
  int64_t bytes[ORC_LEDGER_ENTRIES];
} orc_ledger;
const char* orc_ledger_name(int i);
void orc_ledger_layer(const orc_block_cfg* cfg, int64_t seq_local, int64_t local_heads,
                      int64_t act_bytes, int64_t mask_bytes, orc_ledger* out);

/* ---- full layer ----
 * Simulated-rank tensor+sequence-parallel layer forward (+ optional backward), exactly the
 * reference schedule (block.cpp:512-749) with ranks run serially and rank-ordered sums.
 * x, dy, y, dx are full {s,b,h} tensors (the rank shards are contiguous axis-0 chunks).
 * grads: packed full-layout parameter gradients (assembled as block.cpp:730-746).
 * interior (optional, may be NULL): {a,b,s,s} x3 (softmax_out, mask, dropout_out) of all ranks.
 * Returns 0 on success, 1 invalid_argument, 2 domain_error (non-finite). */
int orc_seqpar_layer(const orc_block_cfg* cfg, int64_t t, const double* params, const double* x,
                     const double* dy, double* y, double* dx, double* grads,
                     double* w1_grad_shards, double* interior, orc_comm_log* fwd_log,
                     orc_comm_log* bwd_log, orc_ledger* rank_ledger);
/* Single-rank reference_block_forward/backward (block.cpp:419-510). dy/dx/grads may be NULL. */
int orc_reference_layer(const orc_block_cfg* cfg, const double* params, const double* x,
                        const double* dy, double* y, double* dx, double* grads,
                        double* q_out, double* k_out, double* interior, orc_ledger* ledger);
const char* orc_last_error(void);

/* Thread count used by the GEMMs (OpenMP); <=0 means all. Returns the count in effect. */
int orc_set_threads(int n);

/* ---- activation-memory accountant (activation_memory.cpp:23-104, 195-200) ----
 * kind: 0 none, 1 full, 2 selective. Returns 0 ok, 1 invalid (validate_or_throw). */
int orc_per_layer_bytes(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                        int sequence_parallel, int64_t act, int64_t mask, int64_t* bytes_out);
/* exact rational value as reduced num/den (int128 internally, must fit int64). */
int orc_per_layer_bytes_exact(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                              int sequence_parallel, int64_t act, int64_t mask, int64_t* num,
                              int64_t* den);
int orc_layer_component_breakdown(int64_t a, int64_t h, int64_t s, int64_t b, int64_t act,
                                  int64_t mask, int64_t out[4]);
int orc_percent_of_baseline(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                            int sequence_parallel, int64_t act, int64_t mask, int64_t* num,
                            int64_t* den);
int orc_total_first_stage_bytes(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                                int sequence_parallel, int64_t layers, int64_t pipeline,
                                int64_t interleave, int64_t act, int64_t mask,
                                int64_t* bytes_out);
/* layer_comm_bytes_tensor_parallel / _sequence (collectives.cpp:75-87) */
int64_t orc_layer_comm_bytes_tp(int64_t s, int64_t b, int64_t h, int64_t t, int64_t elem);
int64_t orc_layer_comm_bytes_sp(int64_t s, int64_t b, int64_t h, int64_t t, int64_t elem);

#ifdef __cplusplus
}
#endif
#endif
