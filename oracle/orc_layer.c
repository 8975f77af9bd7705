/* Transformer-layer restatement in fp64 (TEST INFRASTRUCTURE — see oracle.h).
 *
 * Follows /root/reference/proj/core/src/seqpar/block.cpp op-for-op:
 *   mask ids / mask_slice       block.cpp:34-68   (masks at GLOBAL coordinates, rank-sliced)
 *   apply_dropout / backward    block.cpp:70-79
 *   rowwise softmax             block.cpp:97-107
 *   shard_params                block.cpp:122-135 (expressed as strided views, no copies)
 *   attention_over_values       block.cpp:138-153
 *   attention_interior_backward block.cpp:159-193
 *   ledger_add_layer            block.cpp:195-219
 *   LayerParams::random/zeros   block.cpp:234-291
 *   layer_norm (+backward)      block.cpp:300-360
 *   gelu (+backward)            block.cpp:362-379
 *   attention_interior          block.cpp:381-417
 *   reference_block_forward/backward block.cpp:419-510
 *   seqpar_block_forward/backward    block.cpp:512-749
 * and the simulated collectives of collectives.cpp:21-73 (rank-ordered sums 0..t-1, ring
 * element accounting (n/t)(t-1) per AG/RS, twice per AR). */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "orc_internal.h"

enum { kSoftmaxDrop = 0, kAttnOutDrop = 1, kMlpDrop = 2 };

static char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

static double* dalloc(int64_t n) { return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

/* ------------------------------------------------------------------ params */
int64_t orc_param_layout(int64_t h, int64_t off[ORC_NPARAM], int64_t sz[ORC_NPARAM]) {
  const int64_t s[ORC_NPARAM] = {h * h, h * h, h * h, h, h, h, h * h, h, h * 4 * h, 4 * h,
                                 4 * h * h, h, h, h, h, h};
  int64_t acc = 0;
  for (int i = 0; i < ORC_NPARAM; ++i) {
    if (off) off[i] = acc;
    if (sz) sz[i] = s[i];
    acc += s[i];
  }
  return acc;
}

void orc_params_random(int64_t h, uint64_t seed, double* p) {
  int64_t off[ORC_NPARAM], sz[ORC_NPARAM];
  orc_param_layout(h, off, sz);
  const double w_scale = 1.0 / sqrt((double)h);
  /* salts 1..16 in named order; weights U(±1/sqrt(h)), the rest U(±0.1) (block.cpp:244-259) */
  static const int is_weight[ORC_NPARAM] = {1, 1, 1, 0, 0, 0, 1, 0, 1, 0, 1, 0, 0, 0, 0, 0};
  for (int i = 0; i < ORC_NPARAM; ++i) {
    const uint64_t key = orc_hash_counter(seed, (uint64_t)(i + 1));
    if (is_weight[i])
      orc_random_uniform(key, sz[i], -w_scale, w_scale, p + off[i]);
    else
      orc_random_uniform(key, sz[i], -0.1, 0.1, p + off[i]);
  }
  for (int64_t i = 0; i < h; ++i) {
    p[off[ORC_LN1_GAIN] + i] += 1.0;
    p[off[ORC_LN2_GAIN] + i] += 1.0;
  }
}

void orc_params_zeros(int64_t h, double* p) {
  int64_t off[ORC_NPARAM];
  const int64_t total = orc_param_layout(h, off, NULL);
  memset(p, 0, sizeof(double) * (size_t)total);
  for (int64_t i = 0; i < h; ++i) {
    p[off[ORC_LN1_GAIN] + i] = 1.0;
    p[off[ORC_LN2_GAIN] + i] = 1.0;
  }
}

/* ------------------------------------------------------------------ primitives */
void orc_layer_norm(const double* x, int64_t rows, int64_t h, const double* gain,
                    const double* bias, double eps, double* out, double* mean, double* inv_std) {
  for (int64_t r = 0; r < rows; ++r) {
    const double* row = x + r * h;
    double mu = 0.0;
    for (int64_t c = 0; c < h; ++c) mu += row[c];
    mu /= (double)h;
    double var = 0.0;
    for (int64_t c = 0; c < h; ++c) var += (row[c] - mu) * (row[c] - mu);
    var /= (double)h;
    const double is = 1.0 / sqrt(var + eps);
    if (mean) mean[r] = mu;
    if (inv_std) inv_std[r] = is;
    double* o = out + r * h;
    for (int64_t c = 0; c < h; ++c) o[c] = (row[c] - mu) * is * gain[c] + bias[c];
  }
}

void orc_layer_norm_backward(const double* dy, const double* x, const double* mean,
                             const double* inv_std, int64_t rows, int64_t h, const double* gain,
                             double* dx, double* dgain, double* dbias) {
  const double inv_h = 1.0 / (double)h;
  for (int64_t r = 0; r < rows; ++r) {
    const double* xr = x + r * h;
    const double* dyr = dy + r * h;
    double* dxr = dx + r * h;
    const double mu = mean[r], is = inv_std[r];
    double sum_dxhat = 0.0, sum_dxhat_xhat = 0.0;
    for (int64_t c = 0; c < h; ++c) {
      const double xhat = (xr[c] - mu) * is;
      const double dxhat = dyr[c] * gain[c];
      sum_dxhat += dxhat;
      sum_dxhat_xhat += dxhat * xhat;
      if (dgain) dgain[c] += dyr[c] * xhat;
      if (dbias) dbias[c] += dyr[c];
    }
    for (int64_t c = 0; c < h; ++c) {
      const double xhat = (xr[c] - mu) * is;
      const double dxhat = dyr[c] * gain[c];
      dxr[c] = is * (dxhat - inv_h * sum_dxhat - xhat * inv_h * sum_dxhat_xhat);
    }
  }
}

void orc_gelu(const double* x, int64_t n, double* out) {
  const double rs2 = 1.4142135623730951 / 2.0; /* std::numbers::sqrt2 / 2.0 */
  for (int64_t i = 0; i < n; ++i) out[i] = 0.5 * x[i] * (1.0 + erf(x[i] * rs2));
}

void orc_gelu_backward(const double* dy, const double* x, int64_t n, double* out) {
  const double rs2 = 1.4142135623730951 / 2.0;
  const double inv_sqrt_2pi = 1.0 / sqrt(2.0 * 3.141592653589793);
  for (int64_t i = 0; i < n; ++i) {
    const double cdf = 0.5 * (1.0 + erf(x[i] * rs2));
    const double pdf = inv_sqrt_2pi * exp(-0.5 * x[i] * x[i]);
    out[i] = dy[i] * (cdf + x[i] * pdf);
  }
}

void orc_matmul(const double* a, const double* b, const double* bias, int64_t m, int64_t k,
                int64_t n, double* c) {
  orc_gemm(m, n, k, a, k, 1, b, n, 1, c, n, 0);
  if (bias)
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < n; ++j) c[i * n + j] += bias[j];
}

/* Y[rows, w] = X[rows, kdim] · W[:, col0:col0+w] (+bias[col0:]) — matmul_add on a column slice */
static void mm_colslice(const double* x, int64_t rows, int64_t kdim, const double* w, int64_t ldw,
                        int64_t col0, int64_t wdt, const double* bias, double* y) {
  orc_gemm(rows, wdt, kdim, x, kdim, 1, w + col0, ldw, 1, y, wdt, 0);
  if (bias)
    for (int64_t i = 0; i < rows; ++i)
      for (int64_t j = 0; j < wdt; ++j) y[i * wdt + j] += bias[col0 + j];
}

/* dX[rows, kd] = dY[rows, n] · Wv^T, where Wv(kk, j) = w[kk*ldw + j] is [kd, n] (a view) */
static void mm_trhs(const double* dy, int64_t rows, int64_t n, const double* w, int64_t ldw,
                    int64_t kd, double* dx) {
  orc_gemm(rows, kd, n, dy, n, 1, w, 1, ldw, dx, kd, 0);
}

/* G[kd, n] (ldg) = X[rows, kd]^T · dY[rows, n] */
static void mm_tlhs(const double* x, int64_t rows, int64_t kd, const double* dy, int64_t n,
                    double* g, int64_t ldg) {
  orc_gemm(kd, n, rows, x, 1, kd, dy, n, 1, g, ldg, 0);
}

static void colsum(const double* x, int64_t rows, int64_t n, double* out) {
  for (int64_t j = 0; j < n; ++j) out[j] = 0.0;
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < n; ++j) out[j] += x[i * n + j];
}

/* mask_slice (block.cpp:42-68): slice [index] of [parts] along axis 0 of a tensor whose
 * trailing extent is `inner`; rows_full = full axis extent. */
static void mask_slice(uint64_t folded, int64_t full_axis, int64_t inner, double p, int64_t parts,
                       int64_t index, double* out) {
  const int64_t piece = full_axis / parts;
#pragma omp parallel for schedule(static) num_threads(orc_threads()) if (piece * inner > 65536)
  for (int64_t ai = 0; ai < piece; ++ai) {
    const int64_t global_row = index * piece + ai;
    for (int64_t in = 0; in < inner; ++in) {
      const uint64_t g = (uint64_t)(global_row * inner + in);
      out[ai * inner + in] = orc_uniform01(folded, g) >= p ? 1.0 : 0.0;
    }
  }
}

static void apply_dropout(const double* x, const double* mask, int64_t n, double p, double* out) {
  const double inv_keep = 1.0 / (1.0 - p);
  for (int64_t i = 0; i < n; ++i) out[i] = x[i] * mask[i] * inv_keep;
}

static int all_finite(const double* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return 0;
  return 1;
}

int orc_attention_interior(const orc_block_cfg* cfg, const double* q, const double* k,
                           int64_t head_offset, int64_t lh, double* sm, double* mask,
                           double* sd) {
  const int64_t s = cfg->seq, b = cfg->batch, hd = cfg->hidden / cfg->heads;
  const int64_t lw = lh * hd;
  const double scale = 1.0 / sqrt((double)hd);
  const uint64_t folded =
      orc_mask_key_fold(cfg->seed, cfg->layer_index, kSoftmaxDrop, cfg->microbatch);
  if (cfg->heads % lh != 0) return fail(1, "mask axis not divisible");
  mask_slice(folded, cfg->heads, b * s * s, cfg->dropout_p, cfg->heads / lh, head_offset / lh,
             mask);
  for (int64_t kk = 0; kk < lh; ++kk)
    for (int64_t j = 0; j < b; ++j) {
      double* sc = sm + ((kk * b + j) * s) * s;
      const double* qh = q + j * lw + kk * hd;
      const double* kh = k + j * lw + kk * hd;
      /* scores = Q_h · K_h^T (row stride b*lw), then * scale */
      orc_gemm(s, s, hd, qh, b * lw, 1, kh, 1, b * lw, sc, s, 0);
      for (int64_t i = 0; i < s * s; ++i) sc[i] *= scale;
      if (cfg->causal)
        for (int64_t i1 = 0; i1 < s; ++i1)
          for (int64_t i2 = i1 + 1; i2 < s; ++i2) sc[i1 * s + i2] = -INFINITY;
    }
  /* rowwise softmax with scalar exp (masked -inf -> exact 0) */
  const int64_t nrows = lh * b * s;
#pragma omp parallel for schedule(static) num_threads(orc_threads()) if (nrows * s > 65536)
  for (int64_t r = 0; r < nrows; ++r) {
    double* row = sm + r * s;
    double mx = row[0];
    for (int64_t c = 1; c < s; ++c)
      if (row[c] > mx) mx = row[c];
    double sum = 0.0;
    for (int64_t c = 0; c < s; ++c) {
      row[c] = exp(row[c] - mx);
      sum += row[c];
    }
    for (int64_t c = 0; c < s; ++c) row[c] /= sum;
  }
  const double inv_keep = 1.0 / (1.0 - cfg->dropout_p);
  const int64_t n = lh * b * s * s;
  for (int64_t i = 0; i < n; ++i) sd[i] = sm[i] * mask[i] * inv_keep;
  return 0;
}

/* O(:, j, head) = dropout_out(head, j) · V(:, j, head) */
static void attention_over_values(const orc_block_cfg* cfg, int64_t lh, const double* sd,
                                  const double* v, double* out) {
  const int64_t s = cfg->seq, b = cfg->batch, hd = cfg->hidden / cfg->heads, lw = lh * hd;
  for (int64_t kk = 0; kk < lh; ++kk)
    for (int64_t j = 0; j < b; ++j)
      orc_gemm(s, hd, s, sd + ((kk * b + j) * s) * s, s, 1, v + j * lw + kk * hd, b * lw, 1,
               out + j * lw + kk * hd, b * lw, 0);
}

static void attention_interior_backward(const orc_block_cfg* cfg, int64_t lh, const double* d_out,
                                        const double* sm, const double* mask, const double* sd,
                                        const double* q, const double* k, const double* v,
                                        double* dq, double* dk, double* dv) {
  const int64_t s = cfg->seq, b = cfg->batch, hd = cfg->hidden / cfg->heads, lw = lh * hd;
  const double scale = 1.0 / sqrt((double)hd);
  const double inv_keep = 1.0 / (1.0 - cfg->dropout_p);
  double* d_sd = dalloc(s * s);
  double* dsc = dalloc(s * s);
  double* tmp = dalloc(s * hd);
  for (int64_t kk = 0; kk < lh; ++kk)
    for (int64_t j = 0; j < b; ++j) {
      const int64_t base = ((kk * b + j) * s) * s;
      const int64_t ho = j * lw + kk * hd;
      /* d_sd = dO_h · V_h^T */
      orc_gemm(s, s, hd, d_out + ho, b * lw, 1, v + ho, 1, b * lw, d_sd, s, 0);
      /* dV_h = SD^T · dO_h */
      orc_gemm(s, hd, s, sd + base, 1, s, d_out + ho, b * lw, 1, dv + ho, b * lw, 0);
      for (int64_t i = 0; i < s; ++i) {
        double row_dot = 0.0;
        for (int64_t c = 0; c < s; ++c) {
          const double d_sm = d_sd[i * s + c] * mask[base + i * s + c] * inv_keep;
          d_sd[i * s + c] = d_sm;
          row_dot += d_sm * sm[base + i * s + c];
        }
        for (int64_t c = 0; c < s; ++c)
          dsc[i * s + c] = sm[base + i * s + c] * (d_sd[i * s + c] - row_dot);
      }
      /* dQ_h = dS · K_h * scale ; dK_h = dS^T · Q_h * scale */
      orc_gemm(s, hd, s, dsc, s, 1, k + ho, b * lw, 1, tmp, hd, 0);
      for (int64_t i = 0; i < s; ++i)
        for (int64_t d = 0; d < hd; ++d) dq[ho + i * b * lw + d] = tmp[i * hd + d] * scale;
      orc_gemm(s, hd, s, dsc, 1, s, q + ho, b * lw, 1, tmp, hd, 0);
      for (int64_t i = 0; i < s; ++i)
        for (int64_t d = 0; d < hd; ++d) dk[ho + i * b * lw + d] = tmp[i * hd + d] * scale;
    }
  free(d_sd);
  free(dsc);
  free(tmp);
}

/* ------------------------------------------------------------------ ledger */
static const char* kLedgerNames[ORC_LEDGER_ENTRIES] = {
    "ln1_input",          "qkv_input",           "query",           "key",
    "value",              "softmax_out",         "softmax_dropout_mask",
    "softmax_dropout_out", "attn_proj_input",    "attn_dropout_mask", "ln2_input",
    "mlp_fc1_input",      "gelu_input",          "mlp_fc2_input",   "mlp_dropout_mask"};

const char* orc_ledger_name(int i) {
  return (i >= 0 && i < ORC_LEDGER_ENTRIES) ? kLedgerNames[i] : "";
}

void orc_ledger_layer(const orc_block_cfg* cfg, int64_t seq_local, int64_t lh, int64_t act,
                      int64_t mask, orc_ledger* out) {
  const int64_t b = cfg->batch, h = cfg->hidden, s = cfg->seq;
  const int64_t lw = lh * (cfg->hidden / cfg->heads);
  const int64_t e[ORC_LEDGER_ENTRIES] = {
      seq_local * b * h, seq_local * b * h, s * b * lw,         s * b * lw,
      s * b * lw,        lh * b * s * s,    lh * b * s * s,     lh * b * s * s,
      s * b * lw,        seq_local * b * h, seq_local * b * h,  seq_local * b * h,
      s * b * 4 * lw,    s * b * 4 * lw,    seq_local * b * h};
  const int is_mask[ORC_LEDGER_ENTRIES] = {0, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0, 0, 0, 1};
  for (int i = 0; i < ORC_LEDGER_ENTRIES; ++i) {
    out->elements[i] = e[i];
    out->bytes[i] = e[i] * (is_mask[i] ? mask : act);
  }
}

/* ------------------------------------------------------------------ comm log */
static void log_ring(orc_comm_counters* c, int64_t logical, int64_t ranks, int64_t steps,
                     int which) {
  if (!c) return;
  if (which == 0) c->all_gathers++;
  if (which == 1) c->reduce_scatters++;
  if (which == 2) c->all_reduces++;
  c->ring_elements += steps * (logical / ranks) * (ranks - 1);
}

/* reduce_scatter over axis 0: ordered sum of t partials [t][n], shard r = rows chunk r */
static void ordered_sum(double* const* parts, int64_t t, int64_t n, double* acc) {
  memcpy(acc, parts[0], sizeof(double) * (size_t)n);
  for (int64_t r = 1; r < t; ++r)
    for (int64_t i = 0; i < n; ++i) acc[i] += parts[r][i];
}

/* ------------------------------------------------------------------ layer */
typedef struct {
  double *x, *y1, *mu1, *is1, *q, *k, *v, *sm, *msk, *sd, *api, *amask, *r1, *y2, *mu2, *is2,
      *gin, *fin, *mmask, *y;
} rank_state;

static void free_rank(rank_state* s) {
  double** f = (double**)s;
  for (size_t i = 0; i < sizeof(rank_state) / sizeof(double*); ++i) free(f[i]);
  memset(s, 0, sizeof *s);
}

static int check_cfg(const orc_block_cfg* c, int64_t t) {
  if (t < 1) return fail(1, "t must be >= 1");
  if (c->heads < 1 || c->hidden < 1 || c->seq < 1 || c->batch < 1)
    return fail(1, "shape fields must be >= 1");
  if (c->hidden % c->heads != 0) return fail(1, "hidden not divisible by heads");
  if (c->seq % t != 0 || c->hidden % t != 0) return fail(1, "s and h must be divisible by t");
  if (c->heads % t != 0) return fail(1, "attention heads must be divisible by t");
  if (c->dropout_p < 0.0 || c->dropout_p >= 1.0) return fail(1, "dropout_p must lie in [0,1)");
  return 0;
}

int orc_seqpar_layer(const orc_block_cfg* cfg, int64_t t, const double* P, const double* x,
                     const double* dy, double* y, double* dx, double* G, double* w1_shards,
                     double* interior, orc_comm_log* flog, orc_comm_log* blog, orc_ledger* ledg) {
  int rc = check_cfg(cfg, t);
  if (rc) return rc;
  const int64_t s = cfg->seq, b = cfg->batch, h = cfg->hidden, a = cfg->heads;
  const int64_t lh = a / t, lw = h / t, fw = 4 * h / t;
  const int64_t RL = (s / t) * b, RF = s * b; /* local / full rows */
  const double p = cfg->dropout_p;
  int64_t off[ORC_NPARAM];
  const int64_t np = orc_param_layout(h, off, NULL);
  const double *wq = P + off[ORC_WQ], *wk = P + off[ORC_WK], *wv = P + off[ORC_WV];
  const double *bq = P + off[ORC_BQ], *bk = P + off[ORC_BK], *bv = P + off[ORC_BV];
  const double *wo = P + off[ORC_WO], *bo = P + off[ORC_BO], *w1 = P + off[ORC_W1];
  const double *b1 = P + off[ORC_B1], *w2 = P + off[ORC_W2], *b2 = P + off[ORC_B2];
  const double *g1 = P + off[ORC_LN1_GAIN], *be1 = P + off[ORC_LN1_BIAS];
  const double *g2 = P + off[ORC_LN2_GAIN], *be2 = P + off[ORC_LN2_BIAS];
  const uint64_t k_attn = orc_mask_key_fold(cfg->seed, cfg->layer_index, kAttnOutDrop, cfg->microbatch);
  const uint64_t k_mlp = orc_mask_key_fold(cfg->seed, cfg->layer_index, kMlpDrop, cfg->microbatch);
  if (flog) memset(flog, 0, sizeof *flog);
  if (blog) memset(blog, 0, sizeof *blog);

  rank_state* R = (rank_state*)calloc((size_t)t, sizeof(rank_state));
  double** part = (double**)calloc((size_t)t, sizeof(double*));
  double* full = dalloc(RF * h);  /* gathered / summed {s,b,h} scratch */
  double* full2 = dalloc(RF * h);

  /* ---- forward (block.cpp:546-600) */
  for (int64_t r = 0; r < t; ++r) {
    rank_state* S = &R[r];
    S->x = dalloc(RL * h);
    memcpy(S->x, x + r * RL * h, sizeof(double) * (size_t)(RL * h));
    S->y1 = dalloc(RL * h);
    S->mu1 = dalloc(RL);
    S->is1 = dalloc(RL);
    orc_layer_norm(S->x, RL, h, g1, be1, cfg->ln_eps, S->y1, S->mu1, S->is1);
  }
  for (int64_t r = 0; r < t; ++r) memcpy(full + r * RL * h, R[r].y1, sizeof(double) * (size_t)(RL * h));
  log_ring(flog ? &flog->schedule : NULL, RF * h, t, 1, 0);
  for (int64_t r = 0; r < t; ++r) {
    rank_state* S = &R[r];
    S->q = dalloc(RF * lw);
    S->k = dalloc(RF * lw);
    S->v = dalloc(RF * lw);
    mm_colslice(full, RF, h, wq, h, r * lw, lw, bq, S->q);
    mm_colslice(full, RF, h, wk, h, r * lw, lw, bk, S->k);
    mm_colslice(full, RF, h, wv, h, r * lw, lw, bv, S->v);
    S->sm = dalloc(lh * b * s * s);
    S->msk = dalloc(lh * b * s * s);
    S->sd = dalloc(lh * b * s * s);
    rc = orc_attention_interior(cfg, S->q, S->k, r * lh, lh, S->sm, S->msk, S->sd);
    if (rc) goto done;
    S->api = dalloc(RF * lw);
    attention_over_values(cfg, lh, S->sd, S->v, S->api);
    part[r] = dalloc(RF * h);
    /* proj partial = api · wo[rows r*lw ...] */
    orc_gemm(RF, h, lw, S->api, lw, 1, wo + r * lw * h, h, 1, part[r], h, 0);
  }
  ordered_sum(part, t, RF * h, full2);
  log_ring(flog ? &flog->schedule : NULL, RF * h, t, 1, 1);
  for (int64_t r = 0; r < t; ++r) {
    rank_state* S = &R[r];
    double* shard = full2 + r * RL * h;
    for (int64_t i = 0; i < RL; ++i)
      for (int64_t c = 0; c < h; ++c) shard[i * h + c] += bo[c];
    S->amask = dalloc(RL * h);
    mask_slice(k_attn, s, b * h, p, t, r, S->amask);
    S->r1 = dalloc(RL * h);
    apply_dropout(shard, S->amask, RL * h, p, S->r1);
    for (int64_t i = 0; i < RL * h; ++i) S->r1[i] = S->x[i] + S->r1[i];
    S->y2 = dalloc(RL * h);
    S->mu2 = dalloc(RL);
    S->is2 = dalloc(RL);
    orc_layer_norm(S->r1, RL, h, g2, be2, cfg->ln_eps, S->y2, S->mu2, S->is2);
  }
  for (int64_t r = 0; r < t; ++r) memcpy(full + r * RL * h, R[r].y2, sizeof(double) * (size_t)(RL * h));
  log_ring(flog ? &flog->schedule : NULL, RF * h, t, 1, 0);
  for (int64_t r = 0; r < t; ++r) {
    rank_state* S = &R[r];
    S->gin = dalloc(RF * fw);
    S->fin = dalloc(RF * fw);
    mm_colslice(full, RF, h, w1, 4 * h, r * fw, fw, b1, S->gin);
    orc_gelu(S->gin, RF * fw, S->fin);
    orc_gemm(RF, h, fw, S->fin, fw, 1, w2 + r * fw * h, h, 1, part[r], h, 0);
  }
  ordered_sum(part, t, RF * h, full2);
  log_ring(flog ? &flog->schedule : NULL, RF * h, t, 1, 1);
  for (int64_t r = 0; r < t; ++r) {
    rank_state* S = &R[r];
    double* shard = full2 + r * RL * h;
    for (int64_t i = 0; i < RL; ++i)
      for (int64_t c = 0; c < h; ++c) shard[i * h + c] += b2[c];
    S->mmask = dalloc(RL * h);
    mask_slice(k_mlp, s, b * h, p, t, r, S->mmask);
    S->y = dalloc(RL * h);
    apply_dropout(shard, S->mmask, RL * h, p, S->y);
    for (int64_t i = 0; i < RL * h; ++i) S->y[i] = S->r1[i] + S->y[i];
    if (!all_finite(S->y, RL * h)) {
      rc = fail(2, "seqpar_block_forward produced non-finite values");
      goto done;
    }
    if (y) memcpy(y + r * RL * h, S->y, sizeof(double) * (size_t)(RL * h));
    if (ledg) orc_ledger_layer(cfg, s / t, lh, 2, 1, &ledg[r]);
    if (interior) {
      const int64_t n = lh * b * s * s, all = a * b * s * s;
      memcpy(interior + r * n, S->sm, sizeof(double) * (size_t)n);
      memcpy(interior + all + r * n, S->msk, sizeof(double) * (size_t)n);
      memcpy(interior + 2 * all + r * n, S->sd, sizeof(double) * (size_t)n);
    }
  }
  if (!dy) goto done;

  /* ---- backward (block.cpp:622-749) */
  {
    double* dr1 = dalloc(RF * h); /* d_r1 shards, concatenated */
    memcpy(dr1, dy, sizeof(double) * (size_t)(RF * h));
    double* repl = dalloc(6 * t * h); /* partials: bo, b2, g1, be1, g2, be2 per rank */
#define REPL(kind, r) (repl + ((kind) * t + (r)) * h)
    if (G) memset(G, 0, sizeof(double) * (size_t)np);
    /* MLP branch: dropout bwd + b2 partial on shards, then AG (C5) */
    for (int64_t r = 0; r < t; ++r) {
      apply_dropout(dy + r * RL * h, R[r].mmask, RL * h, p, full + r * RL * h);
      colsum(full + r * RL * h, RL, h, REPL(1, r));
    }
    log_ring(blog ? &blog->schedule : NULL, RF * h, t, 1, 0);
    for (int64_t r = 0; r < t; ++r) memcpy(full2 + r * RL * h, R[r].y2, sizeof(double) * (size_t)(RL * h));
    log_ring(blog ? &blog->regather : NULL, RF * h, t, 1, 0);
    double* dfc2 = dalloc(RF * fw);
    double* dgin = dalloc(RF * fw);
    double* b1g = dalloc(fw);
    for (int64_t r = 0; r < t; ++r) {
      const double* w2r = w2 + r * fw * h; /* [fw, h] rows */
      mm_trhs(full, RF, h, w2r, h, fw, dfc2);
      if (G) mm_tlhs(R[r].fin, RF, fw, full, h, G + off[ORC_W2] + r * fw * h, h);
      orc_gelu_backward(dfc2, R[r].gin, RF * fw, dgin);
      colsum(dgin, RF, fw, b1g);
      if (G) memcpy(G + off[ORC_B1] + r * fw, b1g, sizeof(double) * (size_t)fw);
      if (G) mm_tlhs(full2, RF, h, dgin, fw, G + off[ORC_W1] + r * fw, 4 * h);
      if (w1_shards) mm_tlhs(full2, RF, h, dgin, fw, w1_shards + r * h * fw, fw);
      /* d_y2 partial = dgin · W1_r^T, W1_r(kk, j) = w1[kk*4h + r*fw + j] */
      mm_trhs(dgin, RF, fw, w1 + r * fw, 4 * h, h, part[r]);
    }
    free(dfc2);
    free(b1g);
    ordered_sum(part, t, RF * h, full);
    log_ring(blog ? &blog->schedule : NULL, RF * h, t, 1, 1);
    double* tmp = dalloc(RL * h);
    for (int64_t r = 0; r < t; ++r) {
      orc_layer_norm_backward(full + r * RL * h, R[r].r1, R[r].mu2, R[r].is2, RL, h, g2, tmp,
                              REPL(4, r), REPL(5, r));
      for (int64_t i = 0; i < RL * h; ++i) dr1[r * RL * h + i] += tmp[i];
    }
    /* attention branch */
    for (int64_t r = 0; r < t; ++r) {
      apply_dropout(dr1 + r * RL * h, R[r].amask, RL * h, p, full + r * RL * h);
      colsum(full + r * RL * h, RL, h, REPL(0, r));
    }
    log_ring(blog ? &blog->schedule : NULL, RF * h, t, 1, 0);
    for (int64_t r = 0; r < t; ++r) memcpy(full2 + r * RL * h, R[r].y1, sizeof(double) * (size_t)(RL * h));
    log_ring(blog ? &blog->regather : NULL, RF * h, t, 1, 0);
    double* dproj = dalloc(RF * lw);
    double *dq = dalloc(RF * lw), *dk = dalloc(RF * lw), *dv = dalloc(RF * lw);
    double* bias_g = dalloc(lw);
    double* acc = dalloc(RF * h);
    for (int64_t r = 0; r < t; ++r) {
      rank_state* S = &R[r];
      const double* wor = wo + r * lw * h; /* [lw, h] */
      mm_trhs(full, RF, h, wor, h, lw, dproj);
      if (G) mm_tlhs(S->api, RF, lw, full, h, G + off[ORC_WO] + r * lw * h, h);
      attention_interior_backward(cfg, lh, dproj, S->sm, S->msk, S->sd, S->q, S->k, S->v, dq,
                                  dk, dv);
      if (G) {
        colsum(dq, RF, lw, bias_g);
        memcpy(G + off[ORC_BQ] + r * lw, bias_g, sizeof(double) * (size_t)lw);
        colsum(dk, RF, lw, bias_g);
        memcpy(G + off[ORC_BK] + r * lw, bias_g, sizeof(double) * (size_t)lw);
        colsum(dv, RF, lw, bias_g);
        memcpy(G + off[ORC_BV] + r * lw, bias_g, sizeof(double) * (size_t)lw);
        mm_tlhs(full2, RF, h, dq, lw, G + off[ORC_WQ] + r * lw, h);
        mm_tlhs(full2, RF, h, dk, lw, G + off[ORC_WK] + r * lw, h);
        mm_tlhs(full2, RF, h, dv, lw, G + off[ORC_WV] + r * lw, h);
      }
      mm_trhs(dq, RF, lw, wq + r * lw, h, h, part[r]);
      mm_trhs(dk, RF, lw, wk + r * lw, h, h, acc);
      for (int64_t i = 0; i < RF * h; ++i) part[r][i] = part[r][i] + acc[i];
      mm_trhs(dv, RF, lw, wv + r * lw, h, h, acc);
      for (int64_t i = 0; i < RF * h; ++i) part[r][i] = part[r][i] + acc[i];
    }
    free(dproj);
    free(dq);
    free(dk);
    free(dv);
    free(bias_g);
    free(acc);
    ordered_sum(part, t, RF * h, full);
    log_ring(blog ? &blog->schedule : NULL, RF * h, t, 1, 1);
    for (int64_t r = 0; r < t; ++r) {
      orc_layer_norm_backward(full + r * RL * h, R[r].x, R[r].mu1, R[r].is1, RL, h, g1, tmp,
                              REPL(2, r), REPL(3, r));
      if (dx)
        for (int64_t i = 0; i < RL * h; ++i) dx[r * RL * h + i] = dr1[r * RL * h + i] + tmp[i];
    }
    free(tmp);
    free(dr1);
    /* replicated grads: all_reduce ×6 (C11) in rank order */
    const int kinds[6] = {ORC_BO, ORC_B2, ORC_LN1_GAIN, ORC_LN1_BIAS, ORC_LN2_GAIN, ORC_LN2_BIAS};
    const int src[6] = {0, 1, 2, 3, 4, 5};
    for (int kx = 0; kx < 6; ++kx) {
      double* out = G ? G + off[kinds[kx]] : NULL;
      if (out) {
        memcpy(out, REPL(src[kx], 0), sizeof(double) * (size_t)h);
        for (int64_t r = 1; r < t; ++r)
          for (int64_t c = 0; c < h; ++c) out[c] += REPL(src[kx], r)[c];
      }
      log_ring(blog ? &blog->grad_sync : NULL, h, t, 2, 2);
    }
#undef REPL
    free(repl);
    free(dgin);
  }
done:
  for (int64_t r = 0; r < t; ++r) {
    free_rank(&R[r]);
    free(part[r]);
  }
  free(R);
  free(part);
  free(full);
  free(full2);
  return rc;
}

int orc_reference_layer(const orc_block_cfg* cfg, const double* P, const double* x,
                        const double* dy, double* y, double* dx, double* G, double* q_out,
                        double* k_out, double* interior, orc_ledger* ledger) {
  int rc = check_cfg(cfg, 1);
  if (rc) return rc;
  const int64_t s = cfg->seq, b = cfg->batch, h = cfg->hidden, a = cfg->heads;
  const int64_t RF = s * b, n = RF * h, ni = a * b * s * s;
  const double p = cfg->dropout_p;
  int64_t off[ORC_NPARAM];
  const int64_t np = orc_param_layout(h, off, NULL);
  const uint64_t k_attn = orc_mask_key_fold(cfg->seed, cfg->layer_index, kAttnOutDrop, cfg->microbatch);
  const uint64_t k_mlp = orc_mask_key_fold(cfg->seed, cfg->layer_index, kMlpDrop, cfg->microbatch);
  double *y1 = dalloc(n), *mu1 = dalloc(RF), *is1 = dalloc(RF);
  double *q = dalloc(n), *k = dalloc(n), *v = dalloc(n);
  double *sm = dalloc(ni), *msk = dalloc(ni), *sd = dalloc(ni), *api = dalloc(n);
  double *ao = dalloc(n), *amask = dalloc(n), *r1 = dalloc(n), *y2 = dalloc(n);
  double *mu2 = dalloc(RF), *is2 = dalloc(RF), *gin = dalloc(4 * n), *fin = dalloc(4 * n);
  double *mo = dalloc(n), *mmask = dalloc(n), *yy = dalloc(n);

  orc_layer_norm(x, RF, h, P + off[ORC_LN1_GAIN], P + off[ORC_LN1_BIAS], cfg->ln_eps, y1, mu1, is1);
  orc_matmul(y1, P + off[ORC_WQ], P + off[ORC_BQ], RF, h, h, q);
  orc_matmul(y1, P + off[ORC_WK], P + off[ORC_BK], RF, h, h, k);
  orc_matmul(y1, P + off[ORC_WV], P + off[ORC_BV], RF, h, h, v);
  rc = orc_attention_interior(cfg, q, k, 0, a, sm, msk, sd);
  if (rc) goto out;
  attention_over_values(cfg, a, sd, v, api);
  orc_matmul(api, P + off[ORC_WO], P + off[ORC_BO], RF, h, h, ao);
  mask_slice(k_attn, s, b * h, p, 1, 0, amask);
  apply_dropout(ao, amask, n, p, r1);
  for (int64_t i = 0; i < n; ++i) r1[i] = x[i] + r1[i];
  orc_layer_norm(r1, RF, h, P + off[ORC_LN2_GAIN], P + off[ORC_LN2_BIAS], cfg->ln_eps, y2, mu2, is2);
  orc_matmul(y2, P + off[ORC_W1], P + off[ORC_B1], RF, h, 4 * h, gin);
  orc_gelu(gin, 4 * n, fin);
  orc_matmul(fin, P + off[ORC_W2], P + off[ORC_B2], RF, 4 * h, h, mo);
  mask_slice(k_mlp, s, b * h, p, 1, 0, mmask);
  apply_dropout(mo, mmask, n, p, yy);
  for (int64_t i = 0; i < n; ++i) yy[i] = r1[i] + yy[i];
  if (!all_finite(yy, n)) {
    rc = fail(2, "reference_block_forward produced non-finite values");
    goto out;
  }
  if (y) memcpy(y, yy, sizeof(double) * (size_t)n);
  if (q_out) memcpy(q_out, q, sizeof(double) * (size_t)n);
  if (k_out) memcpy(k_out, k, sizeof(double) * (size_t)n);
  if (interior) {
    memcpy(interior, sm, sizeof(double) * (size_t)ni);
    memcpy(interior + ni, msk, sizeof(double) * (size_t)ni);
    memcpy(interior + 2 * ni, sd, sizeof(double) * (size_t)ni);
  }
  if (ledger) orc_ledger_layer(cfg, s, a, 2, 1, ledger);
  if (dy && (dx || G)) {
    double* g = G ? G : dalloc(np);
    memset(g, 0, sizeof(double) * (size_t)np);
    double *dr1 = dalloc(n), *dmo = dalloc(n), *dfc2 = dalloc(4 * n), *dgin = dalloc(4 * n);
    double *dy2 = dalloc(n), *tmp = dalloc(n), *dao = dalloc(n), *dproj = dalloc(n);
    double *dq = dalloc(n), *dk = dalloc(n), *dv = dalloc(n), *dy1 = dalloc(n);
    memcpy(dr1, dy, sizeof(double) * (size_t)n);
    apply_dropout(dy, mmask, n, p, dmo);
    colsum(dmo, RF, h, g + off[ORC_B2]);
    mm_trhs(dmo, RF, h, P + off[ORC_W2], h, 4 * h, dfc2);
    mm_tlhs(fin, RF, 4 * h, dmo, h, g + off[ORC_W2], h);
    orc_gelu_backward(dfc2, gin, 4 * n, dgin);
    colsum(dgin, RF, 4 * h, g + off[ORC_B1]);
    mm_tlhs(y2, RF, h, dgin, 4 * h, g + off[ORC_W1], 4 * h);
    mm_trhs(dgin, RF, 4 * h, P + off[ORC_W1], 4 * h, h, dy2);
    orc_layer_norm_backward(dy2, r1, mu2, is2, RF, h, P + off[ORC_LN2_GAIN], tmp,
                            g + off[ORC_LN2_GAIN], g + off[ORC_LN2_BIAS]);
    for (int64_t i = 0; i < n; ++i) dr1[i] = dr1[i] + tmp[i];
    apply_dropout(dr1, amask, n, p, dao);
    colsum(dao, RF, h, g + off[ORC_BO]);
    mm_trhs(dao, RF, h, P + off[ORC_WO], h, h, dproj);
    mm_tlhs(api, RF, h, dao, h, g + off[ORC_WO], h);
    attention_interior_backward(cfg, a, dproj, sm, msk, sd, q, k, v, dq, dk, dv);
    colsum(dq, RF, h, g + off[ORC_BQ]);
    colsum(dk, RF, h, g + off[ORC_BK]);
    colsum(dv, RF, h, g + off[ORC_BV]);
    mm_tlhs(y1, RF, h, dq, h, g + off[ORC_WQ], h);
    mm_tlhs(y1, RF, h, dk, h, g + off[ORC_WK], h);
    mm_tlhs(y1, RF, h, dv, h, g + off[ORC_WV], h);
    mm_trhs(dq, RF, h, P + off[ORC_WQ], h, h, dy1);
    mm_trhs(dk, RF, h, P + off[ORC_WK], h, h, tmp);
    for (int64_t i = 0; i < n; ++i) dy1[i] = dy1[i] + tmp[i];
    mm_trhs(dv, RF, h, P + off[ORC_WV], h, h, tmp);
    for (int64_t i = 0; i < n; ++i) dy1[i] = dy1[i] + tmp[i];
    orc_layer_norm_backward(dy1, x, mu1, is1, RF, h, P + off[ORC_LN1_GAIN], tmp,
                            g + off[ORC_LN1_GAIN], g + off[ORC_LN1_BIAS]);
    if (dx)
      for (int64_t i = 0; i < n; ++i) dx[i] = dr1[i] + tmp[i];
    free(dr1); free(dmo); free(dfc2); free(dgin); free(dy2); free(tmp); free(dao); free(dproj);
    free(dq); free(dk); free(dv); free(dy1);
    if (!G) free(g);
  }
out:
  free(y1); free(mu1); free(is1); free(q); free(k); free(v); free(sm); free(msk); free(sd);
  free(api); free(ao); free(amask); free(r1); free(y2); free(mu2); free(is2); free(gin);
  free(fin); free(mo); free(mmask); free(yy);
  return rc;
}
