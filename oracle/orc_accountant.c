/* Activation-memory accountant restatement (TEST INFRASTRUCTURE — see oracle.h).
 * Follows /root/reference/proj/core/src/activation_memory.cpp:
 *   coefficient table   activation_memory.cpp:23-27 (4 replicated acts, 12 sharded acts,
 *                        2 replicated masks per sbh; 2 acts + 1 mask per a·s²·b)
 *   per_layer_bytes     activation_memory.cpp:54-82 (floor once, rational.hpp:32-49)
 *   breakdown           activation_memory.cpp:84-104
 *   percent_of_baseline activation_memory.cpp:195-200
 *   total_first_stage   activation_memory.cpp:106-123 (interleave_factor, x L, floor once)
 * and validate() from config.cpp:86-133 (the shape/layout rules that apply per layer).
 * Boost rationals are replaced by __int128 num/den: every per-layer value has denominator 1
 * or t, so 128-bit arithmetic is exact for all shapes whose byte counts fit int64. */
#include "oracle.h"

typedef __int128 i128;

static int valid_layer(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int64_t act,
                       int64_t mask) {
  if (a < 1 || h < 1 || s < 1 || b < 1 || t < 1) return 0;
  if (h % a != 0) return 0;
  if (h % t != 0) return 0;
  if (s % t != 0) return 0;
  if (act < 1 || mask < 1) return 0;
  return 1;
}

static i128 gcd128(i128 x, i128 y) {
  if (x < 0) x = -x;
  if (y < 0) y = -y;
  while (y != 0) {
    i128 r = x % y;
    x = y;
    y = r;
  }
  return x;
}

/* value = num/den, den > 0 */
static int per_layer_rational(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                              int sp, int64_t act, int64_t mask, i128* num, i128* den) {
  if (!valid_layer(a, h, s, b, t, act, mask)) return 1;
  if (kind < 0 || kind > 2) return 1;
  const i128 sbh = (i128)s * b * h;
  if (kind == 1) { /* Full: only the layer input, not divided by t (activation_memory.cpp:59-63) */
    *num = (i128)act * sbh;
    *den = 1;
    return 0;
  }
  const i128 replicated = ((i128)4 * act + (i128)2 * mask) * sbh;
  const i128 sharded = (i128)12 * act * sbh;
  i128 n = sp ? (replicated + sharded) : (replicated * t + sharded);
  if (kind == 0) {
    const i128 interior = ((i128)2 * act + (i128)mask) * ((i128)a * s * s * b);
    n += interior;
  }
  i128 d = t;
  i128 g = gcd128(n, d);
  if (g > 1) {
    n /= g;
    d /= g;
  }
  *num = n;
  *den = d;
  return 0;
}

static int fits64(i128 v) { return v <= (i128)INT64_MAX && v >= (i128)INT64_MIN; }

int orc_per_layer_bytes(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                        int sequence_parallel, int64_t act, int64_t mask, int64_t* bytes_out) {
  i128 n, d;
  if (per_layer_rational(a, h, s, b, t, kind, sequence_parallel, act, mask, &n, &d)) return 1;
  i128 q = n / d; /* n >= 0: truncation == floor */
  if (!fits64(q)) return 3;
  *bytes_out = (int64_t)q;
  return 0;
}

int orc_per_layer_bytes_exact(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                              int sequence_parallel, int64_t act, int64_t mask, int64_t* num,
                              int64_t* den) {
  i128 n, d;
  if (per_layer_rational(a, h, s, b, t, kind, sequence_parallel, act, mask, &n, &d)) return 1;
  if (!fits64(n) || !fits64(d)) return 3;
  *num = (int64_t)n;
  *den = (int64_t)d;
  return 0;
}

int orc_layer_component_breakdown(int64_t a, int64_t h, int64_t s, int64_t b, int64_t act,
                                  int64_t mask, int64_t out[4]) {
  if (!valid_layer(a, h, s, b, 1, act, mask)) return 1;
  const i128 sbh = (i128)s * b * h;
  const i128 interior = (i128)a * s * s * b;
  i128 attention = (i128)5 * act * sbh + (i128)mask * sbh + ((i128)2 * act + mask) * interior;
  i128 mlp = (i128)9 * act * sbh + (i128)mask * sbh;
  i128 lns = (i128)2 * act * sbh;
  i128 total = attention + mlp + lns;
  if (!fits64(total)) return 3;
  out[0] = (int64_t)attention;
  out[1] = (int64_t)mlp;
  out[2] = (int64_t)lns;
  out[3] = (int64_t)total;
  return 0;
}

int orc_percent_of_baseline(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                            int sequence_parallel, int64_t act, int64_t mask, int64_t* num,
                            int64_t* den) {
  i128 n1, d1, n0, d0;
  if (per_layer_rational(a, h, s, b, t, kind, sequence_parallel, act, mask, &n1, &d1)) return 1;
  if (per_layer_rational(a, h, s, b, t, 0, 0, act, mask, &n0, &d0)) return 1;
  i128 n = n1 * d0, d = d1 * n0;
  i128 g = gcd128(n, d);
  if (g > 1) {
    n /= g;
    d /= g;
  }
  if (!fits64(n) || !fits64(d)) return 3;
  *num = (int64_t)n;
  *den = (int64_t)d;
  return 0;
}

int orc_total_first_stage_bytes(int64_t a, int64_t h, int64_t s, int64_t b, int64_t t, int kind,
                                int sequence_parallel, int64_t layers, int64_t pipeline,
                                int64_t interleave, int64_t act, int64_t mask,
                                int64_t* bytes_out) {
  /* config.cpp:94-117: L, p, m >= 1 and L divisible by p*m */
  if (layers < 1 || pipeline < 1 || interleave < 1) return 1;
  if (layers % (pipeline * interleave) != 0) return 1;
  i128 n, d;
  if (per_layer_rational(a, h, s, b, t, kind, sequence_parallel, act, mask, &n, &d)) return 1;
  n *= layers;
  if (interleave > 1) { /* 1 + (p-1)/(p*m) = (p*m + p - 1)/(p*m), activation_memory.cpp:106-110 */
    n *= (i128)pipeline * interleave + pipeline - 1;
    d *= (i128)pipeline * interleave;
  }
  i128 q = n / d;
  if (!fits64(q)) return 3;
  *bytes_out = (int64_t)q;
  return 0;
}

int64_t orc_layer_comm_bytes_tp(int64_t s, int64_t b, int64_t h, int64_t t, int64_t elem) {
  const i128 bytes = (i128)s * b * h * elem;
  return (int64_t)((i128)4 * 2 * (bytes / t) * (t - 1));
}

int64_t orc_layer_comm_bytes_sp(int64_t s, int64_t b, int64_t h, int64_t t, int64_t elem) {
  const i128 bytes = (i128)s * b * h * elem;
  return (int64_t)((i128)8 * (bytes / t) * (t - 1));
}
