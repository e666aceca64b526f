/*
 * spiketrain_oracle.c -- TEST INFRASTRUCTURE ONLY (see spiketrain_oracle.h).
 *
 * Plain-C restatement of the reference's training step.  Every arithmetic
 * statement follows the reference's operation order so that, compiled with
 * -ffp-contract=off against the same libm, results are bit-identical to the
 * reference (checked by tests/test_oracle.py against oracle/_ref and the
 * golden vectors).  Citations are /root/reference/proj/include/spiketrain/.
 */
#include "spiketrain_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* Host threads for the big-shape parity tests (orc_set_threads; default 1).
 * Every parallel loop below splits OUTPUT elements (rows, samples, neurons or
 * weight rows) across threads and keeps each element's own accumulation in the
 * reference order, so results are bit-identical for any thread count
 * (tests/test_oracle.py::test_threads_are_bit_identical). */
static int g_threads = 1;
void orc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }

/* ------------------------------------------------------------------------ */
/* RNG: rng.hpp:20-48 (mix64, from_seed, bits, child), :62-64 (uniform01). */

static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t orc_key_from_seed(uint64_t seed) { return mix64(seed); }

uint64_t orc_key_child(uint64_t key, uint64_t index) {
  return mix64(key ^ mix64(index + 0xC2B2AE3D27D4EB4Full));
}

uint64_t orc_key_bits(uint64_t key, uint64_t counter) {
  return mix64(key ^ mix64(counter + 0x165667B19E3779F9ull));
}

double orc_uniform01(uint64_t key, uint64_t counter) {
  return (double)(orc_key_bits(key, counter) >> 11) * 0x1.0p-53;
}

/* Fisher-Yates (rng.hpp:78-87). */
void orc_permutation(uint64_t key, size_t n, uint64_t* p) {
  for (size_t i = 0; i < n; ++i) p[i] = i;
  for (size_t i = n; i > 1; --i) {
    const size_t j = (size_t)(orc_key_bits(key, i - 1) % (uint64_t)i);
    const uint64_t tmp = p[i - 1];
    p[i - 1] = p[j];
    p[j] = tmp;
  }
}

/* Box-Muller cosine leg (rng.hpp:92-97). */
static double normal_at(uint64_t key, uint64_t i) {
  const double u1 = 1.0 - orc_uniform01(key, 2 * i);
  const double u2 = orc_uniform01(key, 2 * i + 1);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

/* rng_truncated_normal with +-2 sigma bounds (rng.hpp:123-144). */
void orc_truncated_normal(uint64_t key, size_t n, float mean, float stddev,
                          float* out) {
  const double lo = (double)(-2.0f), hi = (double)(2.0f);
  for (size_t i = 0; i < n; ++i) {
    const uint64_t ek = orc_key_child(key, i);
    double z = 0.0;
    int ok = 0;
    for (uint64_t a = 0; a < 256; ++a) {
      z = normal_at(ek, a);
      if (z >= lo && z <= hi) {
        ok = 1;
        break;
      }
    }
    if (!ok) z = z < lo ? lo : (z > hi ? hi : z);
    out[i] = mean + stddev * (float)z;
  }
}

/* ------------------------------------------------------------------------ */
/* Data: synth_raster (commands.hpp:50-86), pack/unpack (data.hpp:105-149). */

void orc_synth_raster(size_t classes, size_t n, size_t t, size_t f,
                      uint64_t seed, uint8_t* x, int64_t* y) {
  const size_t block = f / classes > 1 ? f / classes : 1;
  const uint64_t master = orc_key_from_seed(seed);
  for (size_t i = 0; i < n; ++i) {
    const size_t label = i % classes;
    y[i] = (int64_t)label;
    const size_t lo = label * block;
    const size_t hi = lo + block < f ? lo + block : f;
    const uint64_t ek = orc_key_child(master, i);
    uint8_t* row = x + i * t * f;
    for (size_t s = 0; s < t; ++s)
      for (size_t j = 0; j < f; ++j) {
        const double rate = (j >= lo && j < hi) ? 0.4 : 0.05;
        row[s * f + j] = orc_uniform01(ek, s * f + j) < rate ? 1 : 0;
      }
  }
}

void orc_pack_time(const uint8_t* x, size_t n, size_t t, size_t f,
                   uint8_t* out) {
  const size_t tp = (t + 7) / 8;
  memset(out, 0, n * tp * f);
  for (size_t o = 0; o < n; ++o)
    for (size_t s = 0; s < t; ++s) {
      const unsigned bit = 7u - (unsigned)(s % 8);
      const uint8_t* src = x + (o * t + s) * f;
      uint8_t* dst = out + (o * tp + s / 8) * f;
      for (size_t k = 0; k < f; ++k)
        if (src[k]) dst[k] |= (uint8_t)(1u << bit);
    }
}

void orc_unpack_time(const uint8_t* packed, size_t n, size_t t, size_t f,
                     uint8_t* out) {
  const size_t tp = (t + 7) / 8;
  for (size_t o = 0; o < n; ++o)
    for (size_t s = 0; s < t; ++s) {
      const unsigned bit = 7u - (unsigned)(s % 8);
      const uint8_t* src = packed + (o * tp + s / 8) * f;
      uint8_t* dst = out + (o * t + s) * f;
      for (size_t k = 0; k < f; ++k) dst[k] = (src[k] >> bit) & 1u;
    }
}

/* ------------------------------------------------------------------------ */
/* Parameter layout (network.hpp:164-226): per hidden block w, [b], beta;
 * then readout w, [b], beta.  Normalised ids: Linear 2j, cell 2j+1.        */

static int is_alif(const orc_net* net, int l) { return l < net->n_hidden && net->cell[l] == 1; }
static int is_rlif(const orc_net* net, int l) { return l < net->n_hidden && net->cell[l] == 2; }
/* the declared cells' extra entry after beta: ALIF gamma [h], RLIF rec [h][h] */
static size_t extra_size(const orc_net* net, int l, size_t h) {
  return is_alif(net, l) ? h : is_rlif(net, l) ? h * h : 0;
}

int orc_entry_count(const orc_net* net) {
  int n = (net->n_hidden + 1) * (net->bias ? 3 : 2);
  for (int l = 0; l < net->n_hidden; ++l) n += extra_size(net, l, 1) ? 1 : 0;
  return n;
}

/* beta entry size of cell l (l == n_hidden: the readout) */
static size_t beta_size(const orc_net* net, int l, size_t h) {
  return net->beta_mode[l] == 0 ? h : 1;
}

/* normalised layer ids (network.hpp:125-157): Linear l, its LIF (or the LI
 * readout) right after, and a monitor after a LIF takes the next id */
static int lin_id(const orc_net* net, int l) {
  int id = 2 * l;
  for (int j = 0; j < l && j < net->n_hidden; ++j) id += net->monitor[j] ? 1 : 0;
  return id;
}

static int layer_in(const orc_net* net, int l) {
  return l == 0 ? net->in : net->hidden[l - 1];
}
static int layer_out(const orc_net* net, int l) {
  return l == net->n_hidden ? net->classes : net->hidden[l];
}

void orc_entry_layout(const orc_net* net, size_t* offsets, size_t* sizes,
                      char (*names)[16]) {
  size_t off = 0;
  int e = 0;
  for (int l = 0; l <= net->n_hidden; ++l) {
    const size_t k = (size_t)layer_in(net, l), h = (size_t)layer_out(net, l);
    const size_t sz[4] = {k * h, h, beta_size(net, l, h), extra_size(net, l, h)};
    const char* leaf[4] = {"w", "b", "beta", is_rlif(net, l) ? "rec" : "gamma"};
    const int lid[4] = {lin_id(net, l), lin_id(net, l), lin_id(net, l) + 1, lin_id(net, l) + 1};
    for (int q = 0; q < 4; ++q) {
      if (q == 1 && !net->bias) continue;
      if (q == 3 && !sz[3]) continue;
      if (offsets) offsets[e] = off;
      if (sizes) sizes[e] = sz[q];
      if (names) snprintf(names[e], 16, "l%d.%s", lid[q], leaf[q]);
      off += sz[q];
      ++e;
    }
  }
}

size_t orc_param_count(const orc_net* net) {
  size_t n = 0;
  for (int l = 0; l <= net->n_hidden; ++l) {
    const size_t k = (size_t)layer_in(net, l), h = (size_t)layer_out(net, l);
    n += k * h + beta_size(net, l, h) + (net->bias ? h : 0) + extra_size(net, l, h);
  }
  return n;
}

typedef struct {
  size_t w, b, beta, gamma; /* offsets; b == SIZE_MAX when no bias, gamma (ALIF gamma or
                               RLIF rec) when the cell has no extra entry */
} layer_off;

static void layer_offsets(const orc_net* net, layer_off* lo) {
  size_t off = 0;
  for (int l = 0; l <= net->n_hidden; ++l) {
    const size_t k = (size_t)layer_in(net, l), h = (size_t)layer_out(net, l);
    lo[l].w = off;
    off += k * h;
    if (net->bias) {
      lo[l].b = off;
      off += h;
    } else {
      lo[l].b = (size_t)-1;
    }
    lo[l].beta = off;
    off += beta_size(net, l, h);
    lo[l].gamma = (size_t)-1;
    if (extra_size(net, l, h)) {
      lo[l].gamma = off;
      off += extra_size(net, l, h);
    }
  }
}

/* init (network.hpp:231-286) with init_lif PerNeuron (neuron.hpp:56-76). */
void orc_init(const orc_net* net, uint64_t key, float* params) {
  layer_off lo[ORC_MAX_HIDDEN + 1];
  layer_offsets(net, lo);
  for (int l = 0; l <= net->n_hidden; ++l) {
    const size_t k = (size_t)layer_in(net, l), h = (size_t)layer_out(net, l);
    const uint64_t lk_lin = orc_key_child(key, (uint64_t)lin_id(net, l));
    const float sd = 1.0f / sqrtf((float)k);
    orc_truncated_normal(orc_key_child(lk_lin, 0), k * h, 0.0f, sd,
                         params + lo[l].w);
    if (net->bias) memset(params + lo[l].b, 0, h * sizeof(float));
    const uint64_t lk_cell = orc_key_child(key, (uint64_t)(lin_id(net, l) + 1));
    if (net->beta_mode[l] == 2) /* Fixed: Tensor::scalar(fixed_beta) */
      params[lo[l].beta] = net->fixed_beta[l];
    else /* PerNeuron [h] or LearnableScalar [] from the same key */
      orc_truncated_normal(orc_key_child(lk_cell, 2), beta_size(net, l, h), 0.5f, 0.25f,
                           params + lo[l].beta);
    if (is_alif(net, l)) /* declared ALIF: gamma ~ TN(0.5, 0.25) from child 3 */
      orc_truncated_normal(orc_key_child(lk_cell, 3), h, 0.5f, 0.25f, params + lo[l].gamma);
    if (is_rlif(net, l)) /* declared RLIF: rec ~ TN(0, 1/sqrt(h)) from child 4 */
      orc_truncated_normal(orc_key_child(lk_cell, 4), h * h, 0.0f, 1.0f / sqrtf((float)h),
                           params + lo[l].gamma);
  }
}

/* ------------------------------------------------------------------------ */
/* Surrogates (surrogate.hpp:59-120), evaluated in float like SpikingActivation<float>. */

static float surrogate_k(int act, float k, float aux, float x) {
  switch (act) {
    case ORC_ACT_SUPERSPIKE: {
      const float d = 1.0f + k * fabsf(x);
      return 1.0f / (d * d);
    }
    case ORC_ACT_TRIANGULAR: {
      const float r = 1.0f - fabsf(k * x);
      return 0.0f < r ? r : 0.0f;
    }
    case ORC_ACT_ARCTAN: {
      const float u = (float)3.141592653589793 * k * x / 2.0f;
      return 1.0f / (1.0f + u * u);
    }
    case ORC_ACT_BOXCAR:
      return fabsf(x) <= k / 2.0f ? aux : 0.0f;
    case ORC_ACT_SIGMOID: {
      /* declared (spiketrain_oracle.h): k e / (1 + e)^2, e = exp(-k|x|) */
      const float e = expf(-(k * fabsf(x)));
      return (k * e) / ((1.0f + e) * (1.0f + e));
    }
    default:
      return 1.0f;
  }
}

static float surrogate(const orc_net* net, float x) {
  return surrogate_k(net->act, net->slope, net->aux, x);
}

void orc_surrogate(int act, float slope, float aux, const float* x, size_t n, float* out) {
  for (size_t i = 0; i < n; ++i) out[i] = surrogate_k(act, slope, aux, x[i]);
}

/* clip(beta, 0, 1) = std::min(1, std::max(0, beta)) (ops.hpp clip). */
static float clip01(float b) {
  const float lo = 0.0f < b ? b : 0.0f;
  return lo < 1.0f ? lo : 1.0f;
}

/* ------------------------------------------------------------------------ */
/* Forward/backward (network.hpp:306-431, objective.hpp:88-134,
 * autodiff.hpp:52-78 and the per-op closures).                            */

/* matmul (ops.hpp:147-174): rows x k times k x n, zero-skip on a. */
static void matmul_rows(const float* a, size_t rows, size_t k, const float* w,
                        size_t n, const float* bias, float* out) {
#pragma omp parallel for schedule(static) num_threads(g_threads)
  for (size_t r = 0; r < rows; ++r) {
    float* o = out + r * n;
    for (size_t j = 0; j < n; ++j) o[j] = 0.0f;
    const float* ar = a + r * k;
    for (size_t kk = 0; kk < k; ++kk) {
      const float av = ar[kk];
      if (av == 0.0f) continue;
      const float* wr = w + kk * n;
      for (size_t j = 0; j < n; ++j) o[j] += av * wr[j];
    }
    if (bias)
      for (size_t j = 0; j < n; ++j) o[j] = o[j] + bias[j];
  }
}

static const orc_train_opts k_default_opts = {0, 0.9f, 0, 0.9f, 0.1f, 0, 0, {0, 0, 0, 0},
                                              0.0f, 1.0f, 0.0f, 0.0f};

/* Activity regularizer of one monitor (objective.hpp:186-227) over the spike
 * raster s [B, T, H]: counts = sum over t (monitor_activity, neuron.hpp:106-114,
 * integer-valued so the per-block sums are exact), the value in the reference's
 * running order over i = b*H + n, and d loss / d count per (b, n). */
static float activity_reg(const orc_train_opts* o, const float* s, size_t B, size_t T, size_t H,
                          float* dcount) {
  const size_t n = B * H;
  float low = 0.0f, high = 0.0f;
  const float gs = 1.0f * 2.0f / ((float)n * (float)T);
  for (size_t b = 0; b < B; ++b)
    for (size_t j = 0; j < H; ++j) {
      float c = 0.0f;
      for (size_t t = 0; t < T; ++t) c += s[(b * T + t) * H + j];
      const float r = c / (float)T;
      const float dl = o->f_min - r > 0.0f ? o->f_min - r : 0.0f;
      const float dh = r - o->f_max > 0.0f ? r - o->f_max : 0.0f;
      low += dl * dl;
      high += dh * dh;
      if (dcount) dcount[b * H + j] = gs * (o->lambda_high * dh - o->lambda_low * dl);
    }
  return o->lambda_low * (low / (float)n) + o->lambda_high * (high / (float)n);
}

static int reg_active(const orc_net* net, const orc_train_opts* o) {
  if (o->lambda_low == 0.0f && o->lambda_high == 0.0f) return 0;
  for (int l = 0; l < net->n_hidden; ++l)
    if (net->monitor[l]) return 1;
  return 0;
}

int orc_forward_backward(const orc_net* net, const float* params,
                         const uint8_t* packed, size_t B, size_t T,
                         const int64_t* targets, float* loss_out,
                         double* acc_out, float* grads, uint8_t* spikes_out,
                         float* vtrace_out, float* trace_out) {
  return orc_forward_backward_ex(net, NULL, params, packed, B, T, targets, loss_out,
                                 acc_out, grads, spikes_out, vtrace_out, trace_out);
}

static int fb_impl(const orc_net* net, const orc_train_opts* opts,
                   const float* params, const uint8_t* packed, size_t B,
                   size_t T, const int64_t* targets, float* loss_out,
                   double* acc_out, float* grads, uint8_t* spikes_out,
                   float* vtrace_out, float* trace_out, const uint8_t* forced);

int orc_forward_backward_ex(const orc_net* net, const orc_train_opts* opts,
                            const float* params, const uint8_t* packed, size_t B,
                            size_t T, const int64_t* targets, float* loss_out,
                            double* acc_out, float* grads, uint8_t* spikes_out,
                            float* vtrace_out, float* trace_out) {
  return fb_impl(net, opts, params, packed, B, T, targets, loss_out, acc_out, grads,
                 spikes_out, vtrace_out, trace_out, NULL);
}

int orc_forward_backward_forced(const orc_net* net, const orc_train_opts* opts,
                                const float* params, const uint8_t* packed, size_t B,
                                size_t T, const int64_t* targets, const uint8_t* forced,
                                float* loss_out, double* acc_out, float* grads,
                                uint8_t* spikes_out, float* vtrace_out, float* trace_out) {
  return fb_impl(net, opts, params, packed, B, T, targets, loss_out, acc_out, grads,
                 spikes_out, vtrace_out, trace_out, forced);
}

static int fb_impl(const orc_net* net, const orc_train_opts* opts,
                   const float* params, const uint8_t* packed, size_t B,
                   size_t T, const int64_t* targets, float* loss_out,
                   double* acc_out, float* grads, uint8_t* spikes_out,
                   float* vtrace_out, float* trace_out, const uint8_t* forced) {
  if (!opts) opts = &k_default_opts;
  if (opts->loss == 1 && (opts->rate_hi < 0.0f || opts->rate_hi > 1.0f ||
                          opts->rate_lo < 0.0f || opts->rate_lo > 1.0f))
    return 3; /* spike_rate_mse: rates must lie in [0,1] (objective.hpp:144-145) */
  const int reg = reg_active(net, opts);
  if (reg && (opts->f_min > opts->f_max || opts->f_min < 0.0f || opts->f_max > 1.0f))
    return 3; /* activity_regularizer: need 0 <= f_min <= f_max <= 1 (objective.hpp:191-192) */
  const int L = net->n_hidden;
  const size_t C = (size_t)net->classes;
  if (B == 0 || T == 0 || L < 1 || L > ORC_MAX_HIDDEN || net->unroll < 1)
    return 1;
  for (size_t b = 0; b < B; ++b)
    if (targets[b] < 0 || (size_t)targets[b] >= C) return 2;
  layer_off lo[ORC_MAX_HIDDEN + 1];
  layer_offsets(net, lo);
  const float theta = net->threshold;
  const size_t M = B * T; /* rows (b,t), b-major */

  /* activations a[l] = input of layer l as float rows [M, in_l] */
  float* act[ORC_MAX_HIDDEN + 1];
  float* vst[ORC_MAX_HIDDEN]; /* membrane entering step t, [B,T,H] */
  float* ast[ORC_MAX_HIDDEN] = {0}; /* ALIF: adaptation entering step t, [B,T,H] */
  {
    const size_t in = (size_t)net->in;
    uint8_t* xb = (uint8_t*)malloc(M * in);
    act[0] = (float*)malloc(M * in * sizeof(float));
    orc_unpack_time(packed, B, T, in, xb);
    for (size_t i = 0; i < M * in; ++i) act[0][i] = xb[i] ? 1.0f : 0.0f;
    free(xb);
  }
  size_t sp_off = 0;
  for (int l = 0; l < L; ++l) {
    const size_t K = (size_t)layer_in(net, l), H = (size_t)net->hidden[l];
    float* cur = (float*)malloc(M * H * sizeof(float));
    matmul_rows(act[l], M, K, params + lo[l].w, H,
                net->bias ? params + lo[l].b : NULL, cur);
    act[l + 1] = (float*)malloc(M * H * sizeof(float));
    vst[l] = (float*)malloc(M * H * sizeof(float));
    const float* beta = params + lo[l].beta;
    const size_t bs = net->beta_mode[l] == 0 ? 1 : 0; /* scalar beta broadcasts */
    if (is_rlif(net, l)) {
      /* declared RLIF (spiketrain_oracle.h): every neuron's spike of step t first,
       * then fb_j = sum_i s_i rec[i][j] over spiking i ascending (a zero-skip
       * matmul row, ops.hpp:163-172), v' = (((v bc) + I) + fb) - s theta */
      const float* rec = params + lo[l].gamma;
#pragma omp parallel num_threads(g_threads)
      {
      float* vv = (float*)malloc(H * sizeof(float));
      float* fb = (float*)malloc(H * sizeof(float));
#pragma omp for schedule(static)
      for (size_t b = 0; b < B; ++b) {
        for (size_t n = 0; n < H; ++n) vv[n] = 0.0f;
        for (size_t t = 0; t < T; ++t) {
          const size_t row = (b * T + t) * H;
          for (size_t n = 0; n < H; ++n) {
            vst[l][row + n] = vv[n];
            const float pre = vv[n] + (-theta);
            act[l + 1][row + n] = (forced ? forced[sp_off + row + n] != 0 : pre >= 0.0f) ? 1.0f : 0.0f;
            fb[n] = 0.0f;
          }
          for (size_t i = 0; i < H; ++i) {
            if (act[l + 1][row + i] == 0.0f) continue;
            const float* ri = rec + i * H;
            for (size_t j = 0; j < H; ++j) fb[j] += ri[j];
          }
          for (size_t n = 0; n < H; ++n) {
            const float vb = clip01(beta[n * bs]);
            const float m = vv[n] * vb;
            const float ai = m + cur[row + n];
            const float af = ai + fb[n];
            const float r = act[l + 1][row + n] * theta;
            vv[n] = af - r;
          }
        }
      }
      free(vv);
      free(fb);
      }
    } else if (is_alif(net, l)) {
      /* declared ALIF (spiketrain_oracle.h): threshold theta + a, reset by it */
      const float* gam = params + lo[l].gamma;
      ast[l] = (float*)malloc(M * H * sizeof(float));
#pragma omp parallel for schedule(static) num_threads(g_threads)
      for (size_t b = 0; b < B; ++b)
        for (size_t n = 0; n < H; ++n) {
          const float vb = clip01(beta[n * bs]);
          const float gc = clip01(gam[n]);
          const float omg = 1.0f - gc;
          float v = 0.0f, a = 0.0f;
          for (size_t t = 0; t < T; ++t) {
            const size_t idx = (b * T + t) * H + n;
            vst[l][idx] = v;
            ast[l][idx] = a;
            const float th = theta + a;
            const float pre = v - th;
            const float s = (forced ? forced[sp_off + idx] != 0 : pre >= 0.0f) ? 1.0f : 0.0f;
            const float m = v * vb;
            const float ai = m + cur[idx];
            const float r = s * th;
            v = ai - r;
            const float ma = a * gc;
            const float sa = omg * s;
            a = ma + sa;
            act[l + 1][idx] = s;
          }
        }
    } else
    /* lif_step_taped (neuron.hpp:127-136), per timestep */
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (size_t b = 0; b < B; ++b)
      for (size_t n = 0; n < H; ++n) {
        const float vb = clip01(beta[n * bs]);
        float v = 0.0f;
        for (size_t t = 0; t < T; ++t) {
          const size_t idx = (b * T + t) * H + n;
          vst[l][idx] = v;
          const float pre = v + (-theta);
          const float s = (forced ? forced[sp_off + idx] != 0 : pre >= 0.0f) ? 1.0f : 0.0f;
          const float m = v * vb;
          const float a = m + cur[idx];
          const float r = s * theta;
          v = a - r;
          act[l + 1][idx] = s;
        }
      }
    if (spikes_out)
      for (size_t i = 0; i < M * H; ++i)
        spikes_out[sp_off + i] = act[l + 1][i] != 0.0f;
    if (vtrace_out) memcpy(vtrace_out + sp_off, vst[l], M * H * sizeof(float));
    sp_off += M * H;
    free(cur);
  }
  /* readout Linear + LI (neuron.hpp:139-144) */
  const size_t HL = (size_t)net->hidden[L - 1];
  float* i3 = (float*)malloc(M * C * sizeof(float));
  matmul_rows(act[L], M, HL, params + lo[L].w, C,
              net->bias ? params + lo[L].b : NULL, i3);
  float* trace = (float*)malloc(M * C * sizeof(float));
  float* v3 = (float*)malloc(M * C * sizeof(float));
  {
    const float* beta = params + lo[L].beta;
    const size_t bs = net->beta_mode[L] == 0 ? 1 : 0;
    for (size_t b = 0; b < B; ++b)
      for (size_t c = 0; c < C; ++c) {
        const float vb = clip01(beta[c * bs]);
        float v = 0.0f;
        for (size_t t = 0; t < T; ++t) {
          const size_t idx = (b * T + t) * C + c;
          v3[idx] = v;
          if (net->readout_lif) {
            /* LIF readout (neuron.hpp:127-136): the trace is its spikes (network.hpp:396) */
            const float pre = v + (-theta);
            const float s = pre >= 0.0f ? 1.0f : 0.0f;
            v = (v * vb + i3[idx]) - s * theta;
            trace[idx] = s;
          } else {
            v = v * vb + i3[idx];
            trace[idx] = v;
          }
        }
      }
  }
  if (trace_out) memcpy(trace_out, trace, M * C * sizeof(float));

  /* integral CE (objective.hpp:40-73, :88-114) and accuracy (:118-134) */
  float* logits = (float*)calloc(B * C, sizeof(float));
  float* probs = (float*)malloc(B * C * sizeof(float));
  for (size_t b = 0; b < B; ++b)
    for (size_t t = 0; t < T; ++t)
      for (size_t c = 0; c < C; ++c)
        logits[b * C + c] += trace[(b * T + t) * C + c];
  float loss = 0.0f;
  size_t hits = 0;
  for (size_t b = 0; b < B; ++b) {
    const float* row = logits + b * C;
    float m = row[0];
    for (size_t j = 1; j < C; ++j) m = (m < row[j]) ? row[j] : m;
    float z = 0.0f;
    for (size_t j = 0; j < C; ++j) z += expf(row[j] - m);
    const float lse = m + logf(z);
    if (opts->loss == 0) loss += lse - row[(size_t)targets[b]];
    for (size_t j = 0; j < C; ++j) probs[b * C + j] = expf(row[j] - m) / z;
    size_t best = 0;
    for (size_t j = 1; j < C; ++j)
      if (row[j] > row[best]) best = j;
    if (best == (size_t)targets[b]) ++hits;
  }
  if (opts->loss == 1) {
    /* spike_rate_mse (objective.hpp:139-158): one running sum over (b, j) */
    for (size_t b = 0; b < B; ++b)
      for (size_t j = 0; j < C; ++j) {
        const float r = logits[b * C + j] / (float)T;
        const float target = (size_t)targets[b] == j ? opts->rate_hi : opts->rate_lo;
        const float d = r - target;
        loss += d * d;
      }
    *loss_out = loss / (float)(B * C);
  } else {
    *loss_out = loss / (float)B;
  }
  /* loss = add(loss, activity_regularizer(monitor)) per monitor in layer order
   * (optimize.hpp:185-191) */
  float* dcount[ORC_MAX_HIDDEN] = {0};
  if (reg)
    for (int l = 0; l < L; ++l) {
      if (!net->monitor[l]) continue;
      const size_t H = (size_t)net->hidden[l];
      dcount[l] = (float*)malloc(B * H * sizeof(float));
      *loss_out = *loss_out + activity_reg(opts, act[l + 1], B, T, H, dcount[l]);
    }
  *acc_out = (double)hits / (double)B;

  if (grads) {
    memset(grads, 0, orc_param_count(net) * sizeof(float));
    const size_t U = (size_t)net->unroll;
    const size_t nblk = (T + U - 1) / U;
    float* delta = (float*)malloc(B * C * sizeof(float));
    if (opts->loss == 1) {
      /* rate-MSE backward (objective.hpp:170-181): gs*(r - target) on every step */
      const float gs = 1.0f * 2.0f / ((float)(B * C) * (float)T);
      for (size_t b = 0; b < B; ++b)
        for (size_t c = 0; c < C; ++c) {
          const float r = logits[b * C + c] / (float)T;
          const float target = (size_t)targets[b] == c ? opts->rate_hi : opts->rate_lo;
          delta[b * C + c] = gs * (r - target);
        }
    } else {
      /* CE backward: d = (p - onehot) * (1/B) on every timestep. */
      const float gs = 1.0f / (float)B;
      for (size_t b = 0; b < B; ++b)
        for (size_t c = 0; c < C; ++c) {
          float d = probs[b * C + c];
          if ((size_t)targets[b] == c) d -= 1.0f;
          d *= gs;
          delta[b * C + c] = d;
        }
    }
    /* LI reverse scan: Gout_t = delta + Gout_{t+1}*bc; dI = Gout. */
    float* dI = (float*)malloc(M * C * sizeof(float));
    {
      const float* beta = params + lo[L].beta;
      float* gbeta = grads + lo[L].beta;
      const int mode = net->beta_mode[L];
      const size_t bs = mode == 0 ? 1 : 0;
      float* gvb = (float*)malloc(C * sizeof(float));
      for (size_t b = 0; b < B; ++b)
        for (size_t c = 0; c < C; ++c) {
          const float vb = clip01(beta[c * bs]);
          float G = 0.0f;
          for (size_t t = T; t-- > 0;) {
            const size_t idx = (b * T + t) * C + c;
            if (net->readout_lif) {
              /* LIF reverse (the hidden layers' closure order) with dS_t = delta:
               * dI_t = G ; G = G bc + (delta + (-G) theta) g(V_t - theta) */
              dI[idx] = G;
              const float gsp = delta[b * C + c] + (-G) * theta;
              const float gpre = gsp * surrogate(net, v3[idx] + (-theta));
              G = G * vb + gpre;
            } else {
              G = (t == T - 1) ? delta[b * C + c] : delta[b * C + c] + G * vb;
              dI[idx] = G;
            }
          }
        }
      /* d(clip01(beta)) per step, summed over b; beta grad in reverse t. */
      /* (mul_bcast backward, autodiff.hpp:191-205: pg[i % inner] += g*a in
       * row-major order -- a scalar beta sums every (b, c) of the step) */
      for (size_t t = T; t-- > 0 && mode != 2;) {
        for (size_t c = 0; c < C; ++c) gvb[c] = 0.0f;
        for (size_t b = 0; b < B; ++b)
          for (size_t c = 0; c < C; ++c) {
            const size_t idx = (b * T + t) * C + c;
            gvb[c * bs] += dI[idx] * v3[idx];
          }
        for (size_t c = 0; c < (bs ? C : 1); ++c)
          if (beta[c] > 0.0f && beta[c] < 1.0f) gbeta[c] += gvb[c];
      }
      free(gvb);
    }
    /* Linear layers top-down; each is per unroll block, blocks in reverse. */
    float* g_out = dI; /* grad of layer-l Linear output, [M, out_l] */
    for (int l = L; l >= 0; --l) {
      const size_t K = (size_t)layer_in(net, l), N = (size_t)layer_out(net, l);
      const float* W = params + lo[l].w;
      const float* A = act[l];
      float* gW = grads + lo[l].w;
      float* D = (float*)malloc(K * N * sizeof(float));
      float* db = (float*)malloc(N * sizeof(float));
      for (size_t blk = nblk; blk-- > 0;) {
        const size_t t0 = blk * U, t1 = t0 + U < T ? t0 + U : T;
        /* matmul_tn over block rows (b, s) ascending (ops.hpp:203-222) */
        memset(D, 0, K * N * sizeof(float));
        memset(db, 0, N * sizeof(float));
        /* threads own disjoint row ranges of D; each element still sums the
         * block's rows (b, t) in ascending order */
        {
          const size_t nth = (size_t)g_threads < K ? (size_t)g_threads : K;
#pragma omp parallel for schedule(static, 1) num_threads(g_threads)
          for (size_t th = 0; th < nth; ++th) {
            const size_t k0 = K * th / nth, k1 = K * (th + 1) / nth;
            for (size_t b = 0; b < B; ++b)
              for (size_t t = t0; t < t1; ++t) {
                const size_t r = b * T + t;
                const float* ar = A + r * K;
                const float* gr = g_out + r * N;
                for (size_t kk = k0; kk < k1; ++kk) {
                  const float av = ar[kk];
                  if (av == 0.0f) continue;
                  float* o = D + kk * N;
                  for (size_t j = 0; j < N; ++j) o[j] += av * gr[j];
                }
              }
          }
        }
        if (net->bias)
          for (size_t b = 0; b < B; ++b)
            for (size_t t = t0; t < t1; ++t) {
              const float* gr = g_out + (b * T + t) * N;
              for (size_t j = 0; j < N; ++j) db[j] += gr[j];
            }
        for (size_t i = 0; i < K * N; ++i) gW[i] += D[i];
        if (net->bias)
          for (size_t j = 0; j < N; ++j) grads[lo[l].b + j] += db[j];
      }
      free(D);
      free(db);
      if (l == 0) break;
      /* dS = matmul_nt(g, W) (ops.hpp:178-199), then the LIF reverse scan. */
      const size_t H = K;
      float* dS = (float*)malloc(M * H * sizeof(float));
#pragma omp parallel for schedule(static) num_threads(g_threads)
      for (size_t r = 0; r < M; ++r) {
        const float* gr = g_out + r * N;
        for (size_t kk = 0; kk < H; ++kk) {
          const float* wr = W + kk * N;
          float accv = 0.0f;
          for (size_t j = 0; j < N; ++j) accv += gr[j] * wr[j];
          dS[r * H + kk] = accv;
        }
      }
      const int hl = l - 1; /* hidden layer whose spikes fed Linear l */
      if (dcount[hl]) /* the monitor's sum_axis1 adds d loss / d count on every step */
        for (size_t b = 0; b < B; ++b)
          for (size_t t = 0; t < T; ++t)
            for (size_t kk = 0; kk < H; ++kk) dS[(b * T + t) * H + kk] += dcount[hl][b * H + kk];
      const float* beta = params + lo[hl].beta;
      float* gbeta = grads + lo[hl].beta;
      const int mode = net->beta_mode[hl];
      const size_t bs = mode == 0 ? 1 : 0;
      const float* V = vst[hl];
      float* dIh = (float*)malloc(M * H * sizeof(float));
      if (is_rlif(net, hl)) {
        /* declared RLIF reverse, per sample, t descending (G = d/dv_{t+1}):
         *   dI_t = G ; rc_i = sum_j rec[i][j] G_j (j ascending)
         *   gs = (dS + (-G) theta) + rc ; G' = G bc + gs g(v_t - theta)
         *   drec[i][j] += s_i(t) G_j (b, t ascending after the sweep: the
         *   spikes x dI product of the layer with itself, like matmul_tn) */
        const float* rec = params + lo[hl].gamma;
        float* grec = grads + lo[hl].gamma;
        const float* Sx = act[hl + 1];
#pragma omp parallel num_threads(g_threads)
        {
        float* G = (float*)malloc(H * sizeof(float));
        float* G2 = (float*)malloc(H * sizeof(float));
#pragma omp for schedule(static)
        for (size_t b = 0; b < B; ++b) {
          for (size_t n = 0; n < H; ++n) G[n] = 0.0f;
          for (size_t t = T; t-- > 0;) {
            const size_t row = (b * T + t) * H;
            for (size_t i = 0; i < H; ++i) {
              dIh[row + i] = G[i];
              const float* ri = rec + i * H;
              float rc = 0.0f;
              for (size_t j = 0; j < H; ++j) rc += ri[j] * G[j];
              const float vb = clip01(beta[i * bs]);
              const float gs = (dS[row + i] + (-G[i]) * theta) + rc;
              const float pre = V[row + i] + (-theta);
              G2[i] = G[i] * vb + gs * surrogate(net, pre);
            }
            for (size_t i = 0; i < H; ++i) G[i] = G2[i];
          }
        }
        free(G);
        free(G2);
        }
        /* rows of drec split across threads, each summing r ascending */
#pragma omp parallel for schedule(static) num_threads(g_threads)
        for (size_t i = 0; i < H; ++i) {
          float* o = grec + i * H;
          for (size_t r = 0; r < M; ++r) {
            if (Sx[r * H + i] == 0.0f) continue;
            const float* gr = dIh + r * H;
            for (size_t j = 0; j < H; ++j) o[j] += gr[j];
          }
        }
      } else if (is_alif(net, hl)) {
        /* declared ALIF reverse: gv = d/dv_{t+1}, ga = d/da_{t+1}, t descending.
         *   dI_t = gv ; gs = (dS + (-gv) th) + ga (1 - gc) ; gp = gs g(pre)
         *   gv' = gv bc + gp ; ga' = ((ga gc) - gp) - s gv
         *   dgamma += ga (a_t - s) (clip mask), per neuron over (b, t) in b-major,
         *   t-descending order; dbeta from dI and V below, exactly as for LIF. */
        const float* gam = params + lo[hl].gamma;
        float* ggam = grads + lo[hl].gamma;
        const float* Av = ast[hl];
        float* sg = (float*)calloc(H, sizeof(float));
        const float* Sx = act[hl + 1];
#pragma omp parallel for schedule(static) num_threads(g_threads)
        for (size_t n = 0; n < H; ++n)
          for (size_t b = 0; b < B; ++b) {
            const float vb = clip01(beta[n * bs]);
            const float gc = clip01(gam[n]);
            const float omg = 1.0f - gc;
            float gv = 0.0f, ga = 0.0f;
            for (size_t t = T; t-- > 0;) {
              const size_t idx = (b * T + t) * H + n;
              dIh[idx] = gv;
              const float th = theta + Av[idx];
              const float pre = V[idx] - th;
              const float s = Sx[idx];  /* = [pre >= 0] unless teacher-forced */
              const float gs = (dS[idx] + (-gv) * th) + ga * omg;
              const float gp = gs * surrogate(net, pre);
              sg[n] += ga * (Av[idx] - s);
              const float ngv = gv * vb + gp;
              ga = (ga * gc - gp) - s * gv;
              gv = ngv;
            }
          }
        for (size_t n = 0; n < H; ++n)
          if (gam[n] > 0.0f && gam[n] < 1.0f) ggam[n] += sg[n];
        free(sg);
      } else {
#pragma omp parallel for schedule(static) num_threads(g_threads)
      for (size_t b = 0; b < B; ++b)
        for (size_t n = 0; n < H; ++n) {
          const float vb = clip01(beta[n * bs]);
          float G = 0.0f; /* grad of v_{t+1} */
          for (size_t t = T; t-- > 0;) {
            const size_t idx = (b * T + t) * H + n;
            dIh[idx] = G;
            const float rg = -G;              /* sub: pg[1] -= g     */
            const float gsp = dS[idx] + rg * theta; /* stack, then scale */
            const float pre = V[idx] + (-theta);
            const float gpre = gsp * surrogate(net, pre);
            G = G * vb + gpre;                /* mul_bcast, add_scalar */
          }
        }
      }
      {
        float* gvb = (float*)malloc(H * sizeof(float));
        for (size_t t = T - 1; t-- > 0 && mode != 2;) {
          for (size_t n = 0; n < H; ++n) gvb[n] = 0.0f;
          for (size_t b = 0; b < B; ++b)
            for (size_t n = 0; n < H; ++n) {
              const size_t idx = (b * T + t) * H + n;
              gvb[n * bs] += dIh[idx] * V[idx];
            }
          for (size_t n = 0; n < (bs ? H : 1); ++n)
            if (beta[n] > 0.0f && beta[n] < 1.0f) gbeta[n] += gvb[n];
        }
        free(gvb);
      }
      free(dS);
      free(g_out);
      g_out = dIh;
    }
    free(g_out);
    free(delta);
  }

  for (int l = 0; l <= L; ++l) free(act[l]);
  for (int l = 0; l < L; ++l) free(vst[l]);
  for (int l = 0; l < L; ++l) free(ast[l]);
  for (int l = 0; l < L; ++l) free(dcount[l]);
  free(i3);
  free(trace);
  free(v3);
  free(logits);
  free(probs);
  return 0;
}

/* adam_update (optimize.hpp:86-111). */
void orc_adam(float* p, const float* g, float* m, float* v, size_t n,
              uint64_t* step, float lr, float beta1, float beta2, float eps) {
  *step += 1;
  const float bc1 = 1.0f - powf(beta1, (float)*step);
  const float bc2 = 1.0f - powf(beta2, (float)*step);
  for (size_t k = 0; k < n; ++k) {
    m[k] = beta1 * m[k] + (1.0f - beta1) * g[k];
    v[k] = beta2 * v[k] + (1.0f - beta2) * g[k] * g[k];
    const float mhat = m[k] / bc1;
    const float vhat = v[k] / bc2;
    p[k] -= lr * mhat / (sqrtf(vhat) + eps);
  }
}

/* sgd_update (optimize.hpp:69-84). */
void orc_sgd(float* p, const float* g, float* m, size_t n, uint64_t* step,
             float lr, float momentum) {
  *step += 1;
  for (size_t k = 0; k < n; ++k) {
    m[k] = momentum * m[k] + g[k];
    p[k] -= lr * m[k];
  }
}

int orc_train_step(const orc_net* net, float* params, float* m, float* v,
                   uint64_t* step, const uint8_t* packed, size_t batch,
                   size_t t_steps, const int64_t* targets, float lr,
                   float* loss, double* acc) {
  return orc_train_step_ex(net, NULL, params, m, v, step, packed, batch, t_steps,
                           targets, lr, loss, acc);
}

int orc_train_step_ex(const orc_net* net, const orc_train_opts* opts,
                      float* params, float* m, float* v, uint64_t* step,
                      const uint8_t* packed, size_t batch, size_t t_steps,
                      const int64_t* targets, float lr, float* loss, double* acc) {
  if (!opts) opts = &k_default_opts;
  const size_t np = orc_param_count(net);
  float* g = (float*)malloc(np * sizeof(float));
  const int rc = orc_forward_backward_ex(net, opts, params, packed, batch, t_steps,
                                         targets, loss, acc, g, NULL, NULL, NULL);
  if (rc == 0) {
    if (opts->optimizer == 1) orc_sgd(params, g, m, np, step, lr, opts->momentum);
    else orc_adam(params, g, m, v, np, step, lr, 0.9f, 0.999f, 1e-8f);
  }
  free(g);
  return rc;
}

int orc_train_epochs(const orc_net* net, float* params, float* m, float* v,
                     uint64_t* step, const uint8_t* packed, const int64_t* y,
                     size_t n, size_t t_steps, size_t batch, size_t epochs,
                     uint64_t seed, float lr, double* metrics) {
  return orc_train_epochs_ex(net, NULL, params, m, v, step, packed, y, n, t_steps, batch,
                             epochs, seed, lr, metrics);
}

int orc_train_epochs_ex(const orc_net* net, const orc_train_opts* opts, float* params,
                        float* m, float* v, uint64_t* step, const uint8_t* packed,
                        const int64_t* y, size_t n, size_t t_steps, size_t batch,
                        size_t epochs, uint64_t seed, float lr, double* metrics) {
  if (!opts) opts = &k_default_opts;
  /* train() rejects the batch / packed-time axes by number (optimize.hpp:241-245);
   * max_shift <= 0 never reaches shift_augment (optimize.hpp:276).  With a flat
   * feature axis the only rolls that stay on features are 2 and -1; -2 / -3
   * (which the reference would apply to time / batch) are refused here. */
  if (opts->n_shift_axes < 0 || opts->n_shift_axes > 4) return 4;
  for (int i = 0; i < opts->n_shift_axes; ++i) {
    const int ax = opts->shift_axes[i];
    if (ax == 0 || ax == 1) return 4;
    if (opts->max_shift > 0 && ax != 2 && ax != -1) return 4;
  }
  if (batch == 0 || batch > n) return 1;
  const size_t ex = ((t_steps + 7) / 8) * (size_t)net->in;
  const uint64_t master = orc_key_from_seed(seed);
  uint64_t* perm = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint8_t* bx = (uint8_t*)malloc(batch * ex);
  int64_t* by = (int64_t*)malloc(batch * sizeof(int64_t));
  const size_t nb = n / batch;
  int rc = 0;
  for (size_t e = 0; e < epochs && rc == 0; ++e) {
    const uint64_t ek = orc_key_child(master, 1 + e);
    orc_permutation(orc_key_child(ek, 0), n, perm);
    double ls = 0, as = 0;
    for (size_t bi = 0; bi < nb && rc == 0; ++bi) {
      for (size_t i = 0; i < batch; ++i) {
        const size_t src = (size_t)perm[bi * batch + i];
        memcpy(bx + i * ex, packed + src * ex, ex);
        by[i] = y[src];
      }
      if (opts->max_shift > 0 && opts->n_shift_axes > 0) {
        /* shift_augment (data.hpp:216-227): roll(bx, shifts, axes), every axis the
         * feature axis, out[(k + s) mod in] = in[k] (ops.hpp:423-453) */
        const uint64_t bk = orc_key_child(ek, 1 + bi);
        const uint64_t range = (uint64_t)(2 * (int64_t)opts->max_shift);
        int64_t sh = 0;
        for (int ax = 0; ax < opts->n_shift_axes; ++ax)
          sh += -(int64_t)opts->max_shift + (int64_t)(orc_key_bits(bk, (uint64_t)ax) % range);
        const int64_t in = net->in;
        sh %= in;
        if (sh < 0) sh += in;
        if (sh) {
          uint8_t* row = (uint8_t*)malloc((size_t)in);
          for (size_t r = 0; r < batch * ((t_steps + 7) / 8); ++r) {
            uint8_t* p = bx + r * (size_t)in;
            for (int64_t k = 0; k < in; ++k) row[(k + sh) % in] = p[k];
            memcpy(p, row, (size_t)in);
          }
          free(row);
        }
      }
      float l;
      double a;
      rc = orc_train_step_ex(net, opts, params, m, v, step, bx, batch, t_steps, by, lr,
                             &l, &a);
      ls += (double)l;
      as += a;
    }
    if (metrics) {
      metrics[2 * e] = ls / (double)(nb ? nb : 1);
      metrics[2 * e + 1] = as / (double)(nb ? nb : 1);
    }
  }
  free(perm);
  free(bx);
  free(by);
  return rc;
}
