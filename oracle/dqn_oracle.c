/* dqn_oracle.c — plain, slow, obviously-correct fp64 CPU oracle of the
 * distributed deep Q-learning hot path (arXiv 1508.04186, Alg. 1 + Alg. 2).
 *
 * TEST INFRASTRUCTURE. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. It shares no code with the
 * CUDA path (paper_1508_04186_b200/csrc) and neither side includes the other.
 *
 * Each function cites the passage it follows (P:n = PAPER.md line n, S:n =
 * SPEC.md line n, A-n = reading n of DESIGN.md §3). Pins live in
 * tests/test_oracle_*.py. Every function here is pinned; none is "parity
 * unpinned" except or_run's end-to-end VALUES, which the paper never prints —
 * or_run is pinned by the invariants of DESIGN.md §4 (serial == 1 replica,
 * N replicas == one batch of N*b, sharding-free update, C=1 == plain Q-learning).
 */
#include "dqn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* threads the per-sample loops may use (1 without OpenMP); or_set_threads(n <= 0): all host cores */
int32_t or_threads(void) {
#ifdef _OPENMP
  return (int32_t)omp_get_max_threads();
#else
  return 1;
#endif
}
void or_set_threads(int32_t n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : omp_get_num_procs());
#else
  (void)n;
#endif
}

/* ------------------------------------------------------------------ shapes */
/* Valid convolution, no padding: out = (in - k)/s + 1 must be a positive
 * integer (A16). ReLU after every conv and hidden FC, linear
 * output layer with one unit per action. */
typedef struct {
  int n_layers;          /* conv + fc + output */
  int kind[12];          /* 0 conv, 1 fc (hidden, ReLU), 2 output (linear) */
  int in_c[12], in_h[12], in_w[12];
  int out_c[12], out_h[12], out_w[12];
  int k[12], s[12];
  int64_t w_off[12], b_off[12], w_cnt[12];
  int64_t P;
} shape_t;

static int build_shapes(const or_net* net, shape_t* sh) {
  memset(sh, 0, sizeof(*sh));
  if (net->frames < 1 || net->height < 1 || net->width < 1) return -1;
  if (net->n_conv < 0 || net->n_conv > 4 || net->n_fc < 0 || net->n_fc > 4 || net->n_actions < 1) return -1;
  int c = net->frames, h = net->height, w = net->width;
  int64_t off = 0;
  int L = 0;
  for (int i = 0; i < net->n_conv; ++i, ++L) {
    int n = net->conv_filters[i], k = net->conv_kernel[i], s = net->conv_stride[i];
    if (n < 1 || k < 1 || s < 1 || k > h || k > w) return -1;
    if ((h - k) % s != 0 || (w - k) % s != 0) return -1;
    sh->kind[L] = 0;
    sh->in_c[L] = c; sh->in_h[L] = h; sh->in_w[L] = w;
    sh->k[L] = k; sh->s[L] = s;
    sh->out_c[L] = n; sh->out_h[L] = (h - k) / s + 1; sh->out_w[L] = (w - k) / s + 1;
    sh->w_off[L] = off; sh->w_cnt[L] = (int64_t)n * c * k * k; off += sh->w_cnt[L];
    sh->b_off[L] = off; off += n;
    c = n; h = sh->out_h[L]; w = sh->out_w[L];
  }
  int d = c * h * w; /* flatten in (C,H,W) order (A18) */
  for (int i = 0; i <= net->n_fc; ++i, ++L) {
    int units = (i < net->n_fc) ? net->fc_units[i] : net->n_actions;
    if (units < 1) return -1;
    sh->kind[L] = (i < net->n_fc) ? 1 : 2;
    sh->in_c[L] = d; sh->in_h[L] = 1; sh->in_w[L] = 1;
    sh->out_c[L] = units; sh->out_h[L] = 1; sh->out_w[L] = 1;
    sh->w_off[L] = off; sh->w_cnt[L] = (int64_t)units * d; off += sh->w_cnt[L];
    sh->b_off[L] = off; off += units;
    d = units;
  }
  sh->n_layers = L;
  sh->P = off;
  return 0;
}

int64_t or_param_count(const or_net* net) {
  shape_t sh;
  if (build_shapes(net, &sh)) return -1;
  return sh.P;
}

int32_t or_tensor_table(const or_net* net, int64_t* offsets, int64_t* counts, int32_t cap) {
  shape_t sh;
  if (build_shapes(net, &sh)) return -1;
  int32_t t = 0;
  for (int l = 0; l < sh.n_layers; ++l) {
    if (t + 2 > cap) return -1;
    offsets[t] = sh.w_off[l]; counts[t] = sh.w_cnt[l]; ++t;
    offsets[t] = sh.b_off[l]; counts[t] = sh.out_c[l]; ++t;
  }
  return t;
}

static int64_t act_size(const shape_t* sh, int l) { /* output elements of layer l */
  return (int64_t)sh->out_c[l] * sh->out_h[l] * sh->out_w[l];
}

/* ------------------------------------------------------------------ sampler */
/* Philox4x32-10 (Salmon et al., Random123), the counter-based generator behind
 * "Uniformly sample minibatch of experiences X from D_k" (A11). */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* O3: idx = floor(u * size / 2^64), u = x0 * 2^32 + x1, with replacement. */
int64_t or_sample_index(uint64_t seed, uint32_t rank, uint64_t T, uint32_t j, int64_t size) {
  uint32_t ctr[4] = {j, (uint32_t)T, (uint32_t)(T >> 32), rank};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t x[4];
  or_philox4x32_10(ctr, key, x);
  uint64_t u = ((uint64_t)x[0] << 32) | x[1];
  unsigned __int128 prod = (unsigned __int128)u * (unsigned __int128)(uint64_t)size;
  return (int64_t)(prod >> 64);
}

/* ------------------------------------------------------------------ layers */
/* Each output is the dot product of a k x k x C window with one filter, plus
 * that filter's bias; valid convolution with stride s. */
void or_conv_forward(const double* in, int C, int H, int W, const double* w, const double* b, int N, int k,
                     int s, double* out) {
  int Ho = (H - k) / s + 1, Wo = (W - k) / s + 1;
  for (int n = 0; n < N; ++n)
    for (int oy = 0; oy < Ho; ++oy)
      for (int ox = 0; ox < Wo; ++ox) {
        double acc = b[n];
        for (int c = 0; c < C; ++c)
          for (int ky = 0; ky < k; ++ky)
            for (int kx = 0; kx < k; ++kx)
              acc += w[(((int64_t)n * C + c) * k + ky) * k + kx] *
                     in[((int64_t)c * H + (oy * s + ky)) * W + (ox * s + kx)];
        out[((int64_t)n * Ho + oy) * Wo + ox] = acc;
      }
}

/* output = weights . input + bias. */
void or_fc_forward(const double* in, int D, const double* w, const double* b, int H, double* out) {
  for (int h = 0; h < H; ++h) {
    double acc = b[h];
    for (int d = 0; d < D; ++d) acc += w[(int64_t)h * D + d] * in[d];
    out[h] = acc;
  }
}

static double relu(double x) { return x > 0.0 ? x : 0.0; } /* f(x) = max(0,x) */

/* Forward pass storing every layer's pre-activation z[l] (ReLU applied after
 * every layer except the output). a_l = relu(z_l). */
static void forward_store(const shape_t* sh, const double* theta, const double* x, double** z) {
  const double* a_in = x;
  double* a_tmp = NULL;
  for (int l = 0; l < sh->n_layers; ++l) {
    const double* w = theta + sh->w_off[l];
    const double* bb = theta + sh->b_off[l];
    if (sh->kind[l] == 0)
      or_conv_forward(a_in, sh->in_c[l], sh->in_h[l], sh->in_w[l], w, bb, sh->out_c[l], sh->k[l], sh->s[l], z[l]);
    else
      or_fc_forward(a_in, sh->in_c[l], w, bb, sh->out_c[l], z[l]);
    if (l + 1 < sh->n_layers) {
      int64_t n = act_size(sh, l);
      free(a_tmp);
      a_tmp = (double*)malloc(sizeof(double) * n);
      for (int64_t i = 0; i < n; ++i) a_tmp[i] = relu(z[l][i]);
      a_in = a_tmp;
    }
  }
  free(a_tmp);
}

static double** alloc_acts(const shape_t* sh) {
  double** z = (double**)malloc(sizeof(double*) * sh->n_layers);
  for (int l = 0; l < sh->n_layers; ++l) z[l] = (double*)malloc(sizeof(double) * act_size(sh, l));
  return z;
}
static void free_acts(const shape_t* sh, double** z) {
  for (int l = 0; l < sh->n_layers; ++l) free(z[l]);
  free(z);
}

/* O4: x = u8 / 255 (A15). */
static void normalise(const uint8_t* s, int64_t n, double* x) {
  for (int64_t i = 0; i < n; ++i) x[i] = (double)s[i] / 255.0;
}

void or_forward(const or_net* net, const double* theta, const double* x, double* q) {
  shape_t sh;
  if (build_shapes(net, &sh)) return;
  double** z = alloc_acts(&sh);
  forward_store(&sh, theta, x, z);
  memcpy(q, z[sh.n_layers - 1], sizeof(double) * net->n_actions);
  free_acts(&sh, z);
}

void or_forward_u8(const or_net* net, const double* theta, const uint8_t* s, double* q) {
  int64_t n = (int64_t)net->frames * net->height * net->width;
  double* x = (double*)malloc(sizeof(double) * n);
  normalise(s, n, x);
  or_forward(net, theta, x, q);
  free(x);
}

/* greedy action argmax_a Q, lowest index on ties (A20). */
static int32_t argmax_lowest(const double* q, int n) {
  int32_t best = 0;
  for (int a = 1; a < n; ++a)
    if (q[a] > q[best]) best = a;
  return best;
}

void or_q_values(const or_net* net, const double* theta, int64_t n, const uint8_t* states, double* q,
                 int32_t* argmax) {
  int64_t sz = (int64_t)net->frames * net->height * net->width;
#pragma omp parallel for schedule(static, 1)
  for (int64_t i = 0; i < n; ++i) {
    or_forward_u8(net, theta, states + i * sz, q + i * net->n_actions);
    if (argmax) argmax[i] = argmax_lowest(q + i * net->n_actions, net->n_actions);
  }
}

/* Smallest |pre-activation| of any ReLU unit over n states (diagnostic for the
 * parity tests: ReLU'(z) is a step function, so two correct evaluations of the
 * gradient in different precisions may differ when some |z| is within rounding
 * distance of 0; reading A30). */
double or_min_abs_preact(const or_net* net, const double* theta, int64_t n, const uint8_t* states) {
  shape_t sh;
  if (build_shapes(net, &sh)) return NAN;
  int64_t sz = (int64_t)net->frames * net->height * net->width;
  double* x = (double*)malloc(sizeof(double) * sz);
  double** z = alloc_acts(&sh);
  double m = INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    normalise(states + i * sz, sz, x);
    forward_store(&sh, theta, x, z);
    for (int l = 0; l + 1 < sh.n_layers; ++l)
      for (int64_t e = 0; e < act_size(&sh, l); ++e)
        if (fabs(z[l][e]) < m) m = fabs(z[l][e]);
  }
  free_acts(&sh, z);
  free(x);
  return m;
}

/* ------------------------------------------------------------------ Alg. 1 */
/* "Set y_j = r_j if phi_{j+1} terminal, r_j + gamma max_a' Q^(phi_{j+1}, a'; theta^) otherwise".
 * A select, never (1 - term) * m (A14). */
void or_targets(const or_net* net, const double* theta_hat, int b, const uint8_t* s_next, const double* r,
                const uint8_t* term, double gamma, double* y, int32_t* argmax_next) {
  int64_t sz = (int64_t)net->frames * net->height * net->width;
#pragma omp parallel for schedule(static, 1)
  for (int j = 0; j < b; ++j) {
    double* q = (double*)malloc(sizeof(double) * net->n_actions);
    or_forward_u8(net, theta_hat, s_next + j * sz, q);
    double m = q[0];
    for (int a = 1; a < net->n_actions; ++a)
      if (q[a] > m) m = q[a];
    if (argmax_next) argmax_next[j] = argmax_lowest(q, net->n_actions);
    y[j] = term[j] ? r[j] : r[j] + gamma * m;
    free(q);
  }
}

/* Delta theta = (1/b) sum_i grad_theta 1/2 (Q(phi_i, a_i; theta) - y_i)^2, written as that sum:
 * sample j's term g_j is computed on its own (sample_grad), then the terms are added in the order j = 0..b-1.
 * dL/dQ_{j,a} = clamp(delta_j, -c, c)/b for a = a_j, else 0; y is a constant (A2, A3).
 * Backprop through ReLU with ReLU'(0) = 0 (A17).
 * The per-sample terms of a block of OR_BLOCK samples may be computed by several threads (OpenMP, when the
 * library is built with it); the sum is always taken in sample order, so the result does not depend on the
 * thread count (bench.py's all-core cpu_baseline). */
#define OR_BLOCK 16

static double sample_grad(const shape_t* sh, const or_net* net, const double* theta, const double* xj, int32_t aj,
                          double yj, double err_clip, int b, double* grad /* zeroed, P */) {
  int L = sh->n_layers;
  double** z = alloc_acts(sh);
  double** dz = alloc_acts(sh);
  double* act_in = NULL;
  forward_store(sh, theta, xj, z);
  double q = z[L - 1][aj];
  double delta = q - yj;
  double dclip = delta;
  if (err_clip > 0.0) {
    if (dclip > err_clip) dclip = err_clip;
    if (dclip < -err_clip) dclip = -err_clip;
  }
  /* output layer: only the taken action's unit receives error */
  for (int i = 0; i < net->n_actions; ++i) dz[L - 1][i] = 0.0;
  dz[L - 1][aj] = dclip / (double)b;
  for (int l = L - 1; l >= 0; --l) {
    /* input activation of layer l */
    int64_t n_in = (int64_t)sh->in_c[l] * sh->in_h[l] * sh->in_w[l];
    free(act_in);
    act_in = (double*)malloc(sizeof(double) * n_in);
    if (l == 0) memcpy(act_in, xj, sizeof(double) * n_in);
    else for (int64_t i = 0; i < n_in; ++i) act_in[i] = relu(z[l - 1][i]);
    double* gw = grad + sh->w_off[l];
    double* gb = grad + sh->b_off[l];
    const double* w = theta + sh->w_off[l];
    double* dprev = (l > 0) ? dz[l - 1] : NULL; /* becomes d(pre-activation) of layer l-1 */
    if (dprev) for (int64_t i = 0; i < n_in; ++i) dprev[i] = 0.0;
    if (sh->kind[l] == 0) {
      int C = sh->in_c[l], H = sh->in_h[l], W = sh->in_w[l], N = sh->out_c[l], k = sh->k[l], s = sh->s[l];
      int Ho = sh->out_h[l], Wo = sh->out_w[l];
      for (int n = 0; n < N; ++n)
        for (int oy = 0; oy < Ho; ++oy)
          for (int ox = 0; ox < Wo; ++ox) {
            double g = dz[l][((int64_t)n * Ho + oy) * Wo + ox];
            gb[n] += g;
            for (int c = 0; c < C; ++c)
              for (int ky = 0; ky < k; ++ky)
                for (int kx = 0; kx < k; ++kx) {
                  int64_t wi = (((int64_t)n * C + c) * k + ky) * k + kx;
                  int64_t xi = ((int64_t)c * H + (oy * s + ky)) * W + (ox * s + kx);
                  gw[wi] += g * act_in[xi];
                  if (dprev) dprev[xi] += g * w[wi];
                }
          }
    } else {
      int D = sh->in_c[l], Hh = sh->out_c[l];
      for (int h = 0; h < Hh; ++h) {
        double g = dz[l][h];
        gb[h] += g;
        for (int d = 0; d < D; ++d) {
          gw[(int64_t)h * D + d] += g * act_in[d];
          if (dprev) dprev[d] += g * w[(int64_t)h * D + d];
        }
      }
    }
    /* through the ReLU of layer l-1: d z_{l-1} = d a_{l-1} * [z_{l-1} > 0] */
    if (dprev)
      for (int64_t i = 0; i < n_in; ++i) dprev[i] = (z[l - 1][i] > 0.0) ? dprev[i] : 0.0;
  }
  free(act_in);
  free_acts(sh, z);
  free_acts(sh, dz);
  return 0.5 * delta * delta;
}

double or_loss_grad_x(const or_net* net, const double* theta, int b, const double* x, const int32_t* a,
                      const double* y, double err_clip, double* grad) {
  shape_t sh;
  if (build_shapes(net, &sh)) return NAN;
  memset(grad, 0, sizeof(double) * sh.P);
  int64_t sz = (int64_t)net->frames * net->height * net->width;
  double* gj = (double*)malloc(sizeof(double) * sh.P * OR_BLOCK);
  double lj[OR_BLOCK];
  double loss = 0.0;
  for (int j0 = 0; j0 < b; j0 += OR_BLOCK) {
    const int nb = b - j0 < OR_BLOCK ? b - j0 : OR_BLOCK;
#pragma omp parallel for schedule(static, 1)
    for (int q = 0; q < nb; ++q) {
      memset(gj + (int64_t)q * sh.P, 0, sizeof(double) * sh.P);
      lj[q] = sample_grad(&sh, net, theta, x + (int64_t)(j0 + q) * sz, a[j0 + q], y[j0 + q], err_clip, b,
                          gj + (int64_t)q * sh.P);
    }
    for (int q = 0; q < nb; ++q) { /* sample order */
      loss += lj[q];
      const double* g = gj + (int64_t)q * sh.P;
      for (int64_t i = 0; i < sh.P; ++i) grad[i] += g[i];
    }
  }
  free(gj);
  return loss / (double)b;
}

double or_loss_grad(const or_net* net, const double* theta, int b, const uint8_t* s, const int32_t* a,
                    const double* y, double err_clip, double* grad) {
  int64_t sz = (int64_t)net->frames * net->height * net->width;
  double* x = (double*)malloc(sizeof(double) * sz * (b > 0 ? b : 1));
  normalise(s, sz * b, x);
  double loss = or_loss_grad_x(net, theta, b, x, a, y, err_clip, grad);
  free(x);
  return loss;
}

/* ------------------------------------------------------------------ Alg. 2 */
/* RMSPropUpdate(Delta theta): r_i <- 0.9 r_i + 0.1 (Delta theta)_i^2,
 * then theta_i <- theta_i - alpha (Delta theta)_i / sqrt(r_i), r first (A5),
 * with eps inside the root (A4). rho = 0.9 in the paper. */
void or_rmsprop(double* theta, double* r, const double* g, int64_t P, double alpha, double rho, double eps) {
  for (int64_t i = 0; i < P; ++i) {
    r[i] = rho * r[i] + (1.0 - rho) * g[i] * g[i];
    theta[i] = theta[i] - alpha * g[i] / sqrt(r[i] + eps);
  }
}

/* ------------------------------------------------------------------ schedule */
typedef struct {
  int64_t cap, count;
  int64_t sz;
  uint8_t *s, *sn, *term;
  int32_t* a;
  double* r;
} ring_t;

/* O2: push i goes to slot (count mod cap); keep only the last N tuples. */
static void ring_push(ring_t* R, const uint8_t* s, int32_t a, double r, const uint8_t* sn, uint8_t term) {
  int64_t slot = R->count % R->cap;
  memcpy(R->s + slot * R->sz, s, R->sz);
  memcpy(R->sn + slot * R->sz, sn, R->sz);
  R->a[slot] = a; R->r[slot] = r; R->term[slot] = term;
  R->count += 1;
}

int or_run(const or_net* net, const or_train_cfg* cfg, int64_t capacity, const int64_t* n_pushed,
           const uint8_t* const* s, const int32_t* const* a, const double* const* r,
           const uint8_t* const* s_next, const uint8_t* const* term, const double* theta0, int64_t steps,
           double* theta_out, double* r_out, int64_t* n_out, double* loss, int64_t* idx, int32_t* amax,
           double* grad0, int64_t* stale_hist) {
  shape_t sh;
  if (build_shapes(net, &sh)) return -1;
  const int N = cfg->n_replicas, b = cfg->minibatch;
  const int64_t P = sh.P;
  const int64_t sz = (int64_t)net->frames * net->height * net->width;
  int rc = 0;

  /* replay memories D_k, one per worker */
  ring_t* rings = (ring_t*)calloc(N, sizeof(ring_t));
  for (int k = 0; k < N; ++k) {
    ring_t* R = &rings[k];
    R->cap = capacity; R->count = 0; R->sz = sz;
    R->s = (uint8_t*)malloc(capacity * sz); R->sn = (uint8_t*)malloc(capacity * sz);
    R->term = (uint8_t*)malloc(capacity); R->a = (int32_t*)malloc(capacity * sizeof(int32_t));
    R->r = (double*)malloc(capacity * sizeof(double));
    for (int64_t i = 0; i < n_pushed[k]; ++i)
      ring_push(R, s[k] + i * sz, a[k][i], r[k][i], s_next[k] + i * sz, term[k][i]);
    if (R->count == 0) rc = -2; /* A13 */
  }
  if (rc) goto out_rings;

  /* server state: theta, r <- 0, n <- 0 (Alg. 2) */
  double* theta = (double*)malloc(sizeof(double) * P);
  double* rms = (double*)calloc(P, sizeof(double));
  memcpy(theta, theta0, sizeof(double) * P);
  int64_t n = 0;
  /* per worker: local theta + n_k, target theta^ + l (Alg. 1 state line P:109), gradient accumulator */
  double** th_local = (double**)malloc(sizeof(double*) * N);
  double** th_hat = (double**)malloc(sizeof(double*) * N);
  double** acc = (double**)malloc(sizeof(double*) * N);
  int64_t* n_local = (int64_t*)calloc(N, sizeof(int64_t));
  int64_t* ell = (int64_t*)calloc(N, sizeof(int64_t));
  for (int k = 0; k < N; ++k) {
    th_local[k] = (double*)malloc(sizeof(double) * P);
    th_hat[k] = (double*)malloc(sizeof(double) * P);
    acc[k] = (double*)calloc(P, sizeof(double));
    memcpy(th_local[k], theta0, sizeof(double) * P);
    memcpy(th_hat[k], theta0, sizeof(double) * P); /* theta^ = theta_0, l = 0 */
  }
  double* g = (double*)malloc(sizeof(double) * P);
  double* gbar = (double*)malloc(sizeof(double) * P);
  /* O13: the server's last published states; a fetch returns theta^(max(n - L, 0)), or the generation the
     realised asynchronous schedule gives it (cfg->fetch_gen, A40) */
  const int L = cfg->fetch_lag > 0 ? cfg->fetch_lag : 0;
  const int64_t depth = cfg->fetch_gen ? 8 : L + 1;
  const int64_t n_fetches = (steps + cfg->n_fetch - 1) / cfg->n_fetch;
  double* hist = (double*)malloc(sizeof(double) * P * depth);
  memcpy(hist, theta0, sizeof(double) * P);
  int64_t* pend = (int64_t*)calloc((size_t)N * cfg->n_push, sizeof(int64_t)); /* n_local per step of the round */
  if (stale_hist) memset(stale_hist, 0, sizeof(int64_t) * 32);
  uint8_t* bs = (uint8_t*)malloc(b * sz);
  uint8_t* bsn = (uint8_t*)malloc(b * sz);
  int32_t* ba = (int32_t*)malloc(sizeof(int32_t) * b);
  double* br = (double*)malloc(sizeof(double) * b);
  uint8_t* bt = (uint8_t*)malloc(b);
  double* y = (double*)malloc(sizeof(double) * b);
  int32_t* am = (int32_t*)malloc(sizeof(int32_t) * b);

  for (int64_t T = 0; T < steps; ++T) {
    /* O12: every replica finishes step T before any starts T+1 */
    for (int k = 0; k < N; ++k) {
      /* O10 "Fetch model theta and iteration number n from server", every n_fetch steps (A9) */
      if (T % cfg->n_fetch == 0) {
        int64_t m = n - L > 0 ? n - L : 0; /* L = 0: the current server theta */
        if (cfg->fetch_gen) {
          m = cfg->fetch_gen[(int64_t)k * n_fetches + T / cfg->n_fetch];
          if (m > n || n - m >= depth || m < 0) { rc = -4; goto out_all; } /* not a published generation */
        }
        memcpy(th_local[k], hist + (m % depth) * P, sizeof(double) * P);
        n_local[k] = m;
        /* O11 target refresh every C generations (A10) */
        if (n_local[k] - ell[k] >= cfg->target_sync) {
          memcpy(th_hat[k], th_local[k], sizeof(double) * P);
          ell[k] = n_local[k];
        }
      }
      /* O3 "Uniformly sample minibatch of experiences X from D_k" */
      ring_t* R = &rings[k];
      int64_t size = R->count < R->cap ? R->count : R->cap;
      for (int j = 0; j < b; ++j) {
        int64_t slot = or_sample_index(cfg->seed, (uint32_t)k, (uint64_t)T, (uint32_t)j, size);
        if (idx) idx[((int64_t)k * steps + T) * b + j] = slot;
        memcpy(bs + j * sz, R->s + slot * sz, sz);
        memcpy(bsn + j * sz, R->sn + slot * sz, sz);
        ba[j] = R->a[slot]; br[j] = R->r[slot]; bt[j] = R->term[slot];
      }
      /* O6 targets with theta^ */
      or_targets(net, th_hat[k], b, bsn, br, bt, cfg->gamma, y, am);
      if (amax) memcpy(amax + ((int64_t)k * steps + T) * b, am, sizeof(int32_t) * b);
      /* O7 gradient at the fetched theta */
      double l = or_loss_grad(net, th_local[k], b, bs, ba, y, cfg->err_clip, g);
      if (loss) loss[(int64_t)k * steps + T] = l;
      if (grad0 && T == 0 && k == 0) memcpy(grad0, g, sizeof(double) * P);
      /* O8 accumulate until the push (A8: no local update) */
      for (int64_t i = 0; i < P; ++i) acc[k][i] += g[i];
      pend[(int64_t)k * cfg->n_push + T % cfg->n_push] = n_local[k]; /* generation this gradient used */
    }
    /* O9 server round when the push is due (A7) */
    if ((T + 1) % cfg->n_push == 0 && cfg->server_rule == 1) {
      /* A33: "for all workers k ... RMSPropUpdate(Delta theta_k); n <- n + 1" in rank order, each
         gradient the mean of that worker's n_push accumulated gradients (A8) */
      if (stale_hist)
        for (int64_t e = 0; e < (int64_t)N * cfg->n_push; ++e) {
          const int64_t s = n - pend[e];
          stale_hist[s < 31 ? s : 31] += 1;
        }
      for (int k = 0; k < N; ++k) {
        for (int64_t i = 0; i < P; ++i) {
          gbar[i] = acc[k][i] / (double)cfg->n_push;
          if (!isfinite(gbar[i])) { rc = -3; continue; }
          or_rmsprop(theta + i, rms + i, gbar + i, 1, cfg->lr, cfg->rms_decay, cfg->rms_eps);
        }
        n += 1;
        memcpy(hist + (n % depth) * P, theta, sizeof(double) * P);
      }
      for (int k = 0; k < N; ++k) memset(acc[k], 0, sizeof(double) * P);
    } else if ((T + 1) % cfg->n_push == 0) {
      for (int64_t i = 0; i < P; ++i) {
        double sum = 0.0;
        for (int k = 0; k < N; ++k) sum += acc[k][i]; /* rank order */
        gbar[i] = sum / ((double)N * (double)cfg->n_push);
      }
      /* A24: a non-finite mean-gradient element is not applied (theta_i, r_i kept) and the round is flagged */
      for (int64_t i = 0; i < P; ++i) {
        if (!isfinite(gbar[i])) { rc = -3; continue; }
        or_rmsprop(theta + i, rms + i, gbar + i, 1, cfg->lr, cfg->rms_decay, cfg->rms_eps);
      }
      /* A25: every replica step of this round contributes n - n_local (its theta's generation) */
      if (stale_hist)
        for (int64_t e = 0; e < (int64_t)N * cfg->n_push; ++e) {
          const int64_t s = n - pend[e];
          stale_hist[s < 31 ? s : 31] += 1;
        }
      n += 1; /* A22 */
      memcpy(hist + (n % depth) * P, theta, sizeof(double) * P);
      for (int k = 0; k < N; ++k) memset(acc[k], 0, sizeof(double) * P);
    }
  }
out_all:
  if (theta_out) memcpy(theta_out, theta, sizeof(double) * P);
  if (r_out) memcpy(r_out, rms, sizeof(double) * P);
  if (n_out) *n_out = n;

  free(g); free(gbar); free(bs); free(bsn); free(ba); free(br); free(bt); free(y); free(am);
  free(hist); free(pend);
  for (int k = 0; k < N; ++k) { free(th_local[k]); free(th_hat[k]); free(acc[k]); }
  free(th_local); free(th_hat); free(acc); free(n_local); free(ell);
  free(theta); free(rms);
out_rings:
  for (int k = 0; k < N; ++k) {
    free(rings[k].s); free(rings[k].sn); free(rings[k].term); free(rings[k].a); free(rings[k].r);
  }
  free(rings);
  return rc;
}


/* ======================================================================= NEXT-3 acting (Snake) */
static void snake_draw(uint64_t seed, uint32_t env, uint64_t t, uint32_t purpose, uint32_t out[4]) {
  const uint32_t ctr[4] = {env, (uint32_t)t, (uint32_t)(t >> 32), purpose};
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  or_philox4x32_10(ctr, key, out);
}

/* the k-th free cell (row-major) with k = floor(x * free / 2^32); -1 if the grid is full */
static int snake_place_apple(const or_snake* g, int n, uint32_t x) {
  char occ[1024];
  memset(occ, 0, sizeof(occ));
  for (int i = 0; i < g->len; ++i) occ[g->body[i]] = 1;
  const int free_cells = n * n - g->len;
  if (free_cells <= 0) return -1;
  int k = (int)(((uint64_t)x * (uint64_t)free_cells) >> 32);
  for (int c = 0; c < n * n; ++c)
    if (!occ[c] && k-- == 0) return c;
  return -1;
}

void or_snake_reset(or_snake* g, int n, uint64_t seed, uint32_t env, uint64_t t) {
  const int c = n / 2;
  g->len = 2;               /* "starts with body length of two", horizontal, heading right */
  g->dir = 1;
  g->since = 0;
  g->body[0] = (int16_t)(c * n + c);
  g->body[1] = (int16_t)(c * n + c - 1);
  uint32_t x[4];
  snake_draw(seed, env, t, 2, x);
  g->apple = snake_place_apple(g, n, x[0]);
}

double or_snake_step(or_snake* g, int n, int action, uint64_t seed, uint32_t env, uint64_t t, int* term) {
  *term = 0;
  if ((action + 2) % 4 != g->dir) g->dir = action; /* a reversing action keeps the direction */
  const int hy = g->body[0] / n, hx = g->body[0] % n;
  const int ny = hy + (g->dir == 2) - (g->dir == 0), nx = hx + (g->dir == 1) - (g->dir == 3);
  if (ny < 0 || ny >= n || nx < 0 || nx >= n) { *term = 1; return -1.0; } /* wall: death (SPEC closure) */
  const int nh = ny * n + nx;
  if (nh == g->apple) { /* eat: grow by one, +1, new apple */
    for (int i = g->len; i > 0; --i) g->body[i] = g->body[i - 1];
    g->body[0] = (int16_t)nh;
    g->len += 1;
    g->since = 0;
    uint32_t x[4];
    snake_draw(seed, env, t, 1, x);
    g->apple = snake_place_apple(g, n, x[0]);
    if (g->apple < 0) *term = 1; /* grid full */
    return 1.0;
  }
  for (int i = 0; i < g->len - 1; ++i) /* the tail cell moves away this step */
    if (g->body[i] == nh) { *term = 1; return -1.0; }
  for (int i = g->len - 1; i > 0; --i) g->body[i] = g->body[i - 1];
  g->body[0] = (int16_t)nh;
  g->since += 1;
  if (g->since >= 200 * n) *term = 1; /* step cap without an apple, reward 0 (SPEC) */
  return 0.0;
}

void or_snake_render(const or_snake* g, int n, int px, uint8_t* frame) {
  uint8_t cell[1024];
  memset(cell, 0, sizeof(cell));
  for (int i = 1; i < g->len; ++i) cell[g->body[i]] = 128;
  cell[g->body[0]] = 191;
  if (g->apple >= 0) cell[g->apple] = 255;
  const int d = n * px;
  for (int y = 0; y < d; ++y)
    for (int x = 0; x < d; ++x) frame[y * d + x] = cell[(y / px) * n + (x / px)];
}

int or_eps_greedy(uint64_t seed, uint32_t env, uint64_t t, uint64_t eps_thr, int greedy) {
  uint32_t x[4];
  snake_draw(seed, env, t, 0, x);
  if ((uint64_t)x[0] < eps_thr) return (int)(x[1] >> 30);
  return greedy;
}

void or_collect(int n, int F, int H, int E, int64_t steps, uint64_t seed, uint64_t eps_thr, const int32_t* greedy,
                int init, or_snake* games, uint8_t* stacks, uint64_t t0, int32_t* a_log, double* r_log,
                uint8_t* t_log, int64_t* episodes) {
  const int px = H / n;
  const int64_t fb = (int64_t)H * H;
  uint8_t* frame = (uint8_t*)malloc(fb);
  if (init)
    for (int e = 0; e < E; ++e) { /* episode start: the first frame replicated F times (SPEC) */
      or_snake_reset(&games[e], n, seed, (uint32_t)e, ~0ULL);
      or_snake_render(&games[e], n, px, frame);
      for (int f = 0; f < F; ++f) memcpy(stacks + ((int64_t)e * F + f) * fb, frame, fb);
    }
  for (int64_t s = 0; s < steps; ++s) {
    const uint64_t t = t0 + (uint64_t)s;
    for (int e = 0; e < E; ++e) {
      const int a = or_eps_greedy(seed, (uint32_t)e, t, eps_thr, greedy ? greedy[s * E + e] : 0);
      int term;
      const double r = or_snake_step(&games[e], n, a, seed, (uint32_t)e, t, &term);
      if (a_log) a_log[s * E + e] = a;
      if (r_log) r_log[s * E + e] = r;
      if (t_log) t_log[s * E + e] = (uint8_t)term;
      /* phi_{t+1}: drop the oldest frame, append the new one (Alg. 1 "preprocess", S:push_frame) */
      uint8_t* st = stacks + (int64_t)e * F * fb;
      memmove(st, st + fb, (size_t)((F - 1) * fb));
      or_snake_render(&games[e], n, px, st + (F - 1) * fb);
      if (term) {
        if (episodes) episodes[e] += 1;
        or_snake_reset(&games[e], n, seed, (uint32_t)e, t);
        or_snake_render(&games[e], n, px, frame);
        for (int f = 0; f < F; ++f) memcpy(st + f * fb, frame, fb);
      }
    }
  }
  free(frame);
}
