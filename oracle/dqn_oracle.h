/* dqn_oracle.h — fp64 CPU oracle for the distributed deep Q-learning hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library. The
 * product path (paper_1508_04186_b200/, libdqn.so) never links, imports or calls
 * it, and this file shares no code, header, table or constant with the CUDA path.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n (arXiv 1508.04186 text),
 * S:n = SPEC.md line n. Readings of ambiguous passages are the A-numbers of
 * DESIGN.md §3 (== SURVEY.md §8(c)).
 *
 * Everything is plain double precision with naive loops, written in the order
 * the paper states the algorithm; no blocking, fusion or reordering.
 */
#ifndef DQN_ORACLE_H
#define DQN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t frames, height, width;                 /* F, d, d of the phi stack */
  int32_t n_conv;                                /* conv layers, ReLU after each */
  int32_t conv_filters[4], conv_kernel[4], conv_stride[4];
  int32_t n_fc;                                  /* hidden FC layers, ReLU after each */
  int32_t fc_units[4];
  int32_t n_actions;                             /* |A|: one linear output per action */
} or_net;

typedef struct {
  int32_t n_replicas;      /* N workers (Alg. 2 "for all workers k") */
  int32_t minibatch;       /* b (Alg. 1) */
  int32_t n_push, n_fetch; /* Downpour push / fetch periods (A8, A9) */
  int64_t target_sync;     /* C; refresh after a fetch when n - l >= C (A10) */
  double gamma;
  double lr;               /* alpha, Alg. 2 */
  double rms_decay;        /* 0.9 in Alg. 2 */
  double rms_eps;          /* inside the root (A4) */
  double err_clip;         /* 0 = off (A3) */
  uint64_t seed;           /* sampler key (A11) */
  int32_t fetch_lag;       /* 0: synchronous; L > 0: a fetch returns theta as it was L rounds ago (O13, A32) */
  int32_t server_rule;     /* 0: mean of the round's N gradients, one RMSProp, n += 1 (A7);
                              1: Alg. 2 literally - each worker's gradient applied in turn (rank order),
                              one RMSProp and n += 1 per gradient (A33) */
  const int64_t* fetch_gen;  /* NULL, or the generation every fetch returns, [N][ceil(steps / n_fetch)] (fetch f
                                of replica k is at step f * n_fetch): the realised schedule of an asynchronous
                                run (O13, A40). Each entry must be a published generation, n - 7 <= m <= n */
} or_train_cfg;

/* ---- shapes (O0) ---- */
int64_t or_param_count(const or_net* net);                 /* -1 on an invalid chain */
/* Per-tensor [offset, count] in the canonical flat order: for each layer W then b. */
int32_t or_tensor_table(const or_net* net, int64_t* offsets, int64_t* counts, int32_t cap);

/* ---- sampler (O3) ---- */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
int64_t or_sample_index(uint64_t seed, uint32_t rank, uint64_t T, uint32_t j, int64_t size);

/* ---- layers (O5) ---- */
void or_conv_forward(const double* in, int C, int H, int W, const double* w, const double* b, int N, int k,
                     int s, double* out /* N x H' x W' pre-activation */);
void or_fc_forward(const double* in, int D, const double* w, const double* b, int H, double* out);

/* ---- network (O4, O5) ---- */
void or_forward(const or_net* net, const double* theta, const double* x, double* q);
void or_forward_u8(const or_net* net, const double* theta, const uint8_t* s, double* q);
/* Q for n u8 states plus argmax (lowest index on ties, P:37 / A20). */
void or_q_values(const or_net* net, const double* theta, int64_t n, const uint8_t* states, double* q,
                 int32_t* argmax);

/* Smallest |pre-activation| of any ReLU unit over n states (parity diagnostic, A30). */
double or_min_abs_preact(const or_net* net, const double* theta, int64_t n, const uint8_t* states);

/* ---- Alg. 1 pieces (O6, O7) ---- */
/* y_j: terminal -> r_j, else r_j + gamma * max_a' Q(phi_{j+1}, a'; theta_hat). */
void or_targets(const or_net* net, const double* theta_hat, int b, const uint8_t* s_next, const double* r,
                const uint8_t* term, double gamma, double* y, int32_t* argmax_next);
/* Delta theta = (1/b) sum grad 1/2 (Q(phi_j,a_j;theta) - y_j)^2. grad is OVERWRITTEN.
 * Returns the unclipped loss (1/b) sum 1/2 delta^2 (A27). */
double or_loss_grad(const or_net* net, const double* theta, int b, const uint8_t* s, const int32_t* a,
                    const double* y, double err_clip, double* grad);
/* Same with states already normalised to doubles (used by the finite-difference pins). */
double or_loss_grad_x(const or_net* net, const double* theta, int b, const double* x, const int32_t* a,
                      const double* y, double err_clip, double* grad);

/* ---- Alg. 2 RMSPropUpdate (O9) ---- */
void or_rmsprop(double* theta, double* r, const double* g, int64_t P, double alpha, double rho, double eps);

/* ---- replay + whole schedule (O2, O8-O12) ---- */
/* Replica k's pushes: n_pushed[k] transitions given in push order (oldest first).
 * s/s_next: [n][F*H*W] u8, a int32, r double, term u8.  capacity: last-N.
 * theta0: P doubles (canonical). Runs `steps` lock-step replica steps starting at
 * replica step T = 0. Outputs (each may be NULL):
 *   theta_out[P]  server theta after the run      r_out[P]  RMSProp accumulator
 *   n_out         server generation n             loss[N*steps] (A27)
 *   idx[N*steps*b] sampled slots                   amax[N*steps*b] target argmax
 *   grad0[P]      replica-0 gradient of step 0 (before any update)
 * Returns 0, or -2 if some replica has an empty replay (A13), -3 if a push round
 * saw a non-finite mean gradient (A24; those elements are not applied). */
int or_run(const or_net* net, const or_train_cfg* cfg, int64_t capacity, const int64_t* n_pushed,
           const uint8_t* const* s, const int32_t* const* a, const double* const* r,
           const uint8_t* const* s_next, const uint8_t* const* term, const double* theta0, int64_t steps,
           double* theta_out, double* r_out, int64_t* n_out, double* loss, int64_t* idx, int32_t* amax,
           double* grad0, int64_t* stale_hist /* [32]: staleness n_apply - n_local per replica step (A25) */);

/* ---- NEXT-3: the acting side of Alg. 1 on the paper's Snake game (rules
 * closed in SPEC S:216-262, readings A34-A36 in DESIGN.md). Actions 0 up, 1 right, 2 down, 3 left;
 * a reversing action keeps the direction. Cells: empty 0, body 128, head 191, apple 255 (u8 of the
 * SPEC's 0 / 0.5 / 0.75 / 1 render, rounded). Frames are the grid scaled by an integer factor
 * (area averaging of whole cells = replication). Random draws: Philox4x32-10 with key = seed,
 * counter (env, t_lo, t_hi, purpose): purpose 0 the eps-greedy draws (x0 explore, x1 action), 1 the
 * apple after eating, 2 the apple of a reset (the initial reset uses t = 2^64 - 1). */
typedef struct {
  int32_t len, dir, apple, since;   /* body length, direction, apple cell, steps since the last apple */
  int16_t body[1024];               /* cells y*n + x, head first (n*n <= 1024) */
} or_snake;
void or_snake_reset(or_snake* g, int n, uint64_t seed, uint32_t env, uint64_t t);
/* one step; returns the reward, sets *term (wall / self collision -1, grid full or 200*n steps
 * without an apple 0); a terminal step leaves the state unchanged */
double or_snake_step(or_snake* g, int n, int action, uint64_t seed, uint32_t env, uint64_t t, int* term);
void or_snake_render(const or_snake* g, int n, int px, uint8_t* frame /* [n*px][n*px] */);
/* eps-greedy: explore iff x0 < eps_thr (eps_thr = floor(eps * 2^32) in [0, 2^32]); the
 * random action is x1 >> 30 (4 actions); else the given greedy action */
int or_eps_greedy(uint64_t seed, uint32_t env, uint64_t t, uint64_t eps_thr, int greedy);
/* E envs, `steps` acting steps of the collector with the greedy actions given per step
 * (greedy[steps][E], may be NULL when eps_thr = 2^32): stacks [E][F][H][W] in/out (F frames,
 * oldest first; created by the initial reset when init != 0), per-step logs (may be NULL). */
void or_collect(int n, int F, int H, int E, int64_t steps, uint64_t seed, uint64_t eps_thr, const int32_t* greedy,
                int init, or_snake* games, uint8_t* stacks, uint64_t t0, int32_t* a_log, double* r_log,
                uint8_t* t_log, int64_t* episodes);

/* threads of the per-sample loops (OpenMP build; 1 otherwise). The results never depend on it: per-sample
 * gradient terms are summed in sample order (or_loss_grad_x). n <= 0: all host cores. */
int32_t or_threads(void);
void or_set_threads(int32_t n);

#ifdef __cplusplus
}
#endif
#endif
