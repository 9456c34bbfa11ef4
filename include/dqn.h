/* dqn.h — C ABI of the B200-native distributed deep Q-learning hot path.
 *
 * Method: Ong, Chavez, Hong, "Distributed Deep Q-Learning", arXiv 1508.04186.
 * Citation keys: P:n = line n of the paper text,
 * A-n = reading n of the paper listed in DESIGN.md §3.
 *
 * One context per process per GPU ("replica k" of Alg. 1, which also
 * owns shard k of the parameter server of Alg. 2). All device state
 * (replay memory D_k, theta working copy, target theta^, gradient buffer,
 * the owned fp32 master shard of theta and of the RMSProp accumulator r) lives
 * in the context and is freed by dqn_destroy.
 *
 * Conventions for every entry point:
 *  - return value: DQN_OK (0) or a negative DQN_E* status; a failed call that
 *    returns DQN_EINVAL or DQN_EEMPTY has not mutated the context.
 *  - buffers are owned by the caller; pointers may be host or device memory
 *    (detected with cudaPointerGetAttributes); inputs are consumed (copied)
 *    before the call returns; outputs are written before it returns.
 *  - calls are synchronous on return, NOT thread-safe on one context.
 *  - "collective" calls must be made by every rank of the group, in the same
 *    order, with the same arguments where stated.
 *  - after DQN_ECUDA or DQN_ENCCL the context is poisoned: every later call
 *    except dqn_last_error / dqn_destroy returns DQN_ESTATE.
 */
#ifndef DQN_H
#define DQN_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dqn_ctx dqn_ctx;

enum {
  DQN_OK = 0,
  DQN_EINVAL = -1,     /* bad config / argument (validated before any mutation) */
  DQN_EEMPTY = -2,     /* train_steps on an empty replay memory (A13)          */
  DQN_ENONFINITE = -3, /* a push round produced a non-finite mean gradient (A24); sticky */
  DQN_ENOMEM = -4,     /* device allocation failed                                */
  DQN_ECUDA = -5,      /* CUDA runtime error; context poisoned                    */
  DQN_ENCCL = -6,      /* NCCL error; context poisoned                            */
  DQN_ESTATE = -7      /* context poisoned by an earlier ECUDA / ENCCL            */
};

/* arithmetic of the replica step (a3-a9 of DESIGN.md §2) */
enum { DQN_FP32 = 0,   /* fp32 SIMT kernels; parity <= 1e-5 vs the fp64 oracle            */
       DQN_BF16 = 1 }; /* bf16 operands on tcgen05 tensor cores, fp32 accumulate; <= 2e-2 */
/* push / fetch schedule (DESIGN.md §2 a11-a13) */
enum { DQN_DETERMINISTIC = 0, /* lock-step: a fetch returns the current server theta                    */
       DQN_ASYNC = 1,         /* Downpour's asynchrony: the server round (push, RMSProp,
                                 publish) runs on a second stream while the replica keeps stepping; a
                                 fetch never waits - it takes the newest generation the server has
                                 published (a device generation flag), so the staleness n_apply - n_base
                                 is whatever the timing makes it (staleness_hist, step_generation)    */
       DQN_ASYNC_LAG1 = 2 };  /* its deterministic twin (O13 / A32): the same streams, but a fetch returns
                                 exactly the server theta of one round earlier (waits for it)         */
/* how a push round combines the N workers' gradients (Alg. 2)
 *   MEAN         : one RMSProp application of the mean of the N*n_push gradients, n += 1 (A7)
 *   PER_GRADIENT : Alg. 2 literally - each worker's gradient (mean of its n_push) applied in turn
 *                  in rank order, one RMSProp application and n += 1 each (A33). N > 1: the fused
 *                  server round (DQN_DETERMINISTIC, n_fetch = 1), or DQN_ASYNC / DQN_ASYNC_LAG1, where
 *                  the round's all-to-all delivers every worker's slice into the owner's inbox on the
 *                  comm stream (only whole rounds are published: fetched generations are multiples
 *                  of N). DQN_DETERMINISTIC with n_fetch > 1 is rejected. */
enum { DQN_SERVER_MEAN = 0, DQN_SERVER_PER_GRADIENT = 1 };

/* which parameter vector dqn_get_params returns */
enum {
  DQN_PARAMS_SERVER = 0, /* global theta of Alg. 2 (fp32 masters, gathered over ranks: collective) */
  DQN_PARAMS_LOCAL = 1,  /* this replica's fetched theta (Alg. 1 "Fetch model theta")       */
  DQN_PARAMS_TARGET = 2, /* this replica's target theta^                             */
  DQN_PARAMS_GRAD = 3,   /* the gradient this replica pushed in its last push round: sum over its
                            n_push steps of Delta theta (A8), before the mean; needs
                            cfg.keep_grad = 1 (DQN_EINVAL otherwise); diagnostic                   */
  DQN_PARAMS_RMS = 4,    /* RMSProp accumulator r of Alg. 2 (gathered: collective)                 */
  DQN_PARAMS_LOCAL_BF16 = 5,  /* DQN_BF16: the bf16 working copy of theta the tensor cores read,
                                 widened to fp32 (exact); diagnostic (DQN_EINVAL on DQN_FP32)       */
  DQN_PARAMS_TARGET_BF16 = 6  /* DQN_BF16: the bf16 working copy of theta^, widened; diagnostic     */
};

/* Problem statement (P:59-67 network, P:87 C, P:99 N, P:121 gamma, P:123 b,
 * P:142-147 RMSProp + init). Layer list: valid convolutions (no padding,
 * (in-k)/s+1 must be a positive integer, A16), ReLU after every conv and every
 * hidden FC, linear output layer with n_actions units. */
typedef struct {
  int32_t frames, height, width;       /* phi stack F x d x d, u8 pixels          */
  int32_t n_conv;                      /* 1..4                                            */
  int32_t conv_filters[4], conv_kernel[4], conv_stride[4];
  int32_t n_fc;                        /* hidden FC layers 0..4                           */
  int32_t fc_units[4];
  int32_t n_actions;                   /* |A| >= 1                                        */
  int32_t minibatch;                   /* b >= 1 (Alg. 1)                           */
  double gamma;                        /* discount                                */
  double lr;                           /* alpha (Alg. 2)                            */
  double rms_decay;                    /* 0.9 in Alg. 2                           */
  double rms_eps;                      /* epsilon inside the square root (A4), e.g. 1e-8  */
  double err_clip;                     /* 0 = off (Alg. 1); c > 0 clamps delta (A3)       */
  int64_t replay_capacity;             /* last-N experiences kept                  */
  int32_t n_push, n_fetch;             /* Downpour periods (A8, A9), >= 1                 */
  int64_t target_sync;                 /* C: refresh theta^ after a fetch when n-l >= C */
  int32_t precision;                   /* DQN_FP32 | DQN_BF16                             */
  int32_t sync_mode;                   /* DQN_DETERMINISTIC                               */
  uint64_t seed;                       /* key of the counter-based sampler (A11)          */
  double init_std;                     /* xi of theta_i ~ N(0, xi) (A19)           */
  uint64_t init_seed;
  const float* init_params;            /* optional: P floats in canonical order (host or device); copied */
  int32_t server_rule;                 /* DQN_SERVER_MEAN (A7, default) | DQN_SERVER_PER_GRADIENT (A33) */
  int32_t replay_dedup;                /* 1: frame-deduplicated replay (NEXT-4): every pushed s' must be
                                          s shifted by one frame plus a new frame (Atari-style stacks);
                                          a slot stores F+1 frames instead of 2F (DQN_EINVAL otherwise) */
  int32_t keep_grad;                   /* 1: the kernels that consume this replica's pushed gradient (the
                                          update / server round, or the acquire that clears it) also store
                                          it into a snapshot that dqn_get_params(DQN_PARAMS_GRAD) returns.
                                          Diagnostic; the step's kernels, launch configuration and
                                          arithmetic are otherwise unchanged (it adds one store per element) */
  double replay_prio_alpha;            /* prioritized replay (NEXT-4, "emphasize transitions from which we
                                          can learn the most"; rule = DESIGN.md A41): 0 = uniform sampling (a1,
                                          default); 1 or 0.5 = draw slot i with probability p_i / sum p, p_i =
                                          (|delta_i| + replay_prio_eps)^alpha written after the step that sampled
                                          it, stored transitions entering with the largest p so far; b stratified
                                          draws per step from a 32-ary fp32 sum tree. Not with dqn_collect */
  double replay_prio_eps;              /* eps_p >= 0 of the priority                                           */
} dqn_config;

typedef struct {
  /* outputs */
  double loss_mean;          /* mean over the call's steps of (1/b) sum 1/2 delta^2 (unclipped, A27) */
  int64_t generation;        /* server iteration number n after the call (Alg. 2)              */
  int64_t steps_done;        /* replica step counter T after the call                                */
  float device_ms;           /* device time of the call (CUDA events on the context stream)          */
  int64_t nonfinite_elems;   /* mean-gradient elements so far that were non-finite and skipped (A24) */
  /* optional caller-owned HOST outputs (NULL = not wanted); valid when k <= 4096 */
  int32_t* sampled_idx;      /* [k][b] replay slots sampled by this replica (a1)                     */
  int32_t* target_argmax;    /* [k][b] argmax_a' Q(phi_{j+1}, a'; theta^), lowest index on ties      */
  float* loss_per_step;      /* [k]                                                                  */
  /* output */
  int64_t kernel_launches;   /* kernels of this library launched by the call (graph kernel nodes)     */
  int64_t staleness_hist[32];/* DQN_ASYNC*: replica steps by staleness n_apply - n_local (A25), since create;
                                bucket 31 collects >= 31. All zero in the deterministic mode.          */
  /* optional caller-owned HOST output (NULL = not wanted); valid when k <= 4096 */
  int64_t* step_generation;  /* [k] generation n_local of the theta each step of the call used: the
                                realised fetch schedule (A40; in DQN_ASYNC it depends on timing)       */
  /* output: the paper's Fig. 3 quantities per replica step, from the most recent
     dqn_profile_steps call on this context (-1 before any): T = gradient computation (sampling,
     forward, TD head, backward), tau = the parameter update, and the communication regions
     (push, fetch, the fused server round, target refresh)                                              */
  double grad_ms, update_ms, comm_ms;
  /* optional caller-owned HOST output (NULL = not wanted); valid when k <= 4096 */
  float* td_error;           /* [k][b] delta_j = Q(phi_j, a_j; theta) - y_j, unclipped (A27)            */
} dqn_step_stats;

/* Per-region device time of the replica step (diagnostic; dqn_profile_steps). */
typedef struct {
  char name[48];             /* step region, e.g. "conv1_fwd", "head_td", "rmsprop_update"            */
  double avg_us;             /* mean device time per step, CUDA events around the region in the graph */
  int32_t kernels;           /* kernels in the region                                                */
  int32_t steps;             /* steps in which the region ran                                        */
} dqn_region_time;

/* Number of parameters P (weights + biases of every layer); -1 if the layer chain
 * is invalid. Pure. Canonical flat order: layer by layer, W then b; conv W is
 * [N][C][k][k], FC W is [H][D] with D flattened in (C,H,W) order (A18). */
int64_t dqn_param_count(const dqn_config* cfg);

/* Bytes of the NCCL unique id (128). dqn_nccl_unique_id writes one into out
 * (call on rank 0, broadcast the bytes to every rank out of band). */
int32_t dqn_nccl_id_bytes(void);
int dqn_nccl_unique_id(void* out);

/* Create the context of `rank` in a group of `world` ranks (collective when
 * world > 1). nccl_unique_id: dqn_nccl_id_bytes() bytes, NULL iff world == 1.
 * cuda_stream: a cudaStream_t all work is ordered on, or NULL for a
 * library-owned stream. The current CUDA device must already be selected.
 * Initial state: theta = init_params (or N(0, init_std^2) from init_seed, the
 * same on every rank), r = 0, n = 0, theta^ = theta, l = 0, T = 0 (Alg. 2). */
int dqn_create(const dqn_config* cfg, int rank, int world, const void* nccl_unique_id, void* cuda_stream,
               dqn_ctx** out);

/* "Store experience (phi_t, a_t, r_t, phi_{t+1}) in D_k" (Alg. 1).
 * n transitions, oldest first: s and s_next [n][F][H][W] u8 (frames oldest
 * first), a [n] in [0, n_actions), r [n] finite, terminal [n] (0/1).
 * Push i goes to slot (count + i) mod capacity (FIFO last-N).
 * DQN_EINVAL (nothing stored) on an out-of-range action or non-finite reward.
 * Host buffers are validated on the host and packed into library-owned pinned
 * staging before the call returns (the caller may reuse them at once); the copy
 * to the device and the ring write are then ordered on the context's stream
 * without a host sync. Device buffers are validated on the device and the call
 * synchronises the stream before returning. */
int dqn_push_transitions(dqn_ctx* ctx, int64_t n, const uint8_t* s, const int32_t* a, const float* r,
                         const uint8_t* s_next, const uint8_t* terminal);

/* Run k replica steps of Alg. 1 with the server rounds of Alg. 2 they trigger
 * (collective: every rank passes the same k). Per step T: fetch when
 * T % n_fetch == 0 (then refresh theta^ when n - l >= C); sample b slots
 * uniformly with replacement; targets with theta^; gradient at the fetched
 * theta; accumulate; when (T+1) % n_push == 0 every shard owner sums the N
 * replicas' gradient slices of its shard in rank order, applies RMSProp to its
 * shard and n += 1. At world > 1 that round is ONE kernel over NVLink peer memory
 * (DQN_DETERMINISTIC with n_fetch = 1: push, update and the delivery of the new
 * theta to every replica); otherwise an NCCL reduce-scatter, the update and an
 * NCCL all-gather (bf16 records on DQN_BF16), on a second stream in DQN_ASYNC*.
 * stats may be NULL. DQN_EEMPTY if the replay memory is empty (nothing run);
 * DQN_ENONFINITE if any round so far produced a non-finite mean gradient. */
int dqn_train_steps(dqn_ctx* ctx, int64_t k, dqn_step_stats* stats);

/* Alg. 1's loop for k iterations, in one call (collective: every rank
 * passes the same k): iteration i stores transition i ("Store experience ... in D",
 * P:117; arguments and layout as dqn_push_transitions, k items) and then runs one
 * replica step exactly as dqn_train_steps(1) (sample from D including that item,
 * gradient, the server round it triggers). Equivalent to k alternating calls
 * dqn_push_transitions(1 item) + dqn_train_steps(1), with one host synchronisation
 * at the end instead of one per iteration. stats as dqn_train_steps (loss_per_step
 * receives the k losses). Errors: as dqn_push_transitions (validated before anything
 * runs) and dqn_train_steps; DQN_EINVAL in the DQN_ASYNC* modes. */
int dqn_store_and_train(dqn_ctx* ctx, int64_t k, const uint8_t* s, const int32_t* a, const float* r,
                        const uint8_t* s_next, const uint8_t* terminal, dqn_step_stats* stats);

/* Diagnostic twin of dqn_train_steps (collective, same semantics: it advances the
 * run by k real steps): the step graphs are captured with CUDA event records
 * around every region, each step is replayed and synchronised, and the mean
 * device time per region is written to out[cap]; *n_regions = regions found. */
int dqn_profile_steps(dqn_ctx* ctx, int64_t k, dqn_region_time* out, int32_t cap, int32_t* n_regions);

/* Q(s, a; theta_local) for n states [n][F][H][W] u8 -> q [n][n_actions] fp32 and
 * (optional) argmax [n] int32, lowest index on ties. Not collective. */
int dqn_q_values(dqn_ctx* ctx, int64_t n, const uint8_t* states, float* q, int32_t* argmax);

/* Copy a parameter vector (DQN_PARAMS_*) in canonical order into out[cap]
 * (cap >= P, host or device). n_params / generation may be NULL.
 * SERVER and RMS are collective when world > 1; so is LOCAL on a bf16 context with
 * world > 1 and the fused server round (DQN_DETERMINISTIC, n_fetch = 1), where the
 * working copy equals the gathered SERVER vector and is returned as such. */
int dqn_get_params(dqn_ctx* ctx, int which, float* out, int64_t cap, int64_t* n_params, uint64_t* generation);

/* NEXT-3 — the acting side of Alg. 1 on the GPU: n_envs parallel games of the paper's
 * Snake (an n x n grid, `grid` = n, rendered at height/n pixels per cell; rules closed as in
 * walls and self-collision end the game with -1, an apple gives +1 and one body
 * length, 200*n steps without an apple end it with 0; A34-A36), played for `steps` steps with
 * the eps-greedy behaviour policy on Q(phi; theta_local) from the network's forward; every
 * step's transition (phi_t, a_t, r_t, phi_{t+1}, terminal) is stored into the replay on the device.
 * Needs n_actions == 4 (up, right, down, left), height == width, height % grid == 0, 4 <= grid <= 32,
 * height*width % 16 == 0 and n_envs <= minibatch. The games persist in the context: the first call
 * creates them from (n_envs, grid, env_seed); later calls must pass the same values and continue.
 * Random draws are Philox4x32-10 keyed by env_seed (counter: env, step, purpose), so runs are
 * reproducible and equal the oracle's or_collect whenever the greedy actions agree (always at eps=1).
 * stats (may be NULL): env_steps, episodes finished, reward sum, device ms, optional per-step
 * logs [steps][n_envs] of actions / rewards / terminals (host or device, NULL to skip). */
typedef struct {
  int64_t env_steps;
  int64_t episodes;
  double reward_sum;
  float device_ms;
  int32_t* actions;
  float* rewards;
  uint8_t* terminals;
} dqn_collect_stats;
int dqn_collect(dqn_ctx* ctx, int32_t n_envs, int32_t grid, int64_t steps, double epsilon, uint64_t env_seed,
                dqn_collect_stats* stats);
/* The current frame stacks of the collector's games, [n_envs][F][H][W] u8 (host or device). */
int dqn_env_stacks(dqn_ctx* ctx, uint8_t* out, int64_t cap_bytes);

/* Replay occupancy: total pushes so far and min(count, capacity). */
int dqn_replay_size(const dqn_ctx* ctx, int64_t* count, int64_t* size);

/* Prioritized replay (cfg.replay_prio_alpha != 0; NEXT-4, A41): the replay_capacity leaf priorities
 * p_i (0 = never stored) into out[cap >= replay_capacity] and the sum-tree total into *total (either may
 * be NULL; host or device pointers). Synchronises the context stream. DQN_EINVAL without prioritized
 * replay or with a short buffer. */
int dqn_get_priorities(dqn_ctx* ctx, float* out, int64_t cap, float* total);

/* Last error message of this context ("" if none); with ctx == NULL, the message of the
 * last failed dqn_create on the calling thread. Never NULL. */
const char* dqn_last_error(const dqn_ctx* ctx);

/* Free every device resource of the context (not collective). NULL is a no-op. */
void dqn_destroy(dqn_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* DQN_H */
