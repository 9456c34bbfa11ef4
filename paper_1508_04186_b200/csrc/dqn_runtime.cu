// dqn_runtime.cu — the C ABI of include/dqn.h: context, replay memory, parameter
// layout and shards, the deterministic push/fetch schedule, CUDA-graph step
// replay, NCCL reduce-scatter (push, a11) and all-gather (fetch, a13).
//
// Method: Alg. 1 (worker) and Alg. 2 (parameter server) of
// arXiv 1508.04186, re-cast for one process per B200: every rank is a replica
// AND the owner of 1/N of the server state.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "../../include/dqn.h"
#include "dqn_internal.h"
#include "step_trace.cuh"
#include "wimg.cuh"

using namespace dqn;

struct dqn_ctx {
  dqn_config cfg{};
  NetShape net{};
  int rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;
  // replay memory D_k: FIFO ring of the last `cap` experiences
  uint8_t *ring_s = nullptr, *ring_sn = nullptr, *ring_t = nullptr;
  // replay slots: `slot_stride` bytes apart; with frame dedup one buffer of F+1 frames per slot,
  // s = frames 0..F-1 (ring_s), s' = frames 1..F (ring_sn = ring_s + one frame, not owned)
  long long slot_stride = 0;
  bool dedup = false;
  int32_t* ring_a = nullptr;
  float* ring_r = nullptr;
  long long cap = 0, count = 0;
  // parameters, canonical flat order, padded to P_pad = ceil(P / 64N) * 64N
  long long P = 0, P_pad = 0, shard = 0;
  float* theta_master = nullptr;  // [shard] fp32 master of the owned shard (world 1: whole vector)
  float* rms = nullptr;           // [shard] RMSProp accumulator r
  float* grad = nullptr;          // [P_pad] gradient accumulator of this replica
  float* g_shard = nullptr;       // [shard] reduce-scatter output (world > 1)
  float* theta_local = nullptr;   // [P_pad] fetched theta (may alias theta_master)
  float* theta_hat = nullptr;     // [P_pad] target theta^
  float* grad_snap = nullptr;     // [P_pad] optional copy of the last pushed gradient (cfg.keep_grad)
  float* gather_tmp = nullptr;    // [P_pad] for get_params(SERVER/RMS) with world > 1
  // activations: conv layer c -> act_conv[c][g] [b][N*Ho*Wo]; hidden fc l -> act_fc[l][g] [b][H]
  float* act_conv[kMaxConv][2] = {};
  float* act_fc[kMaxFc][2] = {};
  float* dz_conv[kMaxConv] = {};
  float* dz_fc[kMaxFc] = {};
  float* partial = nullptr;
  float* head_dq = nullptr;   // [b] per-sample scratch of the TD head
  int* head_act = nullptr;    // [b]
  float* head_loss = nullptr; // [b]
  long long partial_elems = 0;
  int* idx = nullptr;
  DevCounters* ctr = nullptr;
  float* diag_loss = nullptr;
  int* diag_idx = nullptr;
  int* diag_amax = nullptr;
  // bf16 tensor-core path (precision == DQN_BF16)
  bool bf16 = false;
  // generic bf16 conv path (bf16 && not the Mnih stack): per-layer geometry, buffers, pack maps
  bool gpath = false;
  struct GLayer {
    int Hs, Ws, Cs, Th, Tw, Ho, Wo, N, s;   // s: this layer's stride (its input grid is s2d by s)
    long long fwd_pack, dg_pack;            // offsets of the packed weights after P_pad (-1: none)
    int ipc;                                // images per wgrad CTA
    int* w_canon = nullptr;                 // [Th*Tw*Cs]
    __nv_bfloat16* x[2] = {};               // input grid per group (layers >= 2)
    __nv_bfloat16* dz = nullptr;            // output gradient [b][Ho][Wo][N]
  } gl[kMaxConv];
  int2* pack_map = nullptr;                 // [pack_n]: packed slots of each canonical conv parameter
  // the FC layers on the warp-specialised TMA GEMM (kernels_tma.cu; DQN_TGEMM=0: the older tcgen05 GEMMs)
  bool use_tgemm = false;
  TGemmArgs tg_fwd{}, tg_dw{}, tg_dx{};
  // the conv forward on the same TMA GEMM (implicit GEMM over virtual rows); layer 1 reads a bf16 s2d grid
  // gathered from the replay by gather_s2d_kernel (x1[g], [b][441][64])
  bool use_tconv = false;
  TConvArgs tc_fwd[kMaxConv]{}, tc_dgrad[kMaxConv]{}, tc_wgrad[kMaxConv]{};
  GConvWgradArgs tc_wred[kMaxConv]{};
  __nv_bfloat16* x1[2] = {};
  __nv_bfloat16* dzp[kMaxConv] = {};          // dZ of every conv layer in its input-grid geometry (zero borders)
  __nv_bfloat16* dx_canon = nullptr;          // FC dX (masked) in the canonical flatten [b][D], before chw_to_hwc
  float* tc_part = nullptr;                   // every layer's weight-gradient partials, each at its own offset
  float* tc_part_db = nullptr;
  // conv backward on two graph branches: the data-gradient chain (dgrad L-1 .. 1, then wgrad 0) on the main
  // stream, the weight gradients (+ range reductions) of layers L-1 .. 1 on bside, each after its dZ is ready
  cudaStream_t bside = nullptr;
  cudaEvent_t ev_bdz[kMaxConv] = {}, ev_bjoin = nullptr;
  // N = 1, n_push = 1 on the TMA kernels: the head finish and the RMSProp update of the FC / output-layer
  // parameters run on a side stream (graph branch) next to the FC dX and the conv backward
  bool split_update = false;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_dw = nullptr, ev_join = nullptr;
  long long pack_n = 0, gpack_off = -1;
  float* gw_partial = nullptr;
  float* gw_partial_db = nullptr;
  // DQN_ASYNC / DQN_ASYNC_LAG1: the push -> RMSProp -> publish round runs on
  // comm_stream while the replica keeps stepping. Generation m is published in theta_pub[m % 3] and announced
  // by a device flag (adev->pub_gen); a fetch takes the newest one (DQN_ASYNC) or exactly n - 1 (the lag-1 twin)
  bool async = false, async_lag1 = false;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_grad = nullptr, ev_pub[3] = {}, ev_send[2] = {};
  float* g_send[2] = {};                          // [P_pad] gradient handed to round k, by k % 2
  float* inbox = nullptr;                         // [world][shard] DQN_ASYNC* + per-gradient rule: every worker's
                                                  // slice of this rank's shard, applied one by one (A33)
  float* theta_pub[3] = {};                       // [P_pad] published server theta, by generation % 3
  __nv_bfloat16* theta_pub_bf16[3] = {};
  AsyncDev* adev = nullptr;                       // device generation flag, fetch log, staleness histogram
  AsyncDev* h_adev = nullptr;                     // pinned landing zone
  long long n_fetches = 0;                        // fetches issued (host; fetch f is at step f * n_fetch)
  unsigned async_delay_ns = 0;                    // DQN_ASYNC_DELAY_US: diagnostic server delay per round
  // NEXT-1 fused server round over NVLink peer memory (world > 1, deterministic, n_fetch == 1)
  bool fused_comm = false;
  // a13 over NCCL on the bf16 path (world > 1 without the fused round): one all-gather of per-rank records
  // [bf16 shard | fp32 of its entries outside the FC weight]; the FC weight of theta_local / theta_hat
  // then exists only in bf16 (get_params widens it)
  bool fetch_bf16 = false;
  FetchRecord frec{};
  uint8_t* fetch_send = nullptr;
  uint8_t* fetch_recv = nullptr;
  // NEXT-3 collector (dqn_collect): the games persist between calls
  struct Collector {
    int E = 0, n = 0;
    unsigned long long seed = 0, t = 0;
    EnvGame* games = nullptr;
    uint8_t *stacks = nullptr, *s_stage = nullptr, *sn_stage = nullptr, *t_stage = nullptr;
    int32_t* a_stage = nullptr;
    float* r_stage = nullptr;
    long long* episodes = nullptr;
    double* reward_sum = nullptr;
  } env;
  long long n_per_round = 1;  // server generations per push round: 1 (mean rule) or N (per-gradient rule)
  ServerRoundArgs sra{};                          // peer pointers etc., filled at create
  FusedAcquire acq{};                             // the next step's acquire half (acq.ctr == nullptr: off)
  unsigned long long* flags = nullptr;            // [kMaxWorld] barrier A (written by peers)
  unsigned long long* done = nullptr;             // barrier B counter (incremented by peers)
  std::vector<void*> ipc_opened;                  // peer mappings to close at destroy
  __nv_bfloat16* theta_local_bf16 = nullptr;  // [P_bf16] working copy the tensor cores read
  __nv_bfloat16* theta_hat_bf16 = nullptr;    // [P_bf16]
  // every bf16 theta buffer holds P_pad canonical entries followed by the conv weights' forward
  // image (wimg.cuh) at img_off = P_pad
  long long P_bf16 = 0, img_off = -1, w1_off = 0, w2_off = 0;
  __nv_bfloat16* a2_bf16 = nullptr;           // [2b][2592] conv2 activations (s: theta, s': theta^)
  uint8_t* a1_save = nullptr;                 // [b][8][144][16] conv1 activations (s2d planes)
  __nv_bfloat16* dh_bf16 = nullptr;           // [b][H]
  __nv_bfloat16* dz2_bf16 = nullptr;          // [b][2592]
  float* fc_partial = nullptr;                // [2][splits][H][b]
  unsigned* tc_counters = nullptr;            // last-CTA counters (self-resetting)
  float* bwd_partial = nullptr;               // [b][kBwdPart]
  uint8_t* q_stage_s2d = nullptr;             // [b][28224]
  int fc_splits = 1;
  // q_values staging
  uint8_t* q_stage = nullptr;
  float* q_out = nullptr;
  int* q_amax = nullptr;
  // push staging (host inputs)
  // host-buffer pushes: inputs packed into one of two pinned staging buffers, one H2D copy per
  // chunk into d_stage, the ring kernel; no host sync (the inputs are consumed by the pack)
  uint8_t* d_stage = nullptr;  // push_chunk transitions (~4 MB), allocated at create
  uint8_t* h_stage[2] = {};
  cudaEvent_t ev_stage[2] = {};
  // dqn_store_and_train with host buffers: sub-chunks alternate between the two halves of d_stage, copied on
  // copy_stream while the previous sub-chunk's steps run (ev_copied: the half is filled, ev_consumed: its steps
  // are done with it)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {}, ev_consumed[2] = {};
  int stage_flip = 0;
  long long push_chunk = 0;
  // pinned landing zone of dqn_train_steps' per-call outputs
  struct HostOut {
    DevCounters ctr;
    float loss[kDiagSteps];
  }* h_out = nullptr;
  // host mirrors of the deterministic schedule (identical on every rank)
  long long T = 0, n = 0, n_local = 0, ell = 0;
  std::vector<long long> gen_log = std::vector<long long>(kDiagSteps, 0);  // n_local of step T at T % kDiagSteps
  // graphs per (fetch, refresh, push) variant; [8..15]: the same with profiling event records
  cudaGraphExec_t graphs[16] = {};
  long long graph_kernels[16] = {};
  // dqn_store_and_train on the bf16 Mnih path: the Store runs inside the step graphs (variant bit 16)
  StoreCtl* store_ctl = nullptr;
  unsigned long long* store_flag = nullptr;  // the forward's fused Store: T + 1 once step T's item is in the ring
  bool graph_store = false;
  // prioritized replay (NEXT-4, A41; cfg.replay_prio_alpha != 0)
  bool prio = false;
  int prio_alpha_half = 0;
  float prio_eps = 0.0f;
  PrioTree ptree{};
  float* prio_maxp = nullptr;                 // the largest priority written so far (1 initially)
  float* head_delta = nullptr;                // [b] delta_j of the step (TD head -> prio_update)
  float* diag_delta = nullptr;                // [kDiagSteps][b]
  bool store_chunks_ready = false;
  // multi-step graphs: kChunkLog lengths 2^0..2^(kChunkLog-1) of consecutive same-variant steps,
  // so the programmatic (PDL) edges also span step boundaries (a graph boundary serialises)
  static constexpr int kChunkLog = 5;
  cudaGraphExec_t chunk_graphs[32][kChunkLog] = {};
  long long chunk_kernels[32][kChunkLog] = {};
  bool chunks_ready = false;
  // profiling (dqn_profile_steps): event pairs around each step region, per graph variant
  struct ProfMark {
    std::string name;
    cudaEvent_t a, b;
    int kernels;
  };
  std::vector<ProfMark> marks[16];
  int capture_variant = -1;  // >= 8 while capturing a profiling graph
  bool use_graphs = true;
  bool step_trace = false;  // DQN_TRACE_STEP=1
  int num_sms = 148;
  double prof_grad_ms = -1.0, prof_update_ms = -1.0, prof_comm_ms = -1.0;  // last dqn_profile_steps (T, tau, comm)
  bool early_update = true; // N = 1 bf16: FC / output-layer RMSProp inside the conv backward launch (DQN_EARLY_UPDATE=0: off)
  bool keep_grad = false;
  bool alias_local = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::string err;
  bool poisoned = false;
  bool diverged = false;
};

// ------------------------------------------------------------------ helpers
static int set_err(dqn_ctx* c, int code, const std::string& msg) {
  if (c) {
    c->err = msg;
    if (code == DQN_ECUDA || code == DQN_ENCCL) c->poisoned = true;
  }
  return code;
}

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return set_err(ctx, DQN_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)
#define NK(call)                                                                                  \
  do {                                                                                            \
    ncclResult_t r_ = (call);                                                                     \
    if (r_ != ncclSuccess)                                                                        \
      return set_err(ctx, DQN_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));        \
  } while (0)

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Shapes of the layer chain (valid convolutions A16). Returns false when invalid.
static bool build_net(const dqn_config* c, NetShape* s) {
  std::memset(s, 0, sizeof(*s));
  if (!c || c->frames < 1 || c->height < 1 || c->width < 1) return false;
  if (c->n_conv < 0 || c->n_conv > kMaxConv || c->n_fc < 0 || c->n_fc > kMaxFc || c->n_actions < 1) return false;
  s->F = c->frames; s->Hin = c->height; s->Win = c->width;
  s->state_bytes = (long long)c->frames * c->height * c->width;
  int ch = c->frames, h = c->height, w = c->width;
  long long off = 0;
  s->n_conv = c->n_conv;
  for (int i = 0; i < c->n_conv; ++i) {
    ConvShape& L = s->conv[i];
    const int N = c->conv_filters[i], k = c->conv_kernel[i], st = c->conv_stride[i];
    if (N < 1 || k < 1 || st < 1 || k > h || k > w || (h - k) % st || (w - k) % st) return false;
    L.C = ch; L.H = h; L.W = w; L.N = N; L.k = k; L.s = st;
    L.Ho = (h - k) / st + 1; L.Wo = (w - k) / st + 1;
    L.w_off = off; off += (long long)N * ch * k * k;
    L.b_off = off; off += N;
    ch = N; h = L.Ho; w = L.Wo;
  }
  int d = ch * h * w;
  s->n_fc = c->n_fc;
  for (int i = 0; i <= c->n_fc; ++i) {
    FcShape& F = s->fc[i];
    const int units = i < c->n_fc ? c->fc_units[i] : c->n_actions;
    if (units < 1) return false;
    F.D = d; F.H = units;
    F.w_off = off; off += (long long)units * d;
    F.b_off = off; off += units;
    d = units;
  }
  s->A = c->n_actions;
  s->P = off;
  return true;
}

// deterministic N(0, xi^2) init from init_seed (Alg. 2; identical on every rank)
static uint64_t splitmix64(uint64_t& x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static void gaussian_init(std::vector<float>& th, double std_, uint64_t seed) {
  uint64_t st = seed;
  for (size_t i = 0; i < th.size(); i += 2) {
    double u1 = ((splitmix64(st) >> 11) + 1.0) * (1.0 / 9007199254740993.0);
    double u2 = (splitmix64(st) >> 11) * (1.0 / 9007199254740992.0);
    double rad = std::sqrt(-2.0 * std::log(u1));
    th[i] = (float)(std_ * rad * std::cos(2.0 * M_PI * u2));
    if (i + 1 < th.size()) th[i + 1] = (float)(std_ * rad * std::sin(2.0 * M_PI * u2));
  }
}

// the Mnih-2013 conv stack of BASELINE.json configs[0..3] (the specialised bf16 kernels)
static bool is_mnih_stack(const dqn_config* c) {
  return c->frames == 4 && c->height == 84 && c->width == 84 && c->n_conv == 2 && c->conv_filters[0] == 16 &&
         c->conv_kernel[0] == 8 && c->conv_stride[0] == 4 && c->conv_filters[1] == 32 && c->conv_kernel[1] == 4 &&
         c->conv_stride[1] == 2 && c->n_fc == 1;
}

// The generic bf16 conv path's shape contract (kernels_conv.cu); nullptr when supported.
static const char* gpath_unsupported(const NetShape& net, const dqn_config* c) {
  if (!(net.F == 4 && net.Hin == 84 && net.Win == 84)) return "DQN_BF16 needs 84x84x4 frame stacks";
  if (net.n_fc != 1) return "DQN_BF16 needs exactly one hidden FC layer";
  const ConvShape& L0 = net.conv[0];
  if (L0.k != 8 || L0.s != 4) return "DQN_BF16: the first conv must be 8x8 / 4 (the replay ring's s2d layout)";
  for (int i = 0; i < net.n_conv; ++i) {
    const ConvShape& L = net.conv[i];
    if (L.N % 16 != 0 || L.N > 256) return "DQN_BF16: conv filters must be a multiple of 16 and <= 256";
    if (i == 0) continue;
    if (L.s != 1 && L.s != 2) return "DQN_BF16: conv strides after the first must be 1 or 2";
    if (L.k % L.s != 0 || L.H % L.s != 0 || L.W % L.s != 0) return "DQN_BF16: k and the input size must be multiples of the stride";
    if ((L.C * L.s * L.s) % 64 != 0 || L.C * L.s * L.s > 256) return "DQN_BF16: C*s*s must be a multiple of 64 and <= 256";
    if (L.N % 64 != 0) return "DQN_BF16: filters of convs after the first must be a multiple of 64";
  }
  const FcShape& F = net.fc[0];
  if (F.D % 16 != 0 || F.H % 16 != 0 || F.H > 4096) return "DQN_BF16: FC sizes must be multiples of 16 (units <= 4096)";
  if (c->minibatch % 16 != 0 || c->minibatch > 512) return "DQN_BF16 needs minibatch % 16 == 0 and <= 512";
  return nullptr;
}

static int validate_cfg(const dqn_config* c, NetShape* net, std::string* why) {
  if (!build_net(c, net)) { *why = "invalid layer chain (valid convolutions need integer output sizes)"; return DQN_EINVAL; }
  if (c->n_conv < 1) { *why = "at least one convolution layer is required"; return DQN_EINVAL; }
  if (c->minibatch < 1) { *why = "minibatch must be >= 1"; return DQN_EINVAL; }
  if (c->replay_capacity < 1) { *why = "replay_capacity must be >= 1"; return DQN_EINVAL; }
  if (c->n_push < 1 || c->n_fetch < 1) { *why = "n_push and n_fetch must be >= 1"; return DQN_EINVAL; }
  if (c->precision != DQN_FP32 && c->precision != DQN_BF16) { *why = "unknown precision"; return DQN_EINVAL; }
  if (c->sync_mode != DQN_DETERMINISTIC && c->sync_mode != DQN_ASYNC && c->sync_mode != DQN_ASYNC_LAG1) {
    *why = "unknown sync_mode"; return DQN_EINVAL;
  }
  if (c->server_rule != DQN_SERVER_MEAN && c->server_rule != DQN_SERVER_PER_GRADIENT) { *why = "unknown server_rule"; return DQN_EINVAL; }
  if (c->replay_dedup != 0 && (c->replay_dedup != 1 || c->frames < 2)) { *why = "replay_dedup needs 0, or 1 with frames >= 2"; return DQN_EINVAL; }
  if (!(c->replay_prio_alpha == 0.0 || c->replay_prio_alpha == 0.5 || c->replay_prio_alpha == 1.0) ||
      !(c->replay_prio_eps >= 0.0 && std::isfinite(c->replay_prio_eps))) {
    *why = "replay_prio_alpha must be 0, 0.5 or 1 and replay_prio_eps finite >= 0 (A41)"; return DQN_EINVAL;
  }
  if (c->replay_prio_alpha != 0.0 && (c->replay_capacity > (1LL << 30) || c->minibatch > 8192)) {
    *why = "prioritized replay: capacity <= 2^30 and b <= 8192"; return DQN_EINVAL;
  }
  if (!(c->rms_decay >= 0.0 && c->rms_decay < 1.0) || !(c->rms_eps >= 0.0) || !(c->lr >= 0.0) ||
      !std::isfinite(c->gamma) || !(c->err_clip >= 0.0)) {
    *why = "invalid hyper-parameter"; return DQN_EINVAL;
  }
  {  // the TD head keeps the output layers and 32 samples' activations in shared memory
    const FcShape& O = net->fc[net->n_fc];
    if (O.H > 32 || head_smem_bytes(O.H, O.D, c->minibatch) > 226 * 1024) {
      *why = "output layer too large for the TD-head kernel (|A| <= 32)"; return DQN_EINVAL;
    }
  }
  if (c->precision == DQN_BF16) {
    // the tensor-core kernels are specialised to the Mnih-2013 convolution stack (BASELINE.json configs[0..3])
    const bool mnih = is_mnih_stack(c);
    if (mnih) {
      if (c->minibatch % 16 != 0 || c->minibatch > 256) { *why = "DQN_BF16 needs minibatch % 16 == 0 and <= 256"; return DQN_EINVAL; }
      if (c->fc_units[0] % 16 != 0 || c->fc_units[0] > 4096) {
        *why = "DQN_BF16 needs fc units % 16 == 0 and <= 4096"; return DQN_EINVAL;
      }
      return DQN_OK;
    }
    // generic tensor-core conv path (kernels_conv.cu): every conv a stride-1 conv over a s2d grid
    const char* g = gpath_unsupported(*net, c);
    if (g) { *why = g; return DQN_EINVAL; }
    return DQN_OK;
  }
  // fp32 kernels stage one input image (+ one filter chunk) in shared memory
  for (int i = 0; i < net->n_conv; ++i) {
    const ConvShape& L = net->conv[i];
    long long fwd = ((long long)L.C * L.H * L.W + 3) / 4 * 4 + (long long)L.C * L.k * L.k * 16;
    long long dw = ((long long)L.C * L.H * L.W + 3) / 4 * 4 + (long long)L.N * L.Ho * L.Wo;
    long long dx = ((long long)L.N * L.Ho * L.Wo + 3) / 4 * 4 + (long long)L.N * L.k * L.k * 8;
    if (fwd * 4 > 227 * 1024 || dw * 4 > 227 * 1024 || dx * 4 > 227 * 1024) {
      *why = "layer too large for the shared-memory staging of the fp32 kernels"; return DQN_EINVAL;
    }
  }
  return DQN_OK;
}

extern "C" int64_t dqn_param_count(const dqn_config* cfg) {
  NetShape s;
  if (!build_net(cfg, &s)) return -1;
  return s.P;
}

extern "C" int32_t dqn_nccl_id_bytes(void) { return (int32_t)sizeof(ncclUniqueId); }

extern "C" int dqn_nccl_unique_id(void* out) {
  if (!out) return DQN_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return DQN_ENCCL;
  std::memcpy(out, &id, sizeof(id));
  return DQN_OK;
}

template <typename T>
static int dalloc(dqn_ctx* ctx, T** p, long long n) {
  if (n <= 0) n = 1;
  cudaError_t e = cudaMalloc((void**)p, sizeof(T) * (size_t)n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(ctx, DQN_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  return DQN_OK;
}

static void free_all(dqn_ctx* c) {
  for (auto& g : c->graphs)
    if (g) cudaGraphExecDestroy(g);
  for (auto& row : c->chunk_graphs)
    for (auto& g : row)
      if (g) cudaGraphExecDestroy(g);
  for (auto& v : c->marks)
    for (auto& m : v) {
      cudaEventDestroy(m.a);
      cudaEventDestroy(m.b);
    }
  void* ptrs[] = {c->ring_s, c->dedup ? nullptr : c->ring_sn, c->ring_t, c->ring_a, c->ring_r, c->rms, c->grad, c->g_shard,
                  c->theta_hat, c->grad_snap, c->gather_tmp, c->partial, c->idx, c->ctr, c->diag_loss,
                  c->diag_idx, c->diag_amax, c->head_dq, c->head_act, c->head_loss, c->q_stage, c->q_out, c->q_amax, c->d_stage,
                  c->theta_local_bf16, c->theta_hat_bf16, c->a2_bf16, c->a1_save,
                  c->dh_bf16, c->dz2_bf16, c->fc_partial, c->tc_counters, c->bwd_partial, c->q_stage_s2d,
                  c->store_ctl, c->store_flag, c->ptree.node, c->prio_maxp, c->head_delta, c->diag_delta, c->dx_canon, c->inbox};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& G : c->gl) {
    if (G.w_canon) cudaFree(G.w_canon);
    for (auto* x : G.x)
      if (x) cudaFree(x);
    if (G.dz) cudaFree(G.dz);
  }
  if (c->pack_map) cudaFree(c->pack_map);
  {
    void* ep[] = {c->env.games, c->env.stacks, c->env.s_stage, c->env.sn_stage, c->env.t_stage, c->env.a_stage,
                  c->env.r_stage, c->env.episodes, c->env.reward_sum};
    for (void* p : ep)
      if (p) cudaFree(p);
  }
  if (c->gw_partial) cudaFree(c->gw_partial);
  if (c->side) cudaStreamDestroy(c->side);
  for (cudaEvent_t e : {c->ev_fork, c->ev_dw, c->ev_join})
    if (e) cudaEventDestroy(e);
  for (auto* x : c->x1)
    if (x) cudaFree(x);
  for (auto* x : c->dzp)
    if (x) cudaFree(x);
  if (c->tc_part) cudaFree(c->tc_part);
  if (c->bside) cudaStreamDestroy(c->bside);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  for (cudaEvent_t e : c->ev_bdz)
    if (e) cudaEventDestroy(e);
  if (c->ev_bjoin) cudaEventDestroy(c->ev_bjoin);
  if (c->tc_part_db) cudaFree(c->tc_part_db);
  if (c->gw_partial_db) cudaFree(c->gw_partial_db);
  for (int i = 0; i < 2; ++i) {
    if (c->h_stage[i]) cudaFreeHost(c->h_stage[i]);
    if (c->ev_stage[i]) cudaEventDestroy(c->ev_stage[i]);
    if (c->ev_copied[i]) cudaEventDestroy(c->ev_copied[i]);
    if (c->ev_consumed[i]) cudaEventDestroy(c->ev_consumed[i]);
  }
  if (c->h_out) cudaFreeHost(c->h_out);
  if (c->theta_local && !c->alias_local) cudaFree(c->theta_local);
  if (c->theta_master) cudaFree(c->theta_master);
  for (int i = 0; i < kMaxConv; ++i) {
    for (int g = 0; g < 2; ++g)
      if (c->act_conv[i][g]) cudaFree(c->act_conv[i][g]);
    if (c->dz_conv[i]) cudaFree(c->dz_conv[i]);
  }
  for (int i = 0; i < kMaxFc; ++i) {
    for (int g = 0; g < 2; ++g)
      if (c->act_fc[i][g]) cudaFree(c->act_fc[i][g]);
    if (c->dz_fc[i]) cudaFree(c->dz_fc[i]);
  }
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  if (c->sra.trace) cudaFree(c->sra.trace);
  if (c->flags) cudaFree(c->flags);
  if (c->done) cudaFree(c->done);
  if (c->ev_grad) cudaEventDestroy(c->ev_grad);
  for (int i = 0; i < 3; ++i) {
    if (c->ev_pub[i]) cudaEventDestroy(c->ev_pub[i]);
    if (c->theta_pub[i]) cudaFree(c->theta_pub[i]);
    if (c->theta_pub_bf16[i]) cudaFree(c->theta_pub_bf16[i]);
  }
  for (int i = 0; i < 2; ++i) {
    if (c->ev_send[i]) cudaEventDestroy(c->ev_send[i]);
    if (c->g_send[i]) cudaFree(c->g_send[i]);
  }
  if (c->adev) cudaFree(c->adev);
  if (c->h_adev) cudaFreeHost(c->h_adev);
  if (c->fetch_send) cudaFree(c->fetch_send);
  if (c->fetch_recv) cudaFree(c->fetch_recv);
}

// split-K factor so a GEMM fills the machine (148 SMs)
static int pick_splits(int M, int N, int K, int groups) {
  long long tiles = (long long)((M + 63) / 64) * ((N + 63) / 64) * groups;
  int s = 1;
  while (tiles * s < 296 && K / (s * 2) >= 64) s *= 2;
  return s;
}

static thread_local std::string g_create_err;

// NEXT-1 setup: export G, theta_local (+bf16), the barrier arrays with CUDA IPC, exchange the
// handles over the NCCL communicator (one all-gather), map every peer's buffers.
static int setup_fused_comm(dqn_ctx* ctx) {
  const int N = ctx->world, me = ctx->rank;
  int rc;
  if ((rc = dalloc(ctx, &ctx->flags, kMaxWorld))) return rc;
  // done[0]: barrier-B counter (peers add to it), done[1]: the local blocks' join counter,
  // done[2]: conv-release counter (peers add to it), done[3]: the local conv blocks' join counter
  const long long n_done = 4;
  if ((rc = dalloc(ctx, &ctx->done, n_done))) return rc;
  CK(cudaMemset(ctx->flags, 0, sizeof(unsigned long long) * kMaxWorld));
  CK(cudaMemset(ctx->done, 0, sizeof(unsigned long long) * n_done));
  void* mine[5] = {ctx->grad, ctx->theta_local, ctx->theta_local_bf16, ctx->flags, ctx->done};
  constexpr int H = (int)sizeof(cudaIpcMemHandle_t);
  std::vector<char> hbuf(5 * H, 0), all((size_t)N * 5 * H, 0);
  for (int i = 0; i < 5; ++i)
    if (mine[i]) CK(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(hbuf.data() + i * H), mine[i]));
  char* d_all = nullptr;
  CK(cudaMalloc(&d_all, all.size()));
  CK(cudaMemcpy(d_all + (size_t)me * 5 * H, hbuf.data(), 5 * H, cudaMemcpyHostToDevice));
  ncclResult_t nr = ncclAllGather(d_all + (size_t)me * 5 * H, d_all, 5 * H, ncclChar, ctx->comm, ctx->stream);
  cudaError_t ce = cudaStreamSynchronize(ctx->stream);
  if (nr == ncclSuccess && ce == cudaSuccess) ce = cudaMemcpy(all.data(), d_all, all.size(), cudaMemcpyDeviceToHost);
  cudaFree(d_all);
  if (nr != ncclSuccess) return set_err(ctx, DQN_ENCCL, std::string("handle exchange: ") + ncclGetErrorString(nr));
  CK(ce);
  ServerRoundArgs& a = ctx->sra;
  for (int p = 0; p < N; ++p) {
    void* ptr[5] = {};
    for (int i = 0; i < 5; ++i) {
      if (!mine[i]) continue;
      if (p == me) {
        ptr[i] = mine[i];
      } else {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, all.data() + ((size_t)p * 5 + i) * H, H);
        CK(cudaIpcOpenMemHandle(&ptr[i], h, cudaIpcMemLazyEnablePeerAccess));
        ctx->ipc_opened.push_back(ptr[i]);
      }
    }
    a.grad[p] = static_cast<float*>(ptr[0]);
    a.theta_local[p] = static_cast<float*>(ptr[1]);
    a.theta_local_bf16[p] = static_cast<__nv_bfloat16*>(ptr[2]);
    a.flags[p] = static_cast<unsigned long long*>(ptr[3]);
    a.done[p] = static_cast<unsigned long long*>(ptr[4]);
  }
  const dqn_config& c = ctx->cfg;
  a.world = N; a.rank = me; a.n_push = c.n_push;
  a.shard = ctx->shard; a.grad_elems = ctx->P_pad;
  a.my_flags = ctx->flags; a.my_done = ctx->done; a.my_join = ctx->done + 1;
  a.theta_master = ctx->theta_master; a.rms = ctx->rms;
  a.inv_div = (float)(1.0 / ((double)N * c.n_push));
  a.per_gradient = c.server_rule == DQN_SERVER_PER_GRADIENT;
  a.inv_np = (float)(1.0 / (double)c.n_push);
  a.lr = (float)c.lr; a.rho = (float)c.rms_decay; a.omr = (float)(1.0 - c.rms_decay); a.eps = (float)c.rms_eps;
  a.ctr = ctx->ctr;
  a.img_off = ctx->img_off; a.w1_off = ctx->w1_off; a.w2_off = ctx->w2_off;
  if (ctx->bf16) {  // the FC weight is read only through theta_local_bf16
    const FcShape& F = ctx->net.fc[0];
    a.f32_peer_lo = F.w_off;
    a.f32_peer_hi = F.w_off + (long long)F.H * F.D;
  }
  ctx->acq.done = ctx->done;
  ctx->acq.world = N;
  ctx->acq.n_push = c.n_push;
  ctx->acq.grad = ctx->grad;
  ctx->acq.grad_elems = ctx->P_pad;
  ctx->acq.ctr = ctx->ctr;
  ctx->acq.g_snap = ctx->grad_snap;
  // conv-first delivery (bf16 Mnih path, conv parameters = the canonical prefix [0, kBwdPart))
  const char* cf = getenv("DQN_CONV_FIRST");
  const bool mnih_bf16 = ctx->bf16 && !ctx->gpath && ctx->img_off >= 0 && ctx->w1_off == 0 &&
                         ctx->net.conv[1].b_off + ctx->net.conv[1].N == kBwdPart;
  if (mnih_bf16 && !(cf && atoi(cf) == 0)) {
    for (int p = 0; p < N; ++p) a.done_c[p] = a.done[p] + 2;
    a.my_join_c = ctx->done + 3;
    a.conv4 = std::min(ctx->shard / 4, std::max(0LL, ((long long)kBwdPart - (long long)me * ctx->shard) / 4));
    ctx->acq.done_c = ctx->done + 2;
    ctx->acq.n_c = (int)std::min<long long>(N, (kBwdPart + ctx->shard - 1) / ctx->shard);
    ctx->acq.conv_first = 1;
    a.conv_per_block = 64;  // the conv prefix's scattered weight-image stores spread over 4x more blocks (DESIGN 6a)
  }
  const char* tr = getenv("DQN_TRACE_COMM");
  if (tr && atoi(tr)) {
    if ((rc = dalloc(ctx, &a.trace, 64 * 16))) return rc;
    std::vector<unsigned long long> init(64 * 16, 0);
    for (int r = 0; r < 64; ++r) init[r * 16 + 4] = ~0ull;  // atomicMin slot
    CK(cudaMemcpy(a.trace, init.data(), sizeof(unsigned long long) * 64 * 16, cudaMemcpyHostToDevice));
    ctx->acq.trace = a.trace;
  }
  return DQN_OK;
}

// The FC layers (a5, a7) on the warp-specialised TMA GEMM: forward split-K partials (the TD head reduces
// them), dW into G, dX (x ReLU mask) into the last conv layer's NHWC dZ. Tensor maps are built once here (the
// buffers never move); any refusal leaves the older tcgen05 GEMMs in place.
static void setup_tgemm_fc(dqn_ctx* ctx) {
  const char* e = getenv("DQN_TGEMM");
  if ((e && atoi(e) == 0) || !init_tma_kernel_attrs()) return;
  const FcShape& F = ctx->net.fc[0];
  const int b = ctx->cfg.minibatch, D = F.D, H = F.H;
  // the head's split count (A/B at BJ.configs[4]: 7 splits 210.2, 4: 211.4, 2: 214.3 us/step)
  const int sp = ctx->fc_splits;
  const int kper = (((D + 63) / 64 + sp - 1) / sp) * 64;
  if ((sp - 1) * kper >= D) return;  // an empty split
  const __nv_bfloat16* W[2] = {ctx->theta_local_bf16 + F.w_off, ctx->theta_hat_bf16 + F.w_off};
  const dqn_ctx::GLayer& GL = ctx->gl[ctx->net.n_conv - 1];
  bool ok = true;
  TGemmArgs& f = ctx->tg_fwd;  // h^T [H][b] = W [H][D] a2^T, K-major operands
  f.M = H; f.N = b; f.K = D; f.kper = kper; f.splits = sp; f.BN = std::min(128, (b + 15) / 16 * 16);
  f.a_mn = 0; f.b_mn = 0; f.groups = 2; f.epi = TC_EPI_FC_FWD; f.partial = ctx->fc_partial;
  for (int g = 0; g < 2; ++g) {
    ok = ok && make_tmap_bf16(&f.ta[g], W[g], H, D, D, 128);
    ok = ok && make_tmap_bf16(&f.tb[g], ctx->a2_bf16 + (long long)g * b * D, b, D, D, f.BN);
  }
  TGemmArgs& w = ctx->tg_dw;  // dW^T [D][H] = a2^T dH: both operands MN-major over K = b, stored transposed into
  w.M = D; w.N = H; w.K = b; w.kper = b; w.splits = 1; w.BN = 64;  // G's [H][D] (lanes along d: coalesced)
  w.a_mn = 1; w.b_mn = 1; w.groups = 1; w.epi = TC_EPI_ACCUM_T; w.store = ctx->cfg.n_push == 1;
  w.C[0] = ctx->grad + F.w_off; w.ldc = D;
  ok = ok && make_tmap_bf16(&w.ta[0], ctx->a2_bf16, b, D, D, 64);
  ok = ok && make_tmap_bf16(&w.tb[0], ctx->dh_bf16, b, H, H, 64);
  TGemmArgs& x = ctx->tg_dx;  // dZ [b][D] = [a2 > 0] dH W: A = W MN-major over K = H, B = dH K-major
  x.M = D; x.N = b; x.K = H; x.kper = H; x.splits = 1; x.BN = 64;
  x.a_mn = 1; x.b_mn = 0; x.groups = 1; x.epi = TC_EPI_MASK_T;
  x.out_bf16 = GL.dz; x.mask = ctx->a2_bf16; x.ldo = D; x.hwc_HW = GL.Ho * GL.Wo; x.hwc_C = GL.N;
  ok = ok && make_tmap_bf16(&x.ta[0], W[0], H, D, D, 64);
  ok = ok && make_tmap_bf16(&x.tb[0], ctx->dh_bf16, b, H, H, x.BN);
  ctx->use_tgemm = ok;
  if (ok && ctx->world == 1 && ctx->cfg.n_push == 1 && ctx->alias_local && !ctx->async && F.w_off % 4 == 0 &&
      !((e = getenv("DQN_SPLIT_UPDATE")) && atoi(e) == 0) &&
      cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking) == cudaSuccess &&
      cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) == cudaSuccess &&
      cudaEventCreateWithFlags(&ctx->ev_dw, cudaEventDisableTiming) == cudaSuccess &&
      cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) == cudaSuccess)
    ctx->split_update = true;
  if (!ok || ((e = getenv("DQN_TCONV")) && atoi(e) == 0) || !init_tconv_kernel_attrs()) return;
  // every conv layer on the TMA tap-window kernel (kernels_tma.cu): forward (theta on s, theta^ on s'), data
  // gradient of every layer but the first, weight gradient (+ db) as per-range partials reduced in order
  const NetShape& net = ctx->net;
  const int nl = net.n_conv;
  for (int g = 0; g < 2; ++g)
    if (dalloc(ctx, &ctx->x1[g], (long long)b * 441 * 64)) return;
  long long max_part = 0, max_db = 0;
  for (int i = 0; i < nl && ok; ++i) {
    const ConvShape& L = net.conv[i];
    const dqn_ctx::GLayer& G = ctx->gl[i];
    const int T = G.Th * G.Tw, K = T * G.Cs, HsWs = G.Hs * G.Ws, maxshift = (G.Th - 1) * G.Ws + (G.Tw - 1);
    const long long rows = (long long)b * HsWs;
    if (G.Cs % 64 != 0 || L.N % 16 != 0 || L.N > 256 || (i > 0 && L.N % 64 != 0) || 128 + maxshift > 256) {
      ok = false;
      break;
    }
    if (dalloc(ctx, &ctx->dzp[i], rows * L.N)) return;
    if (cudaMemset(ctx->dzp[i], 0, sizeof(__nv_bfloat16) * rows * L.N) != cudaSuccess) return;
    const __nv_bfloat16* x[2] = {i == 0 ? ctx->x1[0] : G.x[0], i == 0 ? ctx->x1[1] : G.x[1]};
    // forward
    TConvArgs& f = ctx->tc_fwd[i];
    f.mode = TCONV_FWD; f.groups = 2; f.M = (int)rows; f.BN = L.N;
    f.T = T; f.Tw = G.Tw; f.Ws = G.Ws; f.HsWs = HsWs; f.Cblk = G.Cs / 64; f.maxshift = maxshift; f.R = 128 + maxshift;
    f.Ho = G.Ho; f.Wo = G.Wo; f.N = L.N; f.s_next = i + 1 < nl ? ctx->gl[i + 1].s : 0;
    f.scale = i == 0 ? 1.0f / 255.0f : 1.0f;
    const __nv_bfloat16* wpk[2] = {ctx->theta_local_bf16 + ctx->gpack_off + G.fwd_pack,
                                   ctx->theta_hat_bf16 + ctx->gpack_off + G.fwd_pack};
    for (int g = 0; g < 2; ++g) {
      ok = ok && make_tmap_bf16(&f.ta[g], x[g], rows, G.Cs, G.Cs, f.R);
      ok = ok && make_tmap_bf16(&f.tb[g], wpk[g], L.N, K, K, L.N);
      f.bias[g] = (g ? ctx->theta_hat : ctx->theta_local) + L.b_off;
      f.cout[g] = i + 1 < nl ? ctx->gl[i + 1].x[g] : ctx->a2_bf16 + (long long)g * b * F.D;
    }
    ok = ok && tconv_smem(f) > 0;
    // weight gradient: M = (tap, c') rows + the all-ones block (db), K = rows split into ranges
    TConvArgs& w = ctx->tc_wgrad[i];
    w.mode = TCONV_WGRAD; w.groups = 1; w.TCs = K; w.M = K + 64; w.BN = 64;
    w.T = T; w.Tw = G.Tw; w.Ws = G.Ws; w.HsWs = HsWs; w.Cblk = G.Cs / 64; w.maxshift = maxshift; w.R = 64 + maxshift;
    w.krows = rows; w.Nout = L.N;
    const long long chunks = (rows + 63) / 64;
    const int m_tiles = (w.M + 127) / 128;
    (void)m_tiles;  // every M tile of a K range shares its staged chunks: one range per CTA
    // one K range per SM (measured at BJ.configs[4]: 1/2, 1/4, 1/8 of the SMs with proportionally longer
    // ranges cost +21 / +74 / +187 us of conv backward: the per-chunk MMA work, not the partials, binds)
    w.ranges = (int)std::max<long long>(1, std::min<long long>(chunks, ctx->num_sms));
    w.kpr = (int)((chunks + w.ranges - 1) / w.ranges);
    w.ranges = (int)((chunks + w.kpr - 1) / w.kpr);
    ok = ok && L.N <= 64 && make_tmap_bf16(&w.ta[0], x[0], rows, G.Cs, G.Cs, w.R);
    ok = ok && make_tmap_bf16(&w.tb[0], ctx->dzp[i], rows, L.N, L.N, 64);
    ok = ok && tconv_smem(w) > 0;
    max_part += (long long)w.ranges * K * L.N;  // per-layer regions: two layers' weight gradients may overlap
    max_db += (long long)w.ranges * L.N;
    GConvWgradArgs& r = ctx->tc_wred[i];
    r.Th = G.Th; r.Tw = G.Tw; r.Cs = G.Cs; r.N = L.N; r.b = w.ranges; r.ipc = 1; r.first = i == 0;
    r.w_canon = G.w_canon; r.w_off = L.w_off; r.w_nstride = (long long)L.C * L.k * L.k; r.b_off = L.b_off;
    r.grad = ctx->grad; r.store = ctx->cfg.n_push == 1; r.part_cm = 1;
    // data gradient (layers after the first): A = this layer's dZ, B = the packed data-gradient weights
    if (i > 0) {
      TConvArgs& d = ctx->tc_dgrad[i];
      const dqn_ctx::GLayer& GP = ctx->gl[i - 1];
      d.mode = TCONV_DGRAD; d.groups = 1; d.M = (int)rows; d.BN = G.Cs;
      d.T = T; d.Tw = G.Tw; d.Ws = G.Ws; d.HsWs = HsWs; d.Cblk = L.N / 64; d.maxshift = maxshift;
      d.R = 128 + maxshift;
      d.xmask = G.x[0]; d.s = G.s; d.Cp = G.Cs / (G.s * G.s); d.Cs = G.Cs;
      d.prevWs = GP.Ws; d.prevHsWs = GP.Hs * GP.Ws;
      ok = ok && G.Cs <= 256 && make_tmap_bf16(&d.ta[0], ctx->dzp[i], rows, L.N, L.N, d.R);
      ok = ok && make_tmap_bf16(&d.tb[0], ctx->theta_local_bf16 + ctx->gpack_off + G.dg_pack, G.Cs, T * L.N,
                                T * L.N, G.Cs);
      ok = ok && tconv_smem(d) > 0;
    }
  }
  if (ok) {
    ok = !dalloc(ctx, &ctx->tc_part, max_part) && !dalloc(ctx, &ctx->tc_part_db, max_db);
    long long po = 0, pdo = 0;
    for (int i = 0; i < nl && ok; ++i) {
      TConvArgs& w = ctx->tc_wgrad[i];
      w.partial = ctx->tc_part + po; w.partial_db = ctx->tc_part_db + pdo;
      ctx->tc_wred[i].partial = w.partial; ctx->tc_wred[i].partial_db = w.partial_db;
      po += (long long)w.ranges * w.TCs * w.Nout;
      pdo += (long long)w.ranges * w.Nout;
      if (i > 0) ctx->tc_dgrad[i].dzprev = ctx->dzp[i - 1];
    }
    const char* cb = getenv("DQN_CONC_BWD");
    if (ok && nl >= 2 && !(cb && atoi(cb) == 0) &&
        cudaStreamCreateWithFlags(&ctx->bside, cudaStreamNonBlocking) == cudaSuccess &&
        cudaEventCreateWithFlags(&ctx->ev_bjoin, cudaEventDisableTiming) == cudaSuccess) {
      for (int i = 0; i < nl; ++i)
        if (cudaEventCreateWithFlags(&ctx->ev_bdz[i], cudaEventDisableTiming) != cudaSuccess) {
          cudaStreamDestroy(ctx->bside);
          ctx->bside = nullptr;
          break;
        }
    }
    // FC dX writes the last conv layer's dZ: coalesced into the canonical flatten, then chw_to_hwc permutes it
    // into the layer's input-grid geometry (a direct NHWC store from the GEMM epilogue is a 2-byte scatter with a
    // C-element stride across the warp: measured 33 us at BJ.configs[4])
    const dqn_ctx::GLayer& GL2 = ctx->gl[nl - 1];
    if (chw_to_hwc_fits(GL2.N, GL2.Ho, GL2.Wo) && !dalloc(ctx, &ctx->dx_canon, (long long)b * F.D)) {
      ctx->tg_dx.out_bf16 = ctx->dx_canon;
      ctx->tg_dx.hwc_HW = 0;
    } else {
      ctx->tg_dx.out_bf16 = ctx->dzp[nl - 1];
      ctx->tg_dx.hwc_Wo = GL2.Wo; ctx->tg_dx.hwc_Ws = GL2.Ws;
      ctx->tg_dx.ldo_out = (long long)GL2.Hs * GL2.Ws * GL2.N;
    }
  }
  ctx->use_tconv = ok;
}

// Generic bf16 conv path (kernels_conv.cu): layer geometry, packed-weight maps, buffers.
static int setup_gpath(dqn_ctx* ctx) {
  const NetShape& net = ctx->net;
  const int b = ctx->cfg.minibatch;
  int rc;
  init_bf16_kernel_attrs();
  init_conv_kernel_attrs();
  const FcShape& F = net.fc[0];
  // FC forward split-K (gemm_pipe): K per split a multiple of 16 dividing D, at most 8 chunks of 64
  ctx->fc_splits = 0;
  for (int sp = 1; sp <= F.D / 16; ++sp)
    if (F.D % sp == 0 && (F.D / sp) % 16 == 0 && F.D / sp <= 512) {
      ctx->fc_splits = sp;
      break;
    }
  if (!ctx->fc_splits || ctx->fc_splits > kHeadMaxSplits)  // the head sums at most kHeadMaxSplits partials
    return set_err(ctx, DQN_EINVAL, "DQN_BF16: the FC input D = " + std::to_string(F.D) + " needs " +
                                        (ctx->fc_splits ? std::to_string(ctx->fc_splits) : std::string("no valid")) +
                                        " split-K partials of <= 512 (a multiple of 16 dividing D); the TD head sums at most " +
                                        std::to_string(kHeadMaxSplits));
  long long pk = 0, max_part = 0, max_db = 0;
  std::vector<int2> map((size_t)(net.conv[net.n_conv - 1].b_off + net.conv[net.n_conv - 1].N), make_int2(-1, -1));
  for (int i = 0; i < net.n_conv; ++i) {
    const ConvShape& L = net.conv[i];
    dqn_ctx::GLayer& G = ctx->gl[i];
    const int s = i == 0 ? 4 : L.s;
    G.s = s;
    G.Hs = i == 0 ? 21 : L.H / s;
    G.Ws = i == 0 ? 21 : L.W / s;
    G.Cs = L.C * s * s;
    G.Th = G.Tw = L.k / s;
    G.Ho = L.Ho; G.Wo = L.Wo; G.N = L.N;
    const int T = G.Th * G.Tw, K = T * G.Cs;
    G.fwd_pack = pk;
    pk += (long long)L.N * K;
    G.dg_pack = -1;
    if (i > 0) {
      G.dg_pack = pk;
      pk += (long long)G.Cs * T * L.N;
    }
    const int mt = (K + 127) / 128;
    // weight-gradient CTAs per layer ≈ wg_ctas (image ranges × M tiles): 4 × 148 measured best on BJ.configs[4]
    // (296: 875 K, 444: 922 K, 592: 924 K, 888: 899 K tr/s); DQN_GCONV_WG_CTAS overrides
    static const int wg_ctas = getenv("DQN_GCONV_WG_CTAS") ? std::max(1, atoi(getenv("DQN_GCONV_WG_CTAS"))) : 592;
    const int ranges = std::max(1, std::min(b, wg_ctas / mt));
    G.ipc = (b + ranges - 1) / ranges;
    while (G.ipc > 1 && !gconv_wgrad_fits(L.N, i == 0, G.ipc, G.Ho * G.Wo)) --G.ipc;  // position table + ring
    if (!gconv_wgrad_fits(L.N, i == 0, G.ipc, G.Ho * G.Wo))
      return set_err(ctx, DQN_EINVAL, "DQN_BF16: conv layer " + std::to_string(i + 1) +
                                          " too large for the weight-gradient kernel's shared memory");
    const long long nr = (b + G.ipc - 1) / G.ipc;
    max_part = std::max(max_part, nr * K * L.N);
    max_db = std::max(max_db, nr * L.N);
    std::vector<int> canon((size_t)K, -1);
    for (int t = 0; t < T; ++t)
      for (int cs = 0; cs < G.Cs; ++cs) {
        int c, iy, ix;
        if (i == 0) {  // the ring's s2d order c' = f*16 + iy*4 + ix
          c = cs / 16; iy = (cs / 4) % 4; ix = cs % 4;
        } else {       // c' = (iy*s + ix)*C + c
          c = cs % L.C; iy = (cs / L.C) / s; ix = (cs / L.C) % s;
        }
        const int ky = (t / G.Tw) * s + iy, kx = (t % G.Tw) * s + ix;
        const int off = (c * L.k + ky) * L.k + kx;
        canon[(size_t)t * G.Cs + cs] = off;
        for (int n = 0; n < L.N; ++n) {
          int2& d = map[(size_t)(L.w_off + (long long)n * L.C * L.k * L.k + off)];
          d.x = (int)(G.fwd_pack + (long long)n * K + (long long)t * G.Cs + cs);
          if (i > 0) d.y = (int)(G.dg_pack + (long long)cs * T * L.N + (long long)t * L.N + n);
        }
      }
    if ((rc = dalloc(ctx, &G.w_canon, K))) return rc;
    CK(cudaMemcpy(G.w_canon, canon.data(), sizeof(int) * K, cudaMemcpyHostToDevice));
    if (i > 0)
      for (int g = 0; g < 2; ++g)
        if ((rc = dalloc(ctx, &G.x[g], (long long)b * G.Hs * G.Ws * G.Cs))) return rc;
    if ((rc = dalloc(ctx, &G.dz, (long long)b * L.Ho * L.Wo * L.N))) return rc;
  }
  ctx->pack_n = (long long)map.size();
  if ((rc = dalloc(ctx, &ctx->pack_map, ctx->pack_n))) return rc;
  CK(cudaMemcpy(ctx->pack_map, map.data(), sizeof(int2) * map.size(), cudaMemcpyHostToDevice));
  ctx->img_off = -1;  // no Mnih weight image
  ctx->gpack_off = ctx->P_pad;
  ctx->P_bf16 = ctx->P_pad + pk;
  if ((rc = dalloc(ctx, &ctx->theta_local_bf16, ctx->P_bf16))) return rc;
  if ((rc = dalloc(ctx, &ctx->theta_hat_bf16, ctx->P_bf16))) return rc;
  if ((rc = dalloc(ctx, &ctx->a2_bf16, 2LL * b * F.D))) return rc;
  if ((rc = dalloc(ctx, &ctx->dh_bf16, (long long)b * F.H))) return rc;
  if ((rc = dalloc(ctx, &ctx->fc_partial, 2LL * ctx->fc_splits * F.H * b))) return rc;
  if ((rc = dalloc(ctx, &ctx->tc_counters, 64))) return rc;
  CK(cudaMemsetAsync(ctx->tc_counters, 0, 64 * sizeof(unsigned), ctx->stream));
  if ((rc = dalloc(ctx, &ctx->q_stage_s2d, (long long)b * kMnihSlot))) return rc;
  if ((rc = dalloc(ctx, &ctx->gw_partial, max_part))) return rc;
  if ((rc = dalloc(ctx, &ctx->gw_partial_db, max_db))) return rc;
  setup_tgemm_fc(ctx);
  return DQN_OK;
}

static long long align16(long long x) { return (x + 15) & ~15LL; }

static int create_impl(dqn_ctx* ctx, const dqn_config* cfg, int rank, int world, const void* nccl_unique_id,
                       void* cuda_stream) {
  ctx->cfg = *cfg;
  ctx->cfg.init_params = nullptr;
  std::string why;
  int rc = validate_cfg(cfg, &ctx->net, &why);
  if (rc) return set_err(ctx, rc, why);
  ctx->rank = rank;
  ctx->world = world;
  const NetShape& net = ctx->net;
  const int b = cfg->minibatch;
  ctx->P = net.P;
  const long long unit = 64LL * world;
  ctx->P_pad = (net.P + unit - 1) / unit * unit;
  ctx->shard = ctx->P_pad / world;
  ctx->cap = cfg->replay_capacity;
  ctx->use_graphs = !(getenv("DQN_NO_GRAPH") && atoi(getenv("DQN_NO_GRAPH")));
  ctx->keep_grad = cfg->keep_grad != 0;
  ctx->async = cfg->sync_mode == DQN_ASYNC || cfg->sync_mode == DQN_ASYNC_LAG1;
  ctx->async_lag1 = cfg->sync_mode == DQN_ASYNC_LAG1;
  ctx->alias_local = (world == 1 && cfg->n_fetch == 1 && !ctx->async);
  ctx->bf16 = cfg->precision == DQN_BF16;
  ctx->gpath = ctx->bf16 && !is_mnih_stack(cfg);

  if (cuda_stream) {
    ctx->stream = (cudaStream_t)cuda_stream;
  } else {
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamDefault));  // blocking: ordered after legacy-stream producers
    ctx->own_stream = true;
  }
  {  // host-push staging (pinned, double-buffered) and the pinned landing zone of train outputs
    const long long sb = ctx->net.state_bytes;
    ctx->push_chunk = std::min<long long>(ctx->cap, std::max<long long>(1, (4LL << 20) / (2 * sb + 12)));
    const long long bytes = align16(2 * ctx->push_chunk * sb) + 3 * align16(4 * ctx->push_chunk);
    if ((rc = dalloc(ctx, &ctx->d_stage, bytes + 256))) return rc;  // (+ the two halves' alignment slack)
    CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CK(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_stage[i]), bytes, cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&ctx->ev_stage[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_copied[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_consumed[i], cudaEventDisableTiming));
    }
    CK(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_out), sizeof(dqn_ctx::HostOut), cudaHostAllocDefault));
  }
  if (const char* v = getenv("DQN_EARLY_UPDATE")) ctx->early_update = atoi(v) != 0;
  {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
      ctx->num_sms = sms;
  }
  if (const char* v = getenv("DQN_TRACE_STEP")) {
    if (atoi(v)) {
      ctx->step_trace = true;
      step_trace_bf16(1, nullptr);
      step_trace_head(1, nullptr);
      step_trace_common(1, nullptr);
      step_trace_comm(1, nullptr);
    }
  }
  CK(cudaEventCreate(&ctx->ev0));
  CK(cudaEventCreate(&ctx->ev1));
  init_f32_kernel_attrs();

  // replay memory: both stacks of every experience, action, reward, terminal flag
  const long long sb = net.state_bytes, fb = sb / net.F;
  ctx->dedup = cfg->replay_dedup != 0;
  ctx->slot_stride = ctx->dedup ? sb + fb : sb;
  if ((rc = dalloc(ctx, &ctx->ring_s, ctx->cap * ctx->slot_stride))) return rc;
  if (ctx->dedup) ctx->ring_sn = ctx->ring_s + fb;
  else if ((rc = dalloc(ctx, &ctx->ring_sn, ctx->cap * sb))) return rc;
  if ((rc = dalloc(ctx, &ctx->ring_t, ctx->cap))) return rc;
  if ((rc = dalloc(ctx, &ctx->ring_a, ctx->cap))) return rc;
  if ((rc = dalloc(ctx, &ctx->ring_r, ctx->cap))) return rc;

  // parameters and server shards
  if ((rc = dalloc(ctx, &ctx->theta_master, ctx->alias_local ? ctx->P_pad : ctx->shard))) return rc;
  if ((rc = dalloc(ctx, &ctx->rms, ctx->shard))) return rc;
  if ((rc = dalloc(ctx, &ctx->grad, ctx->P_pad))) return rc;
  if (world > 1 && (rc = dalloc(ctx, &ctx->g_shard, ctx->shard))) return rc;
  if (world > 1 && (rc = dalloc(ctx, &ctx->gather_tmp, ctx->P_pad))) return rc;
  if (ctx->alias_local) ctx->theta_local = ctx->theta_master;
  else if ((rc = dalloc(ctx, &ctx->theta_local, ctx->P_pad))) return rc;
  if ((rc = dalloc(ctx, &ctx->theta_hat, ctx->P_pad))) return rc;
  if (ctx->keep_grad && (rc = dalloc(ctx, &ctx->grad_snap, ctx->P_pad))) return rc;
  CK(cudaMemsetAsync(ctx->rms, 0, sizeof(float) * ctx->shard, ctx->stream));
  CK(cudaMemsetAsync(ctx->grad, 0, sizeof(float) * ctx->P_pad, ctx->stream));

  // activations / gradients of activations
  long long max_partial = 0;
  for (int i = 0; i < net.n_conv; ++i) {
    const ConvShape& L = net.conv[i];
    const long long per = (long long)L.N * L.Ho * L.Wo;
    for (int g = 0; g < 2; ++g)
      if ((rc = dalloc(ctx, &ctx->act_conv[i][g], per * b))) return rc;
    if ((rc = dalloc(ctx, &ctx->dz_conv[i], per * b))) return rc;
    max_partial = std::max(max_partial, (long long)b * ((long long)L.N * L.C * L.k * L.k + L.N));
  }
  for (int i = 0; i <= net.n_fc; ++i) {
    const FcShape& F = net.fc[i];
    if (i < net.n_fc) {
      for (int g = 0; g < 2; ++g)
        if ((rc = dalloc(ctx, &ctx->act_fc[i][g], (long long)F.H * b))) return rc;
      if ((rc = dalloc(ctx, &ctx->dz_fc[i], (long long)F.H * b))) return rc;
      const int s_fwd = pick_splits(b, F.H, F.D, 2);
      max_partial = std::max(max_partial, 2LL * s_fwd * b * F.H);
      const int s_dx = pick_splits(b, F.D, F.H, 1);
      max_partial = std::max(max_partial, (long long)s_dx * b * F.D);
    }
  }
  const long long qn = std::max(b, 1);
  max_partial = std::max(max_partial, 2LL * pick_splits(qn, net.fc[0].H, net.fc[0].D, 1) * qn * net.fc[0].H);
  ctx->partial_elems = max_partial;
  if ((rc = dalloc(ctx, &ctx->partial, max_partial))) return rc;
  if ((rc = dalloc(ctx, &ctx->idx, b))) return rc;
  if ((rc = dalloc(ctx, &ctx->head_dq, b))) return rc;
  if ((rc = dalloc(ctx, &ctx->head_act, b))) return rc;
  if ((rc = dalloc(ctx, &ctx->head_loss, b))) return rc;
  if ((rc = dalloc(ctx, &ctx->head_delta, b))) return rc;
  if ((rc = dalloc(ctx, &ctx->diag_delta, (long long)kDiagSteps * b))) return rc;
  if (cfg->replay_prio_alpha != 0.0) {  // the 32-ary sum tree: 32^K leaves (0 = never stored), K levels above
    ctx->prio = true;
    ctx->prio_alpha_half = cfg->replay_prio_alpha == 0.5;
    ctx->prio_eps = (float)cfg->replay_prio_eps;
    int K = 1;
    long long L = 32;
    while (L < ctx->cap) { L *= 32; ++K; }
    ctx->ptree.K = K;
    long long off = 0;
    for (int l = 0; l <= K; ++l) {
      ctx->ptree.off[l] = off;
      off += L;
      L /= 32;
    }
    if ((rc = dalloc(ctx, &ctx->ptree.node, off))) return rc;
    CK(cudaMemsetAsync(ctx->ptree.node, 0, sizeof(float) * off, ctx->stream));
    if ((rc = dalloc(ctx, &ctx->prio_maxp, 1))) return rc;
    const float one = 1.0f;
    CK(cudaMemcpyAsync(ctx->prio_maxp, &one, sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  if ((rc = dalloc(ctx, &ctx->ctr, 1))) return rc;
  CK(cudaMemsetAsync(ctx->ctr, 0, sizeof(DevCounters), ctx->stream));
  if ((rc = dalloc(ctx, &ctx->diag_loss, kDiagSteps))) return rc;
  if ((rc = dalloc(ctx, &ctx->diag_idx, (long long)kDiagSteps * b))) return rc;
  if ((rc = dalloc(ctx, &ctx->diag_amax, (long long)kDiagSteps * b))) return rc;
  if ((rc = dalloc(ctx, &ctx->q_stage, qn * sb))) return rc;
  if ((rc = dalloc(ctx, &ctx->q_out, qn * net.A))) return rc;
  if ((rc = dalloc(ctx, &ctx->q_amax, qn))) return rc;
  init_head_kernel_attrs();
  if (ctx->gpath && (rc = setup_gpath(ctx))) return rc;
  if (ctx->bf16 && !ctx->gpath) {
    init_bf16_kernel_attrs();
    init_conv_kernel_attrs();  // gemm_pipe: the FC backward of FC layers too wide for tc_pair
    const int H = net.fc[0].H;
    ctx->fc_splits = 18;  // K = 2592 = 18 x 144
    ctx->img_off = ctx->P_pad;
    ctx->P_bf16 = ctx->P_pad + kWimgElems;
    ctx->w1_off = net.conv[0].w_off;
    ctx->w2_off = net.conv[1].w_off;
    if ((rc = dalloc(ctx, &ctx->theta_local_bf16, ctx->P_bf16))) return rc;
    if ((rc = dalloc(ctx, &ctx->theta_hat_bf16, ctx->P_bf16))) return rc;
    if ((rc = dalloc(ctx, &ctx->a2_bf16, 2LL * b * 2592))) return rc;
    if ((rc = dalloc(ctx, &ctx->a1_save, (long long)b * kA1Bytes))) return rc;
    if ((rc = dalloc(ctx, &ctx->dh_bf16, (long long)b * H))) return rc;
    if ((rc = dalloc(ctx, &ctx->dz2_bf16, (long long)b * 2592))) return rc;
    if ((rc = dalloc(ctx, &ctx->fc_partial, 2LL * ctx->fc_splits * H * b))) return rc;
    if ((rc = dalloc(ctx, &ctx->tc_counters, 64))) return rc;
    CK(cudaMemsetAsync(ctx->tc_counters, 0, 64 * sizeof(unsigned), ctx->stream));
    if ((rc = dalloc(ctx, &ctx->bwd_partial, (long long)b * kBwdPart))) return rc;
    if ((rc = dalloc(ctx, &ctx->q_stage_s2d, (long long)b * kMnihSlot))) return rc;
  }

  // initial theta (Alg. 2): init_params or N(0, xi^2) from init_seed; theta^ = theta
  std::vector<float> th((size_t)ctx->P_pad, 0.0f);
  if (cfg->init_params) {
    if (is_device_ptr(cfg->init_params)) {
      CK(cudaMemcpy(th.data(), cfg->init_params, sizeof(float) * net.P, cudaMemcpyDeviceToHost));
    } else {
      std::memcpy(th.data(), cfg->init_params, sizeof(float) * net.P);
    }
  } else {
    std::vector<float> g((size_t)net.P);
    gaussian_init(g, cfg->init_std, cfg->init_seed);
    std::memcpy(th.data(), g.data(), sizeof(float) * net.P);
  }
  if (ctx->alias_local) {
    CK(cudaMemcpyAsync(ctx->theta_master, th.data(), sizeof(float) * ctx->P_pad, cudaMemcpyHostToDevice, ctx->stream));
  } else {
    CK(cudaMemcpyAsync(ctx->theta_master, th.data() + ctx->shard * rank, sizeof(float) * ctx->shard,
                       cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->theta_local, th.data(), sizeof(float) * ctx->P_pad, cudaMemcpyHostToDevice, ctx->stream));
  }
  CK(cudaMemcpyAsync(ctx->theta_hat, th.data(), sizeof(float) * ctx->P_pad, cudaMemcpyHostToDevice, ctx->stream));
  if (ctx->bf16) {
    launch_f32_to_bf16(ctx->theta_hat, ctx->theta_local_bf16, ctx->P_pad, ctx->stream, ctx->img_off, ctx->w1_off,
                       ctx->w2_off);
    launch_f32_to_bf16(ctx->theta_hat, ctx->theta_hat_bf16, ctx->P_pad, ctx->stream, ctx->img_off, ctx->w1_off,
                       ctx->w2_off);
    if (ctx->gpath) {
      launch_gpack(ctx->theta_hat, ctx->theta_local_bf16, ctx->gpack_off, ctx->pack_map, ctx->pack_n, ctx->stream);
      launch_gpack(ctx->theta_hat, ctx->theta_hat_bf16, ctx->gpack_off, ctx->pack_map, ctx->pack_n, ctx->stream);
    }
    CK(cudaGetLastError());
  }
  if (ctx->async) {  // theta^(0) published in slot 0 (pub_gen = 0); the comm stream and its events
    CK(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_grad, cudaEventDisableTiming));
    for (int i = 0; i < 3; ++i) {
      CK(cudaEventCreateWithFlags(&ctx->ev_pub[i], cudaEventDisableTiming));
      if ((rc = dalloc(ctx, &ctx->theta_pub[i], ctx->P_pad))) return rc;
      if (ctx->bf16 && (rc = dalloc(ctx, &ctx->theta_pub_bf16[i], ctx->P_bf16))) return rc;
    }
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&ctx->ev_send[i], cudaEventDisableTiming));
      if ((rc = dalloc(ctx, &ctx->g_send[i], ctx->P_pad))) return rc;
      CK(cudaEventRecord(ctx->ev_send[i], ctx->stream));
    }
    if (cfg->server_rule == DQN_SERVER_PER_GRADIENT && world > 1 &&
        (rc = dalloc(ctx, &ctx->inbox, (long long)world * ctx->shard)))
      return rc;
    if ((rc = dalloc(ctx, &ctx->adev, 1))) return rc;
    CK(cudaMemsetAsync(ctx->adev, 0, sizeof(AsyncDev), ctx->stream));
    CK(cudaHostAlloc(reinterpret_cast<void**>(&ctx->h_adev), sizeof(AsyncDev), cudaHostAllocDefault));
    std::memset(ctx->h_adev, 0, sizeof(AsyncDev));
    CK(cudaMemcpyAsync(ctx->theta_pub[0], ctx->theta_hat, sizeof(float) * ctx->P_pad, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    if (ctx->bf16)
      CK(cudaMemcpyAsync(ctx->theta_pub_bf16[0], ctx->theta_local_bf16, sizeof(__nv_bfloat16) * ctx->P_bf16,
                         cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaEventRecord(ctx->ev_pub[0], ctx->stream));
    if (const char* v = getenv("DQN_ASYNC_DELAY_US")) ctx->async_delay_ns = (unsigned)std::max(0, atoi(v)) * 1000u;
  }
  CK(cudaStreamSynchronize(ctx->stream));

  if (world > 1) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    // deterministic schedule: the reduce-scatter's summation order must not change from run to run, so the
    // algorithm and protocol are pinned unless the caller set them; NCCL reads both at
    // communicator creation
    if (!ctx->async) {
      setenv("NCCL_ALGO", "Ring", 0);
      setenv("NCCL_PROTO", "Simple", 0);
    }
    NK(ncclCommInitRank(&ctx->comm, world, id, rank));
    const char* fe = getenv("DQN_FUSED_COMM");
    ctx->fused_comm = !ctx->async && cfg->n_fetch == 1 && world <= kMaxWorld && !(fe && atoi(fe) == 0);
    if (cfg->server_rule == DQN_SERVER_PER_GRADIENT && !ctx->fused_comm && !ctx->async)
      return set_err(ctx, DQN_EINVAL, "DQN_SERVER_PER_GRADIENT with N > 1: the fused server round (deterministic, "
                                      "n_fetch = 1) or DQN_ASYNC*");
    if (ctx->fused_comm && (rc = setup_fused_comm(ctx))) return rc;
    if (ctx->bf16 && !ctx->fused_comm) {
      FetchRecord& f = ctx->frec;
      f.world = world; f.rank = rank; f.shard = ctx->shard;
      f.fw_lo = net.fc[0].w_off;
      f.fw_hi = net.fc[0].w_off + (long long)net.fc[0].H * net.fc[0].D;
      long long mx = 0;
      for (int p = 0; p < world; ++p) {
        const long long lo = (long long)p * ctx->shard, hi = lo + ctx->shard;
        const long long fw = std::max(0LL, std::min(hi, f.fw_hi) - std::max(lo, f.fw_lo));
        mx = std::max(mx, ctx->shard - fw);
      }
      f.rec_f32 = (mx + 3) / 4 * 4;
      f.rec_bytes = 2 * ctx->shard + 4 * f.rec_f32;
      f.img_off = ctx->img_off; f.w1_off = ctx->w1_off; f.w2_off = ctx->w2_off;
      if ((rc = dalloc(ctx, &ctx->fetch_send, f.rec_bytes))) return rc;
      if ((rc = dalloc(ctx, &ctx->fetch_recv, f.rec_bytes * world))) return rc;
      ctx->fetch_bf16 = true;
    }
  }
  ctx->n_per_round = cfg->server_rule == DQN_SERVER_PER_GRADIENT ? world : 1;  // n += 1 per applied gradient (A22)
  return DQN_OK;
}

extern "C" int dqn_create(const dqn_config* cfg, int rank, int world, const void* nccl_unique_id, void* cuda_stream,
                          dqn_ctx** out) {
  g_create_err.clear();
  if (!out) return DQN_EINVAL;
  *out = nullptr;
  if (!cfg || world < 1 || rank < 0 || rank >= world || (world > 1 && !nccl_unique_id)) {
    g_create_err = "bad create arguments";
    return DQN_EINVAL;
  }
  dqn_ctx* ctx = new dqn_ctx();
  int rc = create_impl(ctx, cfg, rank, world, nccl_unique_id, cuda_stream);
  if (rc) {
    g_create_err = ctx->err;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    free_all(ctx);
    delete ctx;
    return rc;
  }
  *out = ctx;
  return DQN_OK;
}

// ------------------------------------------------------------------ push (Alg. 1 "Store")
// Items [i0, i0+m) of the call (device pointers to their first element) go to slots
// (count + i0 + i) mod cap; the bf16 path stores conv1's space-to-depth layout.
// items [i0, i0 + m) of this call into their ring slots; the kernel also publishes the replay
// size after them (min(count, cap), read by the sampler)
static void push_ring(dqn_ctx* ctx, long long i0, long long m, const uint8_t* s, const int32_t* a, const float* r,
                      const uint8_t* sn, const uint8_t* t) {
  const long long size = std::min(ctx->count + i0 + m, ctx->cap);
  long long* size_out = &ctx->ctr->ring_size;
  if (ctx->bf16)
    launch_push_s2d(ctx->ring_s, ctx->ring_sn, ctx->ring_a, ctx->ring_r, ctx->ring_t, ctx->cap, ctx->count, i0, m, s,
                    a, r, sn, t, ctx->stream, size_out, size, ctx->slot_stride, ctx->dedup);
  else
    launch_push_canonical(ctx->ring_s, ctx->ring_sn, ctx->ring_a, ctx->ring_r, ctx->ring_t, ctx->cap, ctx->count, 0,
                          i0, m, ctx->net.state_bytes, s, a, r, sn, t, ctx->stream, size_out, size, ctx->slot_stride,
                          ctx->dedup);
  // prioritized replay: the stored slots enter with the largest priority so far (A41)
  if (ctx->prio) launch_prio_push(ctx->ptree, ctx->cap, (ctx->count + i0) % ctx->cap, m, ctx->prio_maxp, ctx->stream);
}


static int run_steps_chunked(dqn_ctx* ctx, long long k, long long* kernels, bool store = false);

// Alg. 1 "Store" of n items (host or device buffers). With `steps` != nullptr (dqn_store_and_train) every
// item is stored and then one replica step runs (Alg. 1's loop): push_ring(item i) followed by
// the one-step graph, no host synchronisation; *steps counts the kernels launched.
static int push_impl(dqn_ctx* ctx, int64_t n, const uint8_t* s, const int32_t* a, const float* r,
                     const uint8_t* s_next, const uint8_t* terminal, long long* steps) {
  if (!ctx) return DQN_EINVAL;
  if (ctx->poisoned) return DQN_ESTATE;
  if (n < 0 || (n > 0 && (!s || !a || !r || !s_next || !terminal))) return set_err(ctx, DQN_EINVAL, "bad push args");
  if (n == 0) return DQN_OK;
  const long long sb = ctx->net.state_bytes;
  const bool dev = is_device_ptr(s);
  if (dev != is_device_ptr(a) || dev != is_device_ptr(r) || dev != is_device_ptr(s_next) ||
      dev != is_device_ptr(terminal))
    return set_err(ctx, DQN_EINVAL, "push buffers must all be host or all be device memory");
  // only the last min(n, cap) items survive; item i goes to slot (count + i) mod cap (interleaved with
  // steps, every item is sampled from before it is overwritten, so all are stored)
  const long long first = n > ctx->cap && !steps ? n - ctx->cap : 0;
  // push items [i0, i0 + m) (device pointers to item i0), then, interleaved, one step after each item
  auto store = [&](long long i0, long long m, const uint8_t* ds, const int32_t* da, const float* dr, const uint8_t* dsn,
                   const uint8_t* dt) -> int {
    if (!steps) {
      push_ring(ctx, i0, m, ds, da, dr, dsn, dt);
      CK(cudaGetLastError());
      return DQN_OK;
    }
    if (ctx->graph_store) {  // the Store runs as the first kernel of each step of the replayed graphs
      launch_store_ctl(ctx->store_ctl, ds, dsn, da, dr, dt, ctx->T, ctx->count + i0, ctx->stream);
      CK(cudaGetLastError());
      *steps += 1;
      const long long c0 = ctx->count;
      ctx->count = c0 + i0 + m;
      const int rc = run_steps_chunked(ctx, m, steps, true);
      ctx->count = c0;
      return rc;
    }
    for (long long j = 0; j < m; ++j) {
      push_ring(ctx, i0 + j, 1, ds + j * sb, da + j, dr + j, dsn + j * sb, dt + j);
      CK(cudaGetLastError());
      const long long c0 = ctx->count;
      ctx->count = c0 + i0 + j + 1;  // the step sees the item (EEMPTY checks, graph planning)
      const int rc = run_steps_chunked(ctx, 1, steps);
      ctx->count = c0;
      if (rc) return rc;
    }
    return DQN_OK;
  };
  if (!dev) {
    for (long long i = 0; i < n; ++i)
      if (a[i] < 0 || a[i] >= ctx->net.A || !std::isfinite(r[i]))
        return set_err(ctx, DQN_EINVAL, "action out of range or non-finite reward at item " + std::to_string(i));
    if (ctx->dedup) {  // s'[0..F-2] must be s[1..F-1] (frames shared; only s'[F-1] is stored)
      const long long fb = sb / ctx->net.F;
      for (long long i = first; i < n; ++i)
        if (std::memcmp(s_next + i * sb, s + i * sb + fb, (size_t)(sb - fb)) != 0)
          return set_err(ctx, DQN_EINVAL, "replay_dedup: s' is not s shifted by one frame at item " + std::to_string(i));
    }
    // chunk layout (host pinned and device): s [m][sb] | s' [m][sb] | a [m] i32 | r [m] f32 | term [m] u8
    if (steps && ctx->copy_stream && ctx->push_chunk >= 2) {  // (two halves of >= 1 item each)
      // Alg. 1's loop: sub-chunks of the caller's transitions are copied (DMA when pinned; the call synchronises
      // before returning) into alternate halves of d_stage on copy_stream, overlapping the previous sub-chunk's
      // steps on the context stream
      const long long sc = std::max<long long>(1, std::min<long long>(16, ctx->push_chunk / 2));
      const long long half = align16(2 * sc * sb) + 3 * align16(4 * sc);
      int buf = 0;
      for (long long i0 = first; i0 < n; i0 += sc, buf ^= 1) {
        const long long m = std::min(sc, n - i0);
        const long long o_sn = m * sb, o_a = align16(2 * m * sb), o_r = o_a + align16(4 * m), o_t = o_r + align16(4 * m);
        uint8_t* d = ctx->d_stage + buf * half;
        cudaStream_t cs = ctx->copy_stream;
        CK(cudaStreamWaitEvent(cs, ctx->ev_consumed[buf], 0));  // the steps of two sub-chunks back are done with it
        CK(cudaMemcpyAsync(d, s + i0 * sb, m * sb, cudaMemcpyHostToDevice, cs));
        CK(cudaMemcpyAsync(d + o_sn, s_next + i0 * sb, m * sb, cudaMemcpyHostToDevice, cs));
        CK(cudaMemcpyAsync(d + o_a, a + i0, m * sizeof(int32_t), cudaMemcpyHostToDevice, cs));
        CK(cudaMemcpyAsync(d + o_r, r + i0, m * sizeof(float), cudaMemcpyHostToDevice, cs));
        CK(cudaMemcpyAsync(d + o_t, terminal + i0, m, cudaMemcpyHostToDevice, cs));
        CK(cudaEventRecord(ctx->ev_copied[buf], cs));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[buf], 0));
        int rc = store(i0, m, d, reinterpret_cast<const int32_t*>(d + o_a), reinterpret_cast<const float*>(d + o_r),
                       d + o_sn, d + o_t);
        if (rc) return rc;
        CK(cudaEventRecord(ctx->ev_consumed[buf], ctx->stream));
      }
      ctx->count += n;
      return DQN_OK;
    }
    for (long long i0 = first; i0 < n; i0 += ctx->push_chunk) {
      const long long m = std::min(ctx->push_chunk, n - i0);
      const long long o_sn = m * sb, o_a = align16(2 * m * sb), o_r = o_a + align16(4 * m), o_t = o_r + align16(4 * m);
      uint8_t* d = ctx->d_stage;
      if (steps) {
        // dqn_store_and_train synchronises before returning, so the copies may read the caller's buffers
        // directly (DMA when they are pinned); no host-side packing
        CK(cudaMemcpyAsync(d, s + i0 * sb, m * sb, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(d + o_sn, s_next + i0 * sb, m * sb, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(d + o_a, a + i0, m * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(d + o_r, r + i0, m * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(d + o_t, terminal + i0, m, cudaMemcpyHostToDevice, ctx->stream));
      } else {
        const int buf = ctx->stage_flip;
        ctx->stage_flip ^= 1;
        CK(cudaEventSynchronize(ctx->ev_stage[buf]));  // its previous H2D copy has drained
        uint8_t* h = ctx->h_stage[buf];
        std::memcpy(h, s + i0 * sb, m * sb);
        std::memcpy(h + o_sn, s_next + i0 * sb, m * sb);
        std::memcpy(h + o_a, a + i0, m * sizeof(int32_t));
        std::memcpy(h + o_r, r + i0, m * sizeof(float));
        std::memcpy(h + o_t, terminal + i0, m);
        CK(cudaMemcpyAsync(d, h, o_t + m, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaEventRecord(ctx->ev_stage[buf], ctx->stream));
      }
      int rc = store(i0, m, d, reinterpret_cast<const int32_t*>(d + o_a), reinterpret_cast<const float*>(d + o_r),
                     d + o_sn, d + o_t);
      if (rc) return rc;
    }
    ctx->count += n;  // enqueued: the sampler of any later step reads the published size in stream order
    return DQN_OK;
  } else {
    CK(cudaMemsetAsync(&ctx->ctr->bad_input, 0, sizeof(unsigned), ctx->stream));
    launch_validate_push(a, r, n, ctx->net.A, ctx->ctr, ctx->stream);
    if (ctx->dedup) launch_validate_dedup(s, s_next, n, sb, sb / ctx->net.F, ctx->ctr, ctx->stream);
    unsigned bad = 0;
    CK(cudaMemcpyAsync(&bad, &ctx->ctr->bad_input, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (bad) return set_err(ctx, DQN_EINVAL, "action out of range, non-finite reward or (replay_dedup) s' not s "
                                               "shifted by one frame in device push");
    for (long long i0 = first; i0 < n; i0 += 65535) {
      const long long m = std::min<long long>(65535, n - i0);
      int rc = store(i0, m, s + i0 * sb, a + i0, r + i0, s_next + i0 * sb, terminal + i0);
      if (rc) return rc;
    }
  }
  ctx->count += n;
  if (!steps) CK(cudaStreamSynchronize(ctx->stream));  // device inputs: read by the ring kernel before returning
  return DQN_OK;
}

extern "C" int dqn_push_transitions(dqn_ctx* ctx, int64_t n, const uint8_t* s, const int32_t* a, const float* r,
                                    const uint8_t* s_next, const uint8_t* terminal) {
  return push_impl(ctx, n, s, a, r, s_next, terminal, nullptr);
}


// ------------------------------------------------------------------ profiling marks
// (only while capturing a profiling variant: bit 8; the in-graph Store variants carry bit 16)
static bool prof_on(const dqn_ctx* ctx) { return ctx->capture_variant >= 0 && (ctx->capture_variant & 8); }
static void prof_begin(dqn_ctx* ctx, const std::string& name, int kernels) {
  if (!prof_on(ctx)) return;
  dqn_ctx::ProfMark m{name, nullptr, nullptr, kernels};
  cudaEventCreate(&m.a);
  cudaEventCreate(&m.b);
  cudaEventRecordWithFlags(m.a, ctx->stream, cudaEventRecordExternal);  // a real event node in the graph
  ctx->marks[ctx->capture_variant & 15].push_back(m);
}
static void prof_end(dqn_ctx* ctx) {
  if (!prof_on(ctx)) return;
  cudaEventRecordWithFlags(ctx->marks[ctx->capture_variant & 15].back().b, ctx->stream, cudaEventRecordExternal);
}
#define PB(name, k) prof_begin(ctx, name, k)
#define PE() prof_end(ctx)

// prioritized replay (A41): the draws of step T (before the forward) and the priority update after the TD head
static void enqueue_prio_sample(dqn_ctx* ctx, cudaStream_t st) {
  PB("prio_sample", 1);
  launch_prio_sample(ctx->ptree, ctx->cfg.minibatch, ctx->cfg.seed, (unsigned)ctx->rank, ctx->ctr, ctx->idx, st);
  PE();
}
static void enqueue_prio_update(dqn_ctx* ctx, cudaStream_t st) {
  if (!ctx->prio) return;
  PB("prio_update", 1);
  launch_prio_update(ctx->ptree, ctx->cfg.minibatch, ctx->idx, ctx->head_delta, ctx->prio_alpha_half, ctx->prio_eps,
                     ctx->prio_maxp, st);
  PE();
}


// a13 on the bf16 path over NCCL: pack this rank's record, one all-gather, unpack every rank's record into
// the working copies (fp32 entries outside the FC weight, bf16 everywhere + the conv weight image)
static int enqueue_fetch_bf16(dqn_ctx* ctx, cudaStream_t st, float* dst, __nv_bfloat16* dst_bf16) {
  launch_fetch_pack(ctx->theta_master, ctx->frec, ctx->fetch_send, st);
  NK(ncclAllGather(ctx->fetch_send, ctx->fetch_recv, (size_t)ctx->frec.rec_bytes, ncclChar, ctx->comm, st));
  launch_fetch_unpack(ctx->fetch_recv, ctx->frec, dst, dst_bf16, st);
  CK(cudaGetLastError());
  return DQN_OK;
}

// ------------------------------------------------------------------ one replica step (fp32 path)
// Enqueue the kernels of one step T on ctx->stream (captured into a graph).
static int enqueue_step_f32(dqn_ctx* ctx, bool fetch, bool refresh, bool push) {
  const NetShape& net = ctx->net;
  const dqn_config& c = ctx->cfg;
  const int b = c.minibatch;
  cudaStream_t st = ctx->stream;
  // a13 fetch + a14 target refresh
  if (fetch) {
    if (ctx->fused_comm) {
      // delivered into theta_local by the previous round's fused server-round kernel (NEXT-1)
    } else if (ctx->world > 1) {
      PB("fetch_all_gather", 0);
      NK(ncclAllGather(ctx->theta_master, ctx->theta_local, (size_t)ctx->shard, ncclFloat, ctx->comm, st));
      PE();
    } else if (!ctx->alias_local) {
      PB("fetch_copy", 0);
      CK(cudaMemcpyAsync(ctx->theta_local, ctx->theta_master, sizeof(float) * ctx->P_pad, cudaMemcpyDeviceToDevice, st));
      PE();
    }
  }
  if (refresh) {  // right after a fetch (the async mode's fetch is enqueued ahead of the graph)
    PB("target_refresh", 0);
    CK(cudaMemcpyAsync(ctx->theta_hat, ctx->theta_local, sizeof(float) * ctx->P_pad, cudaMemcpyDeviceToDevice, st));
    PE();
  }
  if (ctx->fused_comm) {  // the previous round's deliveries into theta_local, then clear G
    PB("server_round_acquire", 1);
    launch_fused_round_acquire(ctx->acq, st);
    PE();
  }
  // a1 sample
  PB("sample", 1);
  if (ctx->prio) launch_prio_sample(ctx->ptree, b, c.seed, (unsigned)ctx->rank, ctx->ctr, ctx->idx, st);
  else launch_sample(ctx->idx, b, c.seed, (unsigned)ctx->rank, ctx->ctr, st);
  PE();
  // a2-a4 convolutions, theta on s and theta^ on s' in one launch per layer
  ImgSrc src0{};
  src0.u8[0] = ctx->ring_s;
  src0.u8[1] = ctx->ring_sn;
  src0.idx = ctx->idx;
  src0.stride = ctx->slot_stride;
  for (int i = 0; i < net.n_conv; ++i) {
    ImgSrc src = src0;
    if (i > 0) {
      src = ImgSrc{};
      src.f32[0] = ctx->act_conv[i - 1][0];
      src.f32[1] = ctx->act_conv[i - 1][1];
      const ConvShape& P = net.conv[i - 1];
      src.stride = (long long)P.N * P.Ho * P.Wo;
    }
    PB("conv" + std::to_string(i + 1) + "_fwd", 1);
    launch_conv_fwd_f32(net.conv[i], src, ctx->theta_local, ctx->theta_hat, ctx->act_conv[i][0], ctx->act_conv[i][1],
                        b, 2, st);
    PE();
  }
  // a5 hidden FC layers
  const ConvShape& LC = net.conv[net.n_conv - 1];
  const float* in[2] = {ctx->act_conv[net.n_conv - 1][0], ctx->act_conv[net.n_conv - 1][1]};
  for (int l = 0; l < net.n_fc; ++l) {
    const FcShape& F = net.fc[l];
    GemmArgs g{};
    g.A[0] = in[0]; g.A[1] = in[1]; g.sam = F.D; g.sak = 1;
    g.B[0] = ctx->theta_local + F.w_off; g.B[1] = ctx->theta_hat + F.w_off; g.sbk = 1; g.sbn = F.D;
    g.C[0] = ctx->act_fc[l][0]; g.C[1] = ctx->act_fc[l][1]; g.scm = F.H; g.scn = 1;
    g.bias[0] = ctx->theta_local + F.b_off; g.bias[1] = ctx->theta_hat + F.b_off;
    g.M = b; g.N = F.H; g.K = F.D; g.groups = 2; g.splits = pick_splits(b, F.H, F.D, 2);
    g.epi = EPI_BIAS_RELU; g.partial = ctx->partial;
    PB("fc" + std::to_string(l + 1) + "_fwd", g.splits > 1 ? 2 : 1);
    launch_gemm_f32(g, st);
    PE();
    in[0] = ctx->act_fc[l][0]; in[1] = ctx->act_fc[l][1];
  }
  (void)LC;
  // a6 head: TD target, loss, output layer gradient, d(previous pre-activation)
  const FcShape& O = net.fc[net.n_fc];
  HeadArgs h{};
  h.act[0] = in[0]; h.act[1] = in[1];
  h.theta = ctx->theta_local; h.theta_hat = ctx->theta_hat;
  h.w_off = O.w_off; h.b_off = O.b_off;
  h.prev_is_fc = net.n_fc > 0;
  h.prev_b_off = net.n_fc > 0 ? net.fc[net.n_fc - 1].b_off : 0;
  h.H = O.D; h.A = O.H; h.b = b;
  h.idx = ctx->idx; h.ring_a = ctx->ring_a; h.ring_r = ctx->ring_r; h.ring_term = ctx->ring_t;
  h.gamma = (float)c.gamma; h.clip = (float)c.err_clip;
  h.grad = ctx->grad;
  h.dH = net.n_fc > 0 ? ctx->dz_fc[net.n_fc - 1] : ctx->dz_conv[net.n_conv - 1];
  h.ctr = ctx->ctr; h.diag_loss = ctx->diag_loss; h.diag_idx = ctx->diag_idx; h.diag_amax = ctx->diag_amax;
  h.s_dq = ctx->head_dq; h.s_act = ctx->head_act; h.s_loss = ctx->head_loss;
  h.s_delta = ctx->head_delta; h.diag_delta = ctx->diag_delta;
  PB("head_td", 2);
  launch_head_f32(h, st);
  PE();
  enqueue_prio_update(ctx, st);
  // a7 hidden FC backward
  for (int l = net.n_fc - 1; l >= 0; --l) {
    const FcShape& F = net.fc[l];
    const float* dz = ctx->dz_fc[l];
    const float* a_in = l > 0 ? ctx->act_fc[l - 1][0] : ctx->act_conv[net.n_conv - 1][0];
    PB("fc" + std::to_string(l + 1) + "_bwd", (l < net.n_fc - 1 ? 1 : 0) + 1 + (pick_splits(b, F.D, F.H, 1) > 1 ? 2 : 1));
    if (l < net.n_fc - 1) launch_bias_grad(dz, b, F.H, ctx->grad + F.b_off, st);
    GemmArgs gw{};  // dW[h][d] += sum_j dz[j][h] a_in[j][d]
    gw.A[0] = dz; gw.sam = 1; gw.sak = F.H;
    gw.B[0] = a_in; gw.sbk = F.D; gw.sbn = 1;
    gw.C[0] = ctx->grad + F.w_off; gw.scm = F.D; gw.scn = 1;
    gw.M = F.H; gw.N = F.D; gw.K = b; gw.groups = 1; gw.splits = 1; gw.epi = EPI_ACCUM;
    launch_gemm_f32(gw, st);
    GemmArgs gx{};  // dz_prev[j][d] = [a_in > 0] sum_h dz[j][h] W[h][d]
    gx.A[0] = dz; gx.sam = F.H; gx.sak = 1;
    gx.B[0] = ctx->theta_local + F.w_off; gx.sbk = F.D; gx.sbn = 1;
    gx.C[0] = l > 0 ? ctx->dz_fc[l - 1] : ctx->dz_conv[net.n_conv - 1]; gx.scm = F.D; gx.scn = 1;
    gx.mask[0] = a_in; gx.smm = F.D; gx.smn = 1;
    gx.M = b; gx.N = F.D; gx.K = F.H; gx.groups = 1; gx.splits = pick_splits(b, F.D, F.H, 1);
    gx.epi = EPI_MASK; gx.partial = ctx->partial;
    launch_gemm_f32(gx, st);
    PE();
  }
  // a8/a9 convolution backward
  for (int i = net.n_conv - 1; i >= 0; --i) {
    const ConvShape& L = net.conv[i];
    ImgSrc src{};
    if (i == 0) {
      src.u8[0] = ctx->ring_s; src.idx = ctx->idx; src.stride = ctx->slot_stride;
    } else {
      src.f32[0] = ctx->act_conv[i - 1][0];
      src.stride = (long long)L.C * L.H * L.W;
    }
    PB("conv" + std::to_string(i + 1) + "_bwd", i > 0 ? 3 : 2);
    launch_conv_bwd_dw_f32(L, ctx->dz_conv[i], src, ctx->partial, b, st);
    launch_reduce_rows(ctx->partial, b, (long long)L.N * L.C * L.k * L.k + L.N, ctx->grad + L.w_off, st);
    if (i > 0) launch_conv_bwd_dx_f32(L, ctx->dz_conv[i], ctx->theta_local, ctx->act_conv[i - 1][0],
                                      ctx->dz_conv[i - 1], b, st);
    PE();
  }
  // a11 push + a12 shard update (Alg. 2 RMSPropUpdate; n <- n + 1)
  if (push) {
    const float div = (float)((double)ctx->world * c.n_push);
    const float rho = (float)c.rms_decay, omr = (float)(1.0 - c.rms_decay);
    if (ctx->fused_comm) {
      PB("server_round_fused", 1);
      launch_server_round(ctx->sra, st);
      PE();
    } else if (ctx->world > 1) {
      PB("push_reduce_scatter", 0);
      if (ctx->grad_snap)
        CK(cudaMemcpyAsync(ctx->grad_snap, ctx->grad, sizeof(float) * ctx->P_pad, cudaMemcpyDeviceToDevice, st));
      NK(ncclReduceScatter(ctx->grad, ctx->g_shard, (size_t)ctx->shard, ncclFloat, ncclSum, ctx->comm, st));
      CK(cudaMemsetAsync(ctx->grad, 0, sizeof(float) * ctx->P_pad, st));
      PE();
      PB("rmsprop_update", 1);
      launch_rmsprop(ctx->theta_master, ctx->rms, ctx->g_shard, ctx->shard, div, (float)c.lr, rho, omr,
                     (float)c.rms_eps, nullptr, nullptr, ctx->ctr, 0, st);
      PE();
    } else {
      PB("rmsprop_update", 1);
      launch_rmsprop(ctx->theta_master, ctx->rms, ctx->grad, ctx->P_pad, div, (float)c.lr, rho, omr,
                     (float)c.rms_eps, nullptr, nullptr, ctx->ctr, 1, st, -1, 0, 0, ctx->grad_snap);
      PE();
    }
  }
  CK(cudaGetLastError());
  return DQN_OK;
}

// ------------------------------------------------------------------ one replica step (bf16 tensor-core path)
// 7 kernels: conv fwd (sample+gather+conv1+conv2, s and s'), FC fwd (split-K, last CTA
// reduces + bias + ReLU), TD head, FC dW, FC dX (+ReLU mask), conv bwd (conv2 dW/dX,
// conv1 dW, biases), RMSProp update (+ bf16 publication).
static int enqueue_step_bf16(dqn_ctx* ctx, bool fetch, bool refresh, bool push, bool store) {
  const NetShape& net = ctx->net;
  const dqn_config& c = ctx->cfg;
  const int b = c.minibatch;
  const FcShape& F = net.fc[0];
  const FcShape& O = net.fc[1];
  const ConvShape& L1 = net.conv[0];
  const ConvShape& L2 = net.conv[1];
  cudaStream_t st = ctx->stream;
  const StoreArgs sa{ctx->ring_s, ctx->ring_sn, ctx->ring_a, ctx->ring_r, ctx->ring_t, ctx->cap, ctx->slot_stride,
                     ctx->dedup ? 1 : 0, ctx->store_ctl, ctx->ctr};
  // N = 1 or the fused server round: the Store runs inside the conv forward (its extra CTAs), so the forward keeps
  // its PDL overlap with the previous kernel and only a draw of the slot being stored waits for it (DQN_STORE_IN_FWD=0: own kernel)
  const char* sf = getenv("DQN_STORE_IN_FWD");
  const bool store_fused = store && (ctx->world == 1 || ctx->fused_comm) && !ctx->dedup && !ctx->prio &&
                           ctx->store_flag && !(sf && atoi(sf) == 0);
  if (store && !store_fused) {  // Alg. 1 "Store" of this iteration's transition (dqn_store_and_train), then the step
    PB("store", 1);
    launch_store_step(sa, st);
    PE();
  }
  if (fetch) {  // a13 + a14
    if (ctx->fused_comm) {
      // delivered into theta_local by the previous round's fused server-round kernel (NEXT-1)
    } else if (ctx->world > 1) {
      PB("fetch_all_gather", 2);
      int rc = enqueue_fetch_bf16(ctx, st, ctx->theta_local, ctx->theta_local_bf16);
      if (rc) return rc;
      PE();
    } else if (!ctx->alias_local) {
      PB("fetch_copy", 1);
      CK(cudaMemcpyAsync(ctx->theta_local, ctx->theta_master, sizeof(float) * ctx->P_pad, cudaMemcpyDeviceToDevice, st));
      launch_f32_to_bf16(ctx->theta_local, ctx->theta_local_bf16, ctx->P_pad, st, ctx->img_off, ctx->w1_off,
                         ctx->w2_off);
      PE();
    }
  }
  if (refresh) {
    PB("target_refresh", 0);
    if (ctx->fused_comm)  // theta_local's fp32 FC weight holds only this rank's slice (kernels_comm.cu)
      NK(ncclAllGather(ctx->theta_master, ctx->theta_hat, (size_t)ctx->shard, ncclFloat, ctx->comm, st));
    else
      CK(cudaMemcpyAsync(ctx->theta_hat, ctx->theta_local, sizeof(float) * ctx->P_pad, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(ctx->theta_hat_bf16, ctx->theta_local_bf16, sizeof(__nv_bfloat16) * ctx->P_bf16,
                       cudaMemcpyDeviceToDevice, st));
    PE();
  }
  // a1-a4: sample + gather + conv1 + conv2 for s (theta) and s' (theta^), tcgen05
  FwdConvArgs fa{};
  fa.ring[0] = ctx->ring_s; fa.ring[1] = ctx->ring_sn;
  fa.theta[0] = ctx->theta_local_bf16; fa.theta[1] = ctx->theta_hat_bf16;
  fa.theta_f32[0] = ctx->theta_local; fa.theta_f32[1] = ctx->theta_hat;
  fa.w1_off = L1.w_off; fa.b1_off = L1.b_off; fa.w2_off = L2.w_off; fa.b2_off = L2.b_off;
  fa.idx = ctx->idx; fa.ctr = ctx->ctr; fa.seed = c.seed; fa.rank = (unsigned)ctx->rank; fa.n = b;
  fa.a2 = ctx->a2_bf16; fa.a1_save = ctx->a1_save;
  fa.acq = ctx->acq;
  fa.img_off = ctx->img_off;
  fa.slot_stride = ctx->slot_stride;
  fa.late = store && !store_fused ? 1 : 0;
  if (store_fused) {
    fa.store_fused = 1;
    fa.store = sa;
    fa.store_flag = ctx->store_flag;
    fa.store_join = reinterpret_cast<unsigned*>(ctx->store_flag + 1);
  }
  if (ctx->prio) {  // the draws come from the sum tree: the forward waits for them (A41)
    enqueue_prio_sample(ctx, st);
    fa.idx_in = ctx->idx;
    fa.late = 1;
  }
  PB("conv_fwd", 1);
  launch_fwd_conv_bf16(fa, 2, st);
  PE();
  // a5: FC fwd, swap-AB: h^T[H][b] = W[H][2592] a2^T, split-K 18 x 144, last CTA adds bias + ReLU
  TcGemmArgs gf{};
  gf.A[0] = ctx->theta_local_bf16 + F.w_off; gf.A[1] = ctx->theta_hat_bf16 + F.w_off; gf.lda = F.D; gf.a_mn = 0;
  gf.B[0] = ctx->a2_bf16; gf.B[1] = ctx->a2_bf16 + (long long)b * F.D; gf.ldb = F.D; gf.b_mn = 0;
  // n-tile: all samples up to 128, else 128 (BJ.c4, b = 256: 2.41 M -> 2.47 M tr/s with the dW tile below)
  gf.M = F.H; gf.N = b; gf.K = F.D; gf.BN = std::min(b, 128); gf.kper = F.D / ctx->fc_splits; gf.splits = ctx->fc_splits;
  gf.st_id = ST_FC_FWD;
  gf.epi = TC_EPI_FC_FWD; gf.partial = ctx->fc_partial; gf.counters = ctx->tc_counters;
  gf.pre_a = 1; gf.pre_b = 0;  // W from the previous step's update; a2 from the predecessor
  gf.bias[0] = ctx->theta_local + F.b_off; gf.bias[1] = ctx->theta_hat + F.b_off;
  if (ctx->acq.conv_first) gf.acq = ctx->acq;  // the previous round's FC deliveries, G cleared
  // (h_out left null: the TD head reduces the split-K partials, adds the bias and applies ReLU)
  PB("fc1_fwd", 1);
  launch_tc_gemm(gf, 2, st);
  PE();
  // a6 head (TD target, loss, output layer, dH)
  HeadArgs h{};
  h.act[0] = ctx->act_fc[0][0]; h.act[1] = ctx->act_fc[0][1];
  h.theta = ctx->theta_local; h.theta_hat = ctx->theta_hat;
  h.w_off = O.w_off; h.b_off = O.b_off;
  h.prev_is_fc = 1; h.prev_b_off = F.b_off;
  h.H = O.D; h.A = O.H; h.b = b;
  h.idx = ctx->idx; h.ring_a = ctx->ring_a; h.ring_r = ctx->ring_r; h.ring_term = ctx->ring_t;
  h.gamma = (float)c.gamma; h.clip = (float)c.err_clip;
  h.grad = ctx->grad; h.dH = ctx->dz_fc[0]; h.dH_bf16 = ctx->dh_bf16;
  h.fc_partial = ctx->fc_partial; h.fc_split_stride = (long long)gf.N * gf.M;
  h.fc_splits = ctx->use_tgemm ? ctx->tg_fwd.splits : gf.splits;
  h.fc_bias[0] = ctx->theta_local + F.b_off; h.fc_bias[1] = ctx->theta_hat + F.b_off;
  h.act_out[0] = ctx->act_fc[0][0]; h.act_out[1] = ctx->act_fc[0][1];
  h.st_id = ST_HEAD;
  h.ctr = ctx->ctr; h.diag_loss = ctx->diag_loss; h.diag_idx = ctx->diag_idx; h.diag_amax = ctx->diag_amax;
  h.s_dq = ctx->head_dq; h.s_act = ctx->head_act; h.s_loss = ctx->head_loss;
  h.s_delta = ctx->head_delta; h.diag_delta = ctx->diag_delta;
  PB("head_sample", 1);
  launch_head_f32(h, st, /*with_finish=*/false);
  PE();
  enqueue_prio_update(ctx, st);
  // a7 FC backward: dW[h][d] += sum_j dH[j][h] a2[j][d]  and  dz2[j][d] = [a2 > 0] sum_h dH[j][h] W[h][d]
  TcGemmArgs gw{};
  gw.A[0] = ctx->dh_bf16; gw.lda = F.H; gw.a_mn = 1;
  gw.B[0] = ctx->a2_bf16; gw.ldb = F.D; gw.b_mn = 1;
  // 54 CTAs at b = 32 (short store epilogues); 128-column tiles from b = 128 on (longer K per tile)
  gw.M = F.H; gw.N = F.D; gw.K = b; gw.BN = b >= 128 ? 128 : 96; gw.kper = b; gw.splits = 1;
  gw.epi = TC_EPI_ACCUM; gw.C[0] = ctx->grad + F.w_off; gw.ldc = F.D;
  gw.pre_a = 0; gw.pre_b = 1;  // dH comes from the predecessor (head_sample), a2 from the conv forward
  gw.store = c.n_push == 1;     // n_push = 1: this step's gradient is the whole accumulator (A8)
  {  // n_push > 1: the tile rows go out as bulk fp32 reduce-adds (BJ.configs[3]: 82.3 -> 81.0 us/step); at
     // n_push = 1 the plain stores measured the same either way (32.4-33.6 vs 33.0-33.1 us/step), so they stay
    const char* ba = getenv("DQN_BULK_ACCUM");
    gw.bulk_accum = ba ? atoi(ba) : c.n_push > 1;
  }
  TcGemmArgs gx{};
  gx.A[0] = ctx->theta_local_bf16 + F.w_off; gx.lda = F.D; gx.a_mn = 1;
  gx.B[0] = ctx->dh_bf16; gx.ldb = F.H; gx.b_mn = 0;
  // n-tiles of 16 samples (b <= 32) or 64: more CTAs, each with a shorter ReLU-mask epilogue (measured:
  // 35.95 -> 35.35 us/step at b = 32; BJ.c4, b = 256: 2.16 M -> 2.40 M tr/s with 64 instead of 256)
  gx.M = F.D; gx.N = b; gx.K = F.H; gx.BN = b <= 32 ? 16 : 64; gx.kper = F.H; gx.splits = 1;
  gx.epi = TC_EPI_MASK_T; gx.out_bf16 = ctx->dz2_bf16; gx.mask = ctx->a2_bf16; gx.ldo = F.D;
  gx.pre_a = 1; gx.pre_b = 0;  // W is published by the previous step's update; dH by the predecessor
  gw.st_id = gx.st_id = ST_FC_BWD;
  gw.st_ph = ST_P3; gx.st_ph = ST_P4;
  if (tc_pair_fits(gw, gx)) {
    PB("fc1_bwd_head_finish", 1);
    launch_tc_pair_with_head(gw, gx, h, st);
    PE();
  } else {  // wide FC layers: K-pipelined GEMMs (any fc), then the head finish
    gw.BN = 64; gx.BN = 64;
    PB("fc1_bwd_head_finish", 3);
    launch_gemm_pipe(gw, 1, st);
    launch_gemm_pipe(gx, 1, st);
    launch_head_finish_warp(h, st);
    PE();
  }
  // a8/a9 conv backward
  BwdConvArgs ba{};
  ba.ring_s = ctx->ring_s; ba.slot_stride = ctx->slot_stride; ba.idx = ctx->idx; ba.a1_save = ctx->a1_save; ba.dz2 = ctx->dz2_bf16;
  ba.theta = ctx->theta_local_bf16;
  ba.w1_off = L1.w_off; ba.b1_off = L1.b_off; ba.w2_off = L2.w_off; ba.b2_off = L2.b_off;
  ba.n = b; ba.partial = ctx->bwd_partial; ba.counter = ctx->tc_counters + 32; ba.grad = ctx->grad;
  // N = 1, n_push = 1: the conv partials' reduction runs inside the update (reduce_update_kernel)
  const bool fuse_reduce = push && ctx->world == 1 && c.n_push == 1 && ctx->alias_local &&
                           L1.w_off == 0 && L2.b_off + L2.N == kBwdPart;
  ReduceUpdateArgs u{};
  if (fuse_reduce) {
    const float div = (float)((double)ctx->world * c.n_push);
    u.b = ba;
    u.theta = ctx->theta_master; u.r = ctx->rms; u.g = ctx->grad; u.n = ctx->P_pad;
    u.inv_div = 1.0f / div; u.lr = (float)c.lr; u.rho = (float)c.rms_decay; u.omr = (float)(1.0 - c.rms_decay);
    u.eps = (float)c.rms_eps;
    u.pub_bf16 = ctx->theta_local_bf16; u.img_off = ctx->img_off; u.ctr = ctx->ctr;
    u.g_snap = ctx->grad_snap;
    u.early = ctx->early_update && b + 32 <= ctx->num_sms ? 1 : 0;  // needs SMs the conv CTAs leave free
  }
  PB("conv_bwd", fuse_reduce ? 1 : 2);
  if (u.early)  // the non-conv update rides on the SMs the per-image conv CTAs leave free
    launch_bwd_conv_update(ba, u, ctx->num_sms - b, st);
  else
    launch_bwd_conv_bf16(ba, st, !fuse_reduce);
  PE();
  // a11 push + a12 shard update
  if (push) {
    const float div = (float)((double)ctx->world * c.n_push);
    const float rho = (float)c.rms_decay, omr = (float)(1.0 - c.rms_decay);
    if (ctx->fused_comm) {
      PB("server_round_fused", 1);
      launch_server_round(ctx->sra, st);
      PE();
    } else if (ctx->world > 1) {
      PB("push_reduce_scatter", 0);
      if (ctx->grad_snap)
        CK(cudaMemcpyAsync(ctx->grad_snap, ctx->grad, sizeof(float) * ctx->P_pad, cudaMemcpyDeviceToDevice, st));
      NK(ncclReduceScatter(ctx->grad, ctx->g_shard, (size_t)ctx->shard, ncclFloat, ncclSum, ctx->comm, st));
      CK(cudaMemsetAsync(ctx->grad, 0, sizeof(float) * ctx->P_pad, st));
      PE();
      PB("rmsprop_update", 1);
      launch_rmsprop(ctx->theta_master, ctx->rms, ctx->g_shard, ctx->shard, div, (float)c.lr, rho, omr,
                     (float)c.rms_eps, nullptr, nullptr, ctx->ctr, 0, st);
      PE();
    } else if (fuse_reduce) {
      PB("reduce_update", 1);
      launch_reduce_update(u, st);
      PE();
    } else {
      PB("rmsprop_update", 1);
      launch_rmsprop(ctx->theta_master, ctx->rms, ctx->grad, ctx->P_pad, div, (float)c.lr, rho, omr,
                     (float)c.rms_eps, nullptr, ctx->alias_local ? ctx->theta_local_bf16 : nullptr, ctx->ctr, 1, st,
                   ctx->alias_local ? ctx->img_off : -1, ctx->w1_off, ctx->w2_off, ctx->grad_snap);
      PE();
    }
  }
  CK(cudaGetLastError());
  return DQN_OK;
}

// ------------------------------------------------------------------ one replica step (generic bf16 conv path)
// gpack (conv weights of theta -> packed images), conv forward per layer (both groups), FC forward
// (split-K), TD head, FC dW + dX (+ReLU mask, NHWC) + head finish, per layer wgrad (+ range
// reduction into G) and dgrad, the update. Kernels: kernels_conv.cu, kernels_bf16.cu (tc_gemm).
// the FC dX's permutation into the last conv layer's input-grid geometry (when it does not store NHWC itself)
static void launch_dx_hwc(dqn_ctx* ctx, cudaStream_t st) {
  if (!ctx->dx_canon) return;
  const dqn_ctx::GLayer& G = ctx->gl[ctx->net.n_conv - 1];
  launch_chw_to_hwc(ctx->dx_canon, ctx->dzp[ctx->net.n_conv - 1], ctx->cfg.minibatch, G.N, G.Ho, G.Wo, G.Ws,
                    G.Hs * G.Ws, st);
}

static int enqueue_step_gpath(dqn_ctx* ctx, bool fetch, bool refresh, bool push) {
  const NetShape& net = ctx->net;
  const dqn_config& c = ctx->cfg;
  const int b = c.minibatch, nl = net.n_conv;
  const FcShape& F = net.fc[0];
  const FcShape& O = net.fc[1];
  cudaStream_t st = ctx->stream;
  if (ctx->fused_comm) {  // the previous round's deliveries into theta_local, then clear G
    PB("server_round_acquire", 1);
    launch_fused_round_acquire(ctx->acq, st);
    PE();
  }
  if (fetch) {  // a13
    if (ctx->fused_comm) {
    } else if (ctx->world > 1) {
      PB("fetch_all_gather", 2);
      int rc = enqueue_fetch_bf16(ctx, st, ctx->theta_local, ctx->theta_local_bf16);
      if (rc) return rc;
      PE();
    } else if (!ctx->alias_local) {
      PB("fetch_copy", 1);
      CK(cudaMemcpyAsync(ctx->theta_local, ctx->theta_master, sizeof(float) * ctx->P_pad, cudaMemcpyDeviceToDevice, st));
      launch_f32_to_bf16(ctx->theta_local, ctx->theta_local_bf16, ctx->P_pad, st);
      PE();
    }
  }
  // packed conv weights of the working theta (changed by every update)
  // N = 1 (deterministic): the update of the previous step wrote the packed images with theta (rmsprop pack_map);
  // otherwise theta_local arrived from the server round / fetch and is packed here
  const bool pack_in_update = ctx->world == 1 && !ctx->async;
  if (!pack_in_update) {
    PB("gpack", 1);
    launch_gpack(ctx->theta_local, ctx->theta_local_bf16, ctx->gpack_off, ctx->pack_map, ctx->pack_n, st);
    PE();
  }
  if (refresh) {  // a14: theta^ <- theta, packed images included
    PB("target_refresh", 0);
    if (ctx->fused_comm)
      NK(ncclAllGather(ctx->theta_master, ctx->theta_hat, (size_t)ctx->shard, ncclFloat, ctx->comm, st));
    else
      CK(cudaMemcpyAsync(ctx->theta_hat, ctx->theta_local, sizeof(float) * ctx->P_pad, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(ctx->theta_hat_bf16, ctx->theta_local_bf16, sizeof(__nv_bfloat16) * ctx->P_bf16,
                       cudaMemcpyDeviceToDevice, st));
    PE();
  }
  // a1-a4s: sample + gather (layer 1) and every conv forward, s with theta and s' with theta^
  if (ctx->prio) enqueue_prio_sample(ctx, st);  // the draws from the sum tree (A41), read by layer 1
  PB("conv_fwd", ctx->use_tconv ? nl + 1 : nl);
  if (ctx->use_tconv) {
    GConvFwdArgs ga{};
    ga.ring[0] = ctx->ring_s; ga.ring[1] = ctx->ring_sn; ga.slot_stride = ctx->slot_stride;
    ga.idx = ctx->idx; ga.ctr = ctx->ctr; ga.seed = c.seed; ga.rank = (unsigned)ctx->rank; ga.b = b;
    ga.idx_in = ctx->prio ? ctx->idx : nullptr;
    launch_gather_s2d(ga, ctx->x1[0], ctx->x1[1], 2, st);
    for (int i = 0; i < nl; ++i) launch_tconv(ctx->tc_fwd[i], ctx->num_sms, st);
  }
  for (int i = 0; i < nl && !ctx->use_tconv; ++i) {
    const ConvShape& L = net.conv[i];
    const dqn_ctx::GLayer& G = ctx->gl[i];
    GConvFwdArgs a{};
    a.first = i == 0;
    if (i == 0) {
      a.ring[0] = ctx->ring_s; a.ring[1] = ctx->ring_sn; a.slot_stride = ctx->slot_stride;
      a.idx = ctx->idx; a.ctr = ctx->ctr; a.seed = c.seed; a.rank = (unsigned)ctx->rank;
      a.idx_in = ctx->prio ? ctx->idx : nullptr;
    } else {
      a.x[0] = G.x[0]; a.x[1] = G.x[1];
    }
    a.b = b; a.Hs = G.Hs; a.Ws = G.Ws; a.Cs = G.Cs; a.Th = G.Th; a.Tw = G.Tw; a.Ho = G.Ho; a.Wo = G.Wo; a.N = L.N;
    a.s_next = i + 1 < nl ? ctx->gl[i + 1].s : 0;
    a.wpk[0] = ctx->theta_local_bf16 + ctx->gpack_off + G.fwd_pack;
    a.wpk[1] = ctx->theta_hat_bf16 + ctx->gpack_off + G.fwd_pack;
    a.bias[0] = ctx->theta_local + L.b_off; a.bias[1] = ctx->theta_hat + L.b_off;
    for (int g = 0; g < 2; ++g) a.out[g] = i + 1 < nl ? ctx->gl[i + 1].x[g] : ctx->a2_bf16 + (long long)g * b * F.D;
    launch_gconv_fwd(a, 2, st);
  }
  PE();
  // a5: FC forward, split-K partials (the head reduces them)
  TcGemmArgs gf{};
  gf.A[0] = ctx->theta_local_bf16 + F.w_off; gf.A[1] = ctx->theta_hat_bf16 + F.w_off; gf.lda = F.D;
  gf.B[0] = ctx->a2_bf16; gf.B[1] = ctx->a2_bf16 + (long long)b * F.D; gf.ldb = F.D;
  gf.M = F.H; gf.N = b; gf.K = F.D; gf.BN = std::min(b, 128); gf.kper = F.D / ctx->fc_splits; gf.splits = ctx->fc_splits;
  gf.epi = TC_EPI_FC_FWD; gf.partial = ctx->fc_partial;
  PB("fc1_fwd", 1);
  if (ctx->use_tgemm) launch_tgemm(ctx->tg_fwd, ctx->num_sms, st);
  else launch_gemm_pipe(gf, 2, st);
  PE();
  // a6 head
  HeadArgs h{};
  h.st_id = ST_HEAD;
  h.act[0] = ctx->act_fc[0][0]; h.act[1] = ctx->act_fc[0][1];
  h.theta = ctx->theta_local; h.theta_hat = ctx->theta_hat;
  h.w_off = O.w_off; h.b_off = O.b_off;
  h.prev_is_fc = 1; h.prev_b_off = F.b_off;
  h.H = O.D; h.A = O.H; h.b = b;
  h.idx = ctx->idx; h.ring_a = ctx->ring_a; h.ring_r = ctx->ring_r; h.ring_term = ctx->ring_t;
  h.gamma = (float)c.gamma; h.clip = (float)c.err_clip;
  h.grad = ctx->grad; h.dH = ctx->dz_fc[0]; h.dH_bf16 = ctx->dh_bf16;
  h.fc_partial = ctx->fc_partial; h.fc_split_stride = (long long)gf.N * gf.M;
  h.fc_splits = ctx->use_tgemm ? ctx->tg_fwd.splits : gf.splits;
  h.fc_bias[0] = ctx->theta_local + F.b_off; h.fc_bias[1] = ctx->theta_hat + F.b_off;
  h.act_out[0] = ctx->act_fc[0][0]; h.act_out[1] = ctx->act_fc[0][1];
  h.ctr = ctx->ctr; h.diag_loss = ctx->diag_loss; h.diag_idx = ctx->diag_idx; h.diag_amax = ctx->diag_amax;
  h.s_dq = ctx->head_dq; h.s_act = ctx->head_act; h.s_loss = ctx->head_loss;
  h.s_delta = ctx->head_delta; h.diag_delta = ctx->diag_delta;
  PB("head_sample", 1);
  launch_head_f32(h, st, false);
  PE();
  enqueue_prio_update(ctx, st);
  // a7: FC dW (plain store at n_push = 1) + FC dX (x ReLU mask, into the last conv's NHWC dZ)
  const dqn_ctx::GLayer& GL = ctx->gl[nl - 1];
  TcGemmArgs gw{};
  gw.A[0] = ctx->dh_bf16; gw.lda = F.H; gw.a_mn = 1;
  gw.B[0] = ctx->a2_bf16; gw.ldb = F.D; gw.b_mn = 1;
  gw.M = F.H; gw.N = F.D; gw.K = b; gw.BN = 64; gw.kper = b; gw.splits = 1;
  gw.epi = TC_EPI_ACCUM; gw.C[0] = ctx->grad + F.w_off; gw.ldc = F.D; gw.store = c.n_push == 1;
  gw.pre_a = 0; gw.pre_b = 1;
  TcGemmArgs gx{};
  gx.A[0] = ctx->theta_local_bf16 + F.w_off; gx.lda = F.D; gx.a_mn = 1;
  gx.B[0] = ctx->dh_bf16; gx.ldb = F.H; gx.b_mn = 0;
  gx.M = F.D; gx.N = b; gx.K = F.H; gx.BN = 64; gx.kper = F.H; gx.splits = 1;
  gx.epi = TC_EPI_MASK_T; gx.out_bf16 = GL.dz; gx.mask = ctx->a2_bf16; gx.ldo = F.D;
  gx.hwc_HW = GL.Ho * GL.Wo; gx.hwc_C = GL.N;
  // one launch: the FC dW and dX tiles plus the head finish CTAs run side by side (tc_pair); the
  // whole K (= b and H <= 512) is staged at once, which the 200 KB budget allows at BN = 64
  gx.pre_a = 1; gx.pre_b = 0; gw.pre_a = 0; gw.pre_b = 1;
  const long long fc0 = F.w_off;  // the non-conv parameters [fc0, P_pad): FC weight and bias, output layer
  if (ctx->use_tgemm && ctx->split_update && push) {
    // side branch: head finish (dW_o, db_o, db_fc, loss, T + 1) next to the FC dW / dX, then the RMSProp update
    // of the non-conv parameters next to the conv backward; joined at the end of the step
    PB("fc1_bwd_head_finish", 2 + (ctx->dx_canon ? 1 : 0));
    CK(cudaEventRecord(ctx->ev_fork, st));
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    launch_head_finish_warp(h, ctx->side);
    launch_tgemm(ctx->tg_dw, ctx->num_sms, st);
    launch_tgemm(ctx->tg_dx, ctx->num_sms, st);  // reads the FC weight the side update is about to write
    CK(cudaEventRecord(ctx->ev_dw, st));
    launch_dx_hwc(ctx, st);
    PE();
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_dw, 0));
    launch_rmsprop(ctx->theta_master + fc0, ctx->rms + fc0, ctx->grad + fc0, ctx->P_pad - fc0, (float)c.n_push,
                   (float)c.lr, (float)c.rms_decay, (float)(1.0 - c.rms_decay), (float)c.rms_eps, nullptr,
                   ctx->theta_local_bf16 + fc0, ctx->ctr, 1, ctx->side, -1, 0, 0,
                   ctx->grad_snap ? ctx->grad_snap + fc0 : nullptr);
    CK(cudaEventRecord(ctx->ev_join, ctx->side));
  } else if (ctx->use_tgemm) {  // the warp-specialised TMA GEMMs, then the head finish
    PB("fc1_bwd_head_finish", 3 + (ctx->dx_canon ? 1 : 0));
    launch_tgemm(ctx->tg_dw, ctx->num_sms, st);
    launch_tgemm(ctx->tg_dx, ctx->num_sms, st);
    launch_dx_hwc(ctx, st);
    launch_head_finish_warp(h, st);
    PE();
  } else if (tc_pair_fits(gw, gx)) {
    PB("fc1_bwd_head_finish", 1);
    launch_tc_pair_with_head(gw, gx, h, st);
    PE();
  } else {  // FC widths whose whole K does not fit tc_pair's staging: K-pipelined GEMMs, then the head finish
    PB("fc1_bwd_head_finish", 3);
    launch_gemm_pipe(gw, 1, st);
    launch_gemm_pipe(gx, 1, st);
    launch_head_finish_warp(h, st);
    PE();
  }
  // a8/a9: per layer, top down: wgrad (+ range reduction into G), then dgrad into the layer below
  PB("conv_bwd", 3 * nl - 1);
  if (ctx->use_tconv && ctx->bside) {
    // the data-gradient chain on the main stream; layer i's weight gradient on bside as soon as dZ_i exists, so it
    // fills the SMs the chain's tails leave idle (they read dZ_i and the layer input, write their own partials
    // and G's conv rows; joined before the update)
    for (int i = nl - 1; i >= 1; --i) {
      CK(cudaEventRecord(ctx->ev_bdz[i], st));  // dZ_i complete (FC dX or the data gradient of layer i + 1)
      CK(cudaStreamWaitEvent(ctx->bside, ctx->ev_bdz[i], 0));
      launch_tconv(ctx->tc_wgrad[i], ctx->num_sms, ctx->bside);
      launch_gconv_wreduce(ctx->tc_wred[i], ctx->bside);
      launch_tconv(ctx->tc_dgrad[i], ctx->num_sms, st);
    }
    launch_tconv(ctx->tc_wgrad[0], ctx->num_sms, st);
    launch_gconv_wreduce(ctx->tc_wred[0], st);
    CK(cudaEventRecord(ctx->ev_bjoin, ctx->bside));
    CK(cudaStreamWaitEvent(st, ctx->ev_bjoin, 0));
  }
  for (int i = nl - 1; i >= 0 && ctx->use_tconv && !ctx->bside; --i) {
    launch_tconv(ctx->tc_wgrad[i], ctx->num_sms, st);
    launch_gconv_wreduce(ctx->tc_wred[i], st);
    if (i > 0) launch_tconv(ctx->tc_dgrad[i], ctx->num_sms, st);
  }
  for (int i = nl - 1; i >= 0 && !ctx->use_tconv; --i) {
    const ConvShape& L = net.conv[i];
    const dqn_ctx::GLayer& G = ctx->gl[i];
    GConvWgradArgs w{};
    w.first = i == 0;
    if (i == 0) { w.ring = ctx->ring_s; w.idx = ctx->idx; w.slot_stride = ctx->slot_stride; } else { w.x = G.x[0]; }
    w.dz = G.dz;
    w.b = b; w.Hs = G.Hs; w.Ws = G.Ws; w.Cs = G.Cs; w.Th = G.Th; w.Tw = G.Tw; w.Ho = G.Ho; w.Wo = G.Wo; w.N = L.N;
    w.ipc = G.ipc; w.partial = ctx->gw_partial; w.partial_db = ctx->gw_partial_db;
    w.w_canon = G.w_canon; w.w_off = L.w_off; w.w_nstride = (long long)L.C * L.k * L.k; w.b_off = L.b_off;
    w.grad = ctx->grad; w.store = c.n_push == 1;
    launch_gconv_wgrad(w, st);
    if (i > 0) {
      GConvDgradArgs d{};
      d.dz = G.dz; d.wpkT = ctx->theta_local_bf16 + ctx->gpack_off + G.dg_pack; d.xmask = G.x[0];
      d.dzprev = ctx->gl[i - 1].dz;
      d.b = b; d.Hs = G.Hs; d.Ws = G.Ws; d.Cs = G.Cs; d.Th = G.Th; d.Tw = G.Tw; d.Ho = G.Ho; d.Wo = G.Wo; d.N = L.N;
      d.s = G.s;
      launch_gconv_dgrad(d, st);
    }
  }
  PE();
  // a11 push + a12 shard update (+ a13 fetch in the fused round)
  if (push) {
    const float div = (float)((double)ctx->world * c.n_push);
    const float rho = (float)c.rms_decay, omr = (float)(1.0 - c.rms_decay);
    if (ctx->fused_comm) {
      PB("server_round_fused", 1);
      launch_server_round(ctx->sra, st);
      PE();
    } else if (ctx->world > 1) {
      PB("push_reduce_scatter", 0);
      if (ctx->grad_snap)
        CK(cudaMemcpyAsync(ctx->grad_snap, ctx->grad, sizeof(float) * ctx->P_pad, cudaMemcpyDeviceToDevice, st));
      NK(ncclReduceScatter(ctx->grad, ctx->g_shard, (size_t)ctx->shard, ncclFloat, ncclSum, ctx->comm, st));
      CK(cudaMemsetAsync(ctx->grad, 0, sizeof(float) * ctx->P_pad, st));
      PE();
      PB("rmsprop_update", 1);
      launch_rmsprop(ctx->theta_master, ctx->rms, ctx->g_shard, ctx->shard, div, (float)c.lr, rho, omr,
                     (float)c.rms_eps, nullptr, nullptr, ctx->ctr, 0, st);
      PE();
    } else if (ctx->use_tgemm && ctx->split_update) {  // the conv parameters here, the rest on the side branch
      PB("rmsprop_update", 1);
      launch_rmsprop(ctx->theta_master, ctx->rms, ctx->grad, fc0, div, (float)c.lr, rho, omr, (float)c.rms_eps,
                     nullptr, ctx->theta_local_bf16, ctx->ctr, 1, st, -1, 0, 0, ctx->grad_snap, ctx->pack_map,
                     ctx->pack_n, ctx->gpack_off);
      CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
      PE();
    } else {
      PB("rmsprop_update", 1);
      launch_rmsprop(ctx->theta_master, ctx->rms, ctx->grad, ctx->P_pad, div, (float)c.lr, rho, omr,
                     (float)c.rms_eps, nullptr, ctx->alias_local ? ctx->theta_local_bf16 : nullptr, ctx->ctr, 1, st, -1, 0,
                     0, ctx->grad_snap, ctx->alias_local ? ctx->pack_map : nullptr, ctx->pack_n, ctx->gpack_off);
      PE();
    }
  }
  CK(cudaGetLastError());
  return DQN_OK;
}

static int enqueue_step(dqn_ctx* ctx, bool fetch, bool refresh, bool push, bool store = false) {
  if (ctx->gpath) return enqueue_step_gpath(ctx, fetch, refresh, push);
  return ctx->bf16 ? enqueue_step_bf16(ctx, fetch, refresh, push, store) : enqueue_step_f32(ctx, fetch, refresh, push);
}

// Capture `len` consecutive steps of variant v (bits: 1 fetch, 2 refresh, 4 push, 8 profiling
// event records, 16 in-graph Store) into one graph; *kernels = its kernel nodes.
static int capture_steps(dqn_ctx* ctx, int v, int len, cudaGraphExec_t* exec, long long* kernels) {
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  ctx->capture_variant = v;
  int rc = DQN_OK;
  for (int i = 0; i < len && rc == DQN_OK; ++i) rc = enqueue_step(ctx, v & 1, v & 2, v & 4, v & 16);
  ctx->capture_variant = -1;
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
  if (rc) return rc;
  if (e != cudaSuccess) return set_err(ctx, DQN_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  size_t n = 0;
  CK(cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  CK(cudaGraphGetNodes(g, nodes.data(), &n));
  long long nk = 0;
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    CK(cudaGraphNodeGetType(nd, &t));
    if (t == cudaGraphNodeTypeKernel) ++nk;
  }
  *kernels = nk;
  e = cudaGraphInstantiate(exec, g, 0);
  cudaGraphDestroy(g);
  CK(e);
  // upload now, so that the first launch (possibly inside a caller's timed region) does not pay for it
  CK(cudaGraphUpload(*exec, ctx->stream));
  return DQN_OK;
}

// Replay the graph of one step variant (captured on first use). profile: the
// variant with event records around each region. *kernels += kernel nodes run.
static int run_step(dqn_ctx* ctx, bool fetch, bool refresh, bool push, bool profile, long long* kernels) {
  if (!ctx->use_graphs && !profile) return enqueue_step(ctx, fetch, refresh, push);
  const int v = (fetch ? 1 : 0) | (refresh ? 2 : 0) | (push ? 4 : 0) | (profile ? 8 : 0);
  int rc;
  if (!ctx->graphs[v] && (rc = capture_steps(ctx, v, 1, &ctx->graphs[v], &ctx->graph_kernels[v]))) return rc;
  CK(cudaGraphLaunch(ctx->graphs[v], ctx->stream));
  if (kernels) *kernels += ctx->graph_kernels[v];
  return DQN_OK;
}

// O10 / O11 / O9 schedule of step T (host mirror; identical on every rank). In the asynchronous modes the
// generation a fetch returns, and with it the refresh, is decided on the device (async_fetch).
static void schedule(dqn_ctx* ctx, bool* fetch, bool* refresh, bool* push) {
  const dqn_config& c = ctx->cfg;
  const long long T = ctx->T;
  *fetch = (T % c.n_fetch) == 0;
  *refresh = false;
  if (*fetch && !ctx->async) {
    ctx->n_local = ctx->n;
    if (ctx->n_local - ctx->ell >= c.target_sync) {
      *refresh = true;
      ctx->ell = ctx->n_local;
    }
  }
  *push = ((T + 1) % c.n_push) == 0;
  if (!ctx->async) ctx->gen_log[T % kDiagSteps] = ctx->n_local;
}

// asynchronous fetch (O10/O11 on the device), enqueued on the compute stream ahead of the step graph: DQN_ASYNC
// takes the newest published generation without waiting; the lag-1 twin waits for generation n - 1
static int async_fetch(dqn_ctx* ctx) {
  long long forced = -1;
  const long long npr = ctx->n_per_round;  // generations per round: 1, or N with the per-gradient rule
  if (ctx->async_lag1) {  // the previous round's result
    forced = std::max(ctx->n - npr, 0LL);
    CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_pub[(forced / npr) % 3], 0));
  }
  launch_async_pick(ctx->adev, forced, ctx->cfg.target_sync, ctx->n_fetches, ctx->stream);
  AsyncCopy cp{};
  for (int i = 0; i < 3; ++i) {
    cp.pub[i] = ctx->theta_pub[i];
    cp.pubb[i] = ctx->theta_pub_bf16[i];
  }
  cp.th = ctx->theta_local; cp.thb = ctx->theta_local_bf16;
  cp.hat = ctx->theta_hat; cp.hatb = ctx->theta_hat_bf16;
  cp.n32 = ctx->P_pad; cp.n16 = ctx->bf16 ? ctx->P_bf16 : 0;
  cp.npr = npr;
  launch_async_copy(ctx->adev, cp, ctx->stream);
  ctx->n_fetches += 1;
  CK(cudaGetLastError());
  return DQN_OK;
}

// asynchronous push of round k (server generation n = k * npr before it): hand the accumulated gradient to the
// comm stream, which runs the whole server round (reduce-scatter, RMSProp on the owned shard, all-gather into
// theta_pub[(k + 1) % 3], publish generation n + npr) while the replica keeps stepping. With the per-gradient
// rule (A33) the reduce-scatter becomes an all-to-all into the owner's inbox and the owner applies the N
// workers' gradients one by one in rank order (npr = N generations per round). All NCCL traffic of this mode
// lives on the comm stream, in rank order.
static int async_push(dqn_ctx* ctx) {
  const dqn_config& c = ctx->cfg;
  cudaStream_t cs = ctx->comm_stream;
  const long long n0 = ctx->n, k = n0 / ctx->n_per_round;
  float* gs = ctx->g_send[k % 2];
  // g_send[k % 2] is read by round k - 2 until that round ends (so the comm stream lags by two rounds at most)
  CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_send[k % 2], 0));
  CK(cudaMemcpyAsync(gs, ctx->grad, sizeof(float) * ctx->P_pad, cudaMemcpyDeviceToDevice, ctx->stream));
  if (ctx->grad_snap)
    CK(cudaMemcpyAsync(ctx->grad_snap, ctx->grad, sizeof(float) * ctx->P_pad, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemsetAsync(ctx->grad, 0, sizeof(float) * ctx->P_pad, ctx->stream));
  CK(cudaEventRecord(ctx->ev_grad, ctx->stream));
  CK(cudaStreamWaitEvent(cs, ctx->ev_grad, 0));
  const float div = (float)((double)ctx->world * c.n_push);
  const float rho = (float)c.rms_decay, omr = (float)(1.0 - c.rms_decay);
  const int s = (int)((k + 1) % 3);
  if (ctx->world > 1) {
    if (ctx->inbox) {  // A33: worker p's slice of every owner's shard to that owner, applied in rank order
      NK(ncclGroupStart());
      for (int p = 0; p < ctx->world; ++p) {
        NK(ncclSend(gs + (long long)p * ctx->shard, (size_t)ctx->shard, ncclFloat, p, ctx->comm, cs));
        NK(ncclRecv(ctx->inbox + (long long)p * ctx->shard, (size_t)ctx->shard, ncclFloat, p, ctx->comm, cs));
      }
      NK(ncclGroupEnd());
      launch_rmsprop_per_gradient(ctx->theta_master, ctx->rms, ctx->inbox, ctx->world, ctx->shard, (float)c.n_push,
                                  (float)c.lr, rho, omr, (float)c.rms_eps, ctx->ctr, cs);
    } else {
      NK(ncclReduceScatter(gs, ctx->g_shard, (size_t)ctx->shard, ncclFloat, ncclSum, ctx->comm, cs));
      launch_rmsprop(ctx->theta_master, ctx->rms, ctx->g_shard, ctx->shard, div, (float)c.lr, rho, omr,
                     (float)c.rms_eps, nullptr, nullptr, ctx->ctr, 0, cs);
    }
    if (ctx->fetch_bf16) {  // a13 in bf16 (+ the fp32 entries outside the FC weight)
      int rc = enqueue_fetch_bf16(ctx, cs, ctx->theta_pub[s], ctx->theta_pub_bf16[s]);
      if (rc) return rc;
    } else {
      NK(ncclAllGather(ctx->theta_master, ctx->theta_pub[s], (size_t)ctx->shard, ncclFloat, ctx->comm, cs));
    }
  } else {
    launch_rmsprop(ctx->theta_master, ctx->rms, gs, ctx->P_pad, div, (float)c.lr, rho, omr,
                   (float)c.rms_eps, ctx->theta_pub[s], nullptr, ctx->ctr, 0, cs);
  }
  if (ctx->bf16 && !ctx->fetch_bf16)
    launch_f32_to_bf16(ctx->theta_pub[s], ctx->theta_pub_bf16[s], ctx->P_pad, cs, ctx->img_off, ctx->w1_off, ctx->w2_off);
  if (ctx->gpath) launch_gpack(ctx->theta_pub[s], ctx->theta_pub_bf16[s], ctx->gpack_off, ctx->pack_map, ctx->pack_n, cs);
  launch_async_publish(ctx->adev, n0, ctx->n_per_round, c.n_push, c.n_fetch, ctx->async_delay_ns, cs);
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev_pub[s], cs));
  CK(cudaEventRecord(ctx->ev_send[k % 2], cs));
  return DQN_OK;
}

// One replica step T: schedule, (async fetch), the step graph, (async push), counters.
static int do_step(dqn_ctx* ctx, bool profile, long long* kernels, bool* out_fetch, bool* out_refresh,
                   bool* out_push) {
  bool fetch, refresh, push;
  schedule(ctx, &fetch, &refresh, &push);
  int rc;
  if (ctx->async && fetch) {
    if ((rc = async_fetch(ctx))) return rc;
    if (kernels) *kernels += 2;
  }
  const bool g_fetch = fetch && !ctx->async, g_push = push && !ctx->async;
  if ((rc = run_step(ctx, g_fetch, refresh, g_push, profile, kernels))) return rc;
  if (ctx->async && push) {
    if ((rc = async_push(ctx))) return rc;
    if (kernels) *kernels += 2 + (ctx->fetch_bf16 ? 2 : 0) + (ctx->bf16 && !ctx->fetch_bf16 ? 1 : 0) + (ctx->gpath ? 1 : 0);
  }
  if (push) ctx->n += ctx->n_per_round;
  ctx->T += 1;
  if (out_fetch) *out_fetch = g_fetch;
  if (out_refresh) *out_refresh = refresh;
  if (out_push) *out_push = g_push;
  return DQN_OK;
}

// Host schedule of one step of the synchronous modes (do_step without the launch): variant bits.
static int plan_step(dqn_ctx* ctx) {
  bool fetch, refresh, push;
  schedule(ctx, &fetch, &refresh, &push);
  if (push) ctx->n += ctx->n_per_round;
  ctx->T += 1;
  return (fetch ? 1 : 0) | (refresh ? 2 : 0) | (push ? 4 : 0);
}

static int launch_chunk(dqn_ctx* ctx, int v, int l, long long* kernels) {
  int rc;
  cudaGraphExec_t& g = ctx->chunk_graphs[v][l];
  if (!g && (rc = capture_steps(ctx, v, 1 << l, &g, &ctx->chunk_kernels[v][l]))) return rc;
  CK(cudaGraphLaunch(g, ctx->stream));
  *kernels += ctx->chunk_kernels[v][l];
  return DQN_OK;
}

// Capture, once, the multi-step graphs the schedule can ask for, so that no capture falls into
// a caller's timed region (a missing one is still captured on first use).
static int prepare_chunks(dqn_ctx* ctx, int extra = 0) {
  const dqn_config& c = ctx->cfg;
  if (extra & 16) ctx->store_chunks_ready = true;
  else ctx->chunks_ready = true;
  for (int v0 = 0; v0 < 8; ++v0) {
    const bool fetch = v0 & 1, refresh = v0 & 2, push = v0 & 4;
    if ((refresh && !fetch) || (c.n_fetch == 1 && !fetch) || (c.n_push == 1 && !push)) continue;
    const int v = v0 | extra;
    const int nl = (refresh && c.target_sync > 1) ? 1 : dqn_ctx::kChunkLog;  // refreshes are >= C rounds apart
    for (int l = 0; l < nl; ++l) {
      if (ctx->chunk_graphs[v][l]) continue;
      int rc = capture_steps(ctx, v, 1 << l, &ctx->chunk_graphs[v][l], &ctx->chunk_kernels[v][l]);
      if (rc) return rc;
    }
  }
  return DQN_OK;
}

// k steps of a synchronous mode as runs of same-variant steps, each run replayed as
// power-of-two multi-step graphs (the kernels of consecutive steps then overlap via PDL).
static int run_steps_chunked(dqn_ctx* ctx, long long k, long long* kernels, bool store) {
  int rc;
  if (!ctx->chunks_ready && (rc = prepare_chunks(ctx))) return rc;
  if (store && !ctx->store_chunks_ready && (rc = prepare_chunks(ctx, 16))) return rc;
  const int max_len = 1 << (dqn_ctx::kChunkLog - 1);
  for (long long s = 0; s < k;) {
    const int v = plan_step(ctx) | (store ? 16 : 0);
    int len = 1;
    while (len < max_len && s + len < k) {
      const long long saved[4] = {ctx->T, ctx->n, ctx->n_local, ctx->ell};
      if ((plan_step(ctx) | (store ? 16 : 0)) != v) {
        ctx->T = saved[0]; ctx->n = saved[1]; ctx->n_local = saved[2]; ctx->ell = saved[3];
        break;
      }
      ++len;
    }
    for (int l = dqn_ctx::kChunkLog - 1; l >= 0; --l)
      if ((len >> l) & 1 && (rc = launch_chunk(ctx, v, l, kernels))) return rc;
    s += len;
  }
  return DQN_OK;
}

extern "C" int dqn_profile_steps(dqn_ctx* ctx, int64_t k, dqn_region_time* out, int32_t cap, int32_t* n_regions) {
  if (!ctx) return DQN_EINVAL;
  if (ctx->poisoned) return DQN_ESTATE;
  if (k < 0) return set_err(ctx, DQN_EINVAL, "k must be >= 0");
  if (ctx->count == 0) return set_err(ctx, DQN_EEMPTY, "replay memory is empty (A13)");
  std::vector<std::string> names;
  std::vector<double> tot;
  std::vector<int> cnt, kern;
  for (long long s = 0; s < k; ++s) {
    bool fetch, refresh, push;
    int rc = do_step(ctx, true, nullptr, &fetch, &refresh, &push);
    if (rc) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    const int v = (fetch ? 1 : 0) | (refresh ? 2 : 0) | (push ? 4 : 0) | 8;
    for (auto& m : ctx->marks[v]) {
      float ms = 0.0f;
      CK(cudaEventElapsedTime(&ms, m.a, m.b));
      size_t i = 0;
      while (i < names.size() && names[i] != m.name) ++i;
      if (i == names.size()) {
        names.push_back(m.name);
        tot.push_back(0.0);
        cnt.push_back(0);
        kern.push_back(m.kernels);
      }
      tot[i] += ms * 1000.0;
      cnt[i] += 1;
    }
  }
  if (n_regions) *n_regions = (int32_t)names.size();
  {  // the paper's Fig. 3 split: gradient time T, update time tau, communication
    double gm = 0.0, um = 0.0, cm = 0.0;
    for (size_t i = 0; i < names.size(); ++i) {
      const double us = tot[i] / cnt[i] * cnt[i] / (double)std::max<long long>(1, k);  // per step
      const std::string& n = names[i];
      if (n == "rmsprop_update" || n == "reduce_update") um += us;
      else if (n == "push_reduce_scatter" || n == "fetch_all_gather" || n == "fetch_copy" || n == "target_refresh" ||
               n == "server_round_fused" || n == "server_round_acquire")
        cm += us;
      else gm += us;
    }
    ctx->prof_grad_ms = gm / 1e3; ctx->prof_update_ms = um / 1e3; ctx->prof_comm_ms = cm / 1e3;
  }
  for (size_t i = 0; i < names.size() && out && (int32_t)i < cap; ++i) {
    std::memset(out[i].name, 0, sizeof(out[i].name));
    std::strncpy(out[i].name, names[i].c_str(), sizeof(out[i].name) - 1);
    out[i].avg_us = tot[i] / cnt[i];
    out[i].kernels = kern[i];
    out[i].steps = cnt[i];
  }
  return DQN_OK;
}

static int finish_steps(dqn_ctx* ctx, long long T0, long long k, long long kernels, dqn_step_stats* stats);

extern "C" int dqn_train_steps(dqn_ctx* ctx, int64_t k, dqn_step_stats* stats) {
  if (!ctx) return DQN_EINVAL;
  if (ctx->poisoned) return DQN_ESTATE;
  if (k < 0) return set_err(ctx, DQN_EINVAL, "k must be >= 0");
  if (ctx->count == 0) return set_err(ctx, DQN_EEMPTY, "replay memory is empty (A13)");
  const long long T0 = ctx->T;
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  long long kernels = 0;
  if (ctx->use_graphs && !ctx->async) {
    int rc = run_steps_chunked(ctx, k, &kernels);
    if (rc) return rc;
  } else {
    for (long long s = 0; s < k; ++s) {
      // O10 / O11: fetch at the start of step T when T % n_fetch == 0, then refresh theta^ when n - l >= C
      int rc = do_step(ctx, false, &kernels, nullptr, nullptr, nullptr);
      if (rc) return rc;
    }
  }
  return finish_steps(ctx, T0, k, kernels, stats);
}

extern "C" int dqn_store_and_train(dqn_ctx* ctx, int64_t k, const uint8_t* s, const int32_t* a, const float* r,
                                   const uint8_t* s_next, const uint8_t* terminal, dqn_step_stats* stats) {
  if (!ctx) return DQN_EINVAL;
  if (ctx->poisoned) return DQN_ESTATE;
  if (k < 0) return set_err(ctx, DQN_EINVAL, "k must be >= 0");
  if (!ctx->use_graphs || ctx->async)
    return set_err(ctx, DQN_EINVAL, "dqn_store_and_train needs the deterministic graph-replayed schedule");
  if (k == 0) return DQN_OK;
  // bf16 Mnih path: the Store becomes the first kernel of every step inside the replayed multi-step
  // graphs (store_step_kernel), so the steps keep their PDL overlap; otherwise one ring kernel plus a
  // one-step graph per iteration (DQN_GRAPH_STORE=0 forces the latter)
  const char* gs = getenv("DQN_GRAPH_STORE");
  if (!ctx->store_ctl && ctx->bf16 && !ctx->gpath && !ctx->prio && !(gs && atoi(gs) == 0)) {
    int rc0 = dalloc(ctx, &ctx->store_ctl, 1);
    if (rc0) return rc0;
    if ((rc0 = dalloc(ctx, &ctx->store_flag, 2))) return rc0;  // monotone T + 1 of the last fused Store | join
    CK(cudaMemsetAsync(ctx->store_flag, 0, 2 * sizeof(unsigned long long), ctx->stream));
    ctx->graph_store = true;
  }
  const long long T0 = ctx->T;
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  long long kernels = 0;
  int rc = push_impl(ctx, k, s, a, r, s_next, terminal, &kernels);
  if (rc) return rc;
  return finish_steps(ctx, T0, k, kernels, stats);
}

// the end of a train call: counters, losses and diagnostics to pinned memory, ONE stream
// synchronisation, device-side error checks, stats
static int finish_steps(dqn_ctx* ctx, long long T0, long long k, long long kernels, dqn_step_stats* stats) {
  const dqn_config& c = ctx->cfg;
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  dqn_ctx::HostOut* ho = ctx->h_out;
  CK(cudaMemcpyAsync(&ho->ctr, ctx->ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, ctx->stream));
  std::vector<float> loss;
  const bool diag_ok = k > 0 && k <= kDiagSteps;
  if (diag_ok) {  // the k loss slots of the ring: at most two contiguous pieces
    const long long s0 = T0 % kDiagSteps, n0 = std::min<long long>(k, kDiagSteps - s0);
    CK(cudaMemcpyAsync(ho->loss, ctx->diag_loss + s0, sizeof(float) * n0, cudaMemcpyDeviceToHost, ctx->stream));
    if (k > n0)
      CK(cudaMemcpyAsync(ho->loss + n0, ctx->diag_loss, sizeof(float) * (k - n0), cudaMemcpyDeviceToHost, ctx->stream));
    if (stats && stats->sampled_idx)
      for (long long s = 0; s < k; ++s)
        CK(cudaMemcpyAsync(stats->sampled_idx + s * c.minibatch,
                           ctx->diag_idx + ((T0 + s) % kDiagSteps) * c.minibatch, sizeof(int) * c.minibatch,
                           cudaMemcpyDeviceToHost, ctx->stream));
    if (stats && stats->target_argmax)
      for (long long s = 0; s < k; ++s)
        CK(cudaMemcpyAsync(stats->target_argmax + s * c.minibatch,
                           ctx->diag_amax + ((T0 + s) % kDiagSteps) * c.minibatch, sizeof(int) * c.minibatch,
                           cudaMemcpyDeviceToHost, ctx->stream));
    if (stats && stats->td_error)
      for (long long s = 0; s < k; ++s)
        CK(cudaMemcpyAsync(stats->td_error + s * c.minibatch,
                           ctx->diag_delta + ((T0 + s) % kDiagSteps) * c.minibatch, sizeof(float) * c.minibatch,
                           cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->async) {  // the rounds this call pushed are applied; the fetch log and histogram come back
    CK(cudaStreamSynchronize(ctx->comm_stream));
    CK(cudaMemcpy(ctx->h_adev, ctx->adev, sizeof(AsyncDev), cudaMemcpyDeviceToHost));
    ctx->n_local = ctx->h_adev->n_local;
    ctx->ell = ctx->h_adev->ell;
  }
  const DevCounters hc = ho->ctr;
  if (ctx->step_trace) {  // DQN_TRACE_STEP=1: the last step's kernel timeline (CTA 0 stamps)
    unsigned long long t[4][ST_N][3] = {}, m[ST_N][3] = {};
    step_trace_bf16(0, &t[0][0][0]);
    step_trace_head(0, &t[1][0][0]);
    step_trace_common(0, &t[2][0][0]);
    step_trace_comm(0, &t[3][0][0]);
    for (int u = 0; u < 4; ++u)
      for (int q = 0; q < ST_N; ++q)
        for (int w = 0; w < 3; ++w)
          if (t[u][q][w]) m[q][w] = t[u][q][w];
    static const char* nm[ST_N] = {"", "conv_fwd", "fc_fwd", "head", "fc_bwd+finish", "conv_bwd", "bwd_reduce",
                                   "update", "server_round", "fwd:staged/conv1 mma/conv1 epi", "fwd:conv2 mma",
                                   "fc dW tile: staged/mma/exit", "fc dX tile: staged/mma/exit",
                                   "head finish: wait/-/exit", "bwd: dZ2 staged/conv2 mma/dZ1 epi", "bwd: db1 done/conv1 dW mma"};
    const unsigned long long t0 = m[ST_FWD][0];
    fprintf(stderr, "[dqn rank %d] step timeline (us from conv_fwd entry: entry / past wait / exit):", ctx->rank);
    for (int q = 1; q < ST_N; ++q)
      if (m[q][0] && t0)
        fprintf(stderr, " %s %.2f/%.2f/%.2f;", nm[q], ((double)m[q][0] - (double)t0) / 1e3,
                ((double)m[q][1] - (double)t0) / 1e3, ((double)m[q][2] - (double)t0) / 1e3);
    fprintf(stderr, "\n");
  }
  if (diag_ok) loss.assign(ho->loss, ho->loss + k);
  if (ctx->sra.trace) {  // DQN_TRACE_COMM=1: phases of the fused server round (block 0), last 64 rounds
    unsigned long long t[1024];
    if (cudaMemcpy(t, ctx->sra.trace, sizeof(t), cudaMemcpyDeviceToHost) == cudaSuccess) {
      // intervals: barrier A, work, release (block 0); first block start -> last release;
      // block 0 release -> next step past pdl_sync; acquire spin
      double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, sc[4] = {0, 0, 0, 0};
      int n = 0, nc = 0;
      for (int r = 0; r < 63; ++r) {  // skip the newest slot (its next-step stamps are not there yet)
        const unsigned long long* q = t + r * 16;
        if (!q[0] || q[3] <= q[0] || !q[7] || q[6] < q[3] || q[4] == ~0ull) continue;
        s[0] += (double)(q[1] - q[0]); s[1] += (double)(q[2] - q[1]); s[2] += (double)(q[3] - q[2]);
        s[3] += (double)(q[5] - q[4]); s[4] += (double)(q[6] - q[3]); s[5] += (double)(q[7] - q[6]);
        if (q[8] && q[10]) {  // the next step's first kernel (bf16): entry, gather landed, past pdl_sync
          s[6] += (double)q[8] - (double)q[5]; s[7] += (double)(q[9] - q[8]); s[8] += (double)(q[10] - q[9]);
        }
        if (q[13] && q[14] && q[14] != ~0ull) {  // spread of barrier A over the blocks; conv blocks' work and release
          sc[0] += (double)q[14] - (double)q[1]; sc[1] += (double)q[13] - (double)q[1];
          if (q[11] && q[12]) { sc[2] += (double)q[12] - (double)q[1]; sc[3] += (double)q[11] - (double)q[1]; ++nc; }
        }
        ++n;
      }
      if (getenv("DQN_TRACE_RAW"))
        for (int r = 0; r < 64; ++r) {
          const unsigned long long* q = t + r * 16;
          fprintf(stderr, "[dqn rank %d] slot %d:", ctx->rank, r);
          for (int k = 0; k < 8; ++k) fprintf(stderr, " %lld", (long long)(q[k] - q[0]));
          fprintf(stderr, "\n");
        }
      if (n)
        fprintf(stderr,
                "[dqn rank %d] fused round (%d rounds): barrier A %.2f us, reduce+update+deliver %.2f us, release %.2f us;"
                " all blocks %.2f us; release -> next kernel %.2f us; acquire %.2f us\n",
                ctx->rank, n, s[0] / n / 1e3, s[1] / n / 1e3, s[2] / n / 1e3, s[3] / n / 1e3, s[4] / n / 1e3,
                s[5] / n / 1e3);
      if (n)
        fprintf(stderr, "[dqn rank %d] relative to block 0 past barrier A: first / last block past it %.2f / %.2f us;"
                " conv blocks' work done %.2f us, conv release %.2f us (%d rounds)\n", ctx->rank, sc[0] / n / 1e3,
                sc[1] / n / 1e3, nc ? sc[2] / nc / 1e3 : 0.0, nc ? sc[3] / nc / 1e3 : 0.0, nc);
      if (n && ctx->bf16)
        fprintf(stderr, "[dqn rank %d] next fwd: entry - last round block %.2f us, gather %.2f us, expand+pdl_sync %.2f us\n",
                ctx->rank, s[6] / n / 1e3, s[7] / n / 1e3, s[8] / n / 1e3);
      fflush(stderr);
    }
  }
  if (hc.bad_input & 0x40000000u)
    return set_err(ctx, DQN_ECUDA, "fused Store: a forward CTA's wait for the stored slot timed out");
  if (hc.bad_input & 0x80000000u)
    return set_err(ctx, DQN_ECUDA, "fused server round: peer barrier timed out (ranks out of step?)");
  if (ctx->bf16 && gconv_error())
    return set_err(ctx, DQN_ECUDA, "generic conv kernel: an MMA completion was never signalled (bounded wait expired)");
  if (hc.T != (unsigned long long)ctx->T)
    return set_err(ctx, DQN_ECUDA, "device step counters diverged from the host schedule");
  if (hc.nonfinite > 0) ctx->diverged = true;
  if (stats) {
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    stats->device_ms = ms;
    stats->generation = ctx->n;
    stats->steps_done = ctx->T;
    stats->nonfinite_elems = hc.nonfinite;
    for (int i = 0; i < 32; ++i) stats->staleness_hist[i] = ctx->async ? ctx->h_adev->hist[i] : 0;
    if (stats->step_generation && diag_ok)
      for (long long t = T0; t < T0 + k; ++t)  // step t used the theta of its last fetch f = t / n_fetch (A40)
        stats->step_generation[t - T0] =
            ctx->async ? ctx->h_adev->fgen_log[(t / c.n_fetch) % kDiagSteps] : ctx->gen_log[t % kDiagSteps];
    stats->kernel_launches = kernels;
    stats->grad_ms = ctx->prof_grad_ms;
    stats->update_ms = ctx->prof_update_ms;
    stats->comm_ms = ctx->prof_comm_ms;
    double lm = 0.0;
    for (float l : loss) lm += l;
    stats->loss_mean = loss.empty() ? 0.0 : lm / (double)loss.size();
    if (stats->loss_per_step && diag_ok) std::memcpy(stats->loss_per_step, loss.data(), sizeof(float) * k);
  }
  if (ctx->diverged) return set_err(ctx, DQN_ENONFINITE, "a push round produced a non-finite mean gradient (A24)");
  return DQN_OK;
}

// ------------------------------------------------------------------ acting boundary (a15)
// The forward of m <= b states already in ctx->q_stage (canonical u8) with theta_local, Q into
// ctx->q_out [m][A] and the greedy actions into ctx->q_amax [m] (lowest index on ties); enqueued on
// the context stream without a host synchronisation (a15; reused by the on-GPU collector).
static int q_enqueue(dqn_ctx* ctx, int m) {
  const NetShape& net = ctx->net;
  const int b = ctx->cfg.minibatch;
  const long long sb = net.state_bytes;
  (void)sb;
  cudaStream_t st = ctx->stream;
  const float* in = nullptr;
  if (ctx->fused_comm && ctx->T > 0 && ctx->T % ctx->cfg.n_push == 0) {
    // the last step pushed: acquire the peers' deliveries of that round into theta_local before reading
    // it (the next step's first kernel would do it; G is cleared here and harmlessly again there)
    FusedAcquire f = ctx->acq;
    f.g_snap = nullptr;  // keep the round's gradient snapshot
    launch_fused_round_acquire(f, st);
  }
  if (ctx->gpath) {  // s2d staging, the generic tensor-core conv forward, FC split-K + reduction
    const FcShape& F = net.fc[0];
    launch_push_s2d(ctx->q_stage_s2d, nullptr, nullptr, nullptr, nullptr, b, 0, 0, m, ctx->q_stage, nullptr,
                    nullptr, nullptr, nullptr, st);
    for (int i = 0; i < net.n_conv; ++i) {
      const ConvShape& L = net.conv[i];
      const dqn_ctx::GLayer& G = ctx->gl[i];
      GConvFwdArgs a{};
      a.first = i == 0;
      if (i == 0) { a.ring[0] = ctx->q_stage_s2d; a.slot_stride = kMnihSlot; }  // ctr == nullptr: image j = slot j
      else a.x[0] = G.x[0];
      a.b = m; a.Hs = G.Hs; a.Ws = G.Ws; a.Cs = G.Cs; a.Th = G.Th; a.Tw = G.Tw; a.Ho = G.Ho; a.Wo = G.Wo; a.N = L.N;
      a.s_next = i + 1 < net.n_conv ? ctx->gl[i + 1].s : 0;
      a.wpk[0] = ctx->theta_local_bf16 + ctx->gpack_off + G.fwd_pack;
      a.bias[0] = ctx->theta_local + L.b_off;
      a.out[0] = i + 1 < net.n_conv ? ctx->gl[i + 1].x[0] : ctx->a2_bf16;
      launch_gconv_fwd(a, 1, st);
    }
    TcGemmArgs gf{};
    gf.A[0] = ctx->theta_local_bf16 + F.w_off; gf.lda = F.D;
    gf.B[0] = ctx->a2_bf16; gf.ldb = F.D;
    gf.M = F.H; gf.N = m; gf.K = F.D; gf.BN = std::min(128, (m + 15) / 16 * 16); gf.kper = F.D / ctx->fc_splits;
    gf.splits = ctx->fc_splits; gf.epi = TC_EPI_FC_FWD; gf.partial = ctx->fc_partial;
    gf.bias[0] = ctx->theta_local + F.b_off; gf.h_out[0] = ctx->act_fc[0][0];
    launch_gemm_pipe(gf, 1, st);
    launch_fc_reduce(gf, 1, st);
    in = ctx->act_fc[0][0];
  } else if (ctx->bf16) {  // conv1's s2d staging, then the tensor-core forward with theta_local
    const FcShape& F = net.fc[0];
    launch_push_s2d(ctx->q_stage_s2d, nullptr, nullptr, nullptr, nullptr, b, 0, 0, m, ctx->q_stage, nullptr,
                    nullptr, nullptr, nullptr, st);
    FwdConvArgs fa{};
    fa.ring[0] = ctx->q_stage_s2d;
    fa.img_off = ctx->img_off;
    fa.slot_stride = kMnihSlot;
    fa.theta[0] = ctx->theta_local_bf16;
    fa.theta_f32[0] = ctx->theta_local;
    fa.w1_off = net.conv[0].w_off; fa.b1_off = net.conv[0].b_off;
    fa.w2_off = net.conv[1].w_off; fa.b2_off = net.conv[1].b_off;
    fa.n = m; fa.a2 = ctx->a2_bf16;
    launch_fwd_conv_bf16(fa, 1, st);
    TcGemmArgs gf{};
    gf.A[0] = ctx->theta_local_bf16 + F.w_off; gf.lda = F.D;
    gf.B[0] = ctx->a2_bf16; gf.ldb = F.D;
    gf.M = F.H; gf.N = m; gf.K = F.D; gf.BN = (m + 15) / 16 * 16; gf.kper = F.D / ctx->fc_splits;
    gf.splits = ctx->fc_splits; gf.epi = TC_EPI_FC_FWD; gf.partial = ctx->fc_partial;
    gf.pre_a = 1; gf.pre_b = 0;
    gf.counters = ctx->tc_counters; gf.bias[0] = ctx->theta_local + F.b_off; gf.h_out[0] = ctx->act_fc[0][0];
    launch_tc_gemm(gf, 1, st);
    in = ctx->act_fc[0][0];
  } else {
  ImgSrc src{};
  src.u8[0] = ctx->q_stage;
  src.stride = sb;
  for (int i = 0; i < net.n_conv; ++i) {
    ImgSrc s2 = src;
    if (i > 0) {
      s2 = ImgSrc{};
      s2.f32[0] = ctx->act_conv[i - 1][0];
      const ConvShape& P = net.conv[i - 1];
      s2.stride = (long long)P.N * P.Ho * P.Wo;
    }
    launch_conv_fwd_f32(net.conv[i], s2, ctx->theta_local, nullptr, ctx->act_conv[i][0], nullptr, m, 1, st);
  }
  in = ctx->act_conv[net.n_conv - 1][0];
  }
  for (int l = 0; l < net.n_fc && !ctx->bf16; ++l) {
    const FcShape& F = net.fc[l];
    GemmArgs g{};
    g.A[0] = in; g.sam = F.D; g.sak = 1;
    g.B[0] = ctx->theta_local + F.w_off; g.sbk = 1; g.sbn = F.D;
    g.C[0] = ctx->act_fc[l][0]; g.scm = F.H; g.scn = 1;
    g.bias[0] = ctx->theta_local + F.b_off;
    g.M = m; g.N = F.H; g.K = F.D; g.groups = 1; g.splits = pick_splits(b, F.H, F.D, 1);
    g.epi = EPI_BIAS_RELU; g.partial = ctx->partial;
    launch_gemm_f32(g, st);
    in = ctx->act_fc[l][0];
  }
  const FcShape& O = net.fc[net.n_fc];
  launch_q_head_f32(in, ctx->theta_local, O.w_off, O.b_off, O.D, O.H, m, ctx->q_out, ctx->q_amax, st);
  CK(cudaGetLastError());
  return DQN_OK;
}

// ------------------------------------------------------------------ NEXT-3: on-GPU acting
extern "C" int dqn_collect(dqn_ctx* ctx, int32_t n_envs, int32_t grid, int64_t steps, double epsilon, uint64_t env_seed,
                           dqn_collect_stats* stats) {
  if (!ctx) return DQN_EINVAL;
  if (ctx->poisoned) return DQN_ESTATE;
  const NetShape& net = ctx->net;
  const int F = net.F, H = net.Hin;
  if (net.A != 4) return set_err(ctx, DQN_EINVAL, "dqn_collect: the Snake game needs n_actions == 4");
  if (ctx->prio) return set_err(ctx, DQN_EINVAL, "dqn_collect stores without priorities: not with replay_prio_alpha");
  if (net.Hin != net.Win || grid < 4 || grid > 32 || H % grid != 0 || ((long long)H * H) % 16 != 0)
    return set_err(ctx, DQN_EINVAL, "dqn_collect: needs square frames, 4 <= grid <= 32, height % grid == 0, H*H % 16 == 0");
  if (n_envs < 1 || n_envs > ctx->cfg.minibatch || n_envs > ctx->cap || steps < 0 || !(epsilon >= 0.0 && epsilon <= 1.0))
    return set_err(ctx, DQN_EINVAL, "dqn_collect: 1 <= n_envs <= min(minibatch, capacity), steps >= 0, eps in [0, 1]");
  dqn_ctx::Collector& C = ctx->env;
  cudaStream_t st = ctx->stream;
  const long long sb = net.state_bytes;
  int rc;
  if (!C.games) {
    C.E = n_envs; C.n = grid; C.seed = env_seed; C.t = 0;
    if ((rc = dalloc(ctx, &C.games, n_envs))) return rc;
    if ((rc = dalloc(ctx, &C.stacks, n_envs * sb))) return rc;
    if ((rc = dalloc(ctx, &C.s_stage, n_envs * sb))) return rc;
    if ((rc = dalloc(ctx, &C.sn_stage, n_envs * sb))) return rc;
    if ((rc = dalloc(ctx, &C.t_stage, n_envs))) return rc;
    if ((rc = dalloc(ctx, &C.a_stage, n_envs))) return rc;
    if ((rc = dalloc(ctx, &C.r_stage, n_envs))) return rc;
    if ((rc = dalloc(ctx, &C.episodes, n_envs))) return rc;
    if ((rc = dalloc(ctx, &C.reward_sum, n_envs))) return rc;
    CK(cudaMemsetAsync(C.episodes, 0, sizeof(long long) * n_envs, st));
    CK(cudaMemsetAsync(C.reward_sum, 0, sizeof(double) * n_envs, st));
    EnvArgs a{};
    a.games = C.games; a.stacks = C.stacks; a.n = grid; a.F = F; a.H = H; a.E = n_envs; a.seed = env_seed;
    launch_env_init(a, st);
    CK(cudaGetLastError());
  } else if (C.E != n_envs || C.n != grid || C.seed != env_seed) {
    return set_err(ctx, DQN_EINVAL, "dqn_collect: n_envs, grid and env_seed must match the first call");
  }
  // per-call logs (device scratch when the caller passes host buffers)
  int32_t* a_log = nullptr;
  float* r_log = nullptr;
  uint8_t* t_log = nullptr;
  const bool want = stats && (stats->actions || stats->rewards || stats->terminals) && steps > 0;
  if (want) {
    if ((rc = dalloc(ctx, &a_log, steps * n_envs))) return rc;
    if ((rc = dalloc(ctx, &r_log, steps * n_envs))) return rc;
    if ((rc = dalloc(ctx, &t_log, steps * n_envs))) return rc;
  }
  std::vector<long long> ep0(n_envs), ep1(n_envs);
  std::vector<double> rs0(n_envs), rs1(n_envs);
  CK(cudaMemcpyAsync(ep0.data(), C.episodes, sizeof(long long) * n_envs, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(rs0.data(), C.reward_sum, sizeof(double) * n_envs, cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(ctx->ev0, st));
  const unsigned long long thr =
      epsilon >= 1.0 ? (1ULL << 32) : (unsigned long long)std::floor(epsilon * 4294967296.0);
  for (long long s = 0; s < steps; ++s) {
    // Q(phi; theta_local) of every game's stack, greedy actions into ctx->q_amax
    CK(cudaMemcpyAsync(ctx->q_stage, C.stacks, n_envs * sb, cudaMemcpyDeviceToDevice, st));
    if ((rc = q_enqueue(ctx, n_envs))) return rc;
    EnvArgs a{};
    a.games = C.games; a.stacks = C.stacks; a.s_stage = C.s_stage; a.sn_stage = C.sn_stage;
    a.a_stage = C.a_stage; a.r_stage = C.r_stage; a.t_stage = C.t_stage; a.greedy = ctx->q_amax;
    a.n = grid; a.F = F; a.H = H; a.E = n_envs; a.seed = env_seed; a.t = C.t; a.eps_thr = thr;
    a.a_log = a_log; a.r_log = r_log; a.t_log = t_log; a.log_row = s;
    a.episodes = C.episodes; a.reward_sum = C.reward_sum;
    launch_env_act(a, st);
    // Store (Alg. 1): the step's transitions into the replay, on the device
    push_ring(ctx, 0, n_envs, C.s_stage, C.a_stage, C.r_stage, C.sn_stage, C.t_stage);
    CK(cudaGetLastError());
    ctx->count += n_envs;
    C.t += 1;
  }
  CK(cudaEventRecord(ctx->ev1, st));
  CK(cudaMemcpyAsync(ep1.data(), C.episodes, sizeof(long long) * n_envs, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(rs1.data(), C.reward_sum, sizeof(double) * n_envs, cudaMemcpyDeviceToHost, st));
  if (want) {
    auto kind = [](const void* p) { return is_device_ptr(p) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost; };
    if (stats->actions)
      CK(cudaMemcpyAsync(stats->actions, a_log, sizeof(int32_t) * steps * n_envs, kind(stats->actions), st));
    if (stats->rewards)
      CK(cudaMemcpyAsync(stats->rewards, r_log, sizeof(float) * steps * n_envs, kind(stats->rewards), st));
    if (stats->terminals)
      CK(cudaMemcpyAsync(stats->terminals, t_log, steps * n_envs, kind(stats->terminals), st));
  }
  CK(cudaStreamSynchronize(st));
  if (want) {
    cudaFree(a_log);
    cudaFree(r_log);
    cudaFree(t_log);
  }
  if (stats) {
    stats->env_steps = steps * n_envs;
    long long de = 0;
    double dr = 0.0;
    for (int e = 0; e < n_envs; ++e) {
      de += ep1[e] - ep0[e];
      dr += rs1[e] - rs0[e];
    }
    stats->episodes = de;
    stats->reward_sum = dr;
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    stats->device_ms = ms;
  }
  return DQN_OK;
}

extern "C" int dqn_env_stacks(dqn_ctx* ctx, uint8_t* out, int64_t cap_bytes) {
  if (!ctx) return DQN_EINVAL;
  if (ctx->poisoned) return DQN_ESTATE;
  if (!ctx->env.games) return set_err(ctx, DQN_ESTATE, "dqn_env_stacks: no games yet (call dqn_collect first)");
  const long long bytes = (long long)ctx->env.E * ctx->net.state_bytes;
  if (!out || cap_bytes < bytes) return set_err(ctx, DQN_EINVAL, "dqn_env_stacks: output smaller than n_envs * F*H*W");
  CK(cudaMemcpyAsync(out, ctx->env.stacks, bytes, is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return DQN_OK;
}

extern "C" int dqn_q_values(dqn_ctx* ctx, int64_t n, const uint8_t* states, float* q, int32_t* argmax) {
  if (!ctx) return DQN_EINVAL;
  if (ctx->poisoned) return DQN_ESTATE;
  if (n < 0 || (n > 0 && (!states || !q))) return set_err(ctx, DQN_EINVAL, "bad q_values args");
  const NetShape& net = ctx->net;
  const int b = ctx->cfg.minibatch;
  const long long sb = net.state_bytes;
  const bool dev_in = is_device_ptr(states), dev_q = is_device_ptr(q), dev_a = argmax && is_device_ptr(argmax);
  cudaStream_t st = ctx->stream;
  for (long long i0 = 0; i0 < n; i0 += b) {
    const int m = (int)std::min<long long>(b, n - i0);
    CK(cudaMemcpyAsync(ctx->q_stage, states + i0 * sb, m * sb, dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       st));
    int rc = q_enqueue(ctx, m);
    if (rc) return rc;
    CK(cudaMemcpyAsync(q + i0 * net.A, ctx->q_out, sizeof(float) * m * net.A,
                       dev_q ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    if (argmax)
      CK(cudaMemcpyAsync(argmax + i0, ctx->q_amax, sizeof(int) * m,
                         dev_a ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return DQN_OK;
}

// ------------------------------------------------------------------ parameter readback
extern "C" int dqn_get_params(dqn_ctx* ctx, int which, float* out, int64_t cap, int64_t* n_params,
                              uint64_t* generation) {
  if (!ctx) return DQN_EINVAL;
  if (ctx->poisoned) return DQN_ESTATE;
  if (n_params) *n_params = ctx->P;
  if (generation)
    *generation = (uint64_t)(which == DQN_PARAMS_LOCAL || which == DQN_PARAMS_LOCAL_BF16 ? ctx->n_local
                             : which == DQN_PARAMS_TARGET || which == DQN_PARAMS_TARGET_BF16 ? ctx->ell
                                                                                             : ctx->n);
  if (!out) return DQN_OK;
  if (cap < ctx->P) return set_err(ctx, DQN_EINVAL, "output buffer smaller than P");
  const cudaMemcpyKind kind = is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  const float* src = nullptr;
  switch (which) {
    case DQN_PARAMS_LOCAL:
      if (!(ctx->fused_comm && ctx->bf16)) {
        src = ctx->theta_local;
        break;
      }
      // fused bf16 round: theta_local's fp32 FC weight holds only this rank's slice, and with
      // n_fetch = 1 the working copy equals the gathered server parameters
      [[fallthrough]];
    case DQN_PARAMS_SERVER:
    case DQN_PARAMS_RMS: {
      float* shard = which == DQN_PARAMS_RMS ? ctx->rms : ctx->theta_master;
      if (ctx->async) {  // let the round in flight finish; the server state lives on the comm stream
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaStreamSynchronize(ctx->comm_stream));
      }
      if (ctx->world > 1) {
        cudaStream_t cs = ctx->async ? ctx->comm_stream : ctx->stream;
        NK(ncclAllGather(shard, ctx->gather_tmp, (size_t)ctx->shard, ncclFloat, ctx->comm, cs));
        CK(cudaStreamSynchronize(cs));
        src = ctx->gather_tmp;
      } else {
        src = shard;
      }
      break;
    }
    case DQN_PARAMS_TARGET: src = ctx->theta_hat; break;
    case DQN_PARAMS_GRAD:
      if (!ctx->grad_snap) return set_err(ctx, DQN_EINVAL, "gradient snapshots need cfg.keep_grad = 1 at create");
      src = ctx->grad_snap;
      break;
    case DQN_PARAMS_LOCAL_BF16:
    case DQN_PARAMS_TARGET_BF16: {  // the canonical entries of a bf16 working copy, widened (exact)
      if (!ctx->bf16) return set_err(ctx, DQN_EINVAL, "bf16 working copies exist only on DQN_BF16");
      float* tmp = nullptr;
      int rc = dalloc(ctx, &tmp, ctx->P);
      if (rc) return rc;
      launch_bf16_to_f32(which == DQN_PARAMS_LOCAL_BF16 ? ctx->theta_local_bf16 : ctx->theta_hat_bf16, tmp, ctx->P,
                         ctx->stream);
      cudaError_t e = cudaMemcpyAsync(out, tmp, sizeof(float) * ctx->P, kind, ctx->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
      cudaFree(tmp);
      CK(e);
      return DQN_OK;
    }
    default: return set_err(ctx, DQN_EINVAL, "unknown parameter vector");
  }
  if (ctx->fetch_bf16 && (which == DQN_PARAMS_LOCAL || which == DQN_PARAMS_TARGET)) {
    // the NCCL bf16 fetch delivers the FC weight in bf16 only: widen it from the working copy
    float* tmp = nullptr;
    int rc = dalloc(ctx, &tmp, ctx->P);
    if (rc) return rc;
    cudaError_t e = cudaMemcpyAsync(tmp, src, sizeof(float) * ctx->P, cudaMemcpyDeviceToDevice, ctx->stream);
    if (e == cudaSuccess) {
      launch_widen_range(which == DQN_PARAMS_LOCAL ? ctx->theta_local_bf16 : ctx->theta_hat_bf16, tmp,
                         ctx->frec.fw_lo, ctx->frec.fw_hi, ctx->stream);
      e = cudaMemcpyAsync(out, tmp, sizeof(float) * ctx->P, kind, ctx->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(tmp);
    CK(e);
    return DQN_OK;
  }
  CK(cudaMemcpyAsync(out, src, sizeof(float) * ctx->P, kind, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return DQN_OK;
}

extern "C" int dqn_get_priorities(dqn_ctx* ctx, float* out, int64_t cap, float* total) {
  if (!ctx) return DQN_EINVAL;
  if (ctx->poisoned) return DQN_ESTATE;
  if (!ctx->prio) return set_err(ctx, DQN_EINVAL, "priorities exist only with replay_prio_alpha != 0");
  if (out && cap < ctx->cap) return set_err(ctx, DQN_EINVAL, "output buffer smaller than replay_capacity");
  if (out)
    CK(cudaMemcpyAsync(out, ctx->ptree.node, sizeof(float) * ctx->cap,
                       is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->stream));
  if (total)
    CK(cudaMemcpyAsync(total, ctx->ptree.node + ctx->ptree.off[ctx->ptree.K], sizeof(float),
                       is_device_ptr(total) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return DQN_OK;
}

extern "C" int dqn_replay_size(const dqn_ctx* ctx, int64_t* count, int64_t* size) {
  if (!ctx) return DQN_EINVAL;
  if (count) *count = ctx->count;
  if (size) *size = std::min(ctx->count, ctx->cap);
  return DQN_OK;
}

// ctx == NULL: message of the last failed dqn_create on this thread
extern "C" const char* dqn_last_error(const dqn_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

extern "C" void dqn_destroy(dqn_ctx* ctx) {
  if (!ctx) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->comm_stream) cudaStreamSynchronize(ctx->comm_stream);
  free_all(ctx);
  delete ctx;
}
