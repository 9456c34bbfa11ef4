// kernels_env.cu — NEXT-3: the acting side of Alg. 1 on the GPU: E parallel Snake
// games (rule closures of SPEC S:216-262, readings A34-A36), the eps-greedy behaviour policy
// on Q from the network's forward (a15), and the Store of every transition into the replay.
//
// One CTA per game. Thread 0 runs the (sequential, tiny) game logic; the CTA renders the grid into
// an F-frame stack (whole-cell replication: area averaging of an integer upscale) and writes the
// transition's s and s' into the push staging. Random draws: Philox4x32-10, key = seed, counter
// (env, t_lo, t_hi, purpose) — purpose 0 eps-greedy (x0 explore, x1 action), 1 the apple after
// eating, 2 the apple of a reset (the initial reset uses t = 2^64 - 1). Same order and arithmetic
// as the oracle's or_collect, so a run is bit-exact against it whenever the greedy actions agree
// (always at eps = 1).
#include "dqn_internal.h"
#include "philox.cuh"

namespace dqn {

namespace {

__device__ __forceinline__ void env_draw(unsigned long long seed, unsigned env, unsigned long long t, unsigned purpose,
                                         uint32_t x[4]) {
  uint32_t c0 = env, c1 = (uint32_t)t, c2 = (uint32_t)(t >> 32), c3 = purpose;
  philox4x32_10(c0, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
  x[0] = c0; x[1] = c1; x[2] = c2; x[3] = c3;
}

// the k-th free cell (row-major), k = floor(x * free / 2^32); -1 when the grid is full
__device__ int place_apple(const EnvGame& g, int n, uint32_t x, uint8_t* occ /* [n*n] scratch */) {
  for (int c = 0; c < n * n; ++c) occ[c] = 0;
  for (int i = 0; i < g.len; ++i) occ[g.body[i]] = 1;
  const int free_cells = n * n - g.len;
  if (free_cells <= 0) return -1;
  int k = (int)(((unsigned long long)x * (unsigned long long)free_cells) >> 32);
  for (int c = 0; c < n * n; ++c)
    if (!occ[c] && k-- == 0) return c;
  return -1;
}

__device__ void game_reset(EnvGame& g, int n, unsigned long long seed, unsigned env, unsigned long long t,
                           uint8_t* occ) {
  const int c = n / 2;
  g.len = 2;
  g.dir = 1;
  g.since = 0;
  g.body[0] = (int16_t)(c * n + c);
  g.body[1] = (int16_t)(c * n + c - 1);
  uint32_t x[4];
  env_draw(seed, env, t, 2, x);
  g.apple = place_apple(g, n, x[0], occ);
}

// one step (thread 0); a terminal step leaves the state unchanged
__device__ float game_step(EnvGame& g, int n, int action, unsigned long long seed, unsigned env, unsigned long long t,
                           int* term, uint8_t* occ) {
  *term = 0;
  if ((action + 2) % 4 != g.dir) g.dir = action;
  const int hy = g.body[0] / n, hx = g.body[0] % n;
  const int ny = hy + (g.dir == 2) - (g.dir == 0), nx = hx + (g.dir == 1) - (g.dir == 3);
  if (ny < 0 || ny >= n || nx < 0 || nx >= n) {
    *term = 1;
    return -1.0f;
  }
  const int nh = ny * n + nx;
  if (nh == g.apple) {
    for (int i = g.len; i > 0; --i) g.body[i] = g.body[i - 1];
    g.body[0] = (int16_t)nh;
    g.len += 1;
    g.since = 0;
    uint32_t x[4];
    env_draw(seed, env, t, 1, x);
    g.apple = place_apple(g, n, x[0], occ);
    if (g.apple < 0) *term = 1;
    return 1.0f;
  }
  for (int i = 0; i < g.len - 1; ++i)
    if (g.body[i] == nh) {
      *term = 1;
      return -1.0f;
    }
  for (int i = g.len - 1; i > 0; --i) g.body[i] = g.body[i - 1];
  g.body[0] = (int16_t)nh;
  g.since += 1;
  if (g.since >= 200 * n) *term = 1;
  return 0.0f;
}

// cell values of the game (empty 0, body 128, head 191, apple 255) into smem
__device__ void cell_map(const EnvGame& g, int n, uint8_t* cell) {
  for (int c = threadIdx.x; c < n * n; c += blockDim.x) cell[c] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < g.len; ++i) cell[g.body[i]] = 128;
    cell[g.body[0]] = 191;
    if (g.apple >= 0) cell[g.apple] = 255;
  }
  __syncthreads();
}

// frame (H x H u8) of the cell map: pixel (y, x) = cell (y / px, x / px)
__device__ void render(const uint8_t* cell, int n, int H, uint8_t* dst) {
  const int px = H / n;
  for (int i = threadIdx.x; i < H * H; i += blockDim.x) dst[i] = cell[(i / H / px) * n + (i % H) / px];
}

}  // namespace

__global__ void __launch_bounds__(256) env_init_kernel(EnvArgs a) {
  __shared__ EnvGame g;
  __shared__ uint8_t occ[1024], cell[1024];
  const int e = blockIdx.x;
  if (threadIdx.x == 0) game_reset(g, a.n, a.seed, (unsigned)e, ~0ULL, occ);
  __syncthreads();
  cell_map(g, a.n, cell);
  const long long fb = (long long)a.H * a.H;
  uint8_t* st = a.stacks + (long long)e * a.F * fb;
  for (int f = 0; f < a.F; ++f) render(cell, a.n, a.H, st + f * fb);
  if (threadIdx.x == 0) a.games[e] = g;
}

// one acting step of every game: eps-greedy action, game step, s / s' / a / r / term into the push
// staging, the stack advanced (or reset after a terminal step)
__global__ void __launch_bounds__(256) env_act_kernel(EnvArgs a) {
  __shared__ EnvGame g;
  __shared__ uint8_t occ[1024], cell[1024];
  __shared__ int s_term;
  const int e = blockIdx.x;
  const long long fb = (long long)a.H * a.H;
  uint8_t* st = a.stacks + (long long)e * a.F * fb;
  uint8_t* ss = a.s_stage + (long long)e * a.F * fb;
  uint8_t* sn = a.sn_stage + (long long)e * a.F * fb;
  if (threadIdx.x == 0) {
    g = a.games[e];
    uint32_t x[4];
    env_draw(a.seed, (unsigned)e, a.t, 0, x);
    const int act = (unsigned long long)x[0] < a.eps_thr ? (int)(x[1] >> 30) : a.greedy[e];
    int term;
    const float r = game_step(g, a.n, act, a.seed, (unsigned)e, a.t, &term, occ);
    s_term = term;
    a.a_stage[e] = act;
    a.r_stage[e] = r;
    a.t_stage[e] = (uint8_t)term;
    if (a.a_log) a.a_log[a.log_row * a.E + e] = act;
    if (a.r_log) a.r_log[a.log_row * a.E + e] = r;
    if (a.t_log) a.t_log[a.log_row * a.E + e] = (uint8_t)term;
    a.reward_sum[e] += (double)r;
    if (term) a.episodes[e] += 1;
  }
  __syncthreads();
  // s = the current stack; s' = frames 1..F-1 and the render of the stepped game (Alg. 1 "preprocess")
  const long long n16 = a.F * fb / 16;
  for (long long v = threadIdx.x; v < n16; v += blockDim.x)
    reinterpret_cast<uint4*>(ss)[v] = reinterpret_cast<const uint4*>(st)[v];
  const long long m16 = (a.F - 1) * fb / 16;
  for (long long v = threadIdx.x; v < m16; v += blockDim.x)
    reinterpret_cast<uint4*>(sn)[v] = reinterpret_cast<const uint4*>(st + fb)[v];
  cell_map(g, a.n, cell);
  render(cell, a.n, a.H, sn + (a.F - 1) * fb);
  __syncthreads();
  if (s_term) {  // a new episode: the first frame replicated F times
    if (threadIdx.x == 0) game_reset(g, a.n, a.seed, (unsigned)e, a.t, occ);
    __syncthreads();
    cell_map(g, a.n, cell);
    for (int f = 0; f < a.F; ++f) render(cell, a.n, a.H, st + f * fb);
  } else {
    for (long long v = threadIdx.x; v < n16; v += blockDim.x)
      reinterpret_cast<uint4*>(st)[v] = reinterpret_cast<const uint4*>(sn)[v];
  }
  if (threadIdx.x == 0) a.games[e] = g;
}

void launch_env_init(const EnvArgs& a, cudaStream_t st) { env_init_kernel<<<a.E, 256, 0, st>>>(a); }
void launch_env_act(const EnvArgs& a, cudaStream_t st) { env_act_kernel<<<a.E, 256, 0, st>>>(a); }

}  // namespace dqn
