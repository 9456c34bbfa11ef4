// dqn_internal.h — shapes, device-side state and kernel launchers shared by the
// runtime (dqn_runtime.cu) and the kernel translation units. Product code only;
// nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <cuda.h>  // CUtensorMap (types only; the encode entry point is fetched from the driver at run time)
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace dqn {

constexpr int kMaxConv = 4;
constexpr int kMaxFc = 4;
constexpr int kDiagSteps = 4096;  // ring of per-step diagnostics (idx, argmax, loss)
constexpr int kHeadMaxSplits = 24;  // FC forward split-K partials the TD head sums (head_sample_kernel)

// One valid convolution layer (A16): in C x H x W, out N x Ho x Wo.
struct ConvShape {
  int C, H, W, N, k, s, Ho, Wo;
  long long w_off, b_off;  // canonical offsets: W [N][C][k][k] then b [N]
};
// One fully connected layer: in D, out H (hidden: ReLU; last: linear output).
struct FcShape {
  int D, H;
  long long w_off, b_off;  // W [H][D] then b [H]
};
struct NetShape {
  int F, Hin, Win;
  int n_conv;
  ConvShape conv[kMaxConv];
  int n_fc;                 // hidden FC layers
  FcShape fc[kMaxFc + 1];   // hidden FCs then the output layer (fc[n_fc])
  int A;                    // |A|
  long long P;
  long long state_bytes;    // F*Hin*Win
};

// Device counters (one struct in device memory per context). Kernels read T at
// the start of a step and the head kernel advances it, so captured CUDA graphs
// are replayable.
struct DevCounters {
  unsigned long long T;         // replica step counter
  long long n;                  // server generation (mirrored on host in deterministic mode)
  unsigned int nonfinite;       // # of non-finite mean-gradient elements seen (sticky)
  unsigned int nonfinite_rounds;
  unsigned int bad_input;       // push validation
  unsigned int nonfinite_last;  // value of `nonfinite` at the end of the previous round
  long long ring_size;          // min(count, capacity), written by the push path
  unsigned int blocks_done;     // last-block-done counter of the update kernel
  unsigned int pad2;
};

// Where the input image of a (group, image) comes from.
// u8 mode: ring[g] + idx[img] * stride (idx == nullptr: image i at i * stride)
// f32 mode: f32[g] + img * stride
struct ImgSrc {
  const uint8_t* u8[2];
  const float* f32[2];
  const int* idx;
  long long stride;
};

enum Epi { EPI_STORE = 0, EPI_ACCUM = 1, EPI_BIAS_RELU = 2, EPI_BIAS = 3, EPI_MASK = 4 };

struct GemmArgs {
  const float* A[2];
  long long sam, sak;  // A(m,k) = A[m*sam + k*sak]
  const float* B[2];
  long long sbk, sbn;  // B(k,n) = B[k*sbk + n*sbn]
  float* C[2];
  long long scm, scn;  // C(m,n) = C[m*scm + n*scn]
  const float* bias[2];       // indexed by n (EPI_BIAS*)
  const float* mask[2];       // EPI_MASK: keep where mask(m,n) > 0
  long long smm, smn;
  int M, N, K;
  int groups;                 // 1 or 2 (independent problems sharing shapes)
  int splits;                 // split-K factor (>1: partial buffer + reduce kernel)
  int epi;
  float* partial;             // [groups][splits][M][N] when splits > 1
};

struct HeadArgs {
  int st_id;                  // DQN_TRACE_STEP slot (step_trace.cuh), 0 = none
  const float* act[2];        // [b][H]: input of the output layer for s (theta) / s' (theta^)
  // bf16 path: act[] is produced here from the FC split-K partials [g][split][b_row][H]
  const float* fc_partial;    // nullptr: act[] given
  int fc_splits;
  long long fc_split_stride;  // floats between splits
  const float* fc_bias[2];
  float* act_out[2];          // where the reduced activations are stored (h of s is reused by the finish)
  // per-sample scratch written by head_sample, read by head_finish
  float* s_dq;                // [b]
  int* s_act;                 // [b]
  float* s_loss;              // [b]
  float* s_delta;             // [b] delta_j (unclipped TD error; the prioritized replay's update reads it)
  const float* theta;         // live theta (fp32, canonical)
  const float* theta_hat;     // target theta^ (fp32, canonical)
  long long w_off, b_off;     // output layer
  long long prev_b_off;       // bias of the previous hidden FC (if prev_is_fc)
  int prev_is_fc;
  int H, A, b;
  const int* idx;
  const int32_t* ring_a;
  const float* ring_r;
  const uint8_t* ring_term;
  float gamma, clip;
  float* grad;                // G (accumulated)
  float* dH;                  // [b][H] d(pre-activation) of the previous layer
  __nv_bfloat16* dH_bf16;     // optional bf16 copy of dH (tensor-core backward operand)
  DevCounters* ctr;
  float* diag_loss;           // [kDiagSteps]
  int* diag_idx;              // [kDiagSteps][b]
  int* diag_amax;             // [kDiagSteps][b]
  float* diag_delta;          // [kDiagSteps][b] delta_j per step (dqn_step_stats.td_error)
};

// prioritized replay (NEXT-4, A41): 32-ary fp32 sum tree, level l at node + off[l], level K = the root
constexpr int kPrioMaxLevels = 6;  // 32^6 slots
struct PrioTree {
  float* node;
  long long off[kPrioMaxLevels + 1];
  int K;
};

// ------------------------------------------------------------------ launchers
// common (kernels_common.cu)
void launch_sample(int* idx, int b, unsigned long long seed, unsigned rank, const DevCounters* ctr,
                   cudaStream_t st);
void launch_validate_push(const int32_t* a, const float* r, long long n, int A, DevCounters* ctr, cudaStream_t st);
void launch_validate_dedup(const uint8_t* s, const uint8_t* sn, long long n, long long sb, long long fb,
                           DevCounters* ctr, cudaStream_t st);
void launch_push_canonical(uint8_t* ring_s, uint8_t* ring_sn, int32_t* ring_a, float* ring_r, uint8_t* ring_t,
                           long long cap, long long count0, long long n_total, long long first, long long n,
                           long long state_bytes, const uint8_t* s, const int32_t* a, const float* r,
                           const uint8_t* sn, const uint8_t* t, cudaStream_t st, long long* ring_size_out = nullptr,
                           long long ring_size = 0, long long stride = 0, int dedup = 0);
// pack_map (generic path, N = 1): also write the updated conv parameters i < pack_n into their packed slots
// pub_bf16[pack_off + map[i].x / .y] (what gpack_kernel does at the start of a step)
void launch_rmsprop(float* theta, float* r, float* g, long long n, float div, float lr, float rho, float omr,
                    float eps, float* pub_f32, __nv_bfloat16* pub_bf16, DevCounters* ctr, int zero_g,
                    cudaStream_t st, long long img_off = -1,
                    long long w1_off = 0, long long w2_off = 0, float* g_snap = nullptr,
                    const int2* pack_map = nullptr, long long pack_n = 0, long long pack_off = 0);
void launch_f32_to_bf16(const float* src, __nv_bfloat16* dst, long long n, cudaStream_t st, long long img_off = -1,
                        long long w1_off = 0, long long w2_off = 0);
void launch_bf16_to_f32(const __nv_bfloat16* src, float* dst, long long n, cudaStream_t st);

// fp32 SIMT path (kernels_f32.cu)
void init_f32_kernel_attrs();
void launch_conv_fwd_f32(const ConvShape& cs, const ImgSrc& src, const float* theta0, const float* theta1,
                         float* out0, float* out1, int b, int groups, cudaStream_t st);
void launch_conv_bwd_dx_f32(const ConvShape& cs, const float* dout, const float* theta, const float* a_in,
                            float* din, int b, cudaStream_t st);
void launch_conv_bwd_dw_f32(const ConvShape& cs, const float* dout, const ImgSrc& src, float* partial, int b,
                            cudaStream_t st);
void launch_reduce_rows(const float* partial, int rows, long long E, float* dst, cudaStream_t st);
void launch_gemm_f32(const GemmArgs& g, cudaStream_t st);
void launch_bias_grad(const float* dz, int b, int H, float* dst, cudaStream_t st);
void launch_head_f32(const HeadArgs& h, cudaStream_t st, bool with_finish = true);
size_t head_smem_bytes(int A, int H, int b);
void launch_q_head_f32(const float* act, const float* theta, long long w_off, long long b_off, int H, int A, int n,
                       float* q, int* argmax, cudaStream_t st);

// NEXT-1: push + RMSProp + fetch in one kernel over NVLink peer memory (kernels_comm.cu)
constexpr int kMaxWorld = 8;
struct ServerRoundArgs {
  int world, rank, n_push;
  long long shard;                              // elements owned per rank (multiple of 64)
  long long grad_elems;                         // P_pad
  float* grad[kMaxWorld];                       // every rank's G (peer pointers; [rank] is local)
  float* theta_local[kMaxWorld];                // every rank's working theta (fp32)
  __nv_bfloat16* theta_local_bf16[kMaxWorld];   // and its bf16 copy (nullptr on the fp32 path)
  long long f32_peer_lo, f32_peer_hi;           // theta range read only as bf16: no fp32 copy to peers
  long long img_off, w1_off, w2_off;            // bf16 path: conv weight image (wimg.cuh), img_off < 0: none
  unsigned long long* flags[kMaxWorld];         // every rank's barrier-A array [world]
  unsigned long long* done[kMaxWorld];          // every rank's barrier-B counter
  unsigned long long* my_flags;
  unsigned long long* my_done;
  unsigned long long* my_join;                  // local gpu-scope join counter of barrier B
  float* theta_master;                          // owned shard
  float* rms;
  float inv_div, lr, rho, omr, eps;
  int per_gradient;                             // A33: apply each worker's gradient in rank order
  float inv_np;                                 // 1 / n_push (per-gradient rule)
  DevCounters* ctr;
  unsigned long long* trace;                    // optional [64][8] globaltimer stamps (DQN_TRACE_COMM=1)
  // conv-first delivery (bf16 Mnih path): the blocks holding the conv parameters (the canonical prefix,
  // conv4 float4s of this rank's shard; 0: none) release them early through a second counter
  long long conv4;
  unsigned long long* done_c[kMaxWorld];        // every rank's conv-release counter
  unsigned long long* my_join_c;                // local join counter of the conv blocks
  int conv_per_block = 256;                     // conv-prefix float4s per block (1..256)
};
void launch_server_round(const ServerRoundArgs& a, cudaStream_t st);
// the acquire half of the round's second barrier, run at the start of the next step
struct FusedAcquire {
  const unsigned long long* done;               // this rank's barrier-B counter (rounds * world)
  int world, n_push;
  float* grad;                                  // this rank's G, cleared once every peer has read it
  long long grad_elems;
  DevCounters* ctr;                             // nullptr: no fused round in this context
  unsigned long long* trace;                    // the server round's trace (slots 6, 7) or nullptr
  // conv-first delivery: the next step's conv forward waits only for the conv parameters (done_c >=
  // rounds * n_c, n_c = ranks owning conv parameters) instead of the round's grid completion, and the
  // FC forward acquires the whole round (done) and clears G
  const unsigned long long* done_c;
  int n_c;
  int conv_first;
  float* g_snap;                                // cfg.keep_grad: G copied here before it is cleared (or nullptr)
};
void launch_fused_round_acquire(const FusedAcquire& f, cudaStream_t st);
// DQN_ASYNC / DQN_ASYNC_LAG1: device state of the asynchronous schedule
struct AsyncDev {
  unsigned long long pub_gen;      // newest generation the comm stream has published (release store)
  long long n_local, ell;          // generation of the working theta / of theta^ (Alg. 1 state line)
  long long fetch_gen;             // the generation the pending fetch copies
  int do_refresh, pad;
  long long hist[32];              // A25: replica steps by staleness n_apply - n_base (31: >= 31)
  long long fgen_log[kDiagSteps];  // generation taken by fetch f, at f % kDiagSteps
};
struct AsyncCopy {
  const float* pub[3];             // published server theta by generation % 3 (fp32, canonical)
  const __nv_bfloat16* pubb[3];    // and its bf16 working image (nullptr on the fp32 path)
  float* th;                       // theta_local
  __nv_bfloat16* thb;
  float* hat;                      // theta^ (copied too when the fetch refreshes, A10)
  __nv_bfloat16* hatb;
  long long n32, n16;              // fp32 / bf16 elements
  long long npr;                   // generations per round (1, or N with the per-gradient rule): slot = m / npr % 3
};
// fetch f: pick the generation (forced >= 0: that one, the lag-1 twin; else the newest published), decide
// the refresh (n - l >= C), log it; then copy it into the working buffers
void launch_async_pick(AsyncDev* d, long long forced, long long C, long long f, cudaStream_t st);
void launch_async_copy(const AsyncDev* d, const AsyncCopy& c, cudaStream_t st);
// comm stream, after round k = n0 / npr's theta is in pub[(k+1) % 3]: staleness of the round's steps (n0 minus
// the generation each used), then publish generation n0 + npr
void launch_async_publish(AsyncDev* d, long long n0, long long npr, int n_push, int n_fetch, unsigned delay_ns,
                          cudaStream_t st);
// A33 over NCCL (DQN_ASYNC*): theta, r of the owned shard updated by the inbox's world gradients in rank order
void launch_rmsprop_per_gradient(float* theta, float* r, const float* inbox, int world, long long shard, float n_push,
                                 float lr, float rho, float omr, float eps, DevCounters* ctr, cudaStream_t st);

// a13 over NCCL on the bf16 path: the per-rank record of one all-gather (kernels_comm.cu)
struct FetchRecord {
  int world, rank;
  long long shard;                 // elements owned per rank
  long long fw_lo, fw_hi;          // the FC weight [fw_lo, fw_hi): delivered as bf16 only
  long long rec_f32;               // fp32 slots per record (max over ranks of shard entries outside the FC weight)
  long long rec_bytes;             // 2 * shard + 4 * rec_f32, a multiple of 16
  long long img_off, w1_off, w2_off;  // Mnih conv weight image (wimg.cuh), img_off < 0: none
};
void launch_fetch_pack(const float* master, const FetchRecord& f, uint8_t* send, cudaStream_t st);
void launch_fetch_unpack(const uint8_t* recv, const FetchRecord& f, float* theta, __nv_bfloat16* theta_bf16,
                         cudaStream_t st);
void launch_widen_range(const __nv_bfloat16* src, float* dst, long long lo, long long hi, cudaStream_t st);
int server_round_blocks(long long shard, long long conv4, int conv_per_block);

// bf16 tensor-core path, Mnih-2013 net (kernels_bf16.cu)
// dqn_store_and_train on the bf16 Mnih path: Alg. 1's Store as the first kernel of every step of the
// replayed step graph. The graph is fixed, so the chunk of transitions and its position come from here
// (written by store_ctl_kernel before the chunk's graphs): step T stores item T - base of the chunk into
// slot (count0 + T - base) mod capacity and publishes the replay size.
struct StoreCtl {
  const uint8_t* s;                // [m][F][H][W] canonical u8 (device staging or caller device memory)
  const uint8_t* sn;
  const int32_t* a;
  const float* r;
  const uint8_t* t;
  long long base;                  // T of the chunk's first step
  long long count0;                // pushes before the chunk's first item
};
struct StoreArgs {
  uint8_t* ring_s;
  uint8_t* ring_sn;
  int32_t* ring_a;
  float* ring_r;
  uint8_t* ring_t;
  long long cap, stride;
  int dedup;
  const StoreCtl* ctl;
  DevCounters* ctr;
};
struct FwdConvArgs {
  const uint8_t* ring[2];          // s / s' rings (s2d) or a staging buffer (ctr == nullptr: image j = slot j)
  const __nv_bfloat16* theta[2];   // canonical bf16 parameters (theta, theta^)
  const float* theta_f32[2];       // canonical fp32 parameters (biases)
  long long w1_off, b1_off, w2_off, b2_off;
  int* idx;                        // out (group 0) [n]
  const DevCounters* ctr;
  unsigned long long seed;
  unsigned rank;
  int n;
  __nv_bfloat16* a2;               // [groups*n][2592]
  uint8_t* a1_save;                // [n][8][144][16] or nullptr
  FusedAcquire acq;                // NEXT-1: the previous round's deliveries (acq.done == nullptr: none)
  long long img_off;               // conv weight image (wimg.cuh) inside theta[g]
  long long slot_stride;           // bytes between replay slots (28,224, or 35,280 with frame dedup)
  int late;                        // 1: sample + gather after the PDL wait (the predecessor wrote the ring)
  const int* idx_in;               // prioritized replay: the slots prio_sample_kernel drew (nullptr: a1's sampler)
  // store_fused (N = 1 dqn_store_and_train): this step's Alg. 1 Store runs in the extra CTA columns x < 14 after the
  // PDL wait, image j in column j + 14; the draws use the replay size the Store makes (StoreCtl, T), and only a CTA
  // that drew the slot being stored waits (store_flag >= T + 1) before its gather
  int store_fused;
  StoreArgs store;
  unsigned long long* store_flag;
  unsigned* store_join;            // the Store CTAs' join counter (monotone)
};
void launch_store_step(const StoreArgs& a, cudaStream_t st);
void launch_store_ctl(StoreCtl* ctl, const uint8_t* s, const uint8_t* sn, const int32_t* a, const float* r,
                      const uint8_t* t, long long base, long long count0, cudaStream_t st);
struct TcGemmArgs {
  const __nv_bfloat16* A[2];
  long long lda;  // A(m,k) = a_mn ? A[k*lda + m] : A[m*lda + k]
  const __nv_bfloat16* B[2];
  long long ldb;  // B(n,k) = b_mn ? B[k*ldb + n] : B[n*ldb + k]
  int a_mn, b_mn;
  int pre_a;      // 1: A is not the immediate predecessor's output (staged before the PDL wait)
  int pre_b;      // same for B
  int M, N, K;
  int BN;         // n-tile (multiple of 16, <= 256)
  int kper;       // K per split (multiple of 16)
  int splits;
  int epi;        // TC_EPI_*
  float* C[2];    // TC_EPI_ACCUM: C[g][m*ldc + n] += D
  long long ldc;
  float* partial;           // TC_EPI_FC_FWD: partial[g][split][m][n]
  unsigned* counters;       // [groups * m_tiles], self-resetting
  const float* bias[2];
  float* h_out[2];          // [N][M] = relu(sum + bias[m])
  __nv_bfloat16* out_bf16;  // TC_EPI_MASK_T: out[n*ldo + m] = mask[n*ldo + m] > 0 ? D : 0
  const __nv_bfloat16* mask;
  long long ldo;
  int st_id;                // DQN_TRACE_STEP slot (step_trace.cuh), 0 = none
  int st_ph;                // DQN_TRACE_STEP phase slot of tile 0 (staged / MMA done), 0 = none
  int store;                // TC_EPI_ACCUM: 1 = C = D (C known to be zero / overwritten), 0 = C += D
  int hwc_HW, hwc_C;        // TC_EPI_MASK_T: write feature m = c*HW + p to p*C + c (NHWC dZ), 0: off
  FusedAcquire acq;         // conv-first delivery (acq.conv_first): the FC forward acquires the round
  int bulk_accum;           // TC_EPI_ACCUM: rows go out as bulk (reduce-)copies from shared memory
};
enum { TC_EPI_ACCUM = 0, TC_EPI_FC_FWD = 1, TC_EPI_MASK_T = 2 };
struct BwdConvArgs {
  const uint8_t* ring_s;
  long long slot_stride;
  const int* idx;
  const uint8_t* a1_save;
  const __nv_bfloat16* dz2;        // [n][2592]
  const __nv_bfloat16* theta;      // bf16 canonical
  long long w1_off, b1_off, w2_off, b2_off;
  int n;
  float* partial;                  // [n][kBwdPart]
  unsigned* counter;
  float* grad;
};
// ---- generic bf16 conv path (kernels_conv.cu): every conv as a stride-1 conv over a s2d grid
struct GConvFwdArgs {
  const __nv_bfloat16* x[2];       // input grid [b][Hs][Ws][Cs] per group (layers >= 2)
  const uint8_t* ring[2];          // layer 1: replay rings (s2d u8 slots) or a staging buffer
  int* idx;                        // layer 1, group 0: sampled slots out (nullptr: not recorded)
  const DevCounters* ctr;          // layer 1: sampler state (nullptr: image j = slot j)
  unsigned long long seed;
  unsigned rank;
  const int* idx_in;               // layer 1, prioritized replay: the drawn slots (nullptr: a1's sampler)
  int first;                       // 1: layer 1 (u8 input, 1/255 folded into the epilogue)
  long long slot_stride;           // layer 1: bytes between replay slots (frame-major s2d)
  int b, Hs, Ws, Cs, Th, Tw, Ho, Wo, N;
  int s_next;                      // stride of the next conv (its s2d factor), 0: canonical flatten out
  const __nv_bfloat16* wpk[2];     // packed forward weights [N][Th*Tw*Cs] per group
  const float* bias[2];            // fp32 canonical biases per group
  __nv_bfloat16* out[2];
};
void launch_gconv_fwd(const GConvFwdArgs& a, int groups, cudaStream_t st);
struct GConvDgradArgs {
  const __nv_bfloat16* dz;         // layer output gradient [b][Ho][Wo][N]
  const __nv_bfloat16* wpkT;       // packed data-gradient weights [Cs][Th*Tw*N]
  const __nv_bfloat16* xmask;      // the layer input activation [b][Hs][Ws][Cs] (post-ReLU)
  __nv_bfloat16* dzprev;           // previous layer's output gradient [b][Hs*s][Ws*s][Cs/s^2]
  int b, Hs, Ws, Cs, Th, Tw, Ho, Wo, N, s;
};
void launch_gconv_dgrad(const GConvDgradArgs& a, cudaStream_t st);
struct GConvWgradArgs {
  const __nv_bfloat16* x;          // layer input grid (group 0), layers >= 2
  const uint8_t* ring;             // layer 1: the s ring and the sampled slots
  const int* idx;
  int first;
  long long slot_stride;
  const __nv_bfloat16* dz;         // [b][Ho][Wo][N]
  int b, Hs, Ws, Cs, Th, Tw, Ho, Wo, N, ipc;  // ipc: images per CTA (K range)
  float* partial;                  // [ranges][Th*Tw*Cs][N], or [ranges][N][Th*Tw*Cs] with part_cm
  float* partial_db;               // [ranges][N]
  int part_cm;                     // 1: partials column-major per range (twgrad_kernel's coalesced epilogue)
  const int* w_canon;              // per dW row (tap, c'): canonical offset at n = 0 (-1: none)
  long long w_off, w_nstride, b_off;
  float* grad;
  int store;                       // 1: G = sum (n_push = 1), 0: G += sum
};
void launch_gconv_wgrad(const GConvWgradArgs& a, cudaStream_t st);
bool gconv_wgrad_fits(int N, int first, int ipc, int HoWo);  // shared memory of a wgrad CTA within the attribute
void launch_gpack(const float* theta, __nv_bfloat16* dst, long long img_off, const int2* map, long long n,
                  cudaStream_t st);
void init_conv_kernel_attrs();
unsigned long long gconv_error();
// warp-specialised persistent TMA GEMM (kernels_tma.cu): the large-batch FC layers. Operand maps are 2-D
// bf16 tensors read in 64-column boxes with the 128-byte swizzle (make_tmap_bf16): a K-major operand's box is
// [128 or BN rows][64 k], an MN-major one's [64 k][64 mn]. Epilogues as TcGemmArgs (TC_EPI_*).
constexpr int kTgMaxStages = 8;
struct TGemmArgs {
  CUtensorMap ta[2], tb[2];        // per group
  int M, N, K;
  int kper, splits;                // K per split (a multiple of 64 when splits > 1), split count
  int BN;                          // n-tile: multiple of 16 (K-major B) or of 64 (MN-major B), <= 256
  int a_mn, b_mn, groups, stages;
  int epi, store;
  float* C[2];
  long long ldc;
  float* partial;
  __nv_bfloat16* out_bf16;
  const __nv_bfloat16* mask;
  long long ldo;
  int hwc_HW, hwc_C;
  int hwc_Wo, hwc_Ws;              // hwc_Ws > 0: the NHWC dZ in the input-grid geometry (row y * Ws + x, not
  long long ldo_out;               //   y * Wo + x), per-sample stride ldo_out (TCONV backward)
};
// tgemm only: C[g][n * ldc + m] = D (store) or += D, the transposed ACCUM (lanes = consecutive m: coalesced)
constexpr int TC_EPI_ACCUM_T = 4;
// ---- TMA implicit-GEMM convolutions with tap windows (kernels_tma.cu). The A source is a 2-D bf16 tensor of
// "virtual rows" (row = img * Hs*Ws + y * Ws + x of a layer's input grid, 64-channel blocks); ONE TMA box of
// R = 128 (or 64) + maxshift rows per channel block feeds every tap: tap t is the same window read from row
// shift(t) = (t / Tw) * Ws + t % Tw on (128-byte-swizzled descriptors stay valid under whole-row shifts).
//   TCONV_FWD   : D[row][n] = sum_t sum_c X[row + shift(t)][c] W_t[n][c]; B = packed forward weights, resident
//   TCONV_DGRAD : D[row][c] = sum_t sum_n dZ[row - shift(t)][n] W_t[n][c] (dZ in the layer's input-grid geometry,
//                 zero outside the Ho x Wo outputs); B = packed data-gradient weights, resident; epilogue
//                 x [X > 0] (ReLU') and inverse space-to-depth into the previous layer's dZ (same geometry)
//   TCONV_WGRAD : D[(t, c)][n] = sum_rows X[row + shift(t)][c] dZ[row][n] over a K range of rows (MN-major
//                 operands, two 64-row (t, c-block) halves per M tile, plus one all-ones half giving db);
//                 per-range partials, reduced in range order by gconv_wreduce (deterministic)
enum { TCONV_FWD = 0, TCONV_DGRAD = 1, TCONV_WGRAD = 2 };
// n / d for a divisor fixed at launch (the epilogues' row -> (image, y, x) decompositions): one multiply-high,
// an add and a shift instead of a ~20-instruction integer division (Granlund-Montgomery; exact for all 32-bit n)
struct FastDiv {
  uint32_t d, m, s;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0u, 0u};
  if (d <= 1) return f;
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  f.m = (uint32_t)((((1ull << 32) * ((1ull << l) - d)) / d) + 1);
  f.s = l - 1;
  return f;
}
#ifdef __CUDACC__
__device__ __forceinline__ uint32_t fdiv(const FastDiv& f, uint32_t n) {
  if (f.d <= 1) return n;
  const uint32_t t = __umulhi(n, f.m);
  return (t + ((n - t) >> 1)) >> f.s;
}
#endif
struct TConvArgs {
  CUtensorMap ta[2];               // the A source rows per group: box {64, R}
  CUtensorMap tb[2];               // FWD / DGRAD: packed weights [BN][T*64*Cblk] (box {64, BN}); WGRAD: dZ rows (box {64, 64})
  int mode, groups;
  int M;                           // FWD / DGRAD: rows (b * Hs*Ws); WGRAD: T * Cs (+ the ones rows)
  int BN;                          // MMA N: FWD N, DGRAD Cs, WGRAD 64
  int T, Tw, Ws, HsWs, Cblk;       // taps, tap width, grid width, grid pixels, 64-channel blocks of A
  int R, maxshift;                 // window rows, largest tap shift
  int stages;
  // FWD epilogue
  int Ho, Wo, N, s_next;
  float scale;
  const float* bias[2];
  __nv_bfloat16* cout[2];
  // DGRAD epilogue
  const __nv_bfloat16* xmask;      // layer input activation [rows][Cs] (post-ReLU: the mask of ReLU')
  __nv_bfloat16* dzprev;           // previous layer's dZ, input-grid geometry [b * prevHsWs][Cp]
  int s, Cp, prevWs, prevHsWs, Cs;
  // WGRAD: K rows = b * Hs*Ws split into ranges of kpr chunks of 64 rows
  long long krows;
  int kpr, ranges, TCs, Nout;
  float* partial;                  // [ranges][TCs][Nout]
  float* partial_db;               // [ranges][Nout]
  int dbg;                         // probe only (tools/probe_tconv): 1 skip epilogue stores, 2 skip MMAs
  FastDiv fd_hsws, fd_ws, fd_sn, fd_cp, fd_s;  // set by launch_tconv from HsWs, Ws, s_next, Cp, s
};
bool init_tconv_kernel_attrs();
size_t tconv_smem(const TConvArgs& a);  // 0: does not fit
void launch_tconv(const TConvArgs& a, int num_sms, cudaStream_t st);
void launch_gconv_wreduce(const GConvWgradArgs& a, cudaStream_t st);
// layer 1 of the generic path: sample (a1) and gather + convert (a2) every s / s' slot of the step into the
// bf16 s2d grid [b][21][21][64] per group, which the TMA convolution reads
void launch_prio_sample(const PrioTree& t, int b, unsigned long long seed, unsigned rank, const DevCounters* ctr,
                        int* idx, cudaStream_t st);
void launch_prio_update(const PrioTree& t, int b, const int* idx, const float* delta, int alpha_half, float eps,
                        float* maxp, cudaStream_t st);
void launch_prio_push(const PrioTree& t, long long cap, long long first, long long m, const float* maxp,
                      cudaStream_t st);
void launch_gather_s2d(const GConvFwdArgs& a, __nv_bfloat16* x1_0, __nv_bfloat16* x1_1, int groups, cudaStream_t st);
// canonical (C,H,W)-flattened images [b][C*Ho*Wo] -> input-grid geometry [b][Hs*Ws][C] (borders untouched)
bool chw_to_hwc_fits(int C, int Ho, int Wo);
void launch_chw_to_hwc(const __nv_bfloat16* src, __nv_bfloat16* dst, int b, int C, int Ho, int Wo, int Ws, int HsWs,
                       cudaStream_t st);
bool make_tmap_bf16(CUtensorMap* m, const void* base, long long rows, long long cols, long long ld, int box_rows);
void launch_tgemm(const TGemmArgs& a, int num_sms, cudaStream_t st);
bool init_tma_kernel_attrs();  // false: the kernel cannot get its shared memory (the older GEMMs are used)
// pipelined tcgen05 GEMM (generic path FC layers): K split into chunks of 64 (kper % 64 == 0)
void launch_gemm_pipe(const TcGemmArgs& a, int groups, cudaStream_t st);
void launch_fc_reduce(const TcGemmArgs& a, int groups, cudaStream_t st);
void launch_head_finish_warp(const HeadArgs& h, cudaStream_t st);

// ---- NEXT-3 on-GPU acting (kernels_env.cu): Snake games, eps-greedy, Store
struct EnvGame {
  int32_t len, dir, apple, since;  // body length, direction (0 up 1 right 2 down 3 left), apple cell, steps since apple
  int16_t body[1024];              // cells y*n + x, head first
};
struct EnvArgs {
  EnvGame* games;
  uint8_t* stacks;                 // [E][F][H][H] current phi of every game
  uint8_t *s_stage, *sn_stage;     // [E][F][H][H] the step's transition (push input)
  int32_t* a_stage;
  float* r_stage;
  uint8_t* t_stage;
  const int* greedy;               // [E] argmax Q of the current stacks
  int n, F, H, E;
  unsigned long long seed, t, eps_thr;
  int32_t* a_log;                  // optional [steps][E] logs (row log_row)
  float* r_log;
  uint8_t* t_log;
  long long log_row;
  long long* episodes;             // [E] finished episodes
  double* reward_sum;              // [E] accumulated reward
};
void launch_env_init(const EnvArgs& a, cudaStream_t st);
void launch_env_act(const EnvArgs& a, cudaStream_t st);

struct ReduceUpdateArgs {
  BwdConvArgs b;                   // the conv partials and offsets
  float* theta;                    // fp32 theta (= theta_local at N = 1)
  float* r;
  float* g;                        // G (non-conv part; cleared after reading)
  long long n;                     // P_pad
  float inv_div, lr, rho, omr, eps;
  __nv_bfloat16* pub_bf16;         // theta_local_bf16 (+ the conv weight image at img_off)
  long long img_off;
  DevCounters* ctr;
  int early;                       // 1: the non-conv part [kBwdPart, n) is updated by the conv backward's
                                   //    extra CTAs (launch_bwd_conv_update); this launch does the conv part only
  float* g_snap;                   // cfg.keep_grad: every consumed gradient element also stored here (or nullptr)
};
void launch_reduce_update(const ReduceUpdateArgs& u, cudaStream_t st);
// N = 1, n_push = 1: the conv backward launch plus `upd_ctas` CTAs that apply the RMSProp update to the
// non-conv parameters [kBwdPart, u.n) (FC, output layer: their gradients are complete when the conv
// backward passes its PDL wait), off the step's critical path; u.early must be 1.
void launch_bwd_conv_update(const BwdConvArgs& a, const ReduceUpdateArgs& u, int upd_ctas, cudaStream_t st);
constexpr int kMnihSlot = 28224;
constexpr int kA1Bytes = 8 * 144 * 16;
constexpr int kBwdPart = 256 * 16 + 256 * 32 + 16 + 32;
void init_bf16_kernel_attrs();
void init_head_kernel_attrs();
// DQN_TRACE_STEP accessors, one per translation unit (step_trace.cuh)
void step_trace_bf16(int on, unsigned long long* out);
void step_trace_head(int on, unsigned long long* out);
void step_trace_common(int on, unsigned long long* out);
void step_trace_comm(int on, unsigned long long* out);
void launch_push_s2d(uint8_t* ring_s, uint8_t* ring_sn, int32_t* ring_a, float* ring_r, uint8_t* ring_t, long long cap,
                     long long count0, long long first, long long n, const uint8_t* s, const int32_t* a,
                     const float* r, const uint8_t* sn, const uint8_t* t, cudaStream_t st,
                     long long* ring_size_out = nullptr, long long ring_size = 0, long long stride = 28224,
                     int dedup = 0);
void launch_fwd_conv_bf16(const FwdConvArgs& a, int groups, cudaStream_t st);
void launch_tc_gemm(const TcGemmArgs& a, int groups, cudaStream_t st);
// one launch: the tiles of GEMM p0, the tiles of GEMM p1 (single split, group 0 each), then the
// cross-sample TD-head finish (head_finish.cuh) — the bf16 path's whole FC backward
void launch_tc_pair_with_head(const TcGemmArgs& p0, const TcGemmArgs& p1, const HeadArgs& head, cudaStream_t st);
// the whole K of both GEMMs fits tc_pair's shared-memory staging (else: gemm_pipe x 2 + head_finish_warp)
bool tc_pair_fits(const TcGemmArgs& p0, const TcGemmArgs& p1);
void launch_bwd_conv_bf16(const BwdConvArgs& a, cudaStream_t st, bool with_reduce = true);

}  // namespace dqn
