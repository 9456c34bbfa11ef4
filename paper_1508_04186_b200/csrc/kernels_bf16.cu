// kernels_bf16.cu — the tensor-core replica step (precision DQN_BF16) for the
// Mnih-2013 network of BASELINE.json configs[0..3] (conv16 8x8/4, conv32 4x4/2,
// fc256, |A| outputs). bf16 operands, fp32 accumulation in TMEM (tcgen05).
//
// Both strided convolutions are rewritten by space-to-depth (s2d) as 2x2
// stride-1 convolutions (conv1: 84x84x4 -> 21x21x64, conv2: 20x20x16 ->
// 10x10x64), so every filter tap is a ROW SHIFT of one shared-memory image:
// with the image stored as UMMA no-swizzle K-major chunk planes
// [channel/8][pixel][8 x bf16], the A operand of tap (dy,dx) is the same planes
// started dy*W+dx pixels later ("virtual rows" m' = oy*W + ox; the column
// ox = W-1 is computed and discarded). The replay ring holds conv1's s2d layout
// directly (pushed once, gathered every step) and conv1's epilogue writes its
// activation straight into conv2's s2d layout, so the whole forward of one
// state (sample -> gather -> conv1 -> conv2) is one CTA with no HBM round trip.
//
// Formulas: P:61-67 (network), P:121 (target network on s'), P:123 (gradient).
#include <algorithm>
#include <cstdio>
#include "dqn_internal.h"
#include "fused_acquire.cuh"
#include "head_finish.cuh"
#include "pdl.cuh"
#include "step_trace.cuh"
#include "wimg.cuh"
#include "philox.cuh"
#include "sm100.cuh"

namespace dqn {
using namespace dqn_sm100;

namespace mnih {
// conv1: 4x84x84 -> s2d(4) 21x21x64 -> 2x2/1 -> 20x20x16
constexpr int X_W = 21, X_PIX = 441, X_ALLOC = 544, C1 = 16, M1V = 420, M1_TILES = 4;
// conv2: 16x20x20 -> s2d(2) 10x10x64 -> 2x2/1 -> 9x9x32
constexpr int A1_W = 10, A1_PIX = 100, A1_ALLOC = 144, C2 = 32, M2V = 90;  // K = 4 taps x 64 ch = 256 for both
constexpr int D = 2592;     // 32 x 9 x 9 flattened (C,H,W)
constexpr int SLOT = 28224; // bytes of one u8 s2d state
__device__ __forceinline__ int tap_shift1(int t) { return (t >> 1) * X_W + (t & 1); }
__device__ __forceinline__ int tap_shift2(int t) { return (t >> 1) * A1_W + (t & 1); }
}  // namespace mnih

static inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// ------------------------------------------------------------------ push: canonical -> s2d ring slots
// Frame-major s2d slots: out[f][p][16] with p = py*21 + px, byte iy*4 + ix  <-  in[f][4py+iy][4px+ix]
// (channel c' = f*16 + iy*4 + ix of conv1's s2d grid), slot stride `stride` bytes. With `dedup` the
// s' ring aliases the s ring one frame later (5 frames per slot: s = frames 0-3, s' = 1-4) and only
// the new frame of s' is written. One thread writes one 16-byte vector (frame f, pixel p).
__global__ void push_s2d_kernel(uint8_t* ring_s, uint8_t* ring_sn, int32_t* ring_a, float* ring_r, uint8_t* ring_t,
                                long long cap, long long count0, long long first, const uint8_t* s,
                                const int32_t* a, const float* r, const uint8_t* sn, const uint8_t* t,
                                long long* ring_size_out, long long ring_size, long long stride, int dedup) {
  const long long i = blockIdx.y;
  if (ring_size_out && i == 0 && blockIdx.x == 0 && threadIdx.x == 0) *ring_size_out = ring_size;
  const long long slot = (count0 + first + i) % cap;
  const int v = blockIdx.x * blockDim.x + threadIdx.x;  // (frame, pixel)
  if (v < mnih::X_PIX * 4) {
    const int f = v / mnih::X_PIX, p = v % mnih::X_PIX;
    const int py = p / 21, px = p % 21;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      if (which == 1 && (ring_sn == nullptr || (dedup && f != 3))) break;  // q staging: states only
      const uint8_t* src = (which ? sn : s) + i * mnih::SLOT + f * 7056 + (4 * py) * 84 + 4 * px;
      uint4 o;
      o.x = *reinterpret_cast<const uint32_t*>(src);
      o.y = *reinterpret_cast<const uint32_t*>(src + 84);
      o.z = *reinterpret_cast<const uint32_t*>(src + 168);
      o.w = *reinterpret_cast<const uint32_t*>(src + 252);
      uint8_t* dst = (which ? ring_sn : ring_s) + slot * stride + f * 7056 + p * 16;
      *reinterpret_cast<uint4*>(dst) = o;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && ring_a != nullptr) {
    ring_a[slot] = a[i];
    ring_r[slot] = r[i];
    ring_t[slot] = t[i] ? 1 : 0;
  }
}

// Alg. 1 "Store" inside the step graph (dqn_store_and_train): step T writes item T - base of the chunk
// (StoreCtl) into its ring slot exactly as push_s2d_kernel does, after the previous step's kernels (which
// read the ring) completed; the conv forward that follows samples and gathers after its own PDL wait.
// one (frame, pixel) 16-byte piece v of item i of the chunk into ring slot `slot` (s and, unless deduplicated, s')
__device__ __forceinline__ void store_piece(const StoreArgs& a, const StoreCtl& c, long long i, long long slot, int v) {
  {
    const int f = v / mnih::X_PIX, p = v % mnih::X_PIX;
    const int py = p / 21, px = p % 21;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      if (which == 1 && a.dedup && f != 3) break;  // frame dedup: only the new frame of s'
      const uint8_t* src = (which ? c.sn : c.s) + i * mnih::SLOT + f * 7056 + (4 * py) * 84 + 4 * px;
      uint4 o;
      o.x = *reinterpret_cast<const uint32_t*>(src);
      o.y = *reinterpret_cast<const uint32_t*>(src + 84);
      o.z = *reinterpret_cast<const uint32_t*>(src + 168);
      o.w = *reinterpret_cast<const uint32_t*>(src + 252);
      *reinterpret_cast<uint4*>((which ? a.ring_sn : a.ring_s) + slot * a.stride + f * 7056 + p * 16) = o;
    }
  }
}

// the item's action, reward, terminal flag and the new replay size (one thread)
__device__ __forceinline__ void store_scalars(const StoreArgs& a, const StoreCtl& c, long long i, long long slot) {
  a.ring_a[slot] = c.a[i];
  a.ring_r[slot] = c.r[i];
  a.ring_t[slot] = c.t[i] ? 1 : 0;
  a.ctr->ring_size = c.count0 + i + 1 < a.cap ? c.count0 + i + 1 : a.cap;
}

__global__ void store_step_kernel(StoreArgs a) {
  pdl_wait();
  // the successor may launch now: the previous step is complete, and the forward reads this kernel's writes only
  // after its own griddepcontrol.wait
  pdl_trigger();
  const StoreCtl c = *a.ctl;
  const long long i = (long long)a.ctr->T - c.base;
  const long long slot = (c.count0 + i) % a.cap;
  const int v = blockIdx.x * blockDim.x + threadIdx.x;  // (frame, pixel)
  if (v < mnih::X_PIX * 4) store_piece(a, c, i, slot, v);
  if (blockIdx.x == 0 && threadIdx.x == 0) store_scalars(a, c, i, slot);
}

// the same Store in the forward's extra CTAs (store_fused): after the PDL wait (the previous step, whose kernels
// read the ring, is complete), then a gpu-scope release of T + 1 for the CTAs that drew this slot
constexpr int kStoreCtas = (mnih::X_PIX * 4 + 127) / 128;  // one 16-byte piece per thread of 128-thread CTAs

__device__ __forceinline__ void store_in_forward(const FwdConvArgs& fa) {
  const StoreArgs& a = fa.store;
  pdl_wait();
  const StoreCtl c = *a.ctl;
  const unsigned long long T = a.ctr->T;
  const long long i = (long long)T - c.base;
  const long long slot = (c.count0 + i) % a.cap;
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < mnih::X_PIX * 4) store_piece(a, c, i, slot, v);
  if (v == 0) store_scalars(a, c, i, slot);
  __syncthreads();
  if (threadIdx.x == 0) {  // the last of the kStoreCtas CTAs to join releases T + 1
    __threadfence();
    const unsigned old = atomicAdd(fa.store_join, 1u);
    if ((old + 1) % kStoreCtas == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(fa.store_flag), "l"(T + 1) : "memory");
    }
  }
}

void launch_store_step(const StoreArgs& a, cudaStream_t st) {
  launch_pdl(store_step_kernel, dim3(cdiv(mnih::X_PIX * 4, 256)), dim3(256), 0, st, a);
}

__global__ void store_ctl_kernel(StoreCtl* ctl, StoreCtl v) { *ctl = v; }

void launch_store_ctl(StoreCtl* ctl, const uint8_t* s, const uint8_t* sn, const int32_t* a, const float* r,
                      const uint8_t* t, long long base, long long count0, cudaStream_t st) {
  store_ctl_kernel<<<1, 1, 0, st>>>(ctl, StoreCtl{s, sn, a, r, t, base, count0});
}

void launch_push_s2d(uint8_t* ring_s, uint8_t* ring_sn, int32_t* ring_a, float* ring_r, uint8_t* ring_t, long long cap,
                     long long count0, long long first, long long n, const uint8_t* s, const int32_t* a,
                     const float* r, const uint8_t* sn, const uint8_t* t, cudaStream_t st, long long* ring_size_out,
                     long long ring_size, long long stride, int dedup) {
  if (n <= 0) return;
  dim3 grid(cdiv(mnih::X_PIX * 4, 256), (unsigned)n);
  push_s2d_kernel<<<grid, 256, 0, st>>>(ring_s, ring_sn, ring_a, ring_r, ring_t, cap, count0, first, s, a, r, sn, t,
                                        ring_size_out, ring_size, stride, dedup);
}

// ------------------------------------------------------------------ shared helpers
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}
// 16 u8 -> 16 exact bf16 (integers < 256 are exact in bf16), as two 16-byte chunks
__device__ __forceinline__ void u8x16_to_bf16(const uint4 q, uint4& lo, uint4& hi) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
  uint32_t o[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float b0 = (float)(w[i] & 0xFF), b1 = (float)((w[i] >> 8) & 0xFF);
    const float b2 = (float)((w[i] >> 16) & 0xFF), b3 = (float)(w[i] >> 24);
    o[2 * i] = pack_bf16(b0, b1);
    o[2 * i + 1] = pack_bf16(b2, b3);
  }
  lo = make_uint4(o[0], o[1], o[2], o[3]);
  hi = make_uint4(o[4], o[5], o[6], o[7]);
}

// Expand one u8 s2d state (already in shared memory, 28224 B) into bf16 chunk planes
// [8][X_ALLOC][16 B] (pixels >= 441 left untouched).
__device__ __forceinline__ void expand_state(uint8_t* sX, const uint8_t* sU8) {
  const uint4* s4 = reinterpret_cast<const uint4*>(sU8);
  for (int v = threadIdx.x; v < mnih::X_PIX * 4; v += blockDim.x) {
    const int q = v / mnih::X_PIX, p = v % mnih::X_PIX;  // frame-major slot: frame q, pixel p
    uint4 lo, hi;
    u8x16_to_bf16(s4[v], lo, hi);
    *reinterpret_cast<uint4*>(sX + ((2 * q) * mnih::X_ALLOC + p) * 16) = lo;
    *reinterpret_cast<uint4*>(sX + ((2 * q + 1) * mnih::X_ALLOC + p) * 16) = hi;
  }
}

// ------------------------------------------------------------------ a1-a4: sample + gather + conv1 + conv2
// grid (n_images, groups): group 0 = s_j with theta (local), group 1 = s'_j with theta^.
// Writes a2[g*n + j][2592] (bf16, canonical (C,H,W) flatten, post-ReLU) and, for group 0,
// a1_save[j] (conv1 activation as conv2's s2d chunk planes, the backward's operand).
constexpr int FWD_SX = 0;
constexpr int FWD_SA1 = FWD_SX + 8 * mnih::X_ALLOC * 16;       // 69632
constexpr int FWD_SW1 = FWD_SA1 + 8 * mnih::A1_ALLOC * 16;     // +18432
constexpr int FWD_SW2 = FWD_SW1 + 32 * mnih::C1 * 16;          // +8192
constexpr int FWD_SMEM = FWD_SW2 + 32 * mnih::C2 * 16;         // +16384 = 112640: two CTAs per SM
// the gathered u8 slot lands over sA1 | sW1 | sW2, which are written only after it was expanded into sX
constexpr int FWD_SU8 = FWD_SA1;
static_assert(FWD_SU8 + mnih::SLOT <= FWD_SMEM, "u8 staging inside the kernel's shared memory");

__global__ void __launch_bounds__(128) fwd_conv_bf16_kernel(FwdConvArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2, bar_ld;
  __shared__ uint32_t tbase;
  if (a.store_fused && blockIdx.x < kStoreCtas) {  // Alg. 1's Store of this step (group 0's extra CTAs)
    if (blockIdx.y == 0) store_in_forward(a);
    return;
  }
  const int j = blockIdx.x - (a.store_fused ? kStoreCtas : 0), g = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  st_stamp(ST_FWD, 0);
  uint8_t* sX = smem + FWD_SX;
  uint8_t* sA1 = smem + FWD_SA1;
  uint8_t* sW1 = smem + FWD_SW1;
  uint8_t* sW2 = smem + FWD_SW2;
  uint8_t* sU8 = smem + FWD_SU8;
  if (a.late) pdl_wait();  // the immediate predecessor (the in-graph Store) wrote the ring and its size
  unsigned long long* tr = nullptr;  // DQN_TRACE_COMM stamps (slots 8-10 of the previous round)
  if (a.acq.trace && j == 0 && g == 0 && threadIdx.x == 0 && a.acq.ctr->T % a.acq.n_push == 0) {
    tr = a.acq.trace + ((a.acq.ctr->T / a.acq.n_push) % 64) * 16;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tr[8]));
  }
  if (threadIdx.x == 0) {
    long long slot = j, size = 0;
    if (a.idx_in) {
      slot = a.idx_in[j];  // prioritized replay (A41): drawn by the predecessor (a.late = 1)
    } else if (a.store_fused) {
      // this step's Store (CTA column 0) puts item T - base into slot (count0 + T - base) mod cap and makes the
      // replay size min(cap, count0 + T - base + 1): the draw needs neither the Store's writes nor its size store
      const unsigned long long T = a.ctr->T;
      const StoreCtl* c = a.store.ctl;
      const long long i = (long long)T - c->base, n_new = c->count0 + i + 1;
      size = n_new < a.store.cap ? n_new : a.store.cap;
      slot = sample_slot(a.seed, a.rank, T, (unsigned)j, size);  // a1
      if (slot == (c->count0 + i) % a.store.cap) {  // drew the slot being stored: wait for the Store's release
        long long spin = 0;
        for (;;) {
          unsigned long long v;
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a.store_flag) : "memory");
          if (v >= T + 1) break;
          __nanosleep(32);
          if (++spin > (1LL << 26)) { atomicOr(&a.store.ctr->bad_input, 0x40000000u); break; }
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy stores before the TMA read
      }
    } else if (a.ctr) {
      slot = sample_slot(a.seed, a.rank, a.ctr->T, (unsigned)j, a.ctr->ring_size);  // a1
    }
    if (g == 0 && a.idx && !a.idx_in) a.idx[j] = (int)slot;
    mbar_init(&bar, 4);   // conv1: one commit per issuing warp
    mbar_init(&bar2, 4);  // conv2: likewise
    mbar_init(&bar_ld, 1);
    fence_mbar_init();
    // a2 gather: the whole u8 state in one TMA bulk copy (28,224 contiguous bytes of the ring slot)
    mbar_arrive_expect_tx(&bar_ld, mnih::SLOT);
    bulk_g2s(sU8, a.ring[g] + slot * a.slot_stride, mnih::SLOT, &bar_ld);
    // the sampler is counter-based: step T+1's slot is known now. Prefetch it into L2 so that the
    // next step's gather is an L2 hit with a warm TLB (a random 28 KB slot of a 56 GB ring
    // otherwise costs a page walk); harmless if a push changes the ring size before T+1.
    if (a.ctr && !a.idx_in) {
      const long long nxt = sample_slot(a.seed, a.rank, a.ctr->T + 1, (unsigned)j, a.store_fused ? size : a.ctr->ring_size);
      bulk_prefetch_l2(a.ring[g] + nxt * a.slot_stride, mnih::SLOT);
    }
  }
  if (warp == 0) tmem_alloc(&tbase, 128);
  __syncthreads();  // barriers initialised before anyone waits on them
  mbar_wait(&bar_ld, 0);
  if (tr) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tr[9]));
  expand_state(sX, sU8);  // u8 -> exact bf16 (1/255 folded into the epilogue)
  __syncthreads();        // every thread has read the u8 slot before the weights land over it
  // everything above overlaps the previous kernel (the update that publishes theta); weights after the wait
  if (fused_round_acquire_conv(a.acq)) {
    // conv-first delivery: the previous step's server round released the conv parameters early; no
    // griddepcontrol.wait on the round's grid (its FC deliveries are acquired by the FC forward)
    st_stamp(ST_FWD, 1);
    if (tr) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tr[10]));
  } else {
    pdl_wait();
    st_stamp(ST_FWD, 1);
    if (tr) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tr[10]));
    fused_round_acquire(a.acq);  // N > 1 fused server round: peers' deliveries into theta_local complete
  }
  pdl_trigger();               // only now: the FC forward reads the delivered weights before its wait
  // conv1 + conv2 B operands: the weight image the update wrote after the canonical entries
  // (wimg.cuh), contiguous with sW1 | sW2 in shared memory: 1,536 16-byte async copies
  static_assert(FWD_SW2 == FWD_SW1 + kW1Elems * 2 && kWimgElems * 2 == 1536 * 16, "weight image layout");
  {
    const uint4* img = reinterpret_cast<const uint4*>(a.theta[g] + a.img_off);
#pragma unroll
    for (int it = 0; it < 1536 / 128; ++it) cp_async16(sW1 + (threadIdx.x + it * 128) * 16, img + threadIdx.x + it * 128);
    cp_async_wait_all();
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  st_stamp(ST_P1, 0);
  const uint32_t tmem = tbase;
  // ---- conv1: 4 M-tiles x 4 taps x 4 K-steps, M = 128, N = 16; warp w issues M-tile w (warp-uniform issue:
  // 16 MMAs per warp instead of 64 from one thread)
  static_assert(mnih::M1_TILES == 4, "one conv1 M-tile per warp");
  {
    const int mt = warp;
    const uint32_t idesc = make_idesc_bf16(128, mnih::C1, 0, 0);
    const uint32_t xb = smem_u32(sX), wb = smem_u32(sW1);
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = make_desc(xb + (2 * kk) * mnih::X_ALLOC * 16 + (mt * 128 + mnih::tap_shift1(t)) * 16,
                                      mnih::X_ALLOC * 16, 128);
        const uint64_t bd = make_desc(wb + (t * 8 + 2 * kk) * mnih::C1 * 16, mnih::C1 * 16, 128);
        mma_bf16_w(tmem + mt * mnih::C1, ad, bd, idesc, (t | kk) != 0);
      }
    mma_commit_w(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  st_stamp(ST_P1, 1);
  // ---- conv1 epilogue: x (1/255) + b1, ReLU, bf16, into conv2's s2d planes
  {
    const float* b1 = a.theta_f32[g] + a.b1_off;
    float bias[mnih::C1];
#pragma unroll
    for (int n = 0; n < mnih::C1; ++n) bias[n] = __ldg(b1 + n);
    for (int mt = 0; mt < mnih::M1_TILES; ++mt) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + mt * mnih::C1, v);
      const int m = mt * 128 + 32 * warp + lane;
      const int oy = m / mnih::X_W, ox = m % mnih::X_W;
      if (m < mnih::M1V && ox < 20) {
        uint32_t o[8];
#pragma unroll
        for (int n = 0; n < 16; n += 2) {
          const float z0 = fmaxf(fmaf(v[n], 1.0f / 255.0f, bias[n]), 0.0f);
          const float z1 = fmaxf(fmaf(v[n + 1], 1.0f / 255.0f, bias[n + 1]), 0.0f);
          o[n >> 1] = pack_bf16(z0, z1);
        }
        const int p2 = (oy >> 1) * mnih::A1_W + (ox >> 1);
        const int j0 = (((oy & 1) << 1) | (ox & 1)) * 2;
        *reinterpret_cast<uint4*>(sA1 + (j0 * mnih::A1_ALLOC + p2) * 16) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(sA1 + ((j0 + 1) * mnih::A1_ALLOC + p2) * 16) = make_uint4(o[4], o[5], o[6], o[7]);
      }
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  st_stamp(ST_P1, 2);
  // ---- conv2: 1 M-tile x 4 taps x 4 K-steps, M = 128, N = 32; warp w issues tap w into its own
  // accumulator (columns 32 w: conv1's, all read above), the epilogue sums the four in tap order
  {
    const int t = warp;
    const uint32_t idesc = make_idesc_bf16(128, mnih::C2, 0, 0);
    const uint32_t ab = smem_u32(sA1), wb = smem_u32(sW2);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t ad = make_desc(ab + (2 * kk) * mnih::A1_ALLOC * 16 + mnih::tap_shift2(t) * 16,
                                    mnih::A1_ALLOC * 16, 128);
      const uint64_t bd = make_desc(wb + (t * 8 + 2 * kk) * mnih::C2 * 16, mnih::C2 * 16, 128);
      mma_bf16_w(tmem + 32 * t, ad, bd, idesc, kk != 0);
    }
    mma_commit_w(&bar2);
  }
  // save conv1's activation (group 0) for the backward while conv2 runs
  if (g == 0 && a.a1_save) {
    const uint4* src = reinterpret_cast<const uint4*>(sA1);
    uint4* dst = reinterpret_cast<uint4*>(a.a1_save + (long long)j * 8 * mnih::A1_ALLOC * 16);
    for (int v = threadIdx.x; v < 8 * mnih::A1_ALLOC; v += blockDim.x) dst[v] = src[v];
  }
  mbar_wait(&bar2, 0);
  st_stamp(ST_P2, 0);
  tc_fence_after();
  // ---- conv2 epilogue: + b2, ReLU, bf16, canonical flatten d = c*81 + oy*9 + ox
  {
    const float* b2 = a.theta_f32[g] + a.b2_off;
    const int m = 32 * warp + lane;
    const int oy = m / mnih::A1_W, ox = m % mnih::A1_W;
    const bool ok = m < mnih::M2V && ox < 9;
    __nv_bfloat16* out = a.a2 + ((long long)g * a.n + j) * mnih::D + oy * 9 + ox;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float v[16], u[16];
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + 16 * h, v);
#pragma unroll
      for (int t = 1; t < 4; ++t) {
        tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + 32 * t + 16 * h, u);
#pragma unroll
        for (int n = 0; n < 16; ++n) v[n] += u[n];
      }
      if (ok) {
#pragma unroll
        for (int n = 0; n < 16; ++n) {
          const int c = 16 * h + n;
          out[c * 81] = __float2bfloat16_rn(fmaxf(v[n] + __ldg(b2 + c), 0.0f));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 128);
  st_stamp(ST_FWD, 2);
}

void launch_fwd_conv_bf16(const FwdConvArgs& a, int groups, cudaStream_t st) {
  dim3 grid(a.n + (a.store_fused ? kStoreCtas : 0), groups);
  launch_pdl(fwd_conv_bf16_kernel, grid, dim3(128), FWD_SMEM, st, a);
}

// ------------------------------------------------------------------ generic small tcgen05 GEMM
// D[m][n] = sum_k A(m,k) B(n,k), bf16 operands from global, fp32 accumulate in TMEM.
// One CTA = one (group, m-tile of 128, n-tile of BN, k-split); the CTA stages its
// whole K slice at once (these GEMMs are latency-bound: M, N <= 2592, K <= 2592).

// the TC_EPI_MASK_T mask tile [BN][128] bf16 is staged in shared memory when it fits the 200 KB budget
__host__ __device__ __forceinline__ bool tc_mask_fits(const TcGemmArgs& a) {
  return (long long)(128 + a.BN) * a.kper * 2 + (long long)a.BN * 256 <= 200 * 1024;
}

// B (BN rows x KC) into [kc][n][8] (K-major) or [n/8][k][8] (MN-major), 16-byte async copies
__device__ __forceinline__ void stage_b_operand(const TcGemmArgs& a, const __nv_bfloat16* Bg, uint8_t* sB, int n0,
                                                int k0, int KC, int kch) {
  const uint4 z4 = make_uint4(0, 0, 0, 0);
  const int bn = a.BN;
  if (!a.b_mn) {
    for (int e = threadIdx.x; e < bn * kch; e += blockDim.x) {
      const int r = e / kch, c = e % kch;
      const int n = n0 + r;
      uint8_t* d = sB + (c * bn + r) * 16;
      if (n < a.N) cp_async16(d, Bg + (long long)n * a.ldb + k0 + 8 * c);
      else *reinterpret_cast<uint4*>(d) = z4;
    }
  } else {
    const int ng = bn / 8;
    for (int e = threadIdx.x; e < ng * KC; e += blockDim.x) {
      const int gi = e % ng, k = e / ng;
      const int n = n0 + 8 * gi;
      uint8_t* d = sB + (gi * KC + k) * 16;
      if (n < a.N) cp_async16(d, Bg + (long long)(k0 + k) * a.ldb + n);
      else *reinterpret_cast<uint4*>(d) = z4;
    }
  }
}

__device__ __forceinline__ void tc_gemm_tile(const TcGemmArgs& a, int tile, int split, int g, uint8_t* smem,
                                             uint64_t& bar, uint32_t& tbase) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles = (a.N + a.BN - 1) / a.BN;
  const int m_tiles = (a.M + 127) / 128;
  const int mt = tile % m_tiles, nt = tile / m_tiles;
  const int m0 = mt * 128, n0 = nt * a.BN;
  const int k0 = split * a.kper;
  const int KC = min(a.kper, a.K - k0);  // multiple of 16 by construction
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * a.kper * 2;
  (void)n_tiles;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 256);
  // conv-first delivery (FC forward after a server round): the round's FC deliveries complete and every
  // peer done reading this rank's G, which is cleared here (before the W staging below)
  if (a.acq.ctr && a.acq.conv_first) fused_round_acquire(a.acq);
  // ---- stage A (128 rows x KC) and B (BN rows x KC), 16-byte vectors
  const __nv_bfloat16* Ag = a.A[g];
  const __nv_bfloat16* Bg = a.B[g];
  const int kch = KC / 8;
  // all 16-byte pieces go out as cp.async (LDGSTS) so a thread keeps dozens of loads in flight;
  // operands older than the immediate predecessor (pre_a / pre_b) are staged before the PDL wait
  const uint4 z4 = make_uint4(0, 0, 0, 0);
  const bool b_first = a.pre_b && !a.pre_a;
  if (b_first) stage_b_operand(a, Bg, sB, n0, k0, KC, kch);
  // TC_EPI_MASK_T: the ReLU mask tile [BN][128] (two or more launches old) lands in shared memory
  // before the wait, so the epilogue has no global loads on its critical path
  unsigned short* sMask = reinterpret_cast<unsigned short*>(smem + (128 + a.BN) * a.kper * 2);
  const bool mask_smem = a.epi == TC_EPI_MASK_T && tc_mask_fits(a);
  if (mask_smem) {
    for (int e = threadIdx.x; e < a.BN * 16; e += blockDim.x) {
      const int nl = e / 16, ch = e % 16;
      const int n = n0 + nl, mm = m0 + 8 * ch;
      uint8_t* d = reinterpret_cast<uint8_t*>(sMask + nl * 128 + 8 * ch);
      if (n < a.N && mm + 8 <= a.M) cp_async16(d, a.mask + (long long)n * a.ldo + mm);
      else *reinterpret_cast<uint4*>(d) = z4;
    }
  }
  if (!a.pre_a) { pdl_sync(); st_stamp(a.st_id, 1); }
  if (!a.a_mn) {  // K-major: smem [kc][row][8]
    for (int e = threadIdx.x; e < 128 * kch; e += blockDim.x) {
      const int r = e / kch, c = e % kch;
      const int m = m0 + r;
      uint8_t* d = sA + (c * 128 + r) * 16;
      if (m < a.M) cp_async16(d, Ag + (long long)m * a.lda + k0 + 8 * c);
      else *reinterpret_cast<uint4*>(d) = z4;
    }
  } else {        // MN-major: smem [row/8][k][8]
    for (int e = threadIdx.x; e < 16 * KC; e += blockDim.x) {
      const int gi = e % 16, k = e / 16;
      const int m = m0 + 8 * gi;
      uint8_t* d = sA + (gi * KC + k) * 16;
      if (m < a.M) cp_async16(d, Ag + (long long)(k0 + k) * a.lda + m);
      else *reinterpret_cast<uint4*>(d) = z4;
    }
  }
  const int bn = a.BN;
  // operands produced by the immediate predecessor are staged after the PDL wait (pre_a / pre_b flags)
  if (a.pre_a && !a.pre_b) { pdl_sync(); st_stamp(a.st_id, 1); }
  if (!b_first) stage_b_operand(a, Bg, sB, n0, k0, KC, kch);
  cp_async_wait_all();
  if (a.pre_a && a.pre_b) { pdl_sync(); st_stamp(a.st_id, 1); }  // the epilogue's outputs may still be read by the predecessor
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const bool ph = a.st_ph && tile == 0 && split == 0 && g == 0;  // DQN_TRACE_STEP phase stamps
  if (ph) st_stamp_here(a.st_ph, 0);
  const uint32_t tmem = tbase;
  if (warp == 0) {  // warp-uniform issue (one elected lane), not a per-lane R2UR loop under threadIdx.x == 0
    const uint32_t idesc = make_idesc_bf16(128, bn, a.a_mn, a.b_mn);
    const uint32_t ab = smem_u32(sA), bb = smem_u32(sB);
    for (int kk = 0; kk < KC / 16; ++kk) {
      const uint64_t ad = a.a_mn ? make_desc(ab + kk * 256, 128, KC * 16) : make_desc(ab + kk * 2 * 128 * 16, 128 * 16, 128);
      const uint64_t bd = a.b_mn ? make_desc(bb + kk * 256, 128, KC * 16) : make_desc(bb + kk * 2 * bn * 16, bn * 16, 128);
      mma_bf16_w(tmem, ad, bd, idesc, kk > 0);
    }
    mma_commit_w(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (ph) st_stamp_here(a.st_ph, 1);
  const int m = m0 + 32 * warp + lane;
  const uint32_t trow = tmem + ((uint32_t)(32 * warp) << 16);
  if (a.epi == TC_EPI_ACCUM && a.store) {
    // plain store: each thread writes its row's bn contiguous floats straight from TMEM (16-byte
    // stores; a warp's 32 rows complete whole 128-byte lines over consecutive chunks)
    float* crow = a.C[g] + (long long)m * a.ldc + n0;
    const bool vec = ((a.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.C[g]) & 15) == 0) && (n0 & 3) == 0;
    for (int c = 0; c < bn; c += 16) {
      float v[16];
      tmem_ld16(trow + c, v);
      if (m >= a.M) continue;
      if (vec && n0 + c + 16 <= a.N) {
#pragma unroll
        for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(crow + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      } else {
        for (int i = 0; i < 16 && n0 + c + i < a.N; ++i) crow[c + i] = v[i];
      }
    }
  } else if (a.epi == TC_EPI_ACCUM) {
    // TMEM -> shared tile [128][bn+4] (the MMAs are complete, so the operand staging area is free),
    // then a coalesced read-modify-write of C by the whole CTA with many 16-byte accesses in flight
    float* sD = reinterpret_cast<float*>(smem);
    const int ld = bn + 4;
    for (int c = 0; c < bn; c += 16) {
      float v[16];
      tmem_ld16(trow + c, v);
      float* row = sD + (32 * warp + lane) * ld + c;
#pragma unroll
      for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(row + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    }
    const int nv = bn / 4;
    const bool vec = (a.ldc % 4) == 0 && ((reinterpret_cast<uintptr_t>(a.C[g]) & 15) == 0);
    const int ncols = min(bn, a.N - n0);
    if (a.bulk_accum && vec && ncols % 4 == 0) {
      // one bulk transfer per tile row: C += row (or C = row) done by the TMA unit at L2, fp32 add with RN
      // (the same rounding as the register path below), no load round trip through the SM
      fence_async_smem();
      __syncthreads();
      const int r = threadIdx.x;
      if (m0 + r < a.M) bulk_s2g_f32(a.C[g] + (long long)(m0 + r) * a.ldc + n0, sD + r * ld, (uint32_t)ncols * 4, !a.store);
      goto epi_done;
    }
    __syncthreads();
    constexpr int BATCH = 12;  // loads of a batch are all issued before any store (C may alias nothing else,
                               // but the compiler cannot know that)
    for (int e0 = threadIdx.x; e0 < 128 * nv; e0 += 128 * BATCH) {
      float4 o[BATCH];
      float* dst[BATCH];
      bool ok[BATCH];
#pragma unroll
      for (int k = 0; k < BATCH; ++k) {
        const int e = e0 + k * 128;
        const int r = e / nv, q = e % nv;
        const int mm = m0 + r, n = n0 + 4 * q;
        ok[k] = e < 128 * nv && mm < a.M && vec && n + 4 <= a.N;
        dst[k] = a.C[g] + (long long)mm * a.ldc + n;
        o[k] = ok[k] && !a.store ? *reinterpret_cast<const float4*>(dst[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int k = 0; k < BATCH; ++k) {
        const int e = e0 + k * 128;
        if (e >= 128 * nv) break;
        const int r = e / nv, q = e % nv;
        const int mm = m0 + r, n = n0 + 4 * q;
        const float4 d = *reinterpret_cast<const float4*>(sD + r * ld + 4 * q);
        if (ok[k]) {
          o[k].x += d.x; o[k].y += d.y; o[k].z += d.z; o[k].w += d.w;
          *reinterpret_cast<float4*>(dst[k]) = o[k];
        } else if (mm < a.M) {
          const float dv[4] = {d.x, d.y, d.z, d.w};
          for (int i = 0; i < 4 && n + i < a.N; ++i) dst[k][i] = a.store ? dv[i] : dst[k][i] + dv[i];
        }
      }
    }
  } else if (a.epi == TC_EPI_MASK_T) {
    // output feature m of sample n goes to n*ldo + om (NHWC re-layout for the generic conv path)
    const long long om = a.hwc_HW ? (long long)(m % a.hwc_HW) * a.hwc_C + m / a.hwc_HW : (long long)m;
    __nv_bfloat16* const orow = a.out_bf16 + om;
    for (int c = 0; c < bn; c += 16) {
      float v[16];
      tmem_ld16(trow + c, v);
      if (m < a.M) {
        unsigned short mk[16];  // from the staged tile, or all 16 global loads in flight
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = n0 + c + i;
          mk[i] = mask_smem ? sMask[(c + i) * 128 + (m - m0)]
                            : (n < a.N ? __ldg(reinterpret_cast<const unsigned short*>(a.mask) + (long long)n * a.ldo + m) : 0);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = n0 + c + i;
          if (n < a.N)  // bf16 > 0 <=> sign bit clear and not +0
            orow[(long long)n * a.ldo] = __float2bfloat16_rn((mk[i] & 0x8000u) == 0 && mk[i] != 0 ? v[i] : 0.0f);
        }
      }
      if (ph && c < 48) st_stamp_here(ST_P6, c / 16);
    }
  } else {  // TC_EPI_FC_FWD: split partials, transposed to [g][split][n][m] (coalesced over m)
    float* pbase = a.partial + ((long long)g * a.splits + split) * (long long)a.N * a.M;
    for (int c = 0; c < bn; c += 16) {
      float v[16];
      tmem_ld16(trow + c, v);
      if (m < a.M) {
        float* prow = pbase + (long long)(n0 + c) * a.M + m;  // split stride is N*M
        if (n0 + c + 16 <= a.N) {
#pragma unroll
          for (int i = 0; i < 16; ++i) prow[(long long)i * a.M] = v[i];
        } else {
          for (int i = 0; i < 16 && n0 + c + i < a.N; ++i) prow[(long long)i * a.M] = v[i];
        }
      }
    }
  }
epi_done:
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

__global__ void __launch_bounds__(128) tc_gemm_kernel(TcGemmArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  st_stamp(a.st_id, 0);
  tc_gemm_tile(a, blockIdx.x, blockIdx.y, blockIdx.z, smem, bar, tbase);
  st_stamp(a.st_id, 2);
}

struct TcPairArgs {
  TcGemmArgs p0, p1;
  int tiles0, tiles1;
  HeadArgs head;
};

__global__ void __launch_bounds__(128) tc_pair_kernel(TcPairArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int bx = blockIdx.x;
  st_stamp(ST_FC_BWD, 0);
  if (bx < a.tiles0) {
    tc_gemm_tile(a.p0, bx, 0, 0, smem, bar, tbase);
    if (bx == 0) st_stamp_here(ST_P3, 2);
  } else if (bx < a.tiles0 + a.tiles1) {
    tc_gemm_tile(a.p1, bx - a.tiles0, 0, 0, smem, bar, tbase);
    if (bx == a.tiles0) st_stamp_here(ST_P4, 2);
  } else {
    pdl_sync();  // the TD head's per-sample outputs come from the predecessor
    if (bx == a.tiles0 + a.tiles1) st_stamp_here(ST_P5, 0);
    const HeadArgs& h = a.head;
    const int n = head_finish_elems(h);
    // the samples' actions and dQ staged in shared memory (this CTA's operand area is unused)
    int* s_act = reinterpret_cast<int*>(smem);
    float* s_dq = reinterpret_cast<float*>(smem) + h.b;
    for (int j = threadIdx.x; j < h.b; j += 128) {
      s_act[j] = h.s_act[j];
      s_dq[j] = h.s_dq[j];
    }
    __syncthreads();
    const bool warp_rows = h.H % 32 == 0;  // a warp's 32 dW_o elements share one action
    const float* h0 = h.fc_partial ? h.act_out[0] : h.act[0];
    for (int e = (bx - a.tiles0 - a.tiles1) * 128 + threadIdx.x; e < n; e += (gridDim.x - a.tiles0 - a.tiles1) * 128) {
      if (warp_rows && e - (threadIdx.x & 31) + 31 < h.A * h.H) {  // the whole warp in the dW_o rows
        const int a_ = e / h.H, u = e % h.H;
        h.grad[h.w_off + e] += head_finish_dwo_warp(h, h0, s_act, s_dq, a_, u);
      } else {
        head_finish_elem(h, e);
      }
    }
    if (bx == a.tiles0 + a.tiles1) st_stamp_here(ST_P5, 2);
  }
  st_stamp(ST_FC_BWD, 2);
}

static size_t tc_smem(const TcGemmArgs& a) {
  size_t smem = (size_t)(128 + a.BN) * a.kper * 2;
  if (a.epi == TC_EPI_MASK_T && tc_mask_fits(a)) smem += (size_t)a.BN * 128 * 2;  // the mask tile
  if (a.epi == TC_EPI_ACCUM) smem = std::max(smem, (size_t)128 * (a.BN + 4) * 4);  // epilogue tile
  return smem;
}

bool tc_pair_fits(const TcGemmArgs& p0, const TcGemmArgs& p1) {
  return std::max(tc_smem(p0), tc_smem(p1)) <= (size_t)200 * 1024;
}

void launch_tc_pair_with_head(const TcGemmArgs& p0, const TcGemmArgs& p1, const HeadArgs& head, cudaStream_t st) {
  TcPairArgs a{p0, p1, cdiv(p0.M, 128) * cdiv(p0.N, p0.BN), cdiv(p1.M, 128) * cdiv(p1.N, p1.BN), head};
  const int head_ctas = cdiv(head.A * head.H + head.A + head.H + 1, 128);
  launch_pdl(tc_pair_kernel, dim3(a.tiles0 + a.tiles1 + head_ctas), dim3(128), std::max(tc_smem(p0), tc_smem(p1)), st,
             a);
}

// h[g][n][m] = relu(sum_split partial[g][split][n][m] + bias[g][m]), splits summed in order
__global__ void fc_reduce_kernel(TcGemmArgs a) {
  pdl_sync();
  const int g = blockIdx.y;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)a.M * a.N) return;
  const int n = (int)(e / a.M), m = (int)(e % a.M);
  const float* p = a.partial + (long long)g * a.splits * a.N * a.M + (long long)n * a.M + m;
  float s = 0.0f;
#pragma unroll 6
  for (int sp = 0; sp < a.splits; ++sp) s += p[(long long)sp * a.N * a.M];
  a.h_out[g][(long long)n * a.M + m] = fmaxf(s + a.bias[g][m], 0.0f);
}

void launch_tc_gemm(const TcGemmArgs& a, int groups, cudaStream_t st) {
  const int m_tiles = cdiv(a.M, 128), n_tiles = cdiv(a.N, a.BN);
  const size_t smem = tc_smem(a);
  dim3 grid(m_tiles * n_tiles, a.splits, groups);
  launch_pdl(tc_gemm_kernel, grid, dim3(128), smem, st, a);
  if (a.epi == TC_EPI_FC_FWD && a.h_out[0] != nullptr) {  // else the TD head reduces the partials itself
    dim3 rg(cdiv((long long)a.M * a.N, 256), groups);
    launch_pdl(fc_reduce_kernel, rg, dim3(256), 0, st, a);
  }
}

// the FC forward's split-K reduction + bias + ReLU alone (after launch_gemm_pipe)
void launch_fc_reduce(const TcGemmArgs& a, int groups, cudaStream_t st) {
  dim3 rg(cdiv((long long)a.M * a.N, 256), groups);
  launch_pdl(fc_reduce_kernel, rg, dim3(256), 0, st, a);
}

// ------------------------------------------------------------------ a8/a9: fused conv backward
// One CTA per image j of the minibatch (group 0: s_j, theta). Per image:
//   conv2 dW  D2[(t,c'')][n2] += sum_{m'} A1(m'+shift_t)[c''] dZ2[m'][n2]      (2 M-tiles, MN-major A and B)
//   conv2 dX  dA1[p][c''] = sum_t sum_n2 dZ2(p - shift_t)[n2] W2[n2][c''][t]     (K-major, zero-padded rows)
//   dZ1 = dA1 * [A1 > 0]  (ReLU'(0) = 0), re-laid out for conv1's virtual rows
//   conv1 dW  D1[(t,c')][n] += sum_{m'} X(m'+shift_t)[c'] dZ1[m'][n]            (2 M-tiles, MN-major A and B)
//   db2 += sum dZ2, db1 += sum dZ1 (SIMT)
// An M = 128 tile spans two taps whose shifts differ by one pixel, so the image
// planes are stored twice (second copy one pixel ahead) and SBO walks 16 planes.
// Per-image partials are reduced in image order by the last CTA (deterministic).
constexpr int BWD_PART_W1 = 256 * 16;            // (t,c') x n
constexpr int BWD_PART_W2 = 256 * 32;            // (t,c'') x n2
constexpr int BWD_PART = kBwdPart;
constexpr int BWD_ROWS1 = 432;                   // conv1 virtual rows 420 padded to K-steps of 16
constexpr int BWD_ROWS2 = 96;                    // conv2 virtual rows 90 padded
constexpr int DZ2_OFF = 11;                      // zero rows ahead of dZ2 (largest tap shift)
constexpr int DZ2_ALLOC = 144;
constexpr int BWD_SX = 0;                                                  // 16 planes x X_ALLOC x 16
constexpr int BWD_SA1 = BWD_SX + 16 * mnih::X_ALLOC * 16;                  // 139264
constexpr int BWD_SDZ2 = BWD_SA1 + 16 * mnih::A1_ALLOC * 16;               // +36864
constexpr int BWD_SDZ1 = BWD_SDZ2 + 4 * DZ2_ALLOC * 16;                    // +9216
constexpr int BWD_SW2 = BWD_SDZ1 + 2 * BWD_ROWS1 * 16;                     // +13824
constexpr int BWD_SMEM = BWD_SW2 + 4 * 4 * 64 * 16;                        // +16384 = 215552

__device__ void rms_tail(const ReduceUpdateArgs& u, int cta, int ctas);

__global__ void __launch_bounds__(128) bwd_conv_bf16_kernel(BwdConvArgs a, ReduceUpdateArgs u) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar_w;
  __shared__ uint32_t tbase;
  __shared__ float s_db1[16], s_db2[32], s_db1_part[4][16];
  const int j = blockIdx.x;
  if (j >= a.n) {  // early-update CTAs (u.early): RMSProp of the non-conv parameters, off the critical path
    rms_tail(u, j - a.n, gridDim.x - a.n);
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  st_stamp(ST_CONV_BWD, 0);
  uint8_t* sX = smem + BWD_SX;
  uint8_t* sA1 = smem + BWD_SA1;
  uint8_t* sDZ2 = smem + BWD_SDZ2;
  uint8_t* sDZ1 = smem + BWD_SDZ1;
  uint8_t* sW2 = smem + BWD_SW2;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 2);    // conv2 dX: one commit per issuing warp (2)
    mbar_init(&bar_w, 6);  // conv2 dW (2 warps) + conv1 dW (4 warps)
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 256);
  // ---- zero the pads the MMAs read (garbage rows are multiplied by zero dZ rows, so must be finite)
  {
    uint4 z = make_uint4(0, 0, 0, 0);
    for (int e = threadIdx.x; e < 16 * (mnih::X_ALLOC - mnih::X_PIX + 1); e += blockDim.x) {
      const int pl = e / (mnih::X_ALLOC - mnih::X_PIX + 1), p = mnih::X_PIX - 1 + e % (mnih::X_ALLOC - mnih::X_PIX + 1);
      *reinterpret_cast<uint4*>(sX + (pl * mnih::X_ALLOC + p) * 16) = z;
    }
    for (int e = threadIdx.x; e < 16 * (mnih::A1_ALLOC - mnih::A1_PIX + 1); e += blockDim.x) {
      const int pl = e / (mnih::A1_ALLOC - mnih::A1_PIX + 1), p = mnih::A1_PIX - 1 + e % (mnih::A1_ALLOC - mnih::A1_PIX + 1);
      *reinterpret_cast<uint4*>(sA1 + (pl * mnih::A1_ALLOC + p) * 16) = z;
    }
    for (int e = threadIdx.x; e < 4 * DZ2_ALLOC; e += blockDim.x) reinterpret_cast<uint4*>(sDZ2)[e] = z;
    for (int e = threadIdx.x; e < 2 * BWD_ROWS1; e += blockDim.x) reinterpret_cast<uint4*>(sDZ1)[e] = z;
  }
  // ---- W2 as the B operand of conv2 dX, per tap: [t][n2/8][c'' 64][8]  (B(c'', n2) = W2[n2][c][ky][kx])
#pragma unroll
  for (int it = 0; it < 4 * 4 * 64 / 128; ++it) {  // 128 threads, all gathers in flight
    const int e = threadIdx.x + it * 128;
    const int c2 = e % 64, kc = (e / 64) % 4, t = e / 256;
    const int q = c2 >> 4, c = c2 & 15;
    const int ky = 2 * (t >> 1) + (q >> 1), kx = 2 * (t & 1) + (q & 1);
    uint32_t o[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int n0 = kc * 8 + 2 * h;
      const uint16_t lo = __bfloat16_as_ushort(a.theta[a.w2_off + ((n0 * 16 + c) * 4 + ky) * 4 + kx]);
      const uint16_t hi = __bfloat16_as_ushort(a.theta[a.w2_off + (((n0 + 1) * 16 + c) * 4 + ky) * 4 + kx]);
      o[h] = lo | ((uint32_t)hi << 16);
    }
    *reinterpret_cast<uint4*>(sW2 + ((t * 4 + kc) * 64 + c2) * 16) = make_uint4(o[0], o[1], o[2], o[3]);
  }
  __syncthreads();
  // ---- X (s_j) into planes 0..7 and the one-pixel-ahead copy into planes 8..15
  {
    // every thread issues all of its loads before the first conversion (latency, not bandwidth, bound)
    constexpr int XIT = (mnih::X_PIX * 4 + 127) / 128, AIT = (8 * mnih::A1_PIX + 127) / 128;
    const uint4* s4 = reinterpret_cast<const uint4*>(a.ring_s + (long long)a.idx[j] * a.slot_stride);
    const uint4* a4 = reinterpret_cast<const uint4*>(a.a1_save + (long long)j * 8 * mnih::A1_ALLOC * 16);
    uint4 xb[XIT], ab[AIT];
#pragma unroll
    for (int it = 0; it < XIT; ++it) {
      const int v = threadIdx.x + it * 128;
      xb[it] = v < mnih::X_PIX * 4 ? __ldg(s4 + v) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int it = 0; it < AIT; ++it) {
      const int v = threadIdx.x + it * 128;
      ab[it] = v < 8 * mnih::A1_PIX ? __ldg(a4 + (v / mnih::A1_PIX) * mnih::A1_ALLOC + v % mnih::A1_PIX)
                                   : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int it = 0; it < XIT; ++it) {
      const int v = threadIdx.x + it * 128;
      if (v >= mnih::X_PIX * 4) break;
      const int q = v / mnih::X_PIX, p = v % mnih::X_PIX;  // frame-major slot: frame q, pixel p
      uint4 lo, hi;
      u8x16_to_bf16(xb[it], lo, hi);
      *reinterpret_cast<uint4*>(sX + ((2 * q) * mnih::X_ALLOC + p) * 16) = lo;
      *reinterpret_cast<uint4*>(sX + ((2 * q + 1) * mnih::X_ALLOC + p) * 16) = hi;
      if (p > 0) {
        *reinterpret_cast<uint4*>(sX + ((8 + 2 * q) * mnih::X_ALLOC + p - 1) * 16) = lo;
        *reinterpret_cast<uint4*>(sX + ((9 + 2 * q) * mnih::X_ALLOC + p - 1) * 16) = hi;
      }
    }
#pragma unroll
    for (int it = 0; it < AIT; ++it) {
      const int v = threadIdx.x + it * 128;
      if (v >= 8 * mnih::A1_PIX) break;
      const int pl = v / mnih::A1_PIX, p = v % mnih::A1_PIX;
      *reinterpret_cast<uint4*>(sA1 + (pl * mnih::A1_ALLOC + p) * 16) = ab[it];
      if (p > 0) *reinterpret_cast<uint4*>(sA1 + ((8 + pl) * mnih::A1_ALLOC + p - 1) * 16) = ab[it];
    }
  }
  __syncthreads();  // zero-filled dZ2 planes before the scatter below
  pdl_sync();       // dZ2 is the predecessor's (FC dX) output; everything above overlapped it
  st_stamp(ST_CONV_BWD, 1);
  // ---- dZ2 (canonical [n2][81]) into planes [n2/8][DZ2_OFF + m'][8], m' = oy*10 + ox; + db2
  {
    const unsigned short* d = reinterpret_cast<const unsigned short*>(a.dz2 + (long long)j * mnih::D);
#pragma unroll
    for (int it = 0; it < (4 * 81 + 127) / 128; ++it) {
      const int e = threadIdx.x + it * 128;
      if (e < 4 * 81) {
        const int kc = e / 81, p = e % 81;
        const int oy = p / 9, ox = p % 9;
        uint32_t o[4];
#pragma unroll
        for (int h = 0; h < 4; ++h)
          o[h] = __ldg(d + (kc * 8 + 2 * h) * 81 + p) | ((uint32_t)__ldg(d + (kc * 8 + 2 * h + 1) * 81 + p) << 16);
        *reinterpret_cast<uint4*>(sDZ2 + (kc * DZ2_ALLOC + DZ2_OFF + oy * 10 + ox) * 16) =
            make_uint4(o[0], o[1], o[2], o[3]);
      }
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  st_stamp(ST_P6, 0);
  const uint32_t tmem = tbase;
  if (warp == 1) {  // db2 = sum of dZ2 over positions (zero rows contribute nothing)
    float s = 0.0f;
    const __nv_bfloat16* col = reinterpret_cast<const __nv_bfloat16*>(sDZ2 + (lane >> 3) * DZ2_ALLOC * 16) + (lane & 7);
    for (int r = DZ2_OFF; r < DZ2_OFF + mnih::M2V; ++r) s += __bfloat162float(col[r * 8]);
    s_db2[lane] = s;
  }
  // TMEM columns: [0,32) conv1 dW (2 tiles x 16, K half 0), [32,96) conv2 dW (2 tiles x 32), [128,192) and
  // [192,256) conv2 dX (taps 0-1, 2-3), then [128,160) conv1 dW K half 1. Warp-uniform issue spread over the
  // four warps: warps 0-1 conv2 dW M-tile w, warps 2-3 conv2 dX tap pair w - 2 (summed in the dZ1 epilogue).
  {
    const uint32_t xa = smem_u32(sA1), dz2 = smem_u32(sDZ2), w2 = smem_u32(sW2);
    if (warp < 2) {
      // conv2 dW: M = (t pair, c'') via 16 planes, K = m' (6 steps), N = 32 (B MN-major: dZ2 planes)
      const uint32_t id_dw2 = make_idesc_bf16(128, 32, 1, 1);
      const int mt = warp, sh = mt * 10;  // taps (0,1) -> shifts 0,1 ; taps (2,3) -> 10,11
#pragma unroll
      for (int kk = 0; kk < BWD_ROWS2 / 16; ++kk) {
        const uint64_t ad = make_desc(xa + (sh + 16 * kk) * 16, 128, mnih::A1_ALLOC * 16);
        const uint64_t bd = make_desc(dz2 + (DZ2_OFF + 16 * kk) * 16, 128, DZ2_ALLOC * 16);
        mma_bf16_w(tmem + 32 + 32 * mt, ad, bd, id_dw2, kk > 0);
      }
      mma_commit_w(&bar_w);
    } else {
      // conv2 dX: M = s2d pixel rows (100 -> 128), K = n2 (2 steps per tap), N = 64 (c'')
      const uint32_t id_dx = make_idesc_bf16(128, 64, 0, 0);
      const int tp = warp - 2;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int t = 2 * tp + (q >> 1), kk = q & 1;
        const uint64_t ad = make_desc(dz2 + (2 * kk) * DZ2_ALLOC * 16 + (DZ2_OFF - mnih::tap_shift2(t)) * 16,
                                      DZ2_ALLOC * 16, 128);
        const uint64_t bd = make_desc(w2 + ((t * 4 + 2 * kk) * 64) * 16, 64 * 16, 128);
        mma_bf16_w(tmem + 128 + 64 * tp, ad, bd, id_dx, q != 0);
      }
      mma_commit_w(&bar);
    }
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  st_stamp(ST_P6, 1);
  // ---- dZ1 = dA1 * [A1 > 0], into conv1 virtual rows m1 = y*21 + x, planes [n/8][m1][8]
  {
    const int p = 32 * warp + lane;  // s2d(2) pixel row of conv2's input
    float v[64];
#pragma unroll
    for (int c = 0; c < 64; c += 16) {
      float u[16];
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + 128 + c, v + c);
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + 192 + c, u);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[c + i] += u[i];
    }
    float dsum[16];  // db1 of this thread's pixel: its four sub-pixels' dZ1, per channel (bf16-rounded as stored)
#pragma unroll
    for (int n = 0; n < 16; ++n) dsum[n] = 0.0f;
    if (p < mnih::A1_PIX) {
      const int py = p / 10, px = p % 10;
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // (iy, ix) sub-pixel
        const uint4 m0 = *reinterpret_cast<const uint4*>(sA1 + ((2 * q) * mnih::A1_ALLOC + p) * 16);
        const uint4 m1 = *reinterpret_cast<const uint4*>(sA1 + ((2 * q + 1) * mnih::A1_ALLOC + p) * 16);
        const uint32_t mw[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
        uint32_t o[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const float a_lo = __uint_as_float(mw[h] << 16), a_hi = __uint_as_float(mw[h] & 0xFFFF0000u);
          const float d_lo = a_lo > 0.0f ? v[16 * q + 2 * h] : 0.0f;
          const float d_hi = a_hi > 0.0f ? v[16 * q + 2 * h + 1] : 0.0f;
          o[h] = pack_bf16(d_lo, d_hi);
          dsum[2 * h] += __uint_as_float(o[h] << 16);
          dsum[2 * h + 1] += __uint_as_float(o[h] & 0xFFFF0000u);
        }
        const int y = 2 * py + (q >> 1), x = 2 * px + (q & 1);
        const int m1r = y * mnih::X_W + x;
        *reinterpret_cast<uint4*>(sDZ1 + (0 * BWD_ROWS1 + m1r) * 16) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(sDZ1 + (1 * BWD_ROWS1 + m1r) * 16) = make_uint4(o[4], o[5], o[6], o[7]);
      }
    }
    // db1: the warp's 32 pixels by a shuffle butterfly per channel, then the 4 warps' sums in warp order
#pragma unroll
    for (int n = 0; n < 16; ++n) {
#pragma unroll
      for (int o2 = 16; o2 > 0; o2 >>= 1) dsum[n] += __shfl_xor_sync(0xffffffffu, dsum[n], o2);
    }
    if (lane < 16) {
      float vsel = dsum[0];
#pragma unroll
      for (int n = 1; n < 16; ++n)
        if (lane == n) vsel = dsum[n];
      s_db1_part[warp][lane] = vsel;
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  st_stamp(ST_P6, 2);
  {
    // conv1 dW: M = (t pair, c') via 16 X planes, K = m1 (27 steps), N = 16 (B MN-major: dZ1 planes);
    // warp w: M-tile w & 1, K half w >> 1 (steps [0,14) into columns 16 mt, [14,27) into 128 + 16 mt)
    const uint32_t xb = smem_u32(sX), dz1 = smem_u32(sDZ1);
    const uint32_t id_dw1 = make_idesc_bf16(128, 16, 1, 1);
    const int mt = warp & 1, kh = warp >> 1;
    const int sh = mt * mnih::X_W;  // taps (0,1) -> 0,1 ; (2,3) -> 21,22
    constexpr int KS = BWD_ROWS1 / 16, KH = (KS + 1) / 2;
    const int k0 = kh * KH, k1 = kh ? KS : KH;
    for (int kk = k0; kk < k1; ++kk) {
      const uint64_t ad = make_desc(xb + (sh + 16 * kk) * 16, 128, mnih::X_ALLOC * 16);
      const uint64_t bd = make_desc(dz1 + (16 * kk) * 16, 128, BWD_ROWS1 * 16);
      mma_bf16_w(tmem + 128 * kh + 16 * mt, ad, bd, id_dw1, kk > k0);
    }
    mma_commit_w(&bar_w);
  }
  // db1 = the 4 warps' sums (computed in the dZ1 epilogue) in warp order (deterministic)
  if (threadIdx.x < 16) s_db1[threadIdx.x] = ((s_db1_part[0][threadIdx.x] + s_db1_part[1][threadIdx.x]) +
                                              s_db1_part[2][threadIdx.x]) + s_db1_part[3][threadIdx.x];
  __syncwarp();
  st_stamp(ST_P7, 0);
  mbar_wait(&bar_w, 0);
  tc_fence_after();
  st_stamp(ST_P7, 1);
  // ---- per-image partials, column-major: [n][row], row = (t, c) of the tile; a warp's 32 rows of one column are
  // 128 contiguous bytes (row-major float4 rows touched 32 lines per store instruction)
  float* part = a.partial + (long long)j * BWD_PART;
  {
    const int r = 32 * warp + lane;  // M row within a tile
    for (int mt = 0; mt < 2; ++mt) {
      float v[32];
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + 16 * mt, v);
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + 128 + 16 * mt, v + 16);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] += v[16 + i];
#pragma unroll
      for (int i = 0; i < 16; ++i) part[i * 256 + mt * 128 + r] = v[i];
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + 32 + 32 * mt, v);
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + 32 + 32 * mt + 16, v + 16);
#pragma unroll
      for (int i = 0; i < 32; ++i) part[BWD_PART_W1 + i * 256 + mt * 128 + r] = v[i];
    }
    if (threadIdx.x < 16) part[BWD_PART_W1 + BWD_PART_W2 + threadIdx.x] = s_db1[threadIdx.x];
    if (threadIdx.x < 32) part[BWD_PART_W1 + BWD_PART_W2 + 16 + threadIdx.x] = s_db2[threadIdx.x];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
  st_stamp(ST_CONV_BWD, 2);
}

// canonical theta index of per-image partial entry e (tap-permuted conv dW rows, then the biases)
__device__ __forceinline__ long long bwd_part_dst(int e, const BwdConvArgs& a) {
  if (e < BWD_PART_W1) {  // column-major (n, mt*128 + r) with r -> tap t = 2*mt + r/64, c' = r%64
    const int row = e % 256, n = e / 256;
    const int t = 2 * (row / 128) + ((row % 128) >> 6), c = row & 63;
    const int f = c >> 4, iy = (c >> 2) & 3, ix = c & 3;
    const int ky = 4 * (t >> 1) + iy, kx = 4 * (t & 1) + ix;
    return a.w1_off + ((n * 4 + f) * 8 + ky) * 8 + kx;
  }
  if (e < BWD_PART_W1 + BWD_PART_W2) {
    const int ee = e - BWD_PART_W1;
    const int row = ee % 256, n = ee / 256;
    const int t = 2 * (row / 128) + ((row % 128) >> 6), c2 = row & 63;
    const int q = c2 >> 4, c = c2 & 15;
    const int ky = 2 * (t >> 1) + (q >> 1), kx = 2 * (t & 1) + (q & 1);
    return a.w2_off + ((n * 16 + c) * 4 + ky) * 4 + kx;
  }
  if (e < BWD_PART_W1 + BWD_PART_W2 + 16) return a.b1_off + (e - BWD_PART_W1 - BWD_PART_W2);
  return a.b2_off + (e - BWD_PART_W1 - BWD_PART_W2 - 16);
}

// the sum over images of partial entry e, in image order (deterministic); conv1's dW carries the
// 1/255 of the integer-valued input (d/dW of (W.u)/255)
// (the loads of 32 images are issued together, then summed in image order: latency, not bandwidth, bound)
__device__ __forceinline__ float bwd_part_sum(int e, const BwdConvArgs& a) {
  float s = 0.0f;
  for (int i0 = 0; i0 < a.n; i0 += 32) {
    float v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = i0 + k < a.n ? __ldcg(a.partial + (long long)(i0 + k) * BWD_PART + e) : 0.0f;
#pragma unroll
    for (int k = 0; k < 32; ++k)
      if (i0 + k < a.n) s += v[k];
  }
  return e < BWD_PART_W1 ? s * (1.0f / 255.0f) : s;
}

// Sum the per-image partials in image order (deterministic) and scatter into G's canonical layout.
// Large b: warp w of the CTA sums images [32 w, 32 w + 32) of 32 consecutive entries in image order (one round
// of 32 loads in flight instead of b / 32 serial rounds), then the CTA adds the warps' subtotals in warp order:
// a fixed two-level order, deterministic run to run. One warp per CTA (b <= 32) is the plain image order.
__global__ void bwd_reduce_kernel(BwdConvArgs a) {
  __shared__ float s_sub[8][32];
  st_stamp(ST_BWD_REDUCE, 0);
  pdl_sync();
  st_stamp(ST_BWD_REDUCE, 1);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  const int per = (a.n + nw - 1) / nw, i_lo = w * per, i_hi = min(a.n, i_lo + per);
  float s = 0.0f;
  if (e < BWD_PART) {
    for (int i0 = i_lo; i0 < i_hi; i0 += 32) {
      float v[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) v[k] = i0 + k < i_hi ? __ldcg(a.partial + (long long)(i0 + k) * BWD_PART + e) : 0.0f;
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (i0 + k < i_hi) s += v[k];
    }
  }
  s_sub[w][lane] = s;
  __syncthreads();
  if (w == 0 && e < BWD_PART) {
    float t = s_sub[0][lane];
    for (int q = 1; q < nw; ++q) t += s_sub[q][lane];
    a.grad[bwd_part_dst(e, a)] += e < BWD_PART_W1 ? t * (1.0f / 255.0f) : t;
  }
  st_stamp(ST_BWD_REDUCE, 2);
}

void launch_bwd_conv_bf16(const BwdConvArgs& a, cudaStream_t st, bool with_reduce) {
  launch_pdl(bwd_conv_bf16_kernel, dim3(a.n), dim3(128), BWD_SMEM, st, a, ReduceUpdateArgs{});
  // warps per 32 entries: image groups of 32, one batch of 32 loads in flight per thread (BJ.configs[3], b = 256:
  // 84.6 -> 82.0 us/step against groups of 64, which took two dependent batches; groups of 16 measured no better)
  const int nw = std::min(8, std::max(1, (a.n + 31) / 32));
  if (with_reduce) launch_pdl(bwd_reduce_kernel, dim3(cdiv(BWD_PART, 32)), dim3(32 * nw), 0, st, a);
}

// N = 1, n_push = 1: the image-order reduction of the conv partials fused into the RMSProp update
// (one launch and one G round trip fewer). Threads [0, BWD_PART) own one conv parameter each (the
// conv parameters are the canonical prefix [0, BWD_PART) of theta); the rest own a float4 of the
// remaining parameters and read G as rmsprop_kernel does. Same arithmetic per element as
// rmsprop_kernel (A4, A5, A24).
// Rounding pinned with explicit intrinsics (no context-dependent FMA contraction), so the update is
// bit-identical whichever launch applies it (reduce_update_kernel or the conv backward's extra CTAs).
__device__ __forceinline__ bool rms_elem(float& th, float& r, float g, const ReduceUpdateArgs& u) {
  const float gb = __fmul_rn(g, u.inv_div);
  if (!isfinite(gb)) return false;
  const float rr = __fmaf_rn(u.rho, r, __fmul_rn(__fmul_rn(u.omr, gb), gb));
  r = rr;
  th = __fmaf_rn(-__fmul_rn(u.lr, gb), rsqrtf(__fadd_rn(rr, u.eps)), th);
  return true;
}

// RMSProp of the float4 i of theta (non-conv part): G read then cleared, theta / r / bf16 published.
// Split into the loads and the rest so that callers can keep several float4s' loads in flight.
struct Rms4 { float4 g, t, r; };
__device__ __forceinline__ Rms4 rms_load4(const ReduceUpdateArgs& u, long long i) {
  return Rms4{reinterpret_cast<const float4*>(u.g)[i], reinterpret_cast<const float4*>(u.theta)[i],
              reinterpret_cast<const float4*>(u.r)[i]};
}
__device__ __forceinline__ unsigned rms_apply4(const ReduceUpdateArgs& u, long long i, const Rms4& x) {
  unsigned bad = 0;
  reinterpret_cast<float4*>(u.g)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (u.g_snap) reinterpret_cast<float4*>(u.g_snap)[i] = x.g;  // cfg.keep_grad (diagnostic)
  float tv[4] = {x.t.x, x.t.y, x.t.z, x.t.w}, rv[4] = {x.r.x, x.r.y, x.r.z, x.r.w};
  const float gv[4] = {x.g.x, x.g.y, x.g.z, x.g.w};
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (!rms_elem(tv[q], rv[q], gv[q], u)) ++bad;
  reinterpret_cast<float4*>(u.theta)[i] = make_float4(tv[0], tv[1], tv[2], tv[3]);
  reinterpret_cast<float4*>(u.r)[i] = make_float4(rv[0], rv[1], rv[2], rv[3]);
  uint2 o;
  o.x = pack_bf16(tv[0], tv[1]);
  o.y = pack_bf16(tv[2], tv[3]);
  reinterpret_cast<uint2*>(u.pub_bf16)[i] = o;
  return bad;
}

// non-conv float4 range of the update, grid-strided over the conv backward's extra CTAs (u.early);
// RMS_BATCH float4s per thread with all their loads issued first
constexpr int RMS_BATCH = 6;
__device__ void rms_tail(const ReduceUpdateArgs& u, int cta, int ctas) {
  pdl_sync();  // the FC / output-layer gradients come from the predecessor (FC backward + head finish)
  unsigned bad = 0;
  const long long n4 = u.n / 4, stride = (long long)ctas * 128;
  for (long long i0 = BWD_PART / 4 + (long long)cta * 128 + threadIdx.x; i0 < n4; i0 += stride * RMS_BATCH) {
    Rms4 x[RMS_BATCH];
#pragma unroll
    for (int k = 0; k < RMS_BATCH; ++k)
      if (i0 + k * stride < n4) x[k] = rms_load4(u, i0 + k * stride);
#pragma unroll
    for (int k = 0; k < RMS_BATCH; ++k)
      if (i0 + k * stride < n4) bad += rms_apply4(u, i0 + k * stride, x[k]);
  }
  if (bad) atomicAdd(&u.ctr->nonfinite, bad);
}

__global__ void __launch_bounds__(256) reduce_update_kernel(ReduceUpdateArgs u) {
  st_stamp(ST_UPDATE, 0);
  pdl_sync();
  st_stamp(ST_UPDATE, 1);
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned bad = 0;
  if (t < BWD_PART) {
    const int e = (int)t;
    const float g = bwd_part_sum(e, u.b);
    const long long d = bwd_part_dst(e, u.b);
    if (u.g_snap) u.g_snap[d] = g;  // cfg.keep_grad (diagnostic)
    float th = u.theta[d], r = u.r[d];
    if (rms_elem(th, r, g, u)) {
      u.theta[d] = th;
      u.r[d] = r;
    } else {
      ++bad;
    }
    const __nv_bfloat16 hb = __float2bfloat16_rn(th);
    u.pub_bf16[d] = hb;
    const int sl = wimg_slot(d, u.b.w1_off, u.b.w2_off);
    if (sl >= 0) u.pub_bf16[u.img_off + sl] = hb;
  } else {
    const long long i = BWD_PART / 4 + (t - BWD_PART);
    if (u.early || i >= u.n / 4) return;  // early: the conv backward's extra CTAs own this part
    bad += rms_apply4(u, i, rms_load4(u, i));
  }
  if (bad) atomicAdd(&u.ctr->nonfinite, bad);
  st_stamp(ST_UPDATE, 2);
}

void launch_reduce_update(const ReduceUpdateArgs& u, cudaStream_t st) {
  const long long threads = BWD_PART + (u.early ? 0 : u.n / 4 - BWD_PART / 4);
  launch_pdl(reduce_update_kernel, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0, st, u);
}

void launch_bwd_conv_update(const BwdConvArgs& a, const ReduceUpdateArgs& u, int upd_ctas, cudaStream_t st) {
  launch_pdl(bwd_conv_bf16_kernel, dim3(a.n + upd_ctas), dim3(128), BWD_SMEM, st, a, u);
}

void init_bf16_kernel_attrs() {
  cudaFuncSetAttribute(fwd_conv_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FWD_SMEM);
  cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(tc_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(bwd_conv_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_SMEM);
}

DQN_STEP_TRACE_HOST(bf16)

}  // namespace dqn
