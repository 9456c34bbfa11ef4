// kernels_common.cu — precision-independent kernels of the hot path:
//   a1  sampler (counter-based Philox4x32-10, integer-only index mapping)
//   push path (validation + FIFO ring writes, "Store experience" of Alg. 1)
//   a12 fused RMSProp shard update of Alg. 2
#include <algorithm>

#include "dqn_internal.h"
#include "pdl.cuh"
#include "philox.cuh"
#include "step_trace.cuh"
#include "wimg.cuh"

namespace dqn {

// ---------------------------------------------------------------- a1 sampler
// "Uniformly sample minibatch of experiences X from D_k" (Alg. 1), with
// replacement (A11): counter (j, T_lo, T_hi, rank), key = seed.
__global__ void sample_kernel(int* idx, int b, unsigned long long seed, unsigned rank, const DevCounters* ctr) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= b) return;
  idx[j] = (int)sample_slot(seed, rank, ctr->T, (unsigned)j, ctr->ring_size);
}

void launch_sample(int* idx, int b, unsigned long long seed, unsigned rank, const DevCounters* ctr,
                   cudaStream_t st) {
  sample_kernel<<<(b + 127) / 128, 128, 0, st>>>(idx, b, seed, rank, ctr);
}

// ---------------------------------------------------------------- push path
__global__ void validate_push_kernel(const int32_t* a, const float* r, long long n, int A, DevCounters* ctr) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (a[i] < 0 || a[i] >= A || !isfinite(r[i])) atomicAdd(&ctr->bad_input, 1u);
}

// replay_dedup: flag any item whose s'[0..F-2] differs from s[1..F-1] (16-byte words when aligned)
__global__ void validate_dedup_kernel(const uint8_t* s, const uint8_t* sn, long long sb, long long fb,
                                      DevCounters* ctr) {
  const long long i = blockIdx.x;
  const uint8_t* a = s + i * sb + fb;
  const uint8_t* b = sn + i * sb;
  const long long n = sb - fb;
  bool diff = false;
  if (((((uintptr_t)a) | ((uintptr_t)b) | n) & 15) == 0) {
    for (long long v = threadIdx.x; v < n / 16; v += blockDim.x) {
      const uint4 x = reinterpret_cast<const uint4*>(a)[v], y = reinterpret_cast<const uint4*>(b)[v];
      diff |= (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
    }
  } else {
    for (long long v = threadIdx.x; v < n; v += blockDim.x) diff |= a[v] != b[v];
  }
  if (diff) atomicOr(&ctr->bad_input, 2u);
}

void launch_validate_dedup(const uint8_t* s, const uint8_t* sn, long long n, long long sb, long long fb,
                           DevCounters* ctr, cudaStream_t st) {
  if (n > 0) validate_dedup_kernel<<<(unsigned)n, 256, 0, st>>>(s, sn, sb, fb, ctr);
}

void launch_validate_push(const int32_t* a, const float* r, long long n, int A, DevCounters* ctr, cudaStream_t st) {
  if (n <= 0) return;
  validate_push_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a, r, n, A, ctr);
}

// Item i of this chunk (global push index n_total_before + first + i) goes to
// slot (count0 + first + i) mod cap. One CTA per transition, 16-byte copies.
// canonical [F][H][W] slots, slot stride `stride` bytes (state_bytes, or (F+1) frames with frame
// dedup: the s' ring then aliases the s ring one frame later and only the new frame of s' is written)
__global__ void push_kernel(uint8_t* ring_s, uint8_t* ring_sn, int32_t* ring_a, float* ring_r, uint8_t* ring_t,
                            long long cap, long long count0, long long first, long long state_bytes,
                            const uint8_t* s, const int32_t* a, const float* r, const uint8_t* sn,
                            const uint8_t* t, long long* ring_size_out, long long ring_size, long long stride,
                            long long frame_bytes) {
  long long i = blockIdx.x;
  if (ring_size_out && i == 0 && threadIdx.x == 0) *ring_size_out = ring_size;
  long long slot = (count0 + first + i) % cap;
  // s: the whole stack; s': the whole stack, or (dedup) only its last frame
  const long long off1 = frame_bytes ? state_bytes - frame_bytes : 0;
  const uint8_t* src0 = s + i * state_bytes;
  const uint8_t* src1 = sn + i * state_bytes + off1;
  uint8_t* dst0 = ring_s + slot * stride;
  uint8_t* dst1 = ring_sn + slot * stride + off1;
  const long long n1 = state_bytes - off1;
  bool vec = ((state_bytes & 15) == 0) && ((n1 & 15) == 0) && ((stride & 15) == 0) &&
             ((((uintptr_t)src0) | ((uintptr_t)src1) | ((uintptr_t)dst0) | ((uintptr_t)dst1)) & 15) == 0;
  if (vec) {
    for (long long v = threadIdx.x; v < state_bytes / 16; v += blockDim.x)
      reinterpret_cast<uint4*>(dst0)[v] = reinterpret_cast<const uint4*>(src0)[v];
    for (long long v = threadIdx.x; v < n1 / 16; v += blockDim.x)
      reinterpret_cast<uint4*>(dst1)[v] = reinterpret_cast<const uint4*>(src1)[v];
  } else {
    for (long long v = threadIdx.x; v < state_bytes; v += blockDim.x) dst0[v] = src0[v];
    for (long long v = threadIdx.x; v < n1; v += blockDim.x) dst1[v] = src1[v];
  }
  if (threadIdx.x == 0) {
    ring_a[slot] = a[i];
    ring_r[slot] = r[i];
    ring_t[slot] = t[i] ? 1 : 0;
  }
}

void launch_push_canonical(uint8_t* ring_s, uint8_t* ring_sn, int32_t* ring_a, float* ring_r, uint8_t* ring_t,
                           long long cap, long long count0, long long n_total, long long first, long long n,
                           long long state_bytes, const uint8_t* s, const int32_t* a, const float* r,
                           const uint8_t* sn, const uint8_t* t, cudaStream_t st, long long* ring_size_out,
                           long long ring_size, long long stride, int dedup) {
  (void)n_total;
  if (n <= 0) return;
  if (stride <= 0) stride = state_bytes;
  push_kernel<<<(unsigned)n, 256, 0, st>>>(ring_s, ring_sn, ring_a, ring_r, ring_t, cap, count0, first, state_bytes,
                                           s, a, r, sn, t, ring_size_out, ring_size, stride,
                                           dedup ? stride - state_bytes : 0);
}

// ---------------------------------------------------------------- a12 update
// RMSPropUpdate (Alg. 2) on the owned shard, fused with the mean over
// N * n_push gradients (A7, A8), the non-finite guard (A24), the publication of
// the working-precision copy that the fetch all-gathers (a13), and the reset of
// the gradient accumulator. r is updated first and theta uses the new r (A5);
// eps sits inside the root (A4).
// One 16-byte vector per thread (n is a multiple of 64): every load is issued up
// front, there is no loop-carried latency and no fence. The round counter n is
// mirrored by the host (deterministic schedule); non-finite elements are counted
// (sticky) with one atomic per offending thread.
struct RmsArgs {
  float* theta;
  float* r;
  float* g;
  long long n;
  float inv_div, lr, rho, omr, eps;
  float* pub_f32;
  __nv_bfloat16* pub_bf16;
  int zero_g;
  long long img_off, w1_off, w2_off;
  float* g_snap;
  const int2* pack_map;
  long long pack_n, pack_off;
};

// one float4 of the update (loads done by the caller); returns the non-finite count
__device__ __forceinline__ unsigned rmsprop_vec(const RmsArgs& u, long long i, float4 g4, float4 t4, float4 r4) {
  if (u.zero_g) reinterpret_cast<float4*>(u.g)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (u.g_snap) reinterpret_cast<float4*>(u.g_snap)[i] = g4;  // cfg.keep_grad (diagnostic)
  float tv[4] = {t4.x, t4.y, t4.z, t4.w};
  float rv[4] = {r4.x, r4.y, r4.z, r4.w};
  const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
  unsigned bad = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float gb = gv[q] * u.inv_div;  // mean over N * n_push gradients (A7, A8)
    if (isfinite(gb)) {
      const float rr = u.rho * rv[q] + u.omr * gb * gb;
      rv[q] = rr;
      tv[q] = tv[q] - u.lr * gb * rsqrtf(rr + u.eps);
    } else {
      ++bad;
    }
  }
  t4 = make_float4(tv[0], tv[1], tv[2], tv[3]);
  reinterpret_cast<float4*>(u.theta)[i] = t4;
  reinterpret_cast<float4*>(u.r)[i] = make_float4(rv[0], rv[1], rv[2], rv[3]);
  if (u.pub_f32) reinterpret_cast<float4*>(u.pub_f32)[i] = t4;
  if (u.pub_bf16) {
    uint2 o;
    __nv_bfloat162 lo = __floats2bfloat162_rn(t4.x, t4.y), hi = __floats2bfloat162_rn(t4.z, t4.w);
    o.x = *reinterpret_cast<uint32_t*>(&lo);
    o.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(u.pub_bf16)[i] = o;
    if (u.pack_map && 4 * i < u.pack_n) {  // the generic path's packed conv images (gpack_kernel, fused at N = 1)
      const float tq[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (4 * i + q >= u.pack_n) break;
        const int2 d = u.pack_map[4 * i + q];
        const __nv_bfloat16 v = __float2bfloat16_rn(tq[q]);
        if (d.x >= 0) u.pub_bf16[u.pack_off + d.x] = v;
        if (d.y >= 0) u.pub_bf16[u.pack_off + d.y] = v;
      }
    }
    if (u.img_off >= 0 && 4 * i + 3 >= min(u.w1_off, u.w2_off) && 4 * i < max(u.w1_off, u.w2_off) + kW2Elems) {
      const float tq[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int sl = wimg_slot(4 * i + q, u.w1_off, u.w2_off);
        if (sl >= 0) u.pub_bf16[u.img_off + sl] = __float2bfloat16_rn(tq[q]);
      }
    }
  }
  return bad;
}

// grid-stride over the float4s, RMS_VECS of them per thread and round with all their loads issued first (large
// vectors run on a few waves of resident threads instead of one thread per float4)
constexpr int RMS_VECS = 4;
__global__ void __launch_bounds__(256) rmsprop_kernel(RmsArgs u, DevCounters* ctr) {
  st_stamp(ST_UPDATE, 0);
  pdl_sync();
  st_stamp(ST_UPDATE, 1);
  const long long n4 = u.n / 4, stride = (long long)gridDim.x * blockDim.x;
  unsigned bad = 0;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n4; i0 += stride * RMS_VECS) {
    float4 g4[RMS_VECS], t4[RMS_VECS], r4[RMS_VECS];
#pragma unroll
    for (int k = 0; k < RMS_VECS; ++k) {
      const long long i = i0 + k * stride;
      if (i < n4) {
        g4[k] = reinterpret_cast<const float4*>(u.g)[i];
        t4[k] = reinterpret_cast<const float4*>(u.theta)[i];
        r4[k] = reinterpret_cast<const float4*>(u.r)[i];
      }
    }
#pragma unroll
    for (int k = 0; k < RMS_VECS; ++k) {
      const long long i = i0 + k * stride;
      if (i < n4) bad += rmsprop_vec(u, i, g4[k], t4[k], r4[k]);
    }
  }
  if (bad) atomicAdd(&ctr->nonfinite, bad);
  st_stamp(ST_UPDATE, 2);
}

void launch_rmsprop(float* theta, float* r, float* g, long long n, float div, float lr, float rho, float omr,
                    float eps, float* pub_f32, __nv_bfloat16* pub_bf16, DevCounters* ctr, int zero_g,
                    cudaStream_t st, long long img_off, long long w1_off, long long w2_off, float* g_snap,
                    const int2* pack_map, long long pack_n, long long pack_off) {
  // one float4 per thread up to 4 resident waves of 256-thread CTAs, a grid-stride loop beyond
  const long long blocks = std::min<long long>((n / 4 + 255) / 256, 4LL * 148);
  const RmsArgs u{theta, r, g, n, 1.0f / div, lr, rho, omr, eps, pub_f32, pub_bf16, zero_g, img_off, w1_off, w2_off,
                  g_snap, pack_map, pack_n, pack_off};
  launch_pdl(rmsprop_kernel, dim3((unsigned)(blocks < 1 ? 1 : blocks)), dim3(256), 0, st, u, ctr);
}


__global__ void f32_to_bf16_kernel(const float* src, __nv_bfloat16* dst, long long n, long long img_off,
                                   long long w1_off, long long w2_off) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    const __nv_bfloat16 v = __float2bfloat16_rn(src[i]);
    dst[i] = v;
    if (img_off >= 0) {  // the conv weights' forward image (wimg.cuh)
      const int sl = wimg_slot(i, w1_off, w2_off);
      if (sl >= 0) dst[img_off + sl] = v;
    }
  }
}

void launch_f32_to_bf16(const float* src, __nv_bfloat16* dst, long long n, cudaStream_t st, long long img_off,
                        long long w1_off, long long w2_off) {
  if (n <= 0) return;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  f32_to_bf16_kernel<<<blocks, 256, 0, st>>>(src, dst, n, img_off, w1_off, w2_off);
}

__global__ void bf16_to_f32_kernel(const __nv_bfloat16* src, float* dst, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) dst[i] = __bfloat162float(src[i]);
}

void launch_bf16_to_f32(const __nv_bfloat16* src, float* dst, long long n, cudaStream_t st) {
  if (n <= 0) return;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  bf16_to_f32_kernel<<<blocks, 256, 0, st>>>(src, dst, n);
}

DQN_STEP_TRACE_HOST(common)

}  // namespace dqn
