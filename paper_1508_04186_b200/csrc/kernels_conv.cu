// kernels_conv.cu — the generic bf16 tensor-core conv path (a3/a4/a4s forward, a8/a9 backward)
// for conv stacks other than the Mnih-2013 one, e.g. the scaled net of BASELINE.json configs[4]
// (conv32 8x8/4, conv64 4x4/2, conv64 3x3/1).
//
// Every k x k / s convolution is a stride-1 convolution with kt = k/s taps per axis over a
// space-to-depth grid (Hs, Ws, Cs = C*s*s), so one implicit-GEMM kernel shape covers all layers.
// Activations live in HBM as [image][y][x][channel] bf16 (channels contiguous: one 16-byte chunk
// = 8 channels of one pixel). Channel order of a s2d grid: layer 1 reads the replay ring's order
// c' = f*16 + iy*4 + ix (push_s2d); later layers use c' = (iy*s + ix)*C + c, written directly by
// the previous layer's epilogue. Weights are read from "packed images" inside the bf16 theta
// buffer (the update writes them; pack maps computed at create): forward [N][K], K = tap*Cs + c'
// and data-gradient [Cs][T*N].
//
// Three tcgen05 kernels, M = 128 rows per CTA, 128 threads, K staged in chunks of 64 with a
// two-stage cp.async pipeline, fp32 accumulators in TMEM:
//   gconv_fwd   rows = output pixels of 128 (image, y, x); K = (tap, c'); N = Cout
//               epilogue: (x 1/255 on layer 1) + bias, ReLU, bf16 into the next layer's grid or
//               the canonical (C,H,W) flatten of the FC input
//   gconv_dgrad rows = input-grid pixels; K = (tap, n) over dZ shifted back by the tap; N = Cs
//               epilogue: x [input activation > 0] (ReLU'), scattered back to the previous
//               layer's output grid (inverse space-to-depth) as its dZ
//   gconv_wgrad rows = (tap, c') of dW; K = (image, output pixel) over a range of images;
//               N = Cout; both operands MN-major; per-range partials (+ db), reduced in range
//               order by gconv_wreduce into G (deterministic)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <unistd.h>
#include "dqn_internal.h"
#include "pdl.cuh"
#include "philox.cuh"
#include "sm100.cuh"
#include "step_trace.cuh"

namespace dqn {
using namespace dqn_sm100;

namespace {

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_n() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst_smem, const void* src_gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst_smem)), "l"(src_gmem) : "memory");
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}
// 4 u8 -> 4 exact bf16 (two words) without I2F: 0x4B0000bb is the float 2^23 + b, minus 2^23 is
// exactly b (< 256), whose low 16 bits are zero, so its upper half is the bf16 of b
__device__ __forceinline__ uint2 u8x4_to_bf16(uint32_t w) {
  const float f0 = __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7440)) - 8388608.0f;
  const float f1 = __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7441)) - 8388608.0f;
  const float f2 = __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7442)) - 8388608.0f;
  const float f3 = __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7443)) - 8388608.0f;
  return make_uint2(__byte_perm(__float_as_uint(f0), __float_as_uint(f1), 0x7632),
                    __byte_perm(__float_as_uint(f2), __float_as_uint(f3), 0x7632));
}
// 8 u8 (two words) -> 8 exact bf16 as one 16-byte chunk
__device__ __forceinline__ uint4 u8x8_to_bf16(uint32_t w0, uint32_t w1) {
  const uint2 a = u8x4_to_bf16(w0), b = u8x4_to_bf16(w1);
  return make_uint4(a.x, a.y, b.x, b.y);
}
// bounded mbarrier wait: a lost MMA completion is recorded (g_gconv_err) and the wait abandoned,
// so a bug cannot hang the GPU; the host reports it (gconv_debug / dqn_train_steps)
__device__ unsigned long long g_gconv_err;
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity, int where) {
  uint32_t done;
  long long n = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (!done && ++n > (1LL << 24)) {
      atomicExch(&g_gconv_err, ((unsigned long long)where << 48) | ((unsigned long long)blockIdx.y << 32) |
                                   ((unsigned long long)blockIdx.x << 8) | parity);
      return;
    }
  } while (!done);
}
// bf16 bits > 0 (sign clear, not +0)
__device__ __forceinline__ bool bf16_pos(uint32_t h) { return (h & 0x8000u) == 0 && (h & 0x7FFFu) != 0; }

constexpr int KCH = 64;                     // K per pipeline chunk
constexpr int NS = 2;                       // pipeline stages (chunks in flight)
constexpr int A_BYTES = 128 * KCH * 2;      // 16 KB
constexpr int U8_BYTES = 128 * KCH;         // layer 1: raw u8 A chunk, converted after its copy lands
// one stage: A [16 KB] | B [nB x 64 bf16] | (layer 1) u8 A [8 KB]
__host__ __device__ constexpr int stage_bytes(int nB, int first) {
  return ((A_BYTES + nB * KCH * 2 + (first ? U8_BYTES : 0)) + 1023) / 1024 * 1024;
}
constexpr int GCONV_SMEM_MAX = NS * stage_bytes(256, 1);
// TMEM columns of an accumulator of n fp32 columns (power of two >= 32): small N leaves room for
// more co-resident CTAs (these kernels are latency-bound per CTA)
__device__ __forceinline__ uint32_t tmem_cols(int n) {
  uint32_t c = 32;
  while (c < (uint32_t)n) c <<= 1;
  return c;
}

// One MMA K-chunk (64 = 4 x K16) from the stage buffers; A and B K-major [kc][rows][8] or
// MN-major [rows/8][k][8] as flagged.
__device__ __forceinline__ void issue_chunk(uint32_t tmem, uint32_t sa, uint32_t sb, int nB, bool a_mn, bool b_mn,
                                            bool first_chunk, int ksteps = KCH / 16) {
  const uint32_t idesc = make_idesc_bf16(128, nB, a_mn, b_mn);
  for (int kk = 0; kk < ksteps; ++kk) {
    const uint64_t ad = a_mn ? make_desc(sa + kk * 256, 128, KCH * 16) : make_desc(sa + (2 * kk) * 128 * 16, 128 * 16, 128);
    const uint64_t bd = b_mn ? make_desc(sb + kk * 256, 128, KCH * 16) : make_desc(sb + (2 * kk) * nB * 16, nB * 16, 128);
    mma_bf16(tmem, ad, bd, idesc, (!first_chunk || kk > 0) ? 1u : 0u);
  }
}

}  // namespace

// DQN_GCONV_DEBUG=1: per-CTA progress codes in mapped host memory, readable while a kernel runs
__device__ unsigned* g_prog;
__device__ __forceinline__ void prog(unsigned code) {
  if (g_prog && threadIdx.x == 0) {
    *(volatile unsigned*)(g_prog + blockIdx.y * 4096 + blockIdx.x) = code;
    __threadfence_system();
  }
}
static unsigned* h_prog = nullptr;

// DQN_GCONV_DEBUG=1: wait for every generic-path launch (bounded) and name a kernel that hangs
static void gconv_debug(const char* what, cudaStream_t st) {
  static int on = -1;
  if (on < 0) on = getenv("DQN_GCONV_DEBUG") ? atoi(getenv("DQN_GCONV_DEBUG")) : 0;
  if (!on) return;
  if (!h_prog) {
    cudaHostAlloc(reinterpret_cast<void**>(&h_prog), 8192 * sizeof(unsigned), cudaHostAllocMapped);
    unsigned* d = nullptr;
    cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), h_prog, 0);
    cudaMemcpyToSymbol(g_prog, &d, sizeof(d));
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fprintf(stderr, "gconv debug: launch of %s: %s\n", what, cudaGetErrorString(e));
  for (int i = 0; i < 5000; ++i) {
    e = cudaStreamQuery(st);
    if (e != cudaErrorNotReady) {
      unsigned long long err = 0;
      cudaMemcpyFromSymbol(&err, g_gconv_err, sizeof(err));
      fprintf(stderr, "gconv debug: %s done (%s) err %llx\n", what, cudaGetErrorString(e), err);
      return;
    }
    usleep(1000);
  }
  fprintf(stderr, "gconv debug: %s still running after 5 s; progress codes:", what);
  for (int i = 0; i < 64; ++i) fprintf(stderr, " %u", h_prog[i]);
  fprintf(stderr, "\n");
  fflush(stderr);
  _exit(3);
}

// ------------------------------------------------------------------ forward
__global__ void __launch_bounds__(128) gconv_fwd_kernel(GConvFwdArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[NS];
  __shared__ uint32_t tbase;
  const int g = blockIdx.y, tid = threadIdx.x, warp = tid >> 5;
  const int HoWo = a.Ho * a.Wo, T = a.Th * a.Tw, cbn = a.Cs / KCH, nch = T * cbn, K = T * a.Cs;
  const long long M = (long long)a.b * HoWo;
  const long long m0 = (long long)blockIdx.x * 128;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  prog(1);
  if (warp == 0) tmem_alloc(&tbase, tmem_cols(a.N));
  prog(2);
  // this thread's A row
  const long long m = m0 + tid;
  const bool row_ok = m < M;
  int img = 0, oy = 0, ox = 0;
  if (row_ok) {
    img = (int)(m / HoWo);
    const int p = (int)(m % HoWo);
    oy = p / a.Wo;
    ox = p % a.Wo;
  }
  pdl_sync();  // the input grid / replay slots and the packed weights come from earlier launches
  prog(3);
  const uint8_t* xrow8 = nullptr;
  const __nv_bfloat16* xrow = nullptr;
  if (row_ok) {
    if (a.first) {
      long long slot;
      if (a.idx_in) {
        slot = a.idx_in[img];  // prioritized replay (A41)
      } else if (a.ctr) {
        slot = sample_slot(a.seed, a.rank, a.ctr->T, (unsigned)img, a.ctr->ring_size);  // a1
        if (g == 0 && oy == 0 && ox == 0 && a.idx) a.idx[img] = (int)slot;
      } else {
        slot = img;  // staging buffer: image j = slot j
      }
      xrow8 = a.ring[g] + slot * a.slot_stride;  // frame-major s2d slot [frame][pixel][16]
    } else {
      xrow = a.x[g] + (long long)img * a.Hs * a.Ws * a.Cs;
    }
  }
  const __nv_bfloat16* W = a.wpk[g];
  const int SB = stage_bytes(a.N, a.first);
  __syncthreads();
  auto stage = [&](int c, int buf) {
    uint8_t* sA = smem + buf * SB;
    uint8_t* sB = sA + A_BYTES;
    const int t = c / cbn, cb = c % cbn;
    const int ty = t / a.Tw, tx = t % a.Tw;
    // A: this thread's row, 64 channels of tap t = 8 chunks -> [kc][128][8]
    if (row_ok) {
      const long long pix = (long long)(oy + ty) * a.Ws + (ox + tx);
      if (a.first) {  // 64 raw bytes of this row into the u8 area; converted once they land
        const uint8_t* src = xrow8 + pix * 16;  // 4 frames x 16 bytes = the 64 s2d channels
        uint8_t* su = sA + A_BYTES + a.N * KCH * 2 + tid * KCH;
#pragma unroll
        for (int q = 0; q < 4; ++q) cp_async16(su + 16 * q, src + (long long)q * a.Hs * a.Ws * 16);
      } else {
        const __nv_bfloat16* src = xrow + pix * a.Cs + cb * KCH;
#pragma unroll
        for (int kc = 0; kc < 8; ++kc) cp_async16(sA + (kc * 128 + tid) * 16, src + 8 * kc);
      }
    } else {
#pragma unroll
      for (int kc = 0; kc < 8; ++kc) *reinterpret_cast<uint4*>(sA + (kc * 128 + tid) * 16) = make_uint4(0, 0, 0, 0);
    }
    // B: N rows x 8 chunks of the packed [N][K] weights
    for (int e = tid; e < a.N * 8; e += 128) {
      const int n = e >> 3, kc = e & 7;
      cp_async16(sB + (kc * a.N + n) * 16, W + (long long)n * K + c * KCH + 8 * kc);
    }
    cp_async_commit();
  };
  for (int c = 0; c < NS - 1; ++c) {  // prologue: chunks 0 .. NS-2 in flight
    if (c < nch) stage(c, c);
    else cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    const int buf = c % NS, cn = c + NS - 1;
    if (cn < nch) {
      if (c >= 1) mbar_wait_bounded(&bar[(c - 1) % NS], ((c - 1) / NS) & 1, 1);  // chunk c-1 released buffer cn % NS
      stage(cn, cn % NS);
    } else {
      cp_async_commit();  // keeps one group per iteration
    }
    cp_async_wait_n<NS - 1>();  // this thread's copies of chunk c have landed
    if (a.first && row_ok) {  // this thread's own row
      uint8_t* sA = smem + buf * SB;
      const uint4* su = reinterpret_cast<const uint4*>(sA + A_BYTES + a.N * KCH * 2 + tid * KCH);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 v = su[q];
        *reinterpret_cast<uint4*>(sA + ((2 * q) * 128 + tid) * 16) = u8x8_to_bf16(v.x, v.y);
        *reinterpret_cast<uint4*>(sA + ((2 * q + 1) * 128 + tid) * 16) = u8x8_to_bf16(v.z, v.w);
      }
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + buf * SB);
      issue_chunk(tbase, sa, sa + A_BYTES, a.N, false, false, c == 0);
      mma_commit(&bar[buf]);
    }
    prog(10 + c);
  }
  mbar_wait_bounded(&bar[(nch - 1) % NS], ((nch - 1) / NS) & 1, 3);
  tc_fence_after();
  prog(100);
  // ---- epilogue: row m, N columns (tcgen05.ld is warp-collective: every lane loads, valid rows store)
  {
    const float* bias = a.bias[g];
    const float scale = a.first ? 1.0f / 255.0f : 1.0f;
    const uint32_t trow = tbase + ((uint32_t)(32 * warp) << 16);
    __nv_bfloat16* out = a.out[g];
    for (int c0 = 0; c0 < a.N; c0 += 16) {
      float v[16];
      tmem_ld16(trow + c0, v);
      if (!row_ok) continue;
      uint32_t o[8];
#pragma unroll
      for (int i = 0; i < 16; i += 2)
        o[i >> 1] = pack2(fmaxf(fmaf(v[i], scale, __ldg(bias + c0 + i)), 0.0f),
                          fmaxf(fmaf(v[i + 1], scale, __ldg(bias + c0 + i + 1)), 0.0f));
      if (a.s_next == 0) {  // canonical (C,H,W) flatten: out[img][n*HoWo + p]
        __nv_bfloat16* dst = out + (long long)img * a.N * HoWo + (long long)oy * a.Wo + ox;
        const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(o);
#pragma unroll
        for (int i = 0; i < 16; ++i) dst[(long long)(c0 + i) * HoWo] = hv[i];
      } else {  // next grid (s2d by s_next): pixel (oy/s, ox/s), channel (iy*s + ix)*N + n
        const int s = a.s_next, Wn = a.Wo / s, Cn = a.N * s * s;
        const int py = oy / s, px = ox / s, q = (oy % s) * s + (ox % s);
        if (oy < (a.Ho / s) * s && ox < Wn * s) {  // rows beyond the next grid are never read
          uint4* dst = reinterpret_cast<uint4*>(out + (((long long)img * (a.Ho / s) + py) * Wn + px) * Cn + q * a.N + c0);
          dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
          dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, tmem_cols(a.N));
}

void launch_gconv_fwd(const GConvFwdArgs& a, int groups, cudaStream_t st) {
  const long long M = (long long)a.b * a.Ho * a.Wo;
  launch_pdl(gconv_fwd_kernel, dim3((unsigned)((M + 127) / 128), groups), dim3(128), NS * stage_bytes(a.N, a.first),
             st, a);
  gconv_debug("gconv_fwd", st);
}

// ------------------------------------------------------------------ data gradient
__global__ void __launch_bounds__(128) gconv_dgrad_kernel(GConvDgradArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[NS];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int T = a.Th * a.Tw, nbn = a.N / KCH, nch = T * nbn, KT = T * a.N;
  const int HsWs = a.Hs * a.Ws;
  const long long M = (long long)a.b * HsWs;
  const long long m = (long long)blockIdx.x * 128 + tid;
  const bool row_ok = m < M;
  int img = 0, py = 0, px = 0;
  if (row_ok) {
    img = (int)(m / HsWs);
    const int p = (int)(m % HsWs);
    py = p / a.Ws;
    px = p % a.Ws;
  }
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, tmem_cols(a.Cs));
  pdl_sync();
  const int SB = stage_bytes(a.Cs, 0);
  __syncthreads();
  auto stage = [&](int c, int buf) {
    uint8_t* sA = smem + buf * SB;
    uint8_t* sB = sA + A_BYTES;
    const int t = c / nbn, nb = c % nbn;
    const int ty = t / a.Tw, tx = t % a.Tw;
    const int oy = py - ty, ox = px - tx;  // dX[i] = sum_t W_t^T dZ[i - t]
    if (row_ok && oy >= 0 && oy < a.Ho && ox >= 0 && ox < a.Wo) {
      const __nv_bfloat16* src = a.dz + (((long long)img * a.Ho + oy) * a.Wo + ox) * a.N + nb * KCH;
#pragma unroll
      for (int kc = 0; kc < 8; ++kc) cp_async16(sA + (kc * 128 + tid) * 16, src + 8 * kc);
    } else {
#pragma unroll
      for (int kc = 0; kc < 8; ++kc) *reinterpret_cast<uint4*>(sA + (kc * 128 + tid) * 16) = make_uint4(0, 0, 0, 0);
    }
    for (int e = tid; e < a.Cs * 8; e += 128) {
      const int n = e >> 3, kc = e & 7;
      cp_async16(sB + (kc * a.Cs + n) * 16, a.wpkT + (long long)n * KT + c * KCH + 8 * kc);
    }
    cp_async_commit();
  };
  for (int c = 0; c < NS - 1; ++c) {
    if (c < nch) stage(c, c);
    else cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    const int buf = c % NS, cn = c + NS - 1;
    if (cn < nch) {
      if (c >= 1) mbar_wait_bounded(&bar[(c - 1) % NS], ((c - 1) / NS) & 1, 2);
      stage(cn, cn % NS);
    } else {
      cp_async_commit();
    }
    cp_async_wait_n<NS - 1>();
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + buf * SB);
      issue_chunk(tbase, sa, sa + A_BYTES, a.Cs, false, false, c == 0);
      mma_commit(&bar[buf]);
    }
  }
  mbar_wait_bounded(&bar[(nch - 1) % NS], ((nch - 1) / NS) & 1, 3);
  tc_fence_after();
  {  // tcgen05.ld is warp-collective: every lane loads, valid rows store
    const uint32_t trow = tbase + ((uint32_t)(32 * warp) << 16);
    const __nv_bfloat16* xm = a.xmask + (long long)m * a.Cs;  // the layer input, same grid
    const int s = a.s, Cp = a.Cs / (s * s), Wp = a.Ws * s, Hp = a.Hs * s;
    for (int c0 = 0; c0 < a.Cs; c0 += 16) {
      float v[16];
      tmem_ld16(trow + c0, v);
      if (!row_ok) continue;
      const uint4 mk0 = *reinterpret_cast<const uint4*>(xm + c0), mk1 = *reinterpret_cast<const uint4*>(xm + c0 + 8);
      const uint32_t mw[8] = {mk0.x, mk0.y, mk0.z, mk0.w, mk1.x, mk1.y, mk1.z, mk1.w};
      uint32_t o[8];
#pragma unroll
      for (int h = 0; h < 8; ++h)
        o[h] = pack2(bf16_pos(mw[h] & 0xFFFFu) ? v[2 * h] : 0.0f, bf16_pos(mw[h] >> 16) ? v[2 * h + 1] : 0.0f);
      // c' = (iy*s + ix)*Cp + c  ->  previous layer's output pixel (py*s + iy, px*s + ix), channel c
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int cc = c0 + 8 * half, q = cc / Cp, ch = cc % Cp;
        const int y = py * s + q / s, x = px * s + q % s;
        uint4* dst = reinterpret_cast<uint4*>(a.dzprev + (((long long)img * Hp + y) * Wp + x) * Cp + ch);
        *dst = make_uint4(o[4 * half], o[4 * half + 1], o[4 * half + 2], o[4 * half + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, tmem_cols(a.Cs));
}

void launch_gconv_dgrad(const GConvDgradArgs& a, cudaStream_t st) {
  const long long M = (long long)a.b * a.Hs * a.Ws;
  launch_pdl(gconv_dgrad_kernel, dim3((unsigned)((M + 127) / 128)), dim3(128), NS * stage_bytes(a.Cs, 0), st, a);
  gconv_debug("gconv_dgrad", st);
}

// ------------------------------------------------------------------ weight gradient
__global__ void __launch_bounds__(128) gconv_wgrad_kernel(GConvWgradArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[NS];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int T = a.Th * a.Tw, HoWo = a.Ho * a.Wo, MK = T * a.Cs;
  const int m0 = blockIdx.x * 128, range = blockIdx.y;
  const int img0 = range * a.ipc, nimg = min(a.ipc, a.b - img0);
  const int npos = nimg * HoWo, nch = (npos + KCH - 1) / KCH;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, tmem_cols(a.N));
  pdl_sync();
  const int SB = stage_bytes(a.N, a.first);
  const int U8OFF = A_BYTES + a.N * KCH * 2;  // layer 1's raw pieces inside a stage
  __syncthreads();
  const int ng = a.N / 8;
  // source offset of every position q of this image range (tap 0, c' = 0), computed once: the
  // staging loops below then need no integer division
  long long* s_pos = reinterpret_cast<long long*>(smem + NS * SB);
  {
    // layer 1: frame-major s2d replay slot [frame][pixel][16]; later layers: [pixel][Cs]
    const long long grid = (long long)a.Hs * a.Ws * a.Cs;
    const int pstride = a.first ? 16 : a.Cs;
    for (int q = tid; q < npos; q += 128) {
      const int im = img0 + q / HoWo, p = q % HoWo;
      const long long base = a.first ? (long long)a.idx[im] * a.slot_stride : (long long)im * grid;
      s_pos[q] = base + ((long long)(p / a.Wo) * a.Ws + (p % a.Wo)) * pstride;
    }
  }
  // this thread's fixed A row group (tid % 16) and tap, fixed B column group (tid % ng)
  const int gi_a = tid % 16, k0_a = tid / 16, r_a = m0 + 8 * gi_a;
  const bool r_ok = r_a < MK;
  const int t_a = r_ok ? r_a / a.Cs : 0, cc_a = r_ok ? r_a % a.Cs : 0;
  const long long tapoff =
      a.first ? ((long long)(t_a / a.Tw) * a.Ws + (t_a % a.Tw)) * 16 + (long long)(cc_a / 16) * a.Hs * a.Ws * 16 + cc_a % 16
              : ((long long)(t_a / a.Tw) * a.Ws + (t_a % a.Tw)) * a.Cs + cc_a;
  const int gi_b = tid % ng, k0_b = tid / ng, kstep_b = 128 / ng;
  const __nv_bfloat16* dzr = a.dz + (long long)img0 * HoWo * a.N + 8 * gi_b;
  __syncthreads();
  // db (m-tile 0 CTAs): column sums of dZ over this range. Thread tid always sees column group
  // tid % ng of the staged B chunks (128 % ng == 0) and keeps 8 running sums; combined at the end
  float dbacc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  auto stage = [&](int c, int buf) {
    uint8_t* sA = smem + buf * SB;
    uint8_t* sB = sA + A_BYTES;
    // A MN-major [16 row groups][64 k][8]: rows (tap, c'), k = position of this chunk; piece
    // e = tid + 128 j is (row group tid % 16, k = tid / 16 + 8 j)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = k0_a + 8 * j, q = c * KCH + k;
      uint8_t* d = sA + (gi_a * KCH + k) * 16;
      if (q < npos && r_ok) {
        const long long off = s_pos[q] + tapoff;
        if (a.first) cp_async8(sA + U8OFF + (tid + 128 * j) * 8, a.ring + off);  // converted after the wait
        else cp_async16(d, a.x + off);
      } else {
        *reinterpret_cast<uint4*>(d) = make_uint4(0, 0, 0, 0);
      }
    }
    // B MN-major [N/8][64 k][8]: dZ rows of the range are contiguous (position-major NHWC)
    for (int k = k0_b; k < KCH; k += kstep_b) {
      const int q = c * KCH + k;
      uint8_t* d = sB + (gi_b * KCH + k) * 16;
      if (q < npos) cp_async16(d, dzr + (long long)q * a.N);
      else *reinterpret_cast<uint4*>(d) = make_uint4(0, 0, 0, 0);
    }
    cp_async_commit();
  };
  for (int c = 0; c < NS - 1; ++c) {
    if (c < nch) stage(c, c);
    else cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    const int buf = c % NS, cn = c + NS - 1;
    if (cn < nch) {
      if (c >= 1) mbar_wait_bounded(&bar[(c - 1) % NS], ((c - 1) / NS) & 1, 2);
      stage(cn, cn % NS);
    } else {
      cp_async_commit();
    }
    cp_async_wait_n<NS - 1>();
    if (a.first && r_ok) {  // convert the pieces this thread copied (same sequence as the stage)
      uint8_t* sA = smem + buf * SB;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = k0_a + 8 * j;
        if (c * KCH + k < npos) {
          const uint2 v = *reinterpret_cast<const uint2*>(sA + U8OFF + (tid + 128 * j) * 8);
          *reinterpret_cast<uint4*>(sA + (gi_a * KCH + k) * 16) = u8x8_to_bf16(v.x, v.y);
        }
      }
    }
    fence_async_smem();
    __syncthreads();
    if (blockIdx.x == 0) {  // db: 16-byte rows of the B chunk, 8 columns at a time
      const uint8_t* sB = smem + buf * SB + A_BYTES;
      for (int e = tid; e < ng * KCH; e += 128) {
        const int gi = e % ng, k = e / ng;
        const uint4 v = *reinterpret_cast<const uint4*>(sB + (gi * KCH + k) * 16);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          dbacc[2 * h] += __uint_as_float(w[h] << 16);
          dbacc[2 * h + 1] += __uint_as_float(w[h] & 0xFFFF0000u);
        }
      }
    }
    if (tid == 0) {
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + buf * SB);
      issue_chunk(tbase, sa, sa + A_BYTES, a.N, true, true, c == 0);
      mma_commit(&bar[buf]);
    }
  }
  if (nch > 0) {
    mbar_wait_bounded(&bar[(nch - 1) % NS], ((nch - 1) / NS) & 1, 3);
    tc_fence_after();
  }
  // ---- partial[range][row][n]
  const int r = m0 + 32 * warp + (tid & 31);
  float* prow = a.partial + ((long long)range * MK + r) * a.N;
  const uint32_t trow = tbase + ((uint32_t)(32 * warp) << 16);
  for (int c0 = 0; c0 < a.N; c0 += 16) {
    float v[16];
    if (nch > 0) tmem_ld16(trow + c0, v);
    else
      for (int i = 0; i < 16; ++i) v[i] = 0.0f;
    if (r < MK) {
#pragma unroll
      for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(prow + c0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    }
  }
  if (blockIdx.x == 0) {  // combine the per-thread sums of each column group in thread order
    float* s_db = reinterpret_cast<float*>(smem);  // the stage buffers are free (all MMAs done)
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 8; ++i) s_db[tid * 8 + i] = dbacc[i];
    __syncthreads();
    if (tid < a.N) {
      const int gi = tid / 8, i = tid % 8;
      float t = 0.0f;
      for (int u = gi; u < 128; u += ng) t += s_db[u * 8 + i];
      a.partial_db[(long long)range * a.N + tid] = t;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, tmem_cols(a.N));
}

// G[canonical] (+)= sum over the ranges of the partials (x 1/255 on layer 1's W). Block = 32
// consecutive entries x 8 range groups: each group sums its ranges in order, then the 8 group sums
// are added in group order (a fixed order: deterministic).
__global__ void __launch_bounds__(256) gconv_wreduce_kernel(GConvWgradArgs a) {
  pdl_sync();
  const int T = a.Th * a.Tw, MK = T * a.Cs;
  const long long nw = (long long)MK * a.N, total = nw + a.N;
  const int el = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const long long e = blockIdx.x * 32LL + el;
  const int nr = (a.b + a.ipc - 1) / a.ipc, per = (nr + 7) / 8;
  const int q0 = grp * per, q1 = min(nr, q0 + per);
  float s = 0.0f;
  // part_cm: e enumerates (n, row) with the row fastest, the column-major partials' order (coalesced reads)
  if (e < total) {  // 8 loads in flight per round, summed in range order
    const float* src = e < nw ? a.partial + e : a.partial_db + (e - nw);
    const long long stride = e < nw ? nw : a.N;
    for (int q = q0; q < q1; q += 8) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = q + k < q1 ? __ldcg(src + (long long)(q + k) * stride) : 0.0f;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (q + k < q1) s += v[k];
    }
  }
  __shared__ float red[8][32];
  red[grp][el] = s;
  __syncthreads();
  if (grp != 0 || e >= total) return;
  float t = 0.0f;
#pragma unroll
  for (int g = 0; g < 8; ++g) t += red[g][el];
  long long dst;
  if (e < nw) {
    const int row = a.part_cm ? (int)(e % MK) : (int)(e / a.N), n = a.part_cm ? (int)(e / MK) : (int)(e % a.N);
    if (a.first) t *= 1.0f / 255.0f;
    if (a.w_canon[row] < 0) return;
    dst = a.w_off + (long long)n * a.w_nstride + a.w_canon[row];
  } else {
    dst = a.b_off + (e - nw);
  }
  if (a.store) a.grad[dst] = t;
  else a.grad[dst] += t;
}

// dynamic shared memory of a weight-gradient CTA: the stage ring plus the position table of its images
static int gconv_wgrad_smem(int N, int first, int ipc, int HoWo) {
  return NS * stage_bytes(N, first) + (ipc * HoWo * 8 + 1023) / 1024 * 1024;
}
static int g_wgrad_smem_cap = 0;  // the kernel's dynamic shared-memory attribute (init_conv_kernel_attrs)
bool gconv_wgrad_fits(int N, int first, int ipc, int HoWo) {
  return gconv_wgrad_smem(N, first, ipc, HoWo) <= g_wgrad_smem_cap;
}

void launch_gconv_wreduce(const GConvWgradArgs& a, cudaStream_t st) {
  const long long n = (long long)a.Th * a.Tw * a.Cs * a.N + a.N;
  launch_pdl(gconv_wreduce_kernel, dim3((unsigned)((n + 31) / 32)), dim3(256), 0, st, a);
  gconv_debug("gconv_wreduce", st);
}

void launch_gconv_wgrad(const GConvWgradArgs& a, cudaStream_t st) {
  const int T = a.Th * a.Tw, MK = T * a.Cs;
  const int ranges = (a.b + a.ipc - 1) / a.ipc;
  launch_pdl(gconv_wgrad_kernel, dim3((MK + 127) / 128, ranges), dim3(128),
             gconv_wgrad_smem(a.N, a.first, a.ipc, a.Ho * a.Wo), st, a);
  gconv_debug("gconv_wgrad", st);
  const long long n = (long long)MK * a.N + a.N;
  launch_pdl(gconv_wreduce_kernel, dim3((unsigned)((n + 31) / 32)), dim3(256), 0, st, a);
  gconv_debug("gconv_wreduce", st);
}

__global__ void __launch_bounds__(128) gemm_pipe_kernel(TcGemmArgs a);

// the recorded lost-MMA-completion word (0: none), read after a synchronisation
unsigned long long gconv_error() {
  unsigned long long e = 0;
  cudaMemcpyFromSymbol(&e, g_gconv_err, sizeof(e));
  return e;
}

void init_conv_kernel_attrs() {
  // the 227 KB opt-in limit includes each kernel's static shared memory
  auto set = [](const void* f, bool full) {
    cudaFuncAttributes at{};
    cudaFuncGetAttributes(&at, f);
    const int cap = 227 * 1024 - (int)at.sharedSizeBytes - 1024;
    const int mx = full ? cap : std::min<int>(GCONV_SMEM_MAX, cap);
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    return mx;
  };
  set((const void*)gconv_fwd_kernel, false);
  set((const void*)gconv_dgrad_kernel, false);
  g_wgrad_smem_cap = set((const void*)gconv_wgrad_kernel, true);  // the ring + the position table
  set((const void*)gemm_pipe_kernel, false);
}

// ------------------------------------------------------------------ pipelined GEMM (generic path FC layers)
// D[m][n] = sum_k A(m,k) B(n,k) over this CTA's K split, in chunks of 64 through the stage ring
// (K-major or MN-major operands as flagged), with the epilogues the FC layers need:
//   TC_EPI_ACCUM + store : C[m*ldc + n] = D           (FC dW, n_push = 1)
//   TC_EPI_ACCUM         : C[m*ldc + n] += D
//   TC_EPI_MASK_T        : out[n*ldo + m'] = mask[n*ldo + m] > 0 ? D : 0, m' = NHWC remap (FC dX)
//   TC_EPI_FC_FWD        : partial[g][split][n][m] = D    (FC forward, reduced by the TD head)
__global__ void __launch_bounds__(128) gemm_pipe_kernel(TcGemmArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[NS];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = blockIdx.z, split = blockIdx.y;
  const int m_tiles = (a.M + 127) / 128;
  const int mt = blockIdx.x % m_tiles, nt = blockIdx.x / m_tiles;
  const int m0 = mt * 128, n0 = nt * a.BN, bn = a.BN;
  const int k0 = split * a.kper, KC = min(a.kper, a.K - k0), nch = (KC + KCH - 1) / KCH;  // KC % 16 == 0
  const int SB = ((A_BYTES + bn * KCH * 2) + 1023) / 1024 * 1024;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, tmem_cols(bn));
  pdl_sync();
  __syncthreads();
  const __nv_bfloat16* Ag = a.A[g];
  const __nv_bfloat16* Bg = a.B[g];
  const uint4 z4 = make_uint4(0, 0, 0, 0);
  auto stage = [&](int c, int buf) {
    uint8_t* sA = smem + buf * SB;
    uint8_t* sB = sA + A_BYTES;
    const int kb = k0 + c * KCH, klen = min(KCH, KC - c * KCH);  // the last chunk may be short
    if (!a.a_mn) {  // [kc][128][8]
      for (int e = tid; e < 128 * 8; e += 128) {
        const int r = e >> 3, kc = e & 7, m = m0 + r;
        uint8_t* d = sA + (kc * 128 + r) * 16;
        if (m < a.M && 8 * kc < klen) cp_async16(d, Ag + (long long)m * a.lda + kb + 8 * kc);
        else *reinterpret_cast<uint4*>(d) = z4;
      }
    } else {        // [16][64 k][8]
      for (int e = tid; e < 16 * KCH; e += 128) {
        const int gi = e & 15, k = e >> 4, m = m0 + 8 * gi;
        uint8_t* d = sA + (gi * KCH + k) * 16;
        if (m < a.M && k < klen) cp_async16(d, Ag + (long long)(kb + k) * a.lda + m);
        else *reinterpret_cast<uint4*>(d) = z4;
      }
    }
    if (!a.b_mn) {  // [kc][bn][8]
      for (int e = tid; e < bn * 8; e += 128) {
        const int r = e >> 3, kc = e & 7, n = n0 + r;
        uint8_t* d = sB + (kc * bn + r) * 16;
        if (n < a.N && 8 * kc < klen) cp_async16(d, Bg + (long long)n * a.ldb + kb + 8 * kc);
        else *reinterpret_cast<uint4*>(d) = z4;
      }
    } else {        // [bn/8][64 k][8]
      const int ng = bn / 8;
      for (int e = tid; e < ng * KCH; e += 128) {
        const int gi = e % ng, k = e / ng, n = n0 + 8 * gi;
        uint8_t* d = sB + (gi * KCH + k) * 16;
        if (n < a.N && k < klen) cp_async16(d, Bg + (long long)(kb + k) * a.ldb + n);
        else *reinterpret_cast<uint4*>(d) = z4;
      }
    }
    cp_async_commit();
  };
  for (int c = 0; c < NS - 1; ++c) {
    if (c < nch) stage(c, c);
    else cp_async_commit();
  }
  for (int c = 0; c < nch; ++c) {
    const int buf = c % NS, cn = c + NS - 1;
    if (cn < nch) {
      if (c >= 1) mbar_wait_bounded(&bar[(c - 1) % NS], ((c - 1) / NS) & 1, 4);
      stage(cn, cn % NS);
    } else {
      cp_async_commit();
    }
    cp_async_wait_n<NS - 1>();
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + buf * SB);
      issue_chunk(tbase, sa, sa + A_BYTES, bn, a.a_mn, a.b_mn, c == 0, (min(KCH, KC - c * KCH) + 15) / 16);
      mma_commit(&bar[buf]);
    }
  }
  mbar_wait_bounded(&bar[(nch - 1) % NS], ((nch - 1) / NS) & 1, 5);
  tc_fence_after();
  const int m = m0 + 32 * warp + lane;
  const uint32_t trow = tbase + ((uint32_t)(32 * warp) << 16);
  for (int c = 0; c < bn; c += 16) {
    float v[16];
    tmem_ld16(trow + c, v);  // warp-collective: every lane loads
    if (m >= a.M) continue;
    if (a.epi == TC_EPI_ACCUM) {
      float* crow = a.C[g] + (long long)m * a.ldc + n0 + c;
      for (int i = 0; i < 16 && n0 + c + i < a.N; ++i) crow[i] = a.store ? v[i] : crow[i] + v[i];
    } else if (a.epi == TC_EPI_MASK_T) {
      const long long om = a.hwc_HW ? (long long)(m % a.hwc_HW) * a.hwc_C + m / a.hwc_HW : (long long)m;
      unsigned short mk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int n = n0 + c + i;
        mk[i] = n < a.N ? __ldg(reinterpret_cast<const unsigned short*>(a.mask) + (long long)n * a.ldo + m) : 0;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int n = n0 + c + i;
        if (n < a.N) a.out_bf16[(long long)n * a.ldo + om] = __float2bfloat16_rn(bf16_pos(mk[i]) ? v[i] : 0.0f);
      }
    } else {  // TC_EPI_FC_FWD
      float* pbase = a.partial + ((long long)g * a.splits + split) * (long long)a.N * a.M;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (n0 + c + i < a.N) pbase[(long long)(n0 + c + i) * a.M + m] = v[i];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, tmem_cols(bn));
}

void launch_gemm_pipe(const TcGemmArgs& a, int groups, cudaStream_t st) {
  const int m_tiles = (a.M + 127) / 128, n_tiles = (a.N + a.BN - 1) / a.BN;
  const int SB = ((A_BYTES + a.BN * KCH * 2) + 1023) / 1024 * 1024;
  launch_pdl(gemm_pipe_kernel, dim3(m_tiles * n_tiles, a.splits, groups), dim3(128), NS * SB, st, a);
  gconv_debug("gemm_pipe", st);
}

// ------------------------------------------------------------------ TD head finish, one warp per element
// The cross-sample sums of head_finish.cuh for large b: lane l sums samples j = l, l+32, ... in
// ascending order, then the 32 lane sums combine in a fixed shuffle tree (deterministic).
// The cross-sample sums of the TD head (head_finish.cuh's elements), coalesced over 32 consecutive outputs:
//   dW_o[a][u0 .. u0+31] : a warp per (a, u0) walks the samples in ascending j; the samples with a_j = a (found
//                          with ballots over the actions staged in shared memory) are batched 8 at a time, so 8
//                          coalesced 128-byte row loads h_j[u0 .. u0+31] are in flight; summed in j order
//   db_fc[u0 .. u0+31]   : a CTA per u0: warp k sums samples [k b/8, (k+1) b/8) of dH with 8 loads in flight,
//                          then the 8 partial sums are added in warp order
//   db_o[a], loss, T + 1 : the last CTA, a warp per output, lanes over the samples, butterfly (fixed order)
// (a warp per output element reading h_j[u] for 32 samples at once touched 32 lines per load)
__global__ void __launch_bounds__(256) head_finish_warp_kernel(HeadArgs h) {
  extern __shared__ float hf_sm[];  // [b] dQ_j | [b] a_j
  __shared__ float s_part[8][32];
  float* s_dq = hf_sm;
  int* s_act = reinterpret_cast<int*>(hf_sm + h.b);
  pdl_sync();
  for (int j = threadIdx.x; j < h.b; j += blockDim.x) {
    s_dq[j] = h.s_dq[j];
    s_act[j] = h.s_act[j];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int H = h.H, A = h.A, UB = (H + 31) / 32, cw = (A * UB + 7) / 8;  // CTAs of dW_o warps
  const float* h0 = h.fc_partial ? h.act_out[0] : h.act[0];
  if ((int)blockIdx.x < cw) {  // dW_o rows
    const int w = blockIdx.x * 8 + warp;
    if (w >= A * UB) return;
    const int a = w / UB, u = (w % UB) * 32 + lane, uc = u < H ? u : H - 1;
    float s = 0.0f;
    int js[8], n = 0;
    auto flush = [&]() {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = k < n ? h0[(long long)js[k] * H + uc] : 0.0f;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < n) s = fmaf(s_dq[js[k]], v[k], s);
      n = 0;
    };
    for (int j0 = 0; j0 < h.b; j0 += 32) {
      unsigned m = __ballot_sync(0xffffffffu, j0 + lane < h.b && s_act[j0 + lane] == a);
      while (m) {
        const int j = j0 + __ffs(m) - 1;
        m &= m - 1;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k == n) js[k] = j;
        if (++n == 8) flush();
      }
    }
    if (n) flush();
    if (u < H) h.grad[h.w_off + (long long)a * H + u] += s;
    return;
  }
  const int cb = (int)blockIdx.x - cw;
  if (cb < UB) {  // db of the previous FC layer, u block cb
    if (!h.prev_is_fc) return;
    const int u = cb * 32 + lane, uc = u < H ? u : H - 1;
    const int per = (h.b + 7) / 8, j_lo = warp * per, j_hi = min(h.b, j_lo + per);
    float s = 0.0f;
    for (int j0 = j_lo; j0 < j_hi; j0 += 8) {
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = j0 + k < j_hi ? h.dH[(long long)(j0 + k) * H + uc] : 0.0f;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (j0 + k < j_hi) s += v[k];
    }
    s_part[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && u < H) {
      float t = s_part[0][lane];
      for (int k = 1; k < 8; ++k) t += s_part[k][lane];
      h.grad[h.prev_b_off + u] += t;
    }
    return;
  }
  // the last CTA: db_o[a] for a < A, then the loss (warp per output, outputs strided over the 8 warps)
  for (int o = warp; o <= A; o += 8) {
    float s = 0.0f;
    if (o < A) {
      for (int j = lane; j < h.b; j += 32)
        if (s_act[j] == o) s += s_dq[j];
    } else {
      for (int j = lane; j < h.b; j += 32) s += h.s_loss[j];
    }
#pragma unroll
    for (int q = 16; q > 0; q >>= 1) s += __shfl_xor_sync(0xffffffffu, s, q);
    if (lane == 0) {
      if (o < A) {
        h.grad[h.b_off + o] += s;
      } else {
        const unsigned long long T = h.ctr->T;
        h.diag_loss[T % kDiagSteps] = s / (float)h.b;
        h.ctr->T = T + 1;  // this step is complete for the sampler
      }
    }
  }
}

void launch_head_finish_warp(const HeadArgs& h, cudaStream_t st) {
  const int UB = (h.H + 31) / 32, ctas = (h.A * UB + 7) / 8 + UB + 1;
  launch_pdl(head_finish_warp_kernel, dim3(ctas), dim3(256), (size_t)h.b * 8, st, h);
  gconv_debug("head_finish_warp", st);
}

// ------------------------------------------------------------------ packed weight images
// dst[img_off + map[i].x] (and .y) = bf16(theta[i]) for the conv parameters i < n (map < 0: none)
__global__ void gpack_kernel(const float* theta, __nv_bfloat16* dst, long long img_off, const int2* map, long long n) {
  pdl_sync();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int2 d = map[i];
  if (d.x < 0 && d.y < 0) return;
  const __nv_bfloat16 v = __float2bfloat16_rn(theta[i]);
  if (d.x >= 0) dst[img_off + d.x] = v;
  if (d.y >= 0) dst[img_off + d.y] = v;
}

void launch_gpack(const float* theta, __nv_bfloat16* dst, long long img_off, const int2* map, long long n,
                  cudaStream_t st) {
  if (n <= 0) return;
  launch_pdl(gpack_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, theta, dst, img_off, map, n);
  gconv_debug("gpack", st);
}

}  // namespace dqn
