// kernels_tma.cu — warp-specialised, persistent tcgen05 GEMM fed by TMA (the FC layers of the large-batch
// configurations, a5 / a7: BASELINE.json configs[3] and [4]).
//
//   D[m][n] = sum_k A(m, k) B(n, k), one 128 x BN output tile per (group, m-tile, n-tile, k-split);
//   A and B are 2-D bf16 tensors read by TMA (cp.async.bulk.tensor) in 64-element boxes with the 128-byte
//   swizzle, i.e. directly in the UMMA SW128 canonical layouts: K-major boxes [rows][64 k] or MN-major
//   boxes [64 k][64 mn] (two / BN/64 of them per stage).
//
// Roles (192 threads): warp 0 = TMA producer (one thread), warp 1 = MMA issuer (one thread; it also owns the
// TMEM allocation), warps 2..5 = epilogue (128 threads = the 128 TMEM lanes: warp w reads lanes 32 (w % 4) ..).
// A ring of `stages` shared-memory stages (full / empty mbarriers) and TWO TMEM accumulators (tfull / tempty):
// the epilogue of tile i overlaps the MMAs of tile i + 1, and a persistent CTA walks tiles
// blockIdx.x, blockIdx.x + gridDim.x, ...
//
// Epilogues (TcGemmArgs semantics, kernels_bf16.cu):
//   TC_EPI_FC_FWD : partial[g][split][n][m] = D            (split-K partials; the TD head reduces them)
//   TC_EPI_ACCUM  : C[g][m * ldc + n] = D (store) or += D   (FC dW into G)
//   TC_EPI_MASK_T : out[n * ldo + m'] = mask[n * ldo + m] > 0 ? D : 0, m' = NHWC remap (FC dX, ReLU')
//   TC_EPI_ACCUM_T: C[g][n * ldc + m] = D or += D                  (FC dW computed as dW^T: coalesced stores)
#include <cuda.h>  // CUtensorMap and the encode entry point's types (fetched from the driver at run time)

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "dqn_internal.h"
#include "pdl.cuh"
#include "philox.cuh"
#include "sm100.cuh"

namespace dqn {
using namespace dqn_sm100;

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn f = nullptr;
  if (!f) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = reinterpret_cast<EncodeTiledFn>(p);
  }
  return f;
}

// ---- warp-uniform issue: the producer and MMA roles run on a WHOLE warp with warp-uniform values, and the
// one-thread instructions (TMA, MMA, commit, expect-tx) carry their own elect.sync inside the asm. Issued from
// under `if (lane == 0)` instead, every tcgen05.mma / TMA operand goes through a per-lane R2UR loop
// (measured: ~110 cycles per MMA, ~1800 cycles per 16-MMA convolution tile of pure issue overhead).
// mma_bf16_w / mma_commit_w live in sm100.cuh (the per-image kernels use them too).
__device__ __forceinline__ void tma_load_2d_w(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "{ .reg .pred e; elect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4]; }" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_w(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{ .reg .pred e; elect.sync _|e, 0xffffffff;\n"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1; }" ::"r"(smem_u32(bar)), "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_w(uint64_t* bar) {
  asm volatile(
      "{ .reg .pred e; elect.sync _|e, 0xffffffff;\n"
      "@e mbarrier.arrive.shared::cta.b64 _, [%0]; }" ::"r"(smem_u32(bar))
      : "memory");
}
constexpr unsigned kEpiSpinNs = 64;  // back-off of the epilogue warps' polling lane (the producer / MMA spin freely)
// spin on mbarrier.test_wait (never suspends: the pipelines here hand off every few hundred cycles, and a
// suspended try_wait was measured to add ~1 us per hand-off on short convolution tiles)
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  while (true) {
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) break;
  }
}
// the epilogue warps' wait: one lane polls (with a short back-off), the warp then proceeds together, so eight
// waiting warps do not flood the shared-memory pipe the producer and MMA threads hand off through
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  if ((threadIdx.x & 31) == 0) {
    uint32_t done;
    while (true) {
      asm volatile(
          "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(bar)), "r"(parity)
          : "memory");
      if (done) break;
      __nanosleep(kEpiSpinNs);
    }
  }
  __syncwarp();
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// UMMA shared-memory descriptor with the 128-byte swizzle (layout type 2, Blackwell version 1)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ bool bf16_gt0(unsigned short h) { return (h & 0x8000u) == 0 && h != 0; }

constexpr int TG_THREADS = 192;
constexpr int TG_A_BYTES = 128 * 64 * 2;  // one A stage: 128 rows x 64 k (or 64 k x 2 x 64 m)

}  // namespace

// DQN_SYNC_DEBUG=1 (with DQN_NO_GRAPH=1): synchronise after every launch of this file and name the first
// kernel that faults
static void sync_debug(const char* what, cudaStream_t st) {
  static const int on = getenv("DQN_SYNC_DEBUG") ? atoi(getenv("DQN_SYNC_DEBUG")) : 0;
  if (!on) return;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  fprintf(stderr, "[sync debug] %s: %s\n", what, cudaGetErrorString(e));
  if (e != cudaSuccess) exit(3);
}

// A 2-D bf16 tensor [rows][cols] (cols contiguous, row pitch ld elements) read in boxes of box_rows x 64
// columns with the 128-byte swizzle. Returns false when the driver entry point is missing or refuses.
bool make_tmap_bf16(CUtensorMap* m, const void* base, long long rows, long long cols, long long ld, int box_rows) {
  EncodeTiledFn f = encode_fn();
  if (!f || (ld * 2) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return f(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__global__ void __launch_bounds__(TG_THREADS, 2) tgemm_kernel(const __grid_constant__ TGemmArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kTgMaxStages], empty[kTgMaxStages], tfull[2], tempty[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = a.stages, BN = a.BN;
  const int B_BYTES = BN * 64 * 2, STAGE = TG_A_BYTES + B_BYTES;
  const uint32_t tcols = BN <= 16 ? 32 : BN <= 32 ? 64 : BN <= 64 ? 128 : BN <= 128 ? 256 : 512;  // 2 accumulators
  const int m_tiles = (a.M + 127) / 128, n_tiles = (a.N + BN - 1) / BN;
  const int tiles = m_tiles * n_tiles * a.splits * a.groups;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tbase, tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_sync();  // operands come from the immediate predecessor; outputs may still be read by it
  auto decode = [&](int t, int& g, int& split, int& m0, int& n0) {
    const int mt = t % m_tiles;
    t /= m_tiles;
    const int nt = t % n_tiles;
    t /= n_tiles;
    split = t % a.splits;
    g = t / a.splits;
    m0 = mt * 128;
    n0 = nt * BN;
  };
  auto n_chunks = [&](int split) { return (min(a.kper, a.K - split * a.kper) + 63) / 64; };

  if (warp == 0) {
    {  // ---- TMA producer (whole warp, warp-uniform; one elected lane issues)
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int g, split, m0, n0;
        decode(t, g, split, m0, n0);
        const int nch = n_chunks(split);
        for (int c = 0; c < nch; ++c, ++it) {
          const int s = it % S;
          mbar_spin(&empty[s], ((it / S) & 1) ^ 1);
          uint8_t* sA = smem + s * STAGE;
          uint8_t* sB = sA + TG_A_BYTES;
          mbar_expect_tx_w(&full[s], STAGE);
          const int kb = split * a.kper + c * 64;
          if (!a.a_mn) {
            tma_load_2d_w(sA, &a.ta[g], kb, m0, &full[s]);
          } else {
            tma_load_2d_w(sA, &a.ta[g], m0, kb, &full[s]);
            tma_load_2d_w(sA + 8192, &a.ta[g], m0 + 64, kb, &full[s]);
          }
          if (!a.b_mn) {
            tma_load_2d_w(sB, &a.tb[g], kb, n0, &full[s]);
          } else {
            for (int j = 0; j < BN / 64; ++j) tma_load_2d_w(sB + j * 8192, &a.tb[g], n0 + 64 * j, kb, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // ---- MMA issuer (whole warp, warp-uniform; one elected lane issues)
      const uint32_t idesc = make_idesc_bf16(128, BN, a.a_mn, a.b_mn);
      int it = 0, tl = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
        int g, split, m0, n0;
        decode(t, g, split, m0, n0);
        const int nch = n_chunks(split);
        const int buf = tl & 1;
        mbar_spin(&tempty[buf], ((tl >> 1) & 1) ^ 1);  // the epilogue has drained this accumulator
        tc_fence_after();
        const uint32_t d = tbase + (uint32_t)(buf * BN);
        for (int c = 0; c < nch; ++c, ++it) {
          const int s = it % S;
          mbar_spin(&full[s], (it / S) & 1);
          // (TMA data: async proxy to async proxy, ordered by the mbarrier; no tcgen05 fence)
          const uint32_t sa = smem_u32(smem + s * STAGE), sb = sa + TG_A_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            // K-major: +32 B per K step inside the swizzled 128-B rows; MN-major: +16 rows of 128 B
            const uint64_t ad = a.a_mn ? desc_sw128(sa + kk * 2048, 8192, 1024) : desc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t bd = a.b_mn ? desc_sw128(sb + kk * 2048, 8192, 1024) : desc_sw128(sb + kk * 32, 16, 1024);
            mma_bf16_w(d, ad, bd, idesc, (c > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit_w(&empty[s]);  // the stage is free once these MMAs have read it
        }
        mma_commit_w(&tfull[buf]);
      }
    }
  } else {  // ---- epilogue: thread = one row (TMEM lane) of the tile
    const int q = warp & 3;
    int tl = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
      int g, split, m0, n0;
      decode(t, g, split, m0, n0);
      const int buf = tl & 1;
      const int m = m0 + 32 * q + lane;
      // TC_EPI_MASK_T: the ReLU mask of the next 16 columns is always in flight (the first batch before the
      // accumulator wait, so it overlaps the mainloop)
      unsigned short mkn[16];
      auto load_mask = [&](int c0) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = n0 + c0 + i;
          mkn[i] = (n < a.N && m < a.M) ? __ldg(reinterpret_cast<const unsigned short*>(a.mask) + (long long)n * a.ldo + m)
                                        : (unsigned short)0;
        }
      };
      if (a.epi == TC_EPI_MASK_T) load_mask(0);
      mbar_wait_warp(&tfull[buf], (tl >> 1) & 1);
      tc_fence_after();
      const uint32_t trow = tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * BN);
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        tmem_ld16(trow + c, v);  // warp-collective
        unsigned short mk[16];
        if (a.epi == TC_EPI_MASK_T) {
#pragma unroll
          for (int i = 0; i < 16; ++i) mk[i] = mkn[i];
          if (c + 16 < BN) load_mask(c + 16);
        }
        if (m >= a.M) continue;
        if (a.epi == TC_EPI_FC_FWD) {
          float* p = a.partial + ((long long)g * a.splits + split) * (long long)a.N * a.M + m;
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (n0 + c + i < a.N) p[(long long)(n0 + c + i) * a.M] = v[i];
        } else if (a.epi == TC_EPI_ACCUM) {
          float* crow = a.C[g] + (long long)m * a.ldc + n0 + c;
          if (n0 + c + 16 <= a.N && a.store) {
#pragma unroll
            for (int i = 0; i < 16; i += 4)
              *reinterpret_cast<float4*>(crow + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)  // (unrolled: v[] must stay in registers)
              if (n0 + c + i < a.N) crow[i] = a.store ? v[i] : crow[i] + v[i];
          }
        } else if (a.epi == TC_EPI_ACCUM_T) {  // C[n][m]: the warp's 32 rows are 128 contiguous bytes per column
          float* ccol = a.C[g] + m;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int n = n0 + c + i;
            if (n < a.N) {
              float* p = ccol + (long long)n * a.ldc;
              *p = a.store ? v[i] : *p + v[i];
            }
          }
        } else {  // TC_EPI_MASK_T: all 16 mask loads in flight before the (possibly aliasing) stores
          long long om = m;
          if (a.hwc_HW) {
            const int pp = m % a.hwc_HW, cc = m / a.hwc_HW;
            om = a.hwc_Ws ? ((long long)(pp / a.hwc_Wo) * a.hwc_Ws + pp % a.hwc_Wo) * a.hwc_C + cc
                          : (long long)pp * a.hwc_C + cc;
          }
          const long long ldo_out = a.ldo_out ? a.ldo_out : a.ldo;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int n = n0 + c + i;
            if (n < a.N) a.out_bf16[(long long)n * ldo_out + om] = __float2bfloat16_rn(bf16_gt0(mk[i]) ? v[i] : 0.0f);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, tcols);
}

// CTAs per SM (1: one persistent CTA with the deepest ring; 2: two CTAs with half the ring each, so that one
// CTA's TMA latency overlaps the other's MMAs and epilogue on small GEMMs) and the stage count that fits
static int tg_ctas_per_sm(int BN) {
  static const int env = getenv("DQN_TG_CTAS") ? atoi(getenv("DQN_TG_CTAS")) : 0;
  if (env >= 1 && env <= 2) return env;
  return BN <= 128 ? 2 : 1;
}

// ================================================================== TMA implicit-GEMM convolutions (TConvArgs)
namespace {
constexpr int kMaxAcc = 8;
__host__ __device__ __forceinline__ int acc_buffers(int BN) {
  int nb = 512 / (BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256);
  return nb > kMaxAcc ? kMaxAcc : nb;
}
constexpr int TC_NMMA = 4;        // MMA-issuing warps: issue cost (~100 cycles per tcgen05.mma with its operand
                                  // broadcast) exceeds a small-N MMA's execution, so 4 warps issue for alternate tiles
constexpr int TC_THREADS = 32 * (1 + TC_NMMA + 8);  // producer warp, MMA warps, 8 epilogue warps (2 per TMEM quadrant)
__host__ __device__ __forceinline__ int win_bytes(int rows) { return (rows * 128 + 1023) / 1024 * 1024; }
}  // namespace

// smem (FWD / DGRAD; the weight gradient is twgrad_kernel): [resident B: T*Cblk chunks x BN rows x 128 B]
// [stages x window of R rows]
__host__ __device__ __forceinline__ int tconv_stage_bytes(const TConvArgs& a) { return win_bytes(a.R); }
__host__ __device__ __forceinline__ int tconv_fixed_bytes(const TConvArgs& a) { return a.T * a.Cblk * a.BN * 128; }

__global__ void __launch_bounds__(TC_THREADS, 1) tconv_kernel(const __grid_constant__ TConvArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kTgMaxStages], empty[kTgMaxStages], bfull, tfull[kMaxAcc], tempty[kMaxAcc];
  __shared__ uint32_t tbase;
  __shared__ __align__(16) float smem_bias[256];  // FWD: the layer's bias (BN <= 256)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = a.stages, BN = a.BN, SB = tconv_stage_bytes(a);
  uint8_t* fixed = smem;  // the resident B operand, then the ring
  uint8_t* ring = smem + tconv_fixed_bytes(a);
  // NB TMEM accumulators (as many as 512 columns hold, at most kMaxAcc): the MMA warp runs up to NB tiles ahead
  // of the epilogue, which hides the commit -> epilogue -> release round trip of short tiles
  const int NB = acc_buffers(BN);
  const uint32_t tcols = 512;
  // work split: tiles of 128 rows, CTA c serving group c % groups (its resident weights)
  const int m_tiles = (a.M + 127) / 128;
  const int g = (int)(blockIdx.x % a.groups);
  const int cta = blockIdx.x / a.groups;
  const int ctas = (gridDim.x - g + a.groups - 1) / a.groups;
  const int tiles = m_tiles;
  if (tid == 0) {
    for (int st = 0; st < S; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
    }
    mbar_init(&bfull, 1);
    for (int b = 0; b < NB; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 8);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(&tbase, tcols);
  // MMA warps: up to TC_NMMA, each owning a sub-ring of Sw stages and every nmma-th tile, so that each stage
  // barrier is always consumed in order (a warp running a whole ring lap ahead of another would otherwise alias
  // an mbarrier phase)
  int nmma = min(min(TC_NMMA, NB), S / a.Cblk);
  if (nmma < 1) nmma = 1;
  const int Sw = S / nmma;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if ((a.dbg & 64) && blockIdx.x == 0 && tid == 0) reinterpret_cast<long long*>(a.partial)[193] = clock64();
  pdl_sync();
  if ((a.dbg & 64) && blockIdx.x == 0 && tid == 0) reinterpret_cast<long long*>(a.partial)[194] = clock64();

  if (warp == 0) {
    {  // ---- TMA producer (whole warp, warp-uniform; one elected lane issues)
      mbar_expect_tx_w(&bfull, (uint32_t)(a.T * a.Cblk * BN * 128));
      for (int ch = 0; ch < a.T * a.Cblk; ++ch) tma_load_2d_w(fixed + ch * BN * 128, &a.tb[g], ch * 64, 0, &bfull);
      int it = 0, tl_local = 0;
      for (int tl = cta; tl < tiles; tl += ctas, ++tl_local) {
        {
          const int m0 = tl * 128, row0 = a.mode == TCONV_FWD ? m0 : m0 - a.maxshift;
          // the stages of MMA warp w's k-th tile: its own sub-ring of Sw stages (consumed in order by that warp)
          const int w = tl_local % nmma, k = tl_local / nmma;
          for (int cb = 0; cb < a.Cblk; ++cb, ++it) {
            const int q = k * a.Cblk + cb, st = w * Sw + q % Sw, ph = (q / Sw) & 1;
            mbar_spin(&empty[st], ph ^ 1);
            if (a.dbg & 4) {
              mbar_arrive_w(&full[st]);
            } else {
              mbar_expect_tx_w(&full[st], (uint32_t)(a.R * 128));
              tma_load_2d_w(ring + st * SB, &a.ta[g], cb * 64, row0, &full[st]);
            }
            if ((a.dbg & 64) && blockIdx.x == 0 && it < 64 && lane == 0) reinterpret_cast<long long*>(a.partial)[it] = clock64();
          }
        }
      }
    }
  } else if (warp <= TC_NMMA) {
    const int j = warp - 1;
    if (j < nmma) {  // ---- MMA issuer j: local tiles j, j + nmma, ... (whole warp, warp-uniform; one lane issues)
      mbar_spin(&bfull, 0);
      const bool fwd = a.mode == TCONV_FWD;
      const int Th = a.T / a.Tw;
      const uint32_t ring_u = smem_u32(ring);
      const uint32_t idesc = make_idesc_bf16(128, BN, 0, 0);
      const uint32_t fx = smem_u32(fixed);
      int it = 0, tl_local = 0;
      for (int tl = cta; tl < tiles; tl += ctas, ++tl_local) {
        if (tl_local % nmma != j) {  // another MMA warp's tile: only its stages are counted
          it += a.Cblk;
          continue;
        }
        const int buf = tl_local % NB;
        if (!(a.dbg & 128)) mbar_spin(&tempty[buf], ((tl_local / NB) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + (uint32_t)(buf * BN);
        {
          const int k = tl_local / nmma;
          for (int cb = 0; cb < a.Cblk; ++cb, ++it) {
            const int q = k * a.Cblk + cb, st = j * Sw + q % Sw;
            mbar_spin(&full[st], (q / Sw) & 1);
            // (TMA data: async proxy to async proxy, ordered by the mbarrier; no tcgen05 fence)
            // descriptors advance by adding to the 14-bit start-address field (16-byte units); every tap is the
            // same window read shift(t) rows later (fwd; maxshift - shift(t) for dgrad), every K step 32 bytes
            // later. Pure loop-counter arithmetic, so the operands stay in uniform registers (no per-MMA R2UR)
            const uint64_t a0 = desc_sw128(ring_u + (uint32_t)(st * SB), 16, 1024);
            const uint64_t b0 = desc_sw128(fx, 16, 1024) + (uint64_t)(cb * BN * 8);
            for (int ty = 0, t = 0; ty < Th; ++ty)
              for (int tx = 0; tx < a.Tw; ++tx, ++t) {
                const int sh = ty * a.Ws + tx, off = fwd ? sh : a.maxshift - sh;
                const uint64_t at = a0 + (uint64_t)(off * 8), bt = b0 + (uint64_t)((t * a.Cblk) * BN * 8);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  if (!(a.dbg & 2)) mma_bf16_w(d, at + 2 * kk, bt + 2 * kk, idesc, (cb > 0 || t > 0 || kk > 0) ? 1u : 0u);
              }
            if (a.dbg & 8) mbar_arrive_w(&empty[st]);
            else mma_commit_w(&empty[st]);
          }
        }
        if (a.dbg & 8) mbar_arrive_w(&tfull[buf]);
        else mma_commit_w(&tfull[buf]);
        if ((a.dbg & 64) && blockIdx.x == 0 && tl_local < 64 && lane == 0) reinterpret_cast<long long*>(a.partial)[64 + tl_local] = clock64();
      }
    }
  } else if (!(a.dbg & 128)) {  // ---- epilogue: thread = one row (TMEM lane) of the tile, half of its columns
    const int q = warp & 3, half = (warp - 1 - TC_NMMA) >> 2, c_lo = half * (BN / 2), c_hi = c_lo + BN / 2;
    // per-thread constants of the epilogue: the next grid's shape (FWD) and the bias in shared memory (the
    // per-element address math and the bias loads were ~30 % of the forward's stall samples)
    const int Nn = a.N, HoWo = a.Ho * a.Wo;
    const int sn = a.s_next > 0 ? a.s_next : 1, Hn = a.Ho / sn, Wn = a.Wo / sn, Cn = Nn * sn * sn;
    const float* s_bias = smem_bias;
    if (a.mode == TCONV_FWD) {  // the 8 epilogue warps stage the bias (after the PDL wait: the update wrote it)
      for (int e = tid - 32 * (1 + TC_NMMA); e < BN; e += 256) smem_bias[e] = __ldg(a.bias[g] + e);
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
    int tl_local = 0;
    for (int tl = cta; tl < tiles; tl += ctas, ++tl_local) {
      const int buf = tl_local % NB;
      mbar_wait_warp(&tfull[buf], (tl_local / NB) & 1);
      tc_fence_after();
      const int mt = tl;
      const int m = mt * 128 + 32 * q + lane;
      // row m -> (image, y, x) of the grid, once per tile
      const int img = (int)fdiv(a.fd_hsws, (uint32_t)m), pq = m - img * a.HsWs;
      const int yy = (int)fdiv(a.fd_ws, (uint32_t)pq), xx = pq - yy * a.Ws;
      const uint32_t trow = tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * BN);
      for (int c = c_lo; c < c_hi; c += 16) {
        float v[16];
        if (a.dbg & 16) continue;
        tmem_ld16(trow + c, v);  // warp-collective
        if (a.dbg & 1) continue;
        if (a.mode == TCONV_FWD) {
          if (m >= a.M) continue;
          const int oy = yy, ox = xx;
          if (oy >= a.Ho || ox >= a.Wo) continue;
          float bz[16];
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            const float4 b4 = *reinterpret_cast<const float4*>(s_bias + c + i);
            bz[i] = b4.x; bz[i + 1] = b4.y; bz[i + 2] = b4.z; bz[i + 3] = b4.w;
          }
          uint32_t o[8];
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(fmaxf(fmaf(v[i], a.scale, bz[i]), 0.0f),
                                                            fmaxf(fmaf(v[i + 1], a.scale, bz[i + 1]), 0.0f));
            o[i >> 1] = *reinterpret_cast<const uint32_t*>(&h2);
          }
          if (a.s_next == 0) {  // canonical (C,H,W) flatten: out[img][n*HoWo + p]
            __nv_bfloat16* dst = a.cout[g] + (long long)img * Nn * HoWo + (long long)oy * a.Wo + ox;
            const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(o);
#pragma unroll
            for (int i = 0; i < 16; ++i) dst[(long long)(c + i) * HoWo] = hv[i];
          } else {  // next grid (s2d by s_next): pixel (oy/s, ox/s), channel (iy*s + ix)*N + n
            const int py = (int)fdiv(a.fd_sn, (uint32_t)oy), px = (int)fdiv(a.fd_sn, (uint32_t)ox);
            const int qq = (oy - py * sn) * sn + (ox - px * sn);
            if (py < Hn && px < Wn) {
              uint4* dst = reinterpret_cast<uint4*>(a.cout[g] + (((long long)img * Hn + py) * Wn + px) * Cn + qq * Nn + c);
              dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
              dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
            }
          }
        } else if (a.mode == TCONV_DGRAD) {  // x [X > 0], inverse space-to-depth into the previous dZ
          if (m >= a.M) continue;
          const int py = yy, px = xx;
          const uint4* xm = reinterpret_cast<const uint4*>(a.xmask + (long long)m * a.Cs + c);
          const uint4 mk0 = __ldg(xm), mk1 = __ldg(xm + 1);
          const uint32_t mw[8] = {mk0.x, mk0.y, mk0.z, mk0.w, mk1.x, mk1.y, mk1.z, mk1.w};
          uint32_t o[8];
#pragma unroll
          for (int h = 0; h < 8; ++h) {
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(bf16_gt0(mw[h] & 0xFFFFu) ? v[2 * h] : 0.0f,
                                                            bf16_gt0(mw[h] >> 16) ? v[2 * h + 1] : 0.0f);
            o[h] = *reinterpret_cast<const uint32_t*>(&h2);
          }
          const int qq = (int)fdiv(a.fd_cp, (uint32_t)c), cc = c - qq * a.Cp;
          const int iy = (int)fdiv(a.fd_s, (uint32_t)qq), ix = qq - iy * a.s;
          const long long row = (long long)img * a.prevHsWs + (long long)(py * a.s + iy) * a.prevWs + (px * a.s + ix);
          uint4* dst = reinterpret_cast<uint4*>(a.dzprev + row * a.Cp + cc);
          dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
          dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
      if ((a.dbg & 64) && blockIdx.x == 0 && tid == 64 && tl_local < 64) reinterpret_cast<long long*>(a.partial)[128 + tl_local] = clock64();
    }
  }
  if ((a.dbg & 64) && blockIdx.x == 0 && tid == 0) reinterpret_cast<long long*>(a.partial)[192] = clock64();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, tcols);
}


// ---- TCONV_WGRAD: one CTA per K range; every 64-row chunk (the Cblk X windows + the dZ tile) is staged ONCE and
// feeds every M tile of dW (tap, c-block pairs + the all-ones db block), each M tile its own TMEM accumulator;
// MMA warp j issues the M tiles j, j + nmma, ... of every chunk (a stage is released when all of them committed)
__host__ __device__ __forceinline__ int twg_stage_bytes(const TConvArgs& a) { return a.Cblk * win_bytes(a.R) + 8192; }

__global__ void __launch_bounds__(TC_THREADS, 1) twgrad_kernel(const __grid_constant__ TConvArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kTgMaxStages], empty[kTgMaxStages], tfull, tempty;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = a.stages, SB = twg_stage_bytes(a);
  uint8_t* ring = smem;
  uint8_t* ones = smem + S * SB;  // above every window: the LBO of an A tile's second half stays positive
  const int m_tiles = (a.M + 127) / 128;
  const int nmma = m_tiles < TC_NMMA ? m_tiles : TC_NMMA;
  if (tid == 0) {
    for (int st = 0; st < S; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], nmma);
    }
    mbar_init(&tfull, nmma);
    mbar_init(&tempty, 8);
    fence_mbar_init();
  }
  for (int e = tid; e < 8192 / 16; e += blockDim.x)
    reinterpret_cast<uint4*>(ones)[e] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
  fence_async_smem();
  if (warp == 1) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_sync();
  auto chunks_of = [&](int r) {
    const long long r0 = (long long)r * a.kpr * 64;
    const long long rows = min((long long)a.kpr * 64, a.krows - r0);
    return (int)((rows + 63) / 64);
  };
  if (warp == 0) {  // ---- TMA producer (whole warp; one elected lane issues)
    int it = 0;
    for (int r = blockIdx.x; r < a.ranges; r += gridDim.x) {
      const int nch = chunks_of(r);
      for (int c = 0; c < nch; ++c, ++it) {
        const int st = it % S;
        const int p0 = (int)((long long)r * a.kpr * 64 + c * 64);
        mbar_spin(&empty[st], ((it / S) & 1) ^ 1);
        mbar_expect_tx_w(&full[st], (uint32_t)(a.Cblk * a.R * 128 + 8192));
        uint8_t* sb = ring + st * SB;
        for (int cb = 0; cb < a.Cblk; ++cb) tma_load_2d_w(sb + cb * win_bytes(a.R), &a.ta[0], cb * 64, p0, &full[st]);
        tma_load_2d_w(sb + a.Cblk * win_bytes(a.R), &a.tb[0], 0, p0, &full[st]);
      }
    }
  } else if (warp <= TC_NMMA) {
    const int j = warp - 1;
    if (j < nmma) {  // ---- MMA warp j: M tiles j, j + nmma, ... of every chunk
      const uint32_t idesc = make_idesc_bf16(128, 64, 1, 1);
      const uint32_t ring_u = smem_u32(ring), ones_u = smem_u32(ones);
      // this warp's (at most 2: M <= 8 tiles, nmma = min(tiles, 4)) M tiles: the stage offsets of their two
      // 64-row halves, a (t, cb) window read from row shift(t), or -1 for the ones block; fixed for the kernel
      int off[2][2], nmt = 0;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int mt = j + k * nmma;
        if (mt < m_tiles) nmt = k + 1;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int mb = 2 * mt + hh;
          if (mt >= m_tiles || mb * 64 >= a.TCs) {
            off[k][hh] = -1;
            continue;
          }
          const int t = mb / a.Cblk, cb = mb - t * a.Cblk;
          off[k][hh] = cb * win_bytes(a.R) + ((t / a.Tw) * a.Ws + t % a.Tw) * 128;
        }
      }
      int it = 0, rl = 0;
      for (int r = blockIdx.x; r < a.ranges; r += gridDim.x, ++rl) {
        mbar_spin(&tempty, (rl & 1) ^ 1);
        tc_fence_after();
        const int nch = chunks_of(r);
        for (int c = 0; c < nch; ++c, ++it) {
          const int st = it % S;
          mbar_spin(&full[st], (it / S) & 1);
          const uint32_t sb = ring_u + (uint32_t)(st * SB);
          const uint32_t bt = sb + (uint32_t)(a.Cblk * win_bytes(a.R));
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            if (k >= nmt) break;
            const uint32_t h0 = off[k][0] < 0 ? ones_u : sb + (uint32_t)off[k][0];
            const uint32_t h1 = off[k][1] < 0 ? ones_u : sb + (uint32_t)off[k][1];
            const uint32_t lbo = h1 > h0 ? h1 - h0 : 0u;  // both halves the ones block: 0, never past it
            const uint32_t d = tbase + (uint32_t)((j + k * nmma) * 64);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16_w(d, desc_sw128(h0 + kk * 2048, lbo, 1024), desc_sw128(bt + kk * 2048, 8192, 1024), idesc,
                         (c > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit_w(&empty[st]);
        }
        mma_commit_w(&tfull);
      }
    }
  } else {  // ---- epilogue: 8 warps, thread = one row of each M tile, half of the 64 columns
    const int q = warp & 3, half = (warp - 1 - TC_NMMA) >> 2;
    int rl = 0;
    for (int r = blockIdx.x; r < a.ranges; r += gridDim.x, ++rl) {
      mbar_wait_warp(&tfull, rl & 1);
      tc_fence_after();
      for (int mt = 0; mt < m_tiles; ++mt) {
        const int m = mt * 128 + 32 * q + lane;
        for (int c = half * 32; c < half * 32 + 32; c += 16) {
          float v[16];
          tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + (uint32_t)(mt * 64 + c), v);
          if (c >= a.Nout) continue;
          if (m < a.TCs) {  // column-major [r][n][m]: a warp's 32 rows are 128 contiguous bytes per column
            float* p = a.partial + ((long long)r * a.Nout + c) * a.TCs + m;
#pragma unroll
            for (int i = 0; i < 16; ++i) p[(long long)i * a.TCs] = v[i];
          } else if (m == a.TCs) {  // the all-ones row: db
            float* p = a.partial_db + (long long)r * a.Nout + c;
#pragma unroll
            for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 512);
}

bool init_tconv_kernel_attrs() {
  const bool ok = cudaFuncSetAttribute(tconv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024) ==
                      cudaSuccess &&
                  cudaFuncSetAttribute(twgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024) ==
                      cudaSuccess;
  cudaGetLastError();
  return ok;
}

// the deepest ring that fits 219 KB next to the resident weights (>= 2 stages), 0: does not fit
size_t tconv_smem(const TConvArgs& a0) {
  if (a0.mode == TCONV_WGRAD) {
    const int sb = twg_stage_bytes(a0), st = std::min(kTgMaxStages, (219 * 1024 - 1024 - 8192) / sb);
    if (st < 2 || (a0.M + 127) / 128 * 64 > 512) return 0;
    return (size_t)st * sb + 8192 + 1024;
  }
  const int fixed = tconv_fixed_bytes(a0), sb = tconv_stage_bytes(a0);
  const int st = std::min(kTgMaxStages, (219 * 1024 - 1024 - fixed) / sb);
  if (st < 2) return 0;
  return (size_t)fixed + (size_t)st * sb + 1024;
}

void launch_tconv(const TConvArgs& a0, int num_sms, cudaStream_t st) {
  TConvArgs a = a0;
  if (a.mode == TCONV_WGRAD) {
    a.stages = std::min(kTgMaxStages, (219 * 1024 - 1024 - 8192) / twg_stage_bytes(a));
    launch_pdl(twgrad_kernel, dim3((unsigned)std::min(a.ranges, num_sms)), dim3(TC_THREADS), tconv_smem(a), st, a);
    sync_debug("tconv wgrad", st);
    return;
  }
  const int fixed = tconv_fixed_bytes(a), sb = tconv_stage_bytes(a);
  a.stages = std::min(kTgMaxStages, (219 * 1024 - 1024 - fixed) / sb);
  a.fd_hsws = make_fastdiv((uint32_t)a.HsWs);
  a.fd_ws = make_fastdiv((uint32_t)a.Ws);
  a.fd_sn = make_fastdiv((uint32_t)(a.s_next > 0 ? a.s_next : 1));
  a.fd_cp = make_fastdiv((uint32_t)(a.Cp > 0 ? a.Cp : 1));
  a.fd_s = make_fastdiv((uint32_t)(a.s > 0 ? a.s : 1));
  const int m_tiles = (a.M + 127) / 128;
  const long long tiles = (long long)m_tiles * a.groups;
  int grid = (int)std::min<long long>(tiles, num_sms);
  grid -= grid % a.groups;  // whole CTA sets per group
  launch_pdl(tconv_kernel, dim3(grid), dim3(TC_THREADS), tconv_smem(a), st, a);
  sync_debug(a.mode == TCONV_FWD ? "tconv fwd" : a.mode == TCONV_DGRAD ? "tconv dgrad" : "tconv wgrad", st);
}

// ---- layer 1 of the generic path: a1 (Philox sample) + a2 (gather, u8 -> exact bf16) into [b][441][64]
// One CTA per (image, group); thread e handles 16 bytes = one frame's 16 s2d channels of one pixel of the
// frame-major slot [frame][441 px][16] and writes them as 16 bf16 at [px][frame*16 ..]. The first CTA row also
// bulk-prefetches the slot the same image index samples next step (the sampler is counter-based).
// a2 gather + expansion: one CTA per (image, group). The 28,224-byte u8 slot arrives in shared memory by one
// TMA bulk copy, 256 threads expand it into the 441 x 128-byte bf16 rows of the conv1 input grid (thread = one
// 16-byte output chunk: 8 u8 of one frame plane -> 8 exact bf16; a warp stores 512 contiguous bytes). 28 KB of
// shared memory per CTA keeps ~7 CTAs per SM, i.e. the whole b = 512 x 2 gather resident in one wave.
constexpr int GATHER_THREADS = 256, GATHER_SLOT = 441 * 64;
constexpr int GATHER_SMEM = GATHER_SLOT + 16;
__global__ void __launch_bounds__(GATHER_THREADS) gather_s2d_kernel(GConvFwdArgs a, __nv_bfloat16* x0,
                                                                     __nv_bfloat16* x1) {
  extern __shared__ __align__(128) uint8_t gsm[];
  uint8_t* sU8 = gsm;
  uint64_t* bar = reinterpret_cast<uint64_t*>(gsm + GATHER_SLOT);
  const int img = blockIdx.x, g = blockIdx.y;
  pdl_sync();  // the ring (pushes) and the replay size come from earlier launches; x is read by the previous step
  if (threadIdx.x == 0) {
    long long slot = img;
    if (a.idx_in) {
      slot = a.idx_in[img];  // prioritized replay (A41): drawn by the predecessor
    } else if (a.ctr) {
      const unsigned long long T = a.ctr->T;
      slot = sample_slot(a.seed, a.rank, T, (unsigned)img, a.ctr->ring_size);  // a1
      if (g == 0) {
        if (a.idx) a.idx[img] = (int)slot;
        // the sampler is counter-based: step T+1's slot is known now; warm L2 and the TLB for it
        const long long nxt = sample_slot(a.seed, a.rank, T + 1, (unsigned)img, a.ctr->ring_size);
        bulk_prefetch_l2(a.ring[0] + nxt * a.slot_stride, GATHER_SLOT);
        bulk_prefetch_l2(a.ring[1] + nxt * a.slot_stride, GATHER_SLOT);
      }
    }
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, GATHER_SLOT);
    bulk_g2s(sU8, a.ring[g] + slot * a.slot_stride, GATHER_SLOT, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  uint4* dst = reinterpret_cast<uint4*>((g ? x1 : x0) + (long long)img * 441 * 64);
  // output chunk c = (pixel px, frame f, half h): bf16 channels 8 (2 f + h) .. +7 of pixel px = bytes
  // 8 h .. 8 h + 7 of pixel px's 16-byte vector in frame plane f (slot layout [f][441][16])
  for (int c = threadIdx.x; c < 441 * 8; c += GATHER_THREADS) {
    const int px = c >> 3, f = (c >> 1) & 3, h = c & 1;
    const uint2 w = *reinterpret_cast<const uint2*>(sU8 + f * 441 * 16 + px * 16 + h * 8);
    const uint32_t ws[2] = {w.x, w.y};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 2; ++q) {  // 4 bytes -> 4 exact bf16 (0..255 are exact)
      const uint32_t v = ws[q];
      const __nv_bfloat162 lo = __floats2bfloat162_rn((float)(v & 0xFFu), (float)((v >> 8) & 0xFFu));
      const __nv_bfloat162 hi = __floats2bfloat162_rn((float)((v >> 16) & 0xFFu), (float)(v >> 24));
      o[2 * q] = *reinterpret_cast<const uint32_t*>(&lo);
      o[2 * q + 1] = *reinterpret_cast<const uint32_t*>(&hi);
    }
    dst[c] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

void launch_gather_s2d(const GConvFwdArgs& a, __nv_bfloat16* x1_0, __nv_bfloat16* x1_1, int groups, cudaStream_t st) {
  launch_pdl(gather_s2d_kernel, dim3(a.b, groups), dim3(GATHER_THREADS), GATHER_SMEM, st, a, x1_0, x1_1);
  sync_debug("gather_s2d", st);
}

// FC dX, second half: the tgemm epilogue wrote dZ of the last conv layer (ReLU mask applied) in the canonical
// (C,H,W) flatten with coalesced stores; this permutes each image into the layer's input-grid geometry
// [py * Ws + px][C] (the zero border is never written). One CTA per image, the image staged in shared memory.
__global__ void __launch_bounds__(256) chw_to_hwc_kernel(const __nv_bfloat16* src, __nv_bfloat16* dst, int C, int Ho,
                                                         int Wo, int Ws, int HsWs) {
  extern __shared__ __align__(16) uint8_t csm[];
  __nv_bfloat16* sx = reinterpret_cast<__nv_bfloat16*>(csm);
  const int img = blockIdx.x, HoWo = Ho * Wo, n = C * HoWo;
  pdl_sync();  // src is the immediate predecessor's output; dst may still be read by the previous step
  const __nv_bfloat16* s = src + (long long)img * n;
  for (int e = threadIdx.x; e < n / 8; e += blockDim.x)
    reinterpret_cast<uint4*>(sx)[e] = __ldg(reinterpret_cast<const uint4*>(s) + e);
  __syncthreads();
  const int c8n = C / 8;
  for (int e = threadIdx.x; e < HoWo * c8n; e += blockDim.x) {
    const int p = e / c8n, c0 = (e - p * c8n) * 8;
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      o[j] = (uint32_t)__bfloat16_as_ushort(sx[(c0 + 2 * j) * HoWo + p]) |
             ((uint32_t)__bfloat16_as_ushort(sx[(c0 + 2 * j + 1) * HoWo + p]) << 16);
    const int oy = p / Wo, ox = p - oy * Wo;
    *reinterpret_cast<uint4*>(dst + ((long long)img * HsWs + (long long)oy * Ws + ox) * C + c0) =
        make_uint4(o[0], o[1], o[2], o[3]);
  }
}

bool chw_to_hwc_fits(int C, int Ho, int Wo) { return C % 8 == 0 && (C * Ho * Wo) % 8 == 0 && C * Ho * Wo * 2 <= 48 * 1024; }

void launch_chw_to_hwc(const __nv_bfloat16* src, __nv_bfloat16* dst, int b, int C, int Ho, int Wo, int Ws, int HsWs,
                       cudaStream_t st) {
  launch_pdl(chw_to_hwc_kernel, dim3(b), dim3(256), (size_t)C * Ho * Wo * 2, st, src, dst, C, Ho, Wo, Ws, HsWs);
  sync_debug("chw_to_hwc", st);
}

int tgemm_stages(int BN) {
  const int stage = TG_A_BYTES + BN * 64 * 2;
  const int budget = tg_ctas_per_sm(BN) == 2 ? 100 * 1024 : 200 * 1024;
  return std::max(2, std::min(kTgMaxStages, budget / stage));
}

size_t tgemm_smem(int BN) { return (size_t)tgemm_stages(BN) * (TG_A_BYTES + BN * 64 * 2) + 1024; }

bool init_tma_kernel_attrs() {
  const bool ok = cudaFuncSetAttribute(tgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       200 * 1024 + 1024) == cudaSuccess &&  // every ring fits 200 KB
                  cudaFuncSetAttribute(gather_s2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GATHER_SMEM) ==
                      cudaSuccess;
  cudaGetLastError();
  return ok;
}

void launch_tgemm(const TGemmArgs& a0, int num_sms, cudaStream_t st) {
  TGemmArgs a = a0;
  a.stages = tgemm_stages(a.BN);
  const long long tiles = (long long)((a.M + 127) / 128) * ((a.N + a.BN - 1) / a.BN) * a.splits * a.groups;
  const int grid = (int)std::min<long long>(tiles, (long long)num_sms * tg_ctas_per_sm(a.BN));
  launch_pdl(tgemm_kernel, dim3(grid), dim3(TG_THREADS), tgemm_smem(a.BN), st, a);
  sync_debug("tgemm", st);
}

}  // namespace dqn
