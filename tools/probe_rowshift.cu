// probe_rowshift.cu — does a tcgen05 SW128 K-major operand descriptor read a tile that starts r rows (r*128 B)
// into a TMA-written 128-byte-swizzled window, with the descriptor's base-offset field = r & 7?
// A window of 136 rows x 64 bf16 (row i = values i*64 + k, small integers) is loaded by one TMA; for each
// shift r in 0..8 one MMA (M = 128, N = 16, K = 16) multiplies rows r..r+127 by a B = [16][16] one-hot (B[n][k]
// = 1 iff k == n), so D[m][n] must equal A[r + m][n]. Prints mismatches per (r, base-offset mode).
#include <cuda.h>
#include <cstdio>
#include <vector>

#include "../paper_1508_04186_b200/csrc/sm100.cuh"

using namespace dqn_sm100;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t base_off) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(base_off & 7) << 49;
  d |= (uint64_t)2 << 61;
  return d;
}

__global__ void probe(const __grid_constant__ CUtensorMap ta, const __nv_bfloat16* gB, float* out, int mode) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                 // 136 rows x 128 B
  uint8_t* sB = smem + 136 * 128 + 1024 - (136 * 128) % 1024;  // B: 16 rows x 32 B, no swizzle K-major
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  // B in the no-swizzle K-major layout [kc 2][16 rows][8 el]: B[n][k]
  for (int e = tid; e < 2 * 16 * 8; e += blockDim.x) {
    const int kc = e / 128, n = (e / 8) % 16, j = e % 8;
    reinterpret_cast<__nv_bfloat16*>(sB)[e] = gB[n * 16 + kc * 8 + j];
  }
  fence_async_smem();
  if (warp == 0) tmem_alloc(&tbase, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mbar_arrive_expect_tx(&bar, 136 * 128);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(sA)),
        "l"(&ta), "r"(0), "r"(0), "r"(smem_u32(&bar))
        : "memory");
  }
  mbar_wait(&bar, 0);
  for (int r = 0; r <= 8; ++r) {
    if (tid == 0) {
      tc_fence_after();
      const uint32_t sa = smem_u32(sA) + r * 128;
      const uint32_t bo = mode == 0 ? 0 : mode == 1 ? (uint32_t)(r & 7) : (uint32_t)((sa >> 7) & 7);
      const uint64_t ad = desc_sw128(sa, 16, 1024, bo);
      const uint64_t bd = make_desc(smem_u32(sB), 16 * 16, 128);
      mma_bf16(tbase, ad, bd, make_idesc_bf16(128, 16, 0, 0), 0u);
      mma_commit(&mbar);
    }
    mbar_wait(&mbar, r & 1);
    tc_fence_after();
    float v[16];
    tmem_ld16(tbase + ((uint32_t)(32 * (warp & 3)) << 16), v);
    for (int n = 0; n < 16; ++n) out[((size_t)r * 128 + tid) * 16 + n] = v[n];
    tc_fence_before();
    __syncthreads();
  }
  if (warp == 0) tmem_dealloc(tbase, 32);
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiledFn enc = reinterpret_cast<EncodeTiledFn>(p);
  std::vector<__nv_bfloat16> hA(136 * 64), hB(16 * 16);
  for (int i = 0; i < 136; ++i)
    for (int k = 0; k < 64; ++k) hA[i * 64 + k] = __float2bfloat16((float)((i * 7 + k * 3) % 200));
  for (int n = 0; n < 16; ++n)
    for (int k = 0; k < 16; ++k) hB[n * 16 + k] = __float2bfloat16(n == k ? 1.0f : 0.0f);
  __nv_bfloat16 *dA, *dB;
  float* dO;
  cudaMalloc(&dA, hA.size() * 2);
  cudaMalloc(&dB, hB.size() * 2);
  cudaMalloc(&dO, 9 * 128 * 16 * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap ta;
  cuuint64_t dims[2] = {64, 136}, strides[1] = {128};
  cuuint32_t box[2] = {64, 136}, es[2] = {1, 1};
  if (enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dA, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  std::vector<float> hO(9 * 128 * 16);
  const char* names[3] = {"base_offset=0", "base_offset=r&7", "base_offset=(addr>>7)&7"};
  for (int mode = 0; mode < 3; ++mode) {
    probe<<<1, 128, 64 * 1024>>>(ta, dB, dO, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: %s\n", names[mode], cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(hO.data(), dO, hO.size() * 4, cudaMemcpyDeviceToHost);
    printf("%s:", names[mode]);
    for (int r = 0; r <= 8; ++r) {
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n)
          if (hO[((size_t)r * 128 + m) * 16 + n] != __bfloat162float(hA[(r + m) * 64 + n])) ++bad;
      printf(" r=%d bad=%d;", r, bad);
    }
    printf("\n");
  }
  return 0;
}
