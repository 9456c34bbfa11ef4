// probe_tcgen05.cu — standalone check of the tcgen05 / TMEM / descriptor encodings
// used by the library (K-major and MN-major no-swizzle operands, row-shifted A
// views, bf16 and tf32 kinds). Prints PASS/FAIL per case; exit code = #fails.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1508_04186_b200/csrc/sm100.cuh"

using namespace dqn_sm100;

// mode bit0: A MN-major, bit1: B MN-major, bit2: tf32 kind
// A logical [rowsA][K] (rowsA >= 128 + shift), B logical [N][K]; D[m][n] = sum_k A[m+shift][k] * B[n][k]
__global__ void probe_kernel(const float* A, const float* B, float* D, int N, int K, int mode, int shift,
                             int rowsA) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const bool a_mn = mode & 1, b_mn = mode & 2, tf32 = mode & 4;
  const int esz = tf32 ? 4 : 2;
  const int epc = 16 / esz;  // elements per 16-byte chunk
  uint8_t* sA = smem;
  uint8_t* sB = smem + (size_t)rowsA * K * esz;
  // ---- stage A
  for (int i = threadIdx.x; i < rowsA * K; i += blockDim.x) {
    int r = i / K, k = i % K;
    size_t off;
    if (!a_mn) off = (size_t)(k / epc) * rowsA * 16 + (size_t)r * 16 + (k % epc) * esz;  // [k/epc][r][epc]
    else off = (size_t)(r / epc) * K * 16 + (size_t)k * 16 + (r % epc) * esz;            // [r/epc][k][epc]
    float v = A[i];
    if (tf32) *reinterpret_cast<float*>(sA + off) = v;
    else *reinterpret_cast<__nv_bfloat16*>(sA + off) = __float2bfloat16(v);
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    int n = i / K, k = i % K;
    size_t off;
    if (!b_mn) off = (size_t)(k / epc) * N * 16 + (size_t)n * 16 + (k % epc) * esz;
    else off = (size_t)(n / epc) * K * 16 + (size_t)k * 16 + (n % epc) * esz;
    float v = B[i];
    if (tf32) *reinterpret_cast<float*>(sB + off) = v;
    else *reinterpret_cast<__nv_bfloat16*>(sB + off) = __float2bfloat16(v);
  }
  fence_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const int kstep = tf32 ? 8 : 16;
    uint32_t idesc = tf32 ? make_idesc_tf32(128, N, a_mn, b_mn) : make_idesc_bf16(128, N, a_mn, b_mn);
    for (int kk = 0; kk < K / kstep; ++kk) {
      uint64_t ad, bd;
      if (!a_mn) ad = make_desc(smem_u32(sA) + kk * 2 * rowsA * 16 + shift * 16, rowsA * 16, 128);
      else ad = make_desc(smem_u32(sA) + kk * 2 * 128, 128, K * 16);
      if (!b_mn) bd = make_desc(smem_u32(sB) + kk * 2 * N * 16, N * 16, 128);
      else bd = make_desc(smem_u32(sB) + kk * 2 * 128, 128, K * 16);
      if (tf32) mma_tf32(tmem, ad, bd, idesc, kk > 0);
      else mma_bf16(tmem, ad, bd, idesc, kk > 0);
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (w < 4) {
    for (int c = 0; c < N; c += 8) {
      float v[8];
      tmem_ld8(tmem + ((uint32_t)(32 * w) << 16) + c, v);
      int m = 32 * w + lane;
      for (int j = 0; j < 8; ++j) D[m * N + c + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

static float bf16r(float x) { return __bfloat162float(__float2bfloat16(x)); }
static float tf32r(float x) {  // truncation toward zero of 13 mantissa bits is one admissible tf32 reading; use tol
  return x;
}

int main() {
  int fails = 0;
  const int K = 64;
  int cases[][3] = {  // N, mode, shift
      {16, 0, 0}, {32, 0, 0}, {64, 0, 0}, {128, 0, 0}, {256, 0, 0}, {16, 1, 0}, {64, 1, 0},
      {16, 2, 0}, {64, 2, 0}, {32, 3, 0}, {16, 0, 3}, {32, 0, 21}, {16, 4, 0}, {64, 4, 0},
      {16, 5, 0}, {32, 6, 0}, {16, 4, 5}};
  for (auto& cs : cases) {
    int N = cs[0], mode = cs[1], shift = cs[2];
    int rowsA = 128 + ((shift + 7) / 8) * 8;
    std::vector<float> A(rowsA * K), B(N * K), D(128 * N);
    srand(1234 + N + mode * 7 + shift);
    for (auto& x : A) x = (float)((rand() % 17) - 8) / 8.0f;
    for (auto& x : B) x = (float)((rand() % 13) - 6) / 4.0f;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, D.size() * 4);
    size_t smem = (size_t)(rowsA + N) * K * 4 + 1024;
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe_kernel<<<1, 128, smem>>>(dA, dB, dD, N, K, mode, shift, rowsA);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("case N=%d mode=%d shift=%d CUDA ERROR %s\n", N, mode, shift, cudaGetErrorString(e)); return 100; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[(m + shift) * K + k] * B[n * K + k];
        maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
      }
    bool ok = maxerr < 1e-3;
    printf("case N=%3d A_mn=%d B_mn=%d tf32=%d shift=%2d  maxerr=%.3g  %s\n", N, mode & 1, (mode >> 1) & 1,
           (mode >> 2) & 1, shift, maxerr, ok ? "PASS" : "FAIL");
    if (!ok) {
      ++fails;
      printf("  D[0][0..3]=%g %g %g %g\n", D[0], D[1], D[2], D[3]);
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
  }
  (void)bf16r; (void)tf32r;
  printf("fails=%d\n", fails);
  return fails;
}
