// probe_tgemm.cu — standalone check + timing of the warp-specialised TMA GEMM (kernels_tma.cu) on one GPU:
// C[M][N] = A B^T for K-major / MN-major operand layouts, sampled entries against a host fp64 reference,
// then TFLOP/s over repeated launches. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I include -I paper_1508_04186_b200/csrc tools/probe_tgemm.cu -o tools/probe_tgemm
// usage: tools/probe_tgemm M N K a_mn b_mn BN [iters]
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../paper_1508_04186_b200/csrc/kernels_tma.cu"

using namespace dqn;

static float bf(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main(int argc, char** argv) {
  if (argc < 7) {
    fprintf(stderr, "usage: %s M N K a_mn b_mn BN [iters]\n", argv[0]);
    return 2;
  }
  const int M = atoi(argv[1]), N = atoi(argv[2]), K = atoi(argv[3]), amn = atoi(argv[4]), bmn = atoi(argv[5]);
  const int BN = atoi(argv[6]), iters = argc > 7 ? atoi(argv[7]) : 20;
  std::vector<uint16_t> hA((size_t)M * K), hB((size_t)N * K);
  srand(1);
  for (auto& x : hA) x = (uint16_t)(0x3c00 + (rand() % 256) - 128);  // bf16 values near 1/128.. scale
  for (auto& x : hB) x = (uint16_t)(0x3c00 + (rand() % 256) - 128);
  // logical A(m,k): K-major stored [M][K]; MN-major stored [K][M]. Same for B with N.
  __nv_bfloat16 *dA, *dB;
  float* dC;
  cudaMalloc(&dA, hA.size() * 2);
  cudaMalloc(&dB, hB.size() * 2);
  cudaMalloc(&dC, (size_t)M * N * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  auto Aat = [&](int m, int k) { return bf(amn ? hA[(size_t)k * M + m] : hA[(size_t)m * K + k]); };
  auto Bat = [&](int n, int k) { return bf(bmn ? hB[(size_t)k * N + n] : hB[(size_t)n * K + k]); };
  TGemmArgs a{};
  a.M = M; a.N = N; a.K = K; a.kper = K; a.splits = 1; a.BN = BN; a.a_mn = amn; a.b_mn = bmn; a.groups = 1;
  a.epi = TC_EPI_ACCUM; a.store = 1; a.C[0] = dC; a.ldc = N;
  bool ok = amn ? make_tmap_bf16(&a.ta[0], dA, K, M, M, 64) : make_tmap_bf16(&a.ta[0], dA, M, K, K, 128);
  ok = ok && (bmn ? make_tmap_bf16(&a.tb[0], dB, K, N, N, 64) : make_tmap_bf16(&a.tb[0], dB, N, K, K, BN));
  if (!ok || !init_tma_kernel_attrs()) {
    fprintf(stderr, "tensor map / attribute setup failed\n");
    return 1;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  launch_tgemm(a, sms, 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "launch: %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> hC((size_t)M * N);
  cudaMemcpy(hC.data(), dC, hC.size() * 4, cudaMemcpyDeviceToHost);
  double worst = 0.0;
  for (int t = 0; t < 256; ++t) {
    const int m = (int)((t * 7919LL) % M), n = (int)((t * 104729LL) % N);
    double r = 0.0;
    for (int k = 0; k < K; ++k) r += (double)Aat(m, k) * Bat(n, k);
    worst = std::max(worst, std::fabs(r - hC[(size_t)m * N + n]) / std::max(1.0, std::fabs(r)));
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) launch_tgemm(a, sms, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1e3 / iters;
  printf("M %d N %d K %d a_mn %d b_mn %d BN %d: max rel err %.2e, %.2f us, %.1f TFLOP/s\n", M, N, K, amn, bmn, BN, worst,
         us, 2.0 * M * N * K / (us * 1e-6) / 1e12);
  return worst < 1e-2 ? 0 : 1;
}
