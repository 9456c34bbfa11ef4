// probe_tconv.cu — timing of the TMA tap-window convolution kernel (kernels_tma.cu) in isolation, on the
// forward geometry of a layer of the scaled net (BASELINE.json configs[4]) with random data:
//   tools/probe_tconv layer b [iters]      layer 1: 21x21x64 grid, 2x2 taps, N 32; 2: 10x10x128, 2x2, N 64;
//                                           3: 9x9x64, 3x3, N 64
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_1508_04186_b200/csrc
//   tools/probe_tconv.cu -o tools/probe_tconv
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1508_04186_b200/csrc/kernels_tma.cu"

using namespace dqn;

int main(int argc, char** argv) {
  const int layer = argc > 1 ? atoi(argv[1]) : 1, b = argc > 2 ? atoi(argv[2]) : 512;
  const int iters = argc > 3 ? atoi(argv[3]) : 20;
  int Hs, Cs, Th, N, s_next, Ho;
  if (layer == 1) { Hs = 21; Cs = 64; Th = 2; N = 32; s_next = 2; }
  else if (layer == 2) { Hs = 10; Cs = 128; Th = 2; N = 64; s_next = 1; }
  else { Hs = 9; Cs = 64; Th = 3; N = 64; s_next = 0; }
  Ho = Hs - Th + 1;
  const long long rows = (long long)b * Hs * Hs;
  const int T = Th * Th, K = T * Cs;
  std::vector<uint16_t> hx((size_t)rows * Cs), hw((size_t)N * K);
  srand(3);
  for (auto& v : hx) v = (uint16_t)(0x3c00 + rand() % 64);
  for (auto& v : hw) v = (uint16_t)(0x3800 + rand() % 64);
  __nv_bfloat16 *dx[2], *dw[2], *dout[2];
  float* bias;
  const long long out_elems = (long long)b * N * Ho * Ho;
  for (int g = 0; g < 2; ++g) {
    cudaMalloc(&dx[g], hx.size() * 2);
    cudaMalloc(&dw[g], hw.size() * 2);
    cudaMalloc(&dout[g], out_elems * 2);
    cudaMemcpy(dx[g], hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dw[g], hw.data(), hw.size() * 2, cudaMemcpyHostToDevice);
  }
  cudaMalloc(&bias, 256 * 4);
  cudaMemset(bias, 0, 256 * 4);
  TConvArgs f{};
  const int maxshift = (Th - 1) * Hs + (Th - 1);
  f.mode = TCONV_FWD; f.groups = 2; f.M = (int)rows; f.BN = N; f.T = T; f.Tw = Th; f.Ws = Hs; f.HsWs = Hs * Hs;
  f.Cblk = Cs / 64; f.maxshift = maxshift; f.R = getenv("TC_R") ? atoi(getenv("TC_R")) : 128 + maxshift; f.Ho = Ho; f.Wo = Ho; f.N = N; f.s_next = s_next;
  f.scale = 1.0f;
  f.dbg = getenv("TC_DBG") ? atoi(getenv("TC_DBG")) : 0;
  long long* dbgbuf;
  cudaMalloc(&dbgbuf, 256 * 8);
  cudaMemset(dbgbuf, 0, 256 * 8);
  f.partial = reinterpret_cast<float*>(dbgbuf);
  bool ok = init_tconv_kernel_attrs();
  for (int g = 0; g < 2; ++g) {
    ok = ok && make_tmap_bf16(&f.ta[g], dx[g], rows, Cs, Cs, f.R);
    ok = ok && make_tmap_bf16(&f.tb[g], dw[g], N, K, K, N);
    f.bias[g] = bias;
    f.cout[g] = dout[g];
  }
  if (!ok || !tconv_smem(f)) {
    fprintf(stderr, "setup failed\n");
    return 1;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  launch_tconv(f, sms, 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "%s\n", cudaGetErrorString(e));
    return 1;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) launch_tconv(f, sms, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1e3 / iters, flop = 2.0 * 2 * (double)b * Ho * Ho * N * K;
  if (f.dbg & 64) {
    long long h[256];
    cudaMemcpy(h, dbgbuf, sizeof(h), cudaMemcpyDeviceToHost);
    const long long t0 = h[193];
    printf("prologue->pdl %lld; producer:", h[194] - t0);
    for (int i = 0; i < 26; ++i) printf(" %lld", h[i] - t0);
    printf("\nmma:");
    for (int i = 0; i < 26; ++i) printf(" %lld", h[64 + i] - t0);
    printf("\nepi:");
    for (int i = 0; i < 26; ++i) printf(" %lld", h[128 + i] - t0);
    printf("\nend %lld\n", h[192] - t0);
  }
  printf("layer %d b %d: %.2f us, %.1f TFLOP/s (useful), window %d rows, stages %d\n", layer, b, us,
         flop / (us * 1e-6) / 1e12, f.R, (int)((219 * 1024 - 1024 - T * f.Cblk * N * 128) / ((f.R * 128 + 1023) / 1024 * 1024)));
  return 0;
}
