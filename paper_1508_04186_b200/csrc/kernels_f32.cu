// kernels_f32.cu — the fp32 SIMT replica step (precision DQN_FP32): the exact
// parity path (<= 1e-5 vs the fp64 oracle). Layer semantics follow P:61-67
// (valid convolutions, ReLU after every conv / hidden FC, linear output) and the
// gradient of Alg. 1. Activations are stored per image in (C,H,W) order,
// parameters in the canonical flat order (layer by layer, W then b).
//
// All reductions run in a fixed order (no float atomics), so a run is bit-for-bit
// reproducible.
#include <cstdio>
#include "dqn_internal.h"

namespace dqn {

static inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// ------------------------------------------------------------------ staging helpers
// x = u8 / 255 (A15): IEEE single division is correctly rounded, so every value
// equals fp32(k/255) exactly.
__device__ __forceinline__ void stage_image(float* s_in, const ImgSrc& src, int g, int img, int n) {
  if (src.u8[g]) {
    const long long slot = src.idx ? (long long)src.idx[img] : (long long)img;
    const uint8_t* p = src.u8[g] + slot * src.stride;
    if ((n & 15) == 0 && (((uintptr_t)p) & 15) == 0) {
      for (int v = threadIdx.x; v < n / 16; v += blockDim.x) {
        uint4 q = reinterpret_cast<const uint4*>(p)[v];
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) s_in[v * 16 + i * 4 + j] = (float)((w[i] >> (8 * j)) & 0xFF) / 255.0f;
      }
    } else {
      for (int i = threadIdx.x; i < n; i += blockDim.x) s_in[i] = (float)p[i] / 255.0f;
    }
  } else {
    const float* p = src.f32[g] + (long long)img * src.stride;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_in[i] = p[i];
  }
}

// ------------------------------------------------------------------ conv forward
// out[img][n][p] = relu(b[n] + sum_{c,ky,kx} W[n][c][ky][kx] * in[img][c][oy*s+ky][ox*s+kx])
// grid (b, groups * n_chunks, z_splits); each thread owns PIX pixels x NCH channels.
template <int NCH, int PIX>
__global__ void __launch_bounds__(128) conv_fwd_f32_kernel(ConvShape cs, ImgSrc src, const float* __restrict__ th0,
                                                           const float* __restrict__ th1, float* out0, float* out1,
                                                           int zsplits) {
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  const int img = blockIdx.x;
  const int nchunks = (cs.N + NCH - 1) / NCH;
  const int g = blockIdx.y / nchunks;
  const int n0 = (blockIdx.y % nchunks) * NCH;
  const float* theta = g ? th1 : th0;
  float* out = g ? out1 : out0;
  const int CHW = cs.C * cs.H * cs.W;
  const int KK = cs.C * cs.k * cs.k;
  float* s_in = sm;
  float* s_w = sm + ((CHW + 3) & ~3);
  stage_image(s_in, src, g, img, CHW);
  for (int e = threadIdx.x; e < KK * NCH; e += blockDim.x) {
    const int nl = e / KK, t = e % KK;
    s_w[t * NCH + nl] = (n0 + nl < cs.N) ? theta[cs.w_off + (long long)(n0 + nl) * KK + t] : 0.0f;
  }
  __syncthreads();
  const int HoWo = cs.Ho * cs.Wo;
  const int per_z = (HoWo + zsplits - 1) / zsplits;
  const int p_begin = blockIdx.z * per_z;
  const int p_end = min(HoWo, p_begin + per_z);
  const int HW = cs.H * cs.W;
  for (int pb = p_begin + threadIdx.x; pb < p_end; pb += blockDim.x * PIX) {
    int base[PIX];
    bool valid[PIX];
#pragma unroll
    for (int i = 0; i < PIX; ++i) {
      const int p = pb + i * blockDim.x;
      valid[i] = p < p_end;
      const int oy = valid[i] ? p / cs.Wo : 0, ox = valid[i] ? p % cs.Wo : 0;
      base[i] = oy * cs.s * cs.W + ox * cs.s;
    }
    float acc[PIX][NCH];
#pragma unroll
    for (int i = 0; i < PIX; ++i)
#pragma unroll
      for (int nl = 0; nl < NCH; ++nl) acc[i][nl] = 0.0f;
    for (int c = 0; c < cs.C; ++c)
      for (int ky = 0; ky < cs.k; ++ky) {
        const int off = c * HW + ky * cs.W;
        const float* wrow = s_w + ((c * cs.k + ky) * cs.k) * NCH;
        for (int kx = 0; kx < cs.k; ++kx) {
          float w[NCH];
#pragma unroll
          for (int q = 0; q < NCH / 4; ++q) {
            float4 v = reinterpret_cast<const float4*>(wrow + kx * NCH)[q];
            w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
          }
#pragma unroll
          for (int i = 0; i < PIX; ++i) {
            const float x = s_in[base[i] + off + kx];
#pragma unroll
            for (int nl = 0; nl < NCH; ++nl) acc[i][nl] = fmaf(w[nl], x, acc[i][nl]);
          }
        }
      }
#pragma unroll
    for (int i = 0; i < PIX; ++i) {
      if (!valid[i]) continue;
      const int p = pb + i * blockDim.x;
#pragma unroll
      for (int nl = 0; nl < NCH; ++nl) {
        const int n = n0 + nl;
        if (n < cs.N) {
          const float v = acc[i][nl] + theta[cs.b_off + n];
          out[((long long)img * cs.N + n) * HoWo + p] = v > 0.0f ? v : 0.0f;
        }
      }
    }
  }
}

void launch_conv_fwd_f32(const ConvShape& cs, const ImgSrc& src, const float* theta0, const float* theta1,
                         float* out0, float* out1, int b, int groups, cudaStream_t st) {
  constexpr int NCH = 16, PIX = 2;
  const int CHW = cs.C * cs.H * cs.W;
  const int KK = cs.C * cs.k * cs.k;
  const size_t smem = (size_t)(((CHW + 3) & ~3) + KK * NCH) * sizeof(float);
  const int nchunks = cdiv(cs.N, NCH);
  const int HoWo = cs.Ho * cs.Wo;
  int z = cdiv(HoWo, 128 * PIX);
  // aim for at least ~1 wave of CTAs
  while ((long long)b * groups * nchunks * z < 148 && z * 64 < HoWo) ++z;
  dim3 grid(b, groups * nchunks, z);
  conv_fwd_f32_kernel<NCH, PIX><<<grid, 128, smem, st>>>(cs, src, theta0, theta1, out0, out1, z);
}

// ------------------------------------------------------------------ conv backward: dX
// din[img][c][y][x] = [a_in > 0] * sum_{n,ky,kx} dout[img][n][(y-ky)/s][(x-kx)/s] W[n][c][ky][kx]
template <int CCH>
__global__ void __launch_bounds__(128) conv_bwd_dx_f32_kernel(ConvShape cs, const float* __restrict__ dout,
                                                              const float* __restrict__ theta,
                                                              const float* __restrict__ a_in, float* din) {
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  const int img = blockIdx.x;
  const int c0 = blockIdx.y * CCH;
  const int HoWo = cs.Ho * cs.Wo;
  const int kk = cs.k * cs.k;
  float* s_d = sm;                               // [N][HoWo]
  float* s_w = sm + ((cs.N * HoWo + 3) & ~3);    // [N][k][k][CCH]
  const float* dimg = dout + (long long)img * cs.N * HoWo;
  for (int i = threadIdx.x; i < cs.N * HoWo; i += blockDim.x) s_d[i] = dimg[i];
  for (int e = threadIdx.x; e < cs.N * kk * CCH; e += blockDim.x) {
    const int cl = e % CCH, t = (e / CCH) % kk, n = e / (CCH * kk);
    const int c = c0 + cl;
    s_w[e] = (c < cs.C) ? theta[cs.w_off + ((long long)n * cs.C + c) * kk + t] : 0.0f;
  }
  __syncthreads();
  const int HW = cs.H * cs.W;
  for (int p = threadIdx.x; p < HW; p += blockDim.x) {
    const int y = p / cs.W, x = p % cs.W;
    float acc[CCH];
#pragma unroll
    for (int cl = 0; cl < CCH; ++cl) acc[cl] = 0.0f;
    for (int ky = y % cs.s; ky < cs.k; ky += cs.s) {
      const int oy = (y - ky) / cs.s;
      if (y - ky < 0 || oy >= cs.Ho) continue;
      for (int kx = x % cs.s; kx < cs.k; kx += cs.s) {
        const int ox = (x - kx) / cs.s;
        if (x - kx < 0 || ox >= cs.Wo) continue;
        const int q = oy * cs.Wo + ox;
        const int t = ky * cs.k + kx;
        for (int n = 0; n < cs.N; ++n) {
          const float d = s_d[n * HoWo + q];
          const float* w = s_w + (n * kk + t) * CCH;
#pragma unroll
          for (int cl = 0; cl < CCH; ++cl) acc[cl] = fmaf(d, w[cl], acc[cl]);
        }
      }
    }
#pragma unroll
    for (int cl = 0; cl < CCH; ++cl) {
      const int c = c0 + cl;
      if (c < cs.C) {
        const long long o = ((long long)img * cs.C + c) * HW + p;
        din[o] = a_in[o] > 0.0f ? acc[cl] : 0.0f;  // ReLU'(0) = 0 (A17)
      }
    }
  }
}

void launch_conv_bwd_dx_f32(const ConvShape& cs, const float* dout, const float* theta, const float* a_in,
                            float* din, int b, cudaStream_t st) {
  constexpr int CCH = 8;
  const size_t smem = (size_t)(((cs.N * cs.Ho * cs.Wo + 3) & ~3) + cs.N * cs.k * cs.k * CCH) * sizeof(float);
  dim3 grid(b, cdiv(cs.C, CCH));
  conv_bwd_dx_f32_kernel<CCH><<<grid, 128, smem, st>>>(cs, dout, theta, a_in, din);
}

// ------------------------------------------------------------------ conv backward: dW, db
// partial[img][(n,c,ky,kx)] = sum_p dout[img][n][p] * in[img][c][oy*s+ky][ox*s+kx]
// partial[img][NCkk + n]    = sum_p dout[img][n][p]
// One thread per (n, c, ky) row with k accumulators over kx.
template <int KMAX>
__global__ void __launch_bounds__(256) conv_bwd_dw_f32_kernel(ConvShape cs, const float* __restrict__ dout,
                                                              ImgSrc src, float* partial) {
  extern __shared__ float4 sm4[];
  float* sm = reinterpret_cast<float*>(sm4);
  const int img = blockIdx.x;
  const int CHW = cs.C * cs.H * cs.W;
  const int HoWo = cs.Ho * cs.Wo;
  float* s_in = sm;
  float* s_d = sm + ((CHW + 3) & ~3);
  stage_image(s_in, src, 0, img, CHW);
  const float* dimg = dout + (long long)img * cs.N * HoWo;
  for (int i = threadIdx.x; i < cs.N * HoWo; i += blockDim.x) s_d[i] = dimg[i];
  __syncthreads();
  const long long E = (long long)cs.N * cs.C * cs.k * cs.k + cs.N;
  float* prow = partial + (long long)img * E;
  const int rows = cs.N * cs.C * cs.k;
  const int row = blockIdx.y * blockDim.x + threadIdx.x;
  if (row < rows) {
    const int ky = row % cs.k, c = (row / cs.k) % cs.C, n = row / (cs.k * cs.C);
    float acc[KMAX];
#pragma unroll
    for (int i = 0; i < KMAX; ++i) acc[i] = 0.0f;
    const float* dn = s_d + n * HoWo;
    const float* ic = s_in + c * cs.H * cs.W + ky * cs.W;
    for (int oy = 0; oy < cs.Ho; ++oy)
      for (int ox = 0; ox < cs.Wo; ++ox) {
        const float d = dn[oy * cs.Wo + ox];
        const float* xin = ic + oy * cs.s * cs.W + ox * cs.s;
#pragma unroll
        for (int kx = 0; kx < KMAX; ++kx)
          if (kx < cs.k) acc[kx] = fmaf(d, xin[kx], acc[kx]);
      }
    for (int kx = 0; kx < cs.k; ++kx) prow[(long long)row * cs.k + kx] = acc[kx];
  }
  if (blockIdx.y == 0) {
    for (int n = threadIdx.x; n < cs.N; n += blockDim.x) {
      float s = 0.0f;
      for (int p = 0; p < HoWo; ++p) s += s_d[n * HoWo + p];
      prow[E - cs.N + n] = s;
    }
  }
}

void launch_conv_bwd_dw_f32(const ConvShape& cs, const float* dout, const ImgSrc& src, float* partial, int b,
                            cudaStream_t st) {
  const int CHW = cs.C * cs.H * cs.W;
  const size_t smem = (size_t)(((CHW + 3) & ~3) + cs.N * cs.Ho * cs.Wo) * sizeof(float);
  const int rows = cs.N * cs.C * cs.k;
  dim3 grid(b, cdiv(rows, 256));
#define DW_CASE(KM) conv_bwd_dw_f32_kernel<KM><<<grid, 256, smem, st>>>(cs, dout, src, partial);
  if (cs.k <= 4) DW_CASE(4)
  else if (cs.k <= 8) DW_CASE(8)
  else DW_CASE(16)
#undef DW_CASE
}

// dst[e] += sum_{row = 0..rows-1} partial[row][e]   (fixed order)
__global__ void reduce_rows_kernel(const float* __restrict__ partial, int rows, long long E, float* dst) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= E) return;
  float s = 0.0f;
  for (int r = 0; r < rows; ++r) s += partial[(long long)r * E + e];
  dst[e] += s;
}

void launch_reduce_rows(const float* partial, int rows, long long E, float* dst, cudaStream_t st) {
  reduce_rows_kernel<<<cdiv(E, 256), 256, 0, st>>>(partial, rows, E, dst);
}

// ------------------------------------------------------------------ generic SIMT GEMM
// C(m,n) (op)= sum_k A(m,k) B(k,n); 64x64 tile, BK = 16, 256 threads, 4x4 per thread.
constexpr int GBM = 64, GBN = 64, GBK = 16;

__device__ __forceinline__ float epi_apply(const GemmArgs& a, int g, int m, int n, float v) {
  switch (a.epi) {
    case EPI_BIAS_RELU: {
      const float t = v + a.bias[g][n];
      return t > 0.0f ? t : 0.0f;
    }
    case EPI_BIAS: return v + a.bias[g][n];
    case EPI_MASK: return a.mask[g][m * a.smm + n * a.smn] > 0.0f ? v : 0.0f;
    default: return v;
  }
}

__global__ void __launch_bounds__(256) gemm_f32_kernel(GemmArgs a) {
  __shared__ float As[GBK][GBM + 4];
  __shared__ float Bs[GBK][GBN + 4];
  const int g = blockIdx.z / a.splits;
  const int split = blockIdx.z % a.splits;
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  const int kper = ((a.K + a.splits - 1) / a.splits + GBK - 1) / GBK * GBK;
  const int kb = split * kper, ke = min(a.K, kb + kper);
  const float* A = a.A[g];
  const float* B = a.B[g];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  float acc[4][4] = {};
  for (int k0 = kb; k0 < ke; k0 += GBK) {
    // A tile: 64 x 16
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * 256;
      int mm, kk;
      if (a.sak == 1) { kk = e % GBK; mm = e / GBK; } else { mm = e % GBM; kk = e / GBM; }
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < a.M && k < ke) ? A[(long long)m * a.sam + (long long)k * a.sak] : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * 256;
      int nn, kk;
      if (a.sbk == 1) { kk = e % GBK; nn = e / GBK; } else { nn = e % GBN; kk = e / GBN; }
      const int n = n0 + nn, k = k0 + kk;
      Bs[kk][nn] = (n < a.N && k < ke) ? B[(long long)k * a.sbk + (long long)n * a.sbn] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      const float4 av = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 bv = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float am[4] = {av.x, av.y, av.z, av.w};
      const float bn[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(am[i], bn[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m >= a.M || n >= a.N) continue;
      if (a.splits > 1) {
        a.partial[(((long long)g * a.splits + split) * a.M + m) * a.N + n] = acc[i][j];
      } else {
        float* c = a.C[g] + (long long)m * a.scm + (long long)n * a.scn;
        const float v = epi_apply(a, g, m, n, acc[i][j]);
        if (a.epi == EPI_ACCUM) *c += v; else *c = v;
      }
    }
}

__global__ void gemm_splitk_reduce_kernel(GemmArgs a) {
  const long long MN = (long long)a.M * a.N;
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int g = blockIdx.y;
  if (e >= MN) return;
  const int m = (int)(e / a.N), n = (int)(e % a.N);
  float s = 0.0f;
  for (int sp = 0; sp < a.splits; ++sp) s += a.partial[((long long)g * a.splits + sp) * MN + e];
  float* c = a.C[g] + (long long)m * a.scm + (long long)n * a.scn;
  const float v = epi_apply(a, g, m, n, s);
  if (a.epi == EPI_ACCUM) *c += v; else *c = v;
}

void launch_gemm_f32(const GemmArgs& g, cudaStream_t st) {
  dim3 grid(cdiv(g.N, GBN), cdiv(g.M, GBM), g.groups * g.splits);
  gemm_f32_kernel<<<grid, 256, 0, st>>>(g);
  if (g.splits > 1) {
    dim3 rg(cdiv((long long)g.M * g.N, 256), g.groups);
    gemm_splitk_reduce_kernel<<<rg, 256, 0, st>>>(g);
  }
}

// dst[h] += sum_j dz[j][h]
__global__ void bias_grad_kernel(const float* __restrict__ dz, int b, int H, float* dst) {
  int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= H) return;
  float s = 0.0f;
  for (int j = 0; j < b; ++j) s += dz[(long long)j * H + h];
  dst[h] += s;
}

void launch_bias_grad(const float* dz, int b, int H, float* dst, cudaStream_t st) {
  bias_grad_kernel<<<cdiv(H, 256), 256, 0, st>>>(dz, b, H, dst);
}

// ------------------------------------------------------------------ a15 acting head (Q only)
__global__ void q_head_f32_kernel(const float* __restrict__ act, const float* __restrict__ theta, long long w_off,
                                  long long b_off, int H, int A, int n, float* q, int* argmax) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= n) return;
  const float* hv = act + (long long)warp * H;
  float best = 0.0f;
  int barg = 0;
  for (int a = 0; a < A; ++a) {
    const float* w = theta + w_off + (long long)a * H;
    float s = 0.0f;
    for (int i = lane; i < H; i += 32) s = fmaf(w[i], hv[i], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float v = s + theta[b_off + a];
    if (lane == 0) q[(long long)warp * A + a] = v;
    if (a == 0 || v > best) { best = v; barg = a; }
  }
  if (lane == 0 && argmax) argmax[warp] = barg;
}

void launch_q_head_f32(const float* act, const float* theta, long long w_off, long long b_off, int H, int A, int n,
                       float* q, int* argmax, cudaStream_t st) {
  q_head_f32_kernel<<<cdiv((long long)n * 32, 256), 256, 0, st>>>(act, theta, w_off, b_off, H, A, n, q, argmax);
}

// Opt every kernel that stages a whole image into up to 227 KB of dynamic shared
// memory. Called once at context creation (never inside a graph capture).
void init_f32_kernel_attrs() {
  const int mx = 227 * 1024;
  cudaFuncSetAttribute(conv_fwd_f32_kernel<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(conv_bwd_dx_f32_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(conv_bwd_dw_f32_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(conv_bwd_dw_f32_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(conv_bwd_dw_f32_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
}

}  // namespace dqn
