// head_finish.cuh — the cross-sample half of the TD head (a6), one output element per call,
// shared by the standalone head_finish kernel (fp32 path) and the fused FC-backward launch
// (bf16 path). Every sum over samples runs in ascending j (deterministic).
//   e in [0, A*H)         dW_o[a][u] += sum_{j: a_j = a} dQ_j h_j[u]
//   e in [A*H, A*H + A)   db_o[a]    += sum_{j: a_j = a} dQ_j
//   next H entries        db_fc[u]   += sum_j dH_j[u]          (previous layer is an FC)
//   e == A*H + A + H      loss = (1/b) sum 1/2 delta_j^2 (A27) into the diagnostics ring; T <- T + 1
#pragma once
#include "dqn_internal.h"

namespace dqn {

__device__ __forceinline__ int head_finish_elems(const HeadArgs& h) { return h.A * h.H + h.A + h.H + 1; }

__device__ __forceinline__ void head_finish_elem(const HeadArgs& h, int e) {
  const int H = h.H, A = h.A;
  const float* h0 = h.fc_partial ? h.act_out[0] : h.act[0];
  if (e < A * H) {
    const int a = e / H, u = e % H;
    float s = 0.0f;
    for (int j = 0; j < h.b; ++j)
      if (h.s_act[j] == a) s = fmaf(h.s_dq[j], h0[(long long)j * H + u], s);
    h.grad[h.w_off + e] += s;
  } else if (e < A * H + A) {
    const int a = e - A * H;
    float s = 0.0f;
    for (int j = 0; j < h.b; ++j)
      if (h.s_act[j] == a) s += h.s_dq[j];
    h.grad[h.b_off + a] += s;
  } else if (e < A * H + A + H) {
    if (h.prev_is_fc) {
      const int u = e - A * H - A;
      float s = 0.0f;
      for (int j = 0; j < h.b; ++j) s += h.dH[(long long)j * H + u];
      h.grad[h.prev_b_off + u] += s;
    }
  } else if (e == A * H + A + H) {
    const unsigned long long T = h.ctr->T;
    float l = 0.0f;
    for (int j = 0; j < h.b; ++j) l += h.s_loss[j];
    h.diag_loss[T % kDiagSteps] = l / (float)h.b;
    h.ctr->T = T + 1;  // this step is complete for the sampler
  }
}

// dW_o[a][u] of a warp whose 32 lanes hold consecutive u of the same action a (H % 32 == 0): the samples with
// a_j = a are found 32 at a time by a ballot over the staged actions and their h_j[u] loads go out 8 at a
// time. The fmaf chain runs over the same samples in the same ascending order as head_finish_elem (bit-identical),
// without one exposed load latency per matching sample.
__device__ __forceinline__ float head_finish_dwo_warp(const HeadArgs& h, const float* h0, const int* s_act,
                                                      const float* s_dq, int a, int u) {
  const int lane = threadIdx.x & 31;
  float s = 0.0f;
  int js[8], nn = 0;
  auto flush = [&]() {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = k < nn ? h0[(long long)js[k] * h.H + u] : 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < nn) s = fmaf(s_dq[js[k]], v[k], s);
    nn = 0;
  };
  for (int j0 = 0; j0 < h.b; j0 += 32) {
    unsigned m = __ballot_sync(0xffffffffu, j0 + lane < h.b && s_act[j0 + lane] == a);
    while (m) {
      const int j = j0 + __ffs(m) - 1;
      m &= m - 1;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k == nn) js[k] = j;
      if (++nn == 8) flush();
    }
  }
  if (nn) flush();
  return s;
}

}  // namespace dqn
