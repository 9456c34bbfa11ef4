// kernels_head.cu — a6, the fused TD head of Alg. 1, shared by both
// precisions. Two launches:
//
// head_sample (one CTA per sample j, so the b samples run in parallel):
//   [bf16 path] h_j, h'_j = ReLU(sum over FC split-K partials + b_fc)   (a5's reduction, fused here)
//   Q'_j = W^_o h'_j + b^_o ; m_j = max_a' Q'_j, g_j = argmax (warp-shuffle reduction; lowest index on ties, A20)
//   y_j = term_j ? r_j : r_j + gamma m_j                              (a select, A14)
//   delta_j = Q(s_j; theta)_{a_j} - y_j ; dQ_j = clamp(delta_j, -c, c) / b at a_j only (A2, A3)
//   dH_j = dQ_j W_o[a_j] * [h_j > 0]        (d pre-activation of the previous layer, ReLU'(0) = 0)
// head_finish (cross-sample sums in ascending j: deterministic):
//   dW_o[a] += sum_{j: a_j = a} dQ_j h_j ; db_o[a] += sum dQ_j ; db_fc += sum_j dH_j
//   loss = (1/b) sum 1/2 delta^2 (A27) ; T <- T + 1 (the sampler's step counter)
#include "dqn_internal.h"
#include "head_finish.cuh"
#include "pdl.cuh"
#include "step_trace.cuh"

namespace dqn {

constexpr int HS_THREADS = 256;
constexpr int HS_AMAX = 32;
constexpr int HS_MAX_SPLITS = kHeadMaxSplits;

// dynamic smem: h [H] | h' [H] | W^_o [A][H] | W_o[a_j] [H]
// CH: FC split-K partials in flight per thread and group (all of them at small b, where the head is on the
// latency-bound critical path; 8 at large b, where 4 CTAs per SM need the register budget)
// MC > 1: the CTAs of a cluster of MC share one read of theta^'s output layer: the cluster's first CTA issues a
// TMA bulk copy multicast into every member's shared memory (one L2 read instead of MC; the layer is the same
// for every sample)
template <int CH, int MINB, int MC>
__global__ void __launch_bounds__(HS_THREADS, MINB) head_sample_kernel(HeadArgs h) {
  extern __shared__ float4 sm4[];
  const int H = h.H, A = h.A, j = blockIdx.x;
  float* s_h0 = reinterpret_cast<float*>(sm4);  // [H]
  float* s_h1 = s_h0 + H;                       // [H]
  float* s_wt = s_h1 + H;                       // [A][H]: theta^'s output layer
  float* s_wa = s_wt + A * H;                   // [H]: theta's output-layer row of the taken action
  __shared__ float s_q[HS_AMAX], s_bt[HS_AMAX];
  __shared__ float s_qa_b, s_qa;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = HS_THREADS / 32;
  st_stamp(h.st_id, 0);
  // everything here is at least two launches old (PDL-safe): the sampled slot and its (a, r,
  // terminal), and the output layers of theta (updated by the previous step) and theta^
  const int slot = __ldg(h.idx + j);
  const int act = __ldg(h.ring_a + slot);
  const float r = __ldg(h.ring_r + slot);
  const uint8_t term = __ldg(h.ring_term + slot);
  __shared__ __align__(8) uint64_t s_mbar;
  if (MC > 1) {
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
    const uint32_t bytes = (uint32_t)(A * H * 4);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    }
    // every member's barrier is initialised and armed before the multicast can complete on it
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (rank == 0 && threadIdx.x == 0) {
      const uint16_t mask = (uint16_t)((1u << MC) - 1);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
          "%4;" ::"r"((uint32_t)__cvta_generic_to_shared(s_wt)),
          "l"(h.theta_hat + h.w_off), "r"(bytes), "r"(bar), "h"(mask)
          : "memory");
    }
  } else {
    for (int e = threadIdx.x; e < A * H; e += HS_THREADS) s_wt[e] = __ldg(h.theta_hat + h.w_off + e);
  }
  for (int u = threadIdx.x; u < H; u += HS_THREADS) s_wa[u] = __ldg(h.theta + h.w_off + (long long)act * H + u);
  if (threadIdx.x < A) s_bt[threadIdx.x] = __ldg(h.theta_hat + h.b_off + threadIdx.x);
  if (threadIdx.x == 0) s_qa_b = __ldg(h.theta + h.b_off + act);
  pdl_sync();
  st_stamp(h.st_id, 1);
  // ---- the two hidden activation rows of sample j
  if (h.fc_partial) {
    const int ns = h.fc_splits;
    for (int u = threadIdx.x; u < H; u += HS_THREADS) {
      // the splits of both groups, CH at a time in flight, summed in split order (zeros past ns are exact)
      float s2[2] = {0.0f, 0.0f};
      for (int s0 = 0; s0 < ns; s0 += CH) {
        float pv[2][CH];
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const float* p = h.fc_partial + (long long)g * ns * h.fc_split_stride + (long long)j * H + u;
#pragma unroll
          for (int k = 0; k < CH; ++k)
            pv[g][k] = s0 + k < ns ? __ldcg(p + (long long)(s0 + k) * h.fc_split_stride) : 0.0f;
        }
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int k = 0; k < CH; ++k) s2[g] += pv[g][k];
      }
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const float s = s2[g];
        const float v = fmaxf(s + __ldg(h.fc_bias[g] + u), 0.0f);
        (g ? s_h1 : s_h0)[u] = v;
        h.act_out[g][(long long)j * H + u] = v;
      }
    }
  } else {
    for (int u = threadIdx.x; u < H; u += HS_THREADS) {
      s_h0[u] = __ldg(h.act[0] + (long long)j * H + u);
      s_h1[u] = __ldg(h.act[1] + (long long)j * H + u);
    }
  }
  if (MC > 1) {  // theta^'s output layer has landed (phase 0 of this CTA's barrier)
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_mbar);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(bar)
                   : "memory");
  }
  __syncthreads();
  // ---- Q'(s'_j; theta^) for every action (warp per action) and Q(s_j; theta)_{a_j}
  for (int a = warp; a <= A; a += nw) {
    const bool target = a < A;
    const float* w = target ? s_wt + a * H : s_wa;
    const float* x = target ? s_h1 : s_h0;
    float s = 0.0f;
    for (int i = lane; i < H; i += 32) s = fmaf(w[i], x[i], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      if (target) s_q[a] = s + s_bt[a];
      else s_qa = s + s_qa_b;
    }
  }
  __syncthreads();
  __shared__ float s_dq;
  if (warp == 0) {
    // m_j = max_a' Q'_j and its argmax by a warp-shuffle reduction over the actions (lane a holds Q'_a,
    // A <= 32); ties keep the lowest index (A20)
    float best = lane < A ? s_q[lane] : -INFINITY;
    int barg = lane < A ? lane : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oa = __shfl_xor_sync(0xffffffffu, barg, o);
      if (ob > best || (ob == best && oa < barg)) { best = ob; barg = oa; }
    }
    if (lane == 0) {
      const float y = term ? r : r + h.gamma * best;  // a select, never (1 - term) * m (A14)
      const float delta = s_qa - y;
      float dc = delta;
      if (h.clip > 0.0f) dc = fminf(fmaxf(dc, -h.clip), h.clip);  // error clip (A3)
      const float dq = dc / (float)h.b;
      s_dq = dq;
      h.s_dq[j] = dq;
      h.s_act[j] = act;
      h.s_loss[j] = 0.5f * delta * delta;
      h.s_delta[j] = delta;
      const int dslot = (int)(h.ctr->T % kDiagSteps);
      h.diag_idx[(long long)dslot * h.b + j] = slot;
      h.diag_amax[(long long)dslot * h.b + j] = barg;
      h.diag_delta[(long long)dslot * h.b + j] = delta;
    }
  }
  __syncthreads();
  const float dq = s_dq;
  for (int u = threadIdx.x; u < H; u += HS_THREADS) {
    const float d = s_h0[u] > 0.0f ? dq * s_wa[u] : 0.0f;
    h.dH[(long long)j * H + u] = d;
    if (h.dH_bf16) h.dH_bf16[(long long)j * H + u] = __float2bfloat16_rn(d);
  }
  st_stamp(h.st_id, 2);
}

// Cross-sample sums; e in [0, A*H) -> dW_o, [A*H, A*H + A) -> db_o, then H entries of db_fc.
__global__ void head_finish_kernel(HeadArgs h) {
  pdl_sync();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < head_finish_elems(h)) head_finish_elem(h, e);
}

size_t head_smem_bytes(int A, int H, int b) {
  (void)b;
  return (size_t)(3 + A) * H * sizeof(float);
}

void init_head_kernel_attrs() {
  // the 227 KB opt-in limit includes the kernel's static shared memory
  cudaFuncSetAttribute(head_sample_kernel<HS_MAX_SPLITS, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  cudaFuncSetAttribute(head_sample_kernel<8, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  cudaFuncSetAttribute(head_sample_kernel<8, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  cudaGetLastError();  // an attribute refusal only limits the largest head; validate_cfg bounds it
}

void launch_head_f32(const HeadArgs& h, cudaStream_t st, bool with_finish) {
  const size_t smem = head_smem_bytes(h.A, h.H, h.b);
  if (h.b <= 128)
    launch_pdl(head_sample_kernel<HS_MAX_SPLITS, 1, 1>, dim3(h.b), dim3(HS_THREADS), smem, st, h);
  else if (h.b % 4 == 0 && h.w_off % 4 == 0 && (h.A * h.H) % 4 == 0)  // 16-byte bulk copies
    launch_pdl_cluster(head_sample_kernel<8, 4, 4>, dim3(h.b), dim3(HS_THREADS), smem, 4, st, h);
  else
    launch_pdl(head_sample_kernel<8, 4, 1>, dim3(h.b), dim3(HS_THREADS), smem, st, h);
  if (!with_finish) return;  // the bf16 path runs the finish inside its fused FC-backward launch
  const int n = h.A * h.H + h.A + h.H + 1;
  launch_pdl(head_finish_kernel, dim3((n + 255) / 256), dim3(256), 0, st, h);
}

DQN_STEP_TRACE_HOST(head)

}  // namespace dqn
