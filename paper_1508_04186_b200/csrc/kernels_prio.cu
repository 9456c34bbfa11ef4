// kernels_prio.cu — the prioritized replay variant (NEXT-4; "a more sophisticated sampling strategy might
// emphasize transitions from which we can learn the most"; the rule is DESIGN.md reading A41).
//
// A 32-ary sum tree over the replay slots in HBM: level 0 = the 32^K leaf priorities, node i of level l + 1 = the
// fp32 butterfly sum of its 32 children (one warp: v += shfl_xor(v, o), o = 16 .. 1). A warp per tree node is the
// natural B200 shape: the 32 children are one coalesced 128-byte load, the sum one shuffle butterfly, and K = 4
// levels cover a 1M-slot replay (a binary tree would need 20 dependent L2 round trips per draw).
//   prio_sample  : warp per draw; t_j = ((j + u_j) / b) S (stratified), then a fixed-order scan of each node's
//                  32 children from the root down. Every compare / add is an explicit round-to-nearest fp32 op
//                  in the oracle's order (oracle/prio.py), so draws are bit-identical given the same leaves.
//   prio_update  : one CTA after the TD head: p_j = (|delta_j| + eps)^alpha into the slot's leaf, the max priority,
//                  then the changed nodes level by level, 8 per warp with their loads in flight.
//   prio_push    : one CTA after a Store: the stored slots' leaves = the max priority, their ancestors rebuilt.
#include "dqn_internal.h"
#include "pdl.cuh"
#include "philox.cuh"

namespace dqn {

namespace {
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float butterfly32(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// node i of level l (warp-collective): the butterfly sum of its 32 children at level l - 1, stored by lane 0
__device__ __forceinline__ void rebuild_node(const PrioTree& t, int l, long long i) {
  const float c = __ldcg(t.node + t.off[l - 1] + i * 32 + (threadIdx.x & 31));
  const float s = butterfly32(c);
  if ((threadIdx.x & 31) == 0) t.node[t.off[l] + i] = s;
}
}  // namespace

__global__ void __launch_bounds__(256) prio_sample_kernel(PrioTree t, int b, unsigned long long seed, unsigned rank,
                                                          const DevCounters* ctr, int* idx) {
  pdl_sync();  // the tree: the previous step's update and any Store came before
  const int lane = threadIdx.x & 31, j = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (j >= b) return;
  const unsigned long long T = ctr->T;
  uint32_t c0 = (uint32_t)j, c1 = (uint32_t)T, c2 = (uint32_t)(T >> 32), c3 = rank;
  philox4x32_10(c0, c1, c2, c3, (uint32_t)seed, (uint32_t)(seed >> 32));
  const float u = (float)(c2 >> 8) * (1.0f / 16777216.0f);  // word 2, top 24 bits: exact in fp32
  const float S = __ldcg(t.node + t.off[t.K]);
  float r = __fmul_rn(__fadd_rn((float)j, u), __fdiv_rn(S, (float)b));
  long long node = 0;
  for (int l = t.K; l >= 1; --l) {
    const float c = __ldcg(t.node + t.off[l - 1] + node * 32 + lane);
    // the scan of A41, executed identically by every lane on the broadcast children
    float s = 0.0f, pick_s = 0.0f, last_s = 0.0f;
    int pick = -1, last = -1;
    for (int k = 0; k < 32; ++k) {
      const float ck = __shfl_sync(kFull, c, k);
      if (pick < 0) {
        if (ck > 0.0f) {
          if (r < __fadd_rn(s, ck)) {
            pick = k;
            pick_s = s;
          } else {
            last = k;
            last_s = s;
          }
        }
        if (pick < 0) s = __fadd_rn(s, ck);
      }
    }
    if (pick < 0) {
      pick = last;
      pick_s = last_s;
    }
    if (pick < 0) {
      pick = 0;
      pick_s = 0.0f;
    }
    r = __fsub_rn(r, pick_s);
    node = node * 32 + pick;
  }
  if (lane == 0) idx[j] = (int)node;
}

// Duplicates of a slot in one minibatch carry the same transition and theta, hence the same delta and the same
// priority: every draw writes its leaf (the rule "the largest j writes" of A41 is unobservable), and a tree node
// shared by several draws is rebuilt once when the draws are sorted (the stratified descent is monotone in j,
// so equal parents are adjacent) and harmlessly more than once otherwise.
__global__ void __launch_bounds__(1024) prio_update_kernel(PrioTree t, int b, const int* idx, const float* delta,
                                                           int alpha_half, float eps, float* maxp) {
  extern __shared__ int s_idx[];  // [b]
  __shared__ float s_max[32];
  pdl_sync();  // delta and idx of this step (the TD head, the sampler)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  float m = 0.0f;
  for (int j = tid; j < b; j += blockDim.x) {
    const int i = idx[j];
    s_idx[j] = i;
    float p = __fadd_rn(fabsf(delta[j]), eps);
    if (alpha_half) p = __fsqrt_rn(p);
    t.node[t.off[0] + i] = p;
    m = fmaxf(m, p);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
  if (lane == 0) s_max[warp] = m;
  __syncthreads();  // also orders the leaf stores before the level-1 reads of other warps
  if (tid == 0) {
    float mm = *maxp;
    for (int w = 0; w < nw; ++w) mm = fmaxf(mm, s_max[w]);
    *maxp = mm;
  }
  constexpr int PW = 8;  // parents per warp and round: their 8 coalesced child loads in flight together
  for (int l = 1; l <= t.K; ++l) {
    const int sh = 5 * l;
    for (int j0 = warp * PW; j0 < b; j0 += nw * PW) {
      float c[PW];
      long long par[PW];
      bool need[PW];
#pragma unroll
      for (int q = 0; q < PW; ++q) {
        const int j = j0 + q;
        par[q] = j < b ? (long long)s_idx[j] >> sh : -1;
        need[q] = j < b && (j == 0 || ((long long)s_idx[j - 1] >> sh) != par[q]);
        c[q] = need[q] ? __ldcg(t.node + t.off[l - 1] + par[q] * 32 + lane) : 0.0f;
      }
#pragma unroll
      for (int q = 0; q < PW; ++q) {
        if (!need[q]) continue;
        const float sum = butterfly32(c[q]);
        if (lane == 0) t.node[t.off[l] + par[q]] = sum;
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) prio_push_kernel(PrioTree t, long long cap, long long first, long long m,
                                                         const float* maxp) {
  pdl_sync();  // the max priority of the previous step's update
  const float p = *maxp;
  const int tid = threadIdx.x, warp = tid >> 5, nw = blockDim.x >> 5;
  if (m > cap) m = cap;
  for (long long i = tid; i < m; i += blockDim.x) t.node[t.off[0] + (first + i) % cap] = p;
  __syncthreads();
  // the stored slots are one or two contiguous ranges (ring wrap): rebuild their ancestors level by level
  const long long a0 = first, a1 = (first + m < cap ? first + m : cap) - 1;
  const long long b1 = first + m > cap ? first + m - cap - 1 : -1;
  for (int l = 1; l <= t.K; ++l) {
    const long long lo = a0 >> (5 * l), hi = a1 >> (5 * l);
    for (long long i = lo + warp; i <= hi; i += nw) rebuild_node(t, l, i);
    if (b1 >= 0)
      for (long long i = warp; i <= (b1 >> (5 * l)); i += nw)
        if (i < lo || i > hi) rebuild_node(t, l, i);
    __syncthreads();
  }
}

void launch_prio_sample(const PrioTree& t, int b, unsigned long long seed, unsigned rank, const DevCounters* ctr,
                        int* idx, cudaStream_t st) {
  launch_pdl(prio_sample_kernel, dim3((b + 7) / 8), dim3(256), 0, st, t, b, seed, rank, ctr, idx);
}

void launch_prio_update(const PrioTree& t, int b, const int* idx, const float* delta, int alpha_half, float eps,
                        float* maxp, cudaStream_t st) {
  launch_pdl(prio_update_kernel, dim3(1), dim3(1024), (size_t)b * sizeof(int), st, t, b, idx, delta, alpha_half, eps,
             maxp);
}

void launch_prio_push(const PrioTree& t, long long cap, long long first, long long m, const float* maxp,
                      cudaStream_t st) {
  if (m <= 0) return;
  launch_pdl(prio_push_kernel, dim3(1), dim3(1024), 0, st, t, cap, first, m, maxp);
}

}  // namespace dqn
