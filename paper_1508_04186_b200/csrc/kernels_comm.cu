// kernels_comm.cu — NEXT-1: the whole server round of Alg. 2 in ONE kernel over
// NVLink peer memory (one process per GPU, buffers mapped with CUDA IPC):
//
//   push   : every rank reads the slice it owns, [rank*S, (rank+1)*S), of EVERY
//            replica's gradient accumulator G_p directly from the peers' HBM and sums it
//            in rank order p = 0..N-1 (deterministic; the oracle sums in rank order too)
//   update : mean over N*n_push, RMSProp on the owned shard (A4/A5/A7/A24)
//   fetch  : the updated shard is stored straight into every replica's working copy
//            theta_local (fp32 and, on the bf16 path, bf16) on every peer
//
// replacing ncclReduceScatter + update kernel + ncclAllGather (+ the bf16 conversion).
// Two cross-GPU barriers with monotone counters (no reset, graph-replayable):
//   A (gradients complete): each rank stores `round` into flags[rank] on every peer
//     (release, system scope) and waits until all N entries of its own flags reach it;
//   B (shards delivered): every block adds 1 to done[] on every peer after its remote
//     stores (release). The acquire half (done >= rounds * N * blocks, then clear G — all
//     peers have read it by then) runs in the next step's first kernel
//     (fused_acquire.cuh), so stragglers overlap the next forward's replay gather.
// Every spin is bounded; on timeout the kernel records an error and falls through, so
// a desynchronised group cannot hang the GPU.
#include <algorithm>
#include "dqn_internal.h"
#include "fused_acquire.cuh"
#include "pdl.cuh"

namespace dqn {

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(k) \
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[(round_idx % 64) * 4 + (k)] = gtimer()

__global__ void __launch_bounds__(256) server_round_kernel(ServerRoundArgs a) {
  pdl_wait();     // G of this rank is complete (the backward kernels precede in stream order)
  pdl_trigger();  // the next step's gather does not depend on this round
  // round id and round index from the step counter (identical on every rank): the head has
  // already advanced T to (step + 1), and push rounds end exactly at (step + 1) % n_push == 0
  const unsigned long long T = a.ctr->T;
  const unsigned long long round_idx = T / (unsigned long long)a.n_push;
  TRACE(0);
  // ---- barrier A
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      __threadfence_system();
      for (int p = 0; p < a.world; ++p) st_release_sys(a.flags[p] + a.rank, T);
    }
    for (int p = 0; p < a.world; ++p) {
      long long spin = 0;
      while (ld_acquire_sys(a.my_flags + p) < T) {
        __nanosleep(32);
        if (++spin > kSpinLimit) {
          atomicOr(&a.ctr->bad_input, 0x80000000u);  // peer barrier timeout (reported as ECUDA by the host)
          break;
        }
      }
    }
  }
  __syncthreads();
  TRACE(1);
  // ---- reduce (rank order) + RMSProp + deliver, 16-byte vectors, grid-stride over the owned shard
  const long long n4 = a.shard / 4;
  const long long base = (long long)a.rank * a.shard;
  unsigned bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    // all N peer loads in flight at once (NVLink latency ~1-2 us), then summed in rank order
    float4 v[kMaxWorld];
#pragma unroll
    for (int p = 0; p < kMaxWorld; ++p)
      if (p < a.world) v[p] = __ldcg(reinterpret_cast<const float4*>(a.grad[p] + base) + i);
    float4 acc = v[0];
#pragma unroll
    for (int p = 1; p < kMaxWorld; ++p)
      if (p < a.world) { acc.x += v[p].x; acc.y += v[p].y; acc.z += v[p].z; acc.w += v[p].w; }
    float4 t4 = reinterpret_cast<const float4*>(a.theta_master)[i];
    float4 r4 = reinterpret_cast<const float4*>(a.rms)[i];
    float tv[4] = {t4.x, t4.y, t4.z, t4.w}, rv[4] = {r4.x, r4.y, r4.z, r4.w};
    const float gv[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float gb = gv[q] * a.inv_div;
      if (isfinite(gb)) {
        const float rr = a.rho * rv[q] + a.omr * gb * gb;
        rv[q] = rr;
        tv[q] = tv[q] - a.lr * gb * rsqrtf(rr + a.eps);
      } else {
        ++bad;
      }
    }
    t4 = make_float4(tv[0], tv[1], tv[2], tv[3]);
    reinterpret_cast<float4*>(a.theta_master)[i] = t4;
    reinterpret_cast<float4*>(a.rms)[i] = make_float4(rv[0], rv[1], rv[2], rv[3]);
    uint2 h;
    {
      __nv_bfloat162 lo = __floats2bfloat162_rn(t4.x, t4.y), hi = __floats2bfloat162_rn(t4.z, t4.w);
      h.x = *reinterpret_cast<uint32_t*>(&lo);
      h.y = *reinterpret_cast<uint32_t*>(&hi);
    }
    for (int p = 0; p < a.world; ++p) {
      reinterpret_cast<float4*>(a.theta_local[p] + base)[i] = t4;
      if (a.theta_local_bf16[p]) reinterpret_cast<uint2*>(a.theta_local_bf16[p] + base)[i] = h;
    }
  }
  if (bad) atomicAdd(&a.ctr->nonfinite, bad);
  // ---- barrier B, release half: the CTA barrier orders every thread's remote stores before
  // thread 0's system-scope release, which is cumulative (no per-thread system fence needed)
  __syncthreads();
  TRACE(2);
  if (threadIdx.x == 0)
    for (int p = 0; p < a.world; ++p) red_release_sys_add(a.done[p], 1ull);
  TRACE(3);
}

// fp32 path: the acquire half as its own (tiny) kernel at the start of a step
__global__ void fused_round_acquire_kernel(FusedAcquire f) {
  pdl_sync();
  fused_round_acquire(f);
}

void launch_fused_round_acquire(const FusedAcquire& f, cudaStream_t st) {
  launch_pdl(fused_round_acquire_kernel, dim3(148), dim3(256), 0, st, f);
}

// one 16-byte vector per thread (no cross-block waits inside the kernel, so no residency bound)
int server_round_blocks(long long shard) {
  const long long b = (shard / 4 + 255) / 256;
  return (int)(b < 1 ? 1 : b);
}

void launch_server_round(const ServerRoundArgs& a, cudaStream_t st) {
  launch_pdl(server_round_kernel, dim3(server_round_blocks(a.shard)), dim3(256), 0, st, a);
}

}  // namespace dqn
