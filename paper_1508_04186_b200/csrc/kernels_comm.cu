// kernels_comm.cu — NEXT-1: the whole server round of Alg. 2 in ONE kernel over
// NVLink peer memory (one process per GPU, buffers mapped with CUDA IPC):
//
//   push   : every rank reads the slice it owns, [rank*S, (rank+1)*S), of EVERY
//            replica's gradient accumulator G_p directly from the peers' HBM and sums it
//            in rank order p = 0..N-1 (deterministic; the oracle sums in rank order too)
//   update : mean over N*n_push, RMSProp on the owned shard (A4/A5/A7/A24)
//   fetch  : the updated shard is stored straight into every replica's working copy
//            theta_local (fp32 and, on the bf16 path, bf16) on every peer; on the bf16 path
//            the FC weight (98% of P) is read only as bf16, so its fp32 copy stays local
//            (theta_hat's fp32 copy and dqn_get_params gather it from the masters instead)
//
// replacing ncclReduceScatter + update kernel + ncclAllGather (+ the bf16 conversion).
// Two cross-GPU barriers with monotone counters (no reset, graph-replayable), built so that
// each rank issues ONE system-scope release per barrier (a system-scope fence costs
// microseconds and serialises when hundreds of CTAs issue it; measured in DESIGN.md):
//   A (gradients complete): block 0 fences (acq_rel, system scope) — G was completed by
//     the preceding kernels — and stores `T` into flags[rank] on every peer (relaxed);
//     every block polls its own flags with ld.acquire.sys until all N entries reach T;
//   B (shards delivered): the blocks join on a local counter at gpu scope (acq_rel RMW);
//     the last block to join fences at system scope and adds 1 to done[] on every peer:
//     by cumulativity every block's peer stores happen-before that add. The acquire half
//     (ld.acquire.sys polling until done >= rounds * N, then clear G — all peers have read
//     it by then) runs in the next step's first kernel (fused_acquire.cuh), so it overlaps
//     the next forward's replay gather.
// Every spin is bounded; on timeout the kernel records an error and falls through, so
// a desynchronised group cannot hang the GPU.
#include <algorithm>
#include "dqn_internal.h"
#include "fused_acquire.cuh"
#include "pdl.cuh"
#include "step_trace.cuh"
#include "wimg.cuh"

namespace dqn {

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// trace slots per round: 0-3 block 0 after pdl_wait / barrier A / work / release, 4 earliest
// block start, 5 latest block release, 6-7 next step's first kernel after pdl_wait / acquire,
// 8-10 next forward's entry / replay gather landed / past pdl_wait
#define TRACE(k) \
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[(round_idx % 64) * 16 + (k)] = gtimer()

__global__ void __launch_bounds__(256) server_round_kernel(ServerRoundArgs a) {
  st_stamp(ST_ROUND, 0);
  pdl_wait();     // G of this rank is complete (the backward kernels precede in stream order)
  st_stamp(ST_ROUND, 1);
  pdl_trigger();  // the next step's gather does not depend on this round
  // round id and round index from the step counter (identical on every rank): the head has
  // already advanced T to (step + 1), and push rounds end exactly at (step + 1) % n_push == 0
  const unsigned long long T = a.ctr->T;
  const unsigned long long round_idx = T / (unsigned long long)a.n_push;
  TRACE(0);
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    a.trace[((round_idx + 1) % 64) * 16 + 4] = ~0ull;
    a.trace[((round_idx + 1) % 64) * 16 + 14] = ~0ull;
  }
  if (a.trace && threadIdx.x == 0) atomicMin(a.trace + (round_idx % 64) * 16 + 4, gtimer());
  // ---- barrier A
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      fence_acq_rel_sys();
      for (int p = 0; p < a.world; ++p) st_relaxed_sys(a.flags[p] + a.rank, T);
    }
    for (int p = 0; p < a.world; ++p) spin_acquire_sys(a.my_flags + p, T, a.ctr);
  }
  __syncthreads();
  TRACE(1);
  if (a.trace && threadIdx.x == 0) {  // 13 / 14: last / first block past barrier A
    atomicMax(a.trace + (round_idx % 64) * 16 + 13, gtimer());
    atomicMin(a.trace + (round_idx % 64) * 16 + 14, gtimer());
  }
  // ---- reduce (rank order) + RMSProp + deliver, 16-byte vectors, grid-stride over the owned shard
  const long long n4 = a.shard / 4;
  const long long base = (long long)a.rank * a.shard;
  unsigned bad = 0;
  // one float4 per thread; with a conv prefix (conv4 > 0) its float4s are spread conv_per_block per block over the
  // first nb_c blocks (the weight image's scattered peer stores then come from nb_c SMs instead of conv4 / 256),
  // the rest of those blocks and all later blocks take the remaining float4s in order
  const int cpb = a.conv_per_block;
  const long long nb_c = (a.conv4 + cpb - 1) / cpb;
  long long i;
  if ((long long)blockIdx.x < nb_c)
    i = (int)threadIdx.x < cpb ? (blockIdx.x * (long long)cpb + threadIdx.x < a.conv4 ? blockIdx.x * (long long)cpb + threadIdx.x : n4)
                               : a.conv4 + blockIdx.x * (long long)(256 - cpb) + (threadIdx.x - cpb);
  else
    i = a.conv4 + nb_c * (256 - cpb) + (blockIdx.x - nb_c) * 256LL + threadIdx.x;
  if (i < n4) {
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
    if (a.per_gradient) {  // A33: Alg. 2 literally, worker p's gradient then p+1's (rank order)
#pragma unroll
      for (int p = 0; p < kMaxWorld; ++p) {
        if (p >= a.world) break;
        const float gp[4] = {v[p].x, v[p].y, v[p].z, v[p].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float gb = gp[q] * a.inv_np;
          if (isfinite(gb)) {
            const float rr = a.rho * rv[q] + a.omr * gb * gb;
            rv[q] = rr;
            tv[q] = tv[q] - a.lr * gb * rsqrtf(rr + a.eps);
          } else {
            ++bad;
          }
        }
      }
    } else {
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
    const long long e = base + 4 * i;
    const bool f32_all = e < a.f32_peer_lo || e + 4 > a.f32_peer_hi;
    for (int p = 0; p < a.world; ++p) {
      if (p == a.rank || f32_all) reinterpret_cast<float4*>(a.theta_local[p] + base)[i] = t4;
      if (a.theta_local_bf16[p]) reinterpret_cast<uint2*>(a.theta_local_bf16[p] + base)[i] = h;
    }
    if (a.img_off >= 0 && e + 3 >= min(a.w1_off, a.w2_off) && e < max(a.w1_off, a.w2_off) + kW2Elems) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int sl = wimg_slot(e + q, a.w1_off, a.w2_off);
        if (sl < 0) continue;
        const __nv_bfloat16 v = __float2bfloat16_rn(tv[q]);
        for (int p = 0; p < a.world; ++p) a.theta_local_bf16[p][a.img_off + sl] = v;
      }
    }
  }
  if (bad) atomicAdd(&a.ctr->nonfinite, bad);
  // ---- barrier B, release half: the CTA barrier orders every thread's stores before thread 0's
  // gpu-scope release into the join counter; the last block releases once at system scope
  __syncthreads();
  TRACE(2);
  // conv-first delivery: the blocks holding conv parameters (the first nb_c blocks of the owner(s) of
  // the canonical prefix) first join their own counter; the last of them releases the conv weights to
  // every peer (done_c), so the next step's conv forward can start before this round ends
  if (threadIdx.x == 0 && (long long)blockIdx.x < nb_c) {
    if (a.trace) atomicMax(a.trace + (round_idx % 64) * 16 + 12, gtimer());  // 12: last conv block's work done
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(a.my_join_c), "l"(1ull) : "memory");
    if (old == round_idx * (unsigned long long)nb_c - 1) {
      fence_acq_rel_sys();
      for (int p = 0; p < a.world; ++p)
        asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(a.done_c[p]), "l"(1ull) : "memory");
      if (a.trace) a.trace[(round_idx % 64) * 16 + 11] = gtimer();  // 11: conv parameters released
    }
  }
  if (threadIdx.x == 0) {
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(a.my_join), "l"(1ull) : "memory");
    if (old == round_idx * (unsigned long long)gridDim.x - 1) {
      fence_acq_rel_sys();
      for (int p = 0; p < a.world; ++p)
        asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(a.done[p]), "l"(1ull) : "memory");
    }
  }
  TRACE(3);
  if (a.trace && threadIdx.x == 0) atomicMax(a.trace + (round_idx % 64) * 16 + 5, gtimer());
  st_stamp(ST_ROUND, 2);
}

// fp32 path: the acquire half as its own (tiny) kernel at the start of a step
__global__ void fused_round_acquire_kernel(FusedAcquire f) {
  pdl_wait();
  fused_round_acquire(f);
  pdl_trigger();
}

void launch_fused_round_acquire(const FusedAcquire& f, cudaStream_t st) {
  launch_pdl(fused_round_acquire_kernel, dim3(148), dim3(256), 0, st, f);
}

// one 16-byte vector per thread (no cross-block waits inside the kernel, so no residency bound); the conv prefix
// spread cpb per block over the first blocks
int server_round_blocks(long long shard, long long conv4, int cpb) {
  const long long n4 = shard / 4, nb_c = (conv4 + cpb - 1) / cpb;
  const long long rest = std::max(0LL, n4 - conv4 - nb_c * (256 - cpb));
  const long long b = nb_c + (rest + 255) / 256;
  return (int)(b < 1 ? 1 : b);
}

void launch_server_round(const ServerRoundArgs& a, cudaStream_t st) {
  launch_pdl(server_round_kernel, dim3(server_round_blocks(a.shard, a.conv4, a.conv_per_block)), dim3(256), 0, st, a);
}

// ---- NCCL fetch on the bf16 path (a13, n_fetch > 1 or DQN_ASYNC): one all-gather of a per-rank record
// [bf16 of the owned shard | fp32 of the shard's entries outside the FC weight]. The tensor cores read the
// FC weight only as bf16 (98 % of P on the Mnih net); the biases, conv weights and the output layer are read
// in fp32 too (epilogues, TD head, packed conv images), so they travel in both precisions.
__device__ __forceinline__ long long fetch_piece1(const FetchRecord& f, int s) {  // entries before the FC weight
  const long long lo = (long long)s * f.shard, hi = lo + f.shard;
  return max(0LL, min(hi, f.fw_lo) - lo);
}

__global__ void fetch_pack_kernel(const float* __restrict__ master, FetchRecord f, uint8_t* __restrict__ send) {
  pdl_wait();
  pdl_trigger();
  __nv_bfloat16* rb = reinterpret_cast<__nv_bfloat16*>(send);
  float* rf = reinterpret_cast<float*>(send + 2 * f.shard);
  const long long lo = (long long)f.rank * f.shard, n1 = fetch_piece1(f, f.rank);
  const long long lo2 = max(lo, f.fw_hi);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < f.shard; i += (long long)gridDim.x * blockDim.x) {
    const float v = master[i];
    rb[i] = __float2bfloat16_rn(v);
    const long long g = lo + i;
    if (g < f.fw_lo) rf[g - lo] = v;
    else if (g >= f.fw_hi) rf[n1 + (g - lo2)] = v;
  }
}

__global__ void fetch_unpack_kernel(const uint8_t* __restrict__ recv, FetchRecord f, float* __restrict__ th,
                                    __nv_bfloat16* __restrict__ thb) {
  pdl_wait();
  pdl_trigger();
  const long long n = f.shard * f.world;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n; g += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(g / f.shard);
    const long long i = g - (long long)s * f.shard;
    const uint8_t* rec = recv + (long long)s * f.rec_bytes;
    const __nv_bfloat16 v = reinterpret_cast<const __nv_bfloat16*>(rec)[i];
    thb[g] = v;
    if (f.img_off >= 0) {
      const int sl = wimg_slot(g, f.w1_off, f.w2_off);
      if (sl >= 0) thb[f.img_off + sl] = v;
    }
    const float* rf = reinterpret_cast<const float*>(rec + 2 * f.shard);
    if (g < f.fw_lo) th[g] = rf[i];
    else if (g >= f.fw_hi) th[g] = rf[fetch_piece1(f, s) + (g - max((long long)s * f.shard, f.fw_hi))];
  }
}

void launch_fetch_pack(const float* master, const FetchRecord& f, uint8_t* send, cudaStream_t st) {
  const int blocks = (int)std::min<long long>((f.shard + 255) / 256, 148 * 4);
  launch_pdl(fetch_pack_kernel, dim3(blocks), dim3(256), 0, st, master, f, send);
}

void launch_fetch_unpack(const uint8_t* recv, const FetchRecord& f, float* theta, __nv_bfloat16* theta_bf16,
                         cudaStream_t st) {
  const int blocks = (int)std::min<long long>((f.shard * f.world + 255) / 256, 148 * 8);
  launch_pdl(fetch_unpack_kernel, dim3(blocks), dim3(256), 0, st, recv, f, theta, theta_bf16);
}

// the bf16 working copy of [lo, hi) widened into out (get_params of the FC weight on the NCCL bf16 path)
__global__ void widen_range_kernel(const __nv_bfloat16* src, float* dst, long long lo, long long hi) {
  for (long long g = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; g < hi; g += (long long)gridDim.x * blockDim.x)
    dst[g] = __bfloat162float(src[g]);
}
void launch_widen_range(const __nv_bfloat16* src, float* dst, long long lo, long long hi, cudaStream_t st) {
  if (hi <= lo) return;
  widen_range_kernel<<<(int)std::min<long long>((hi - lo + 255) / 256, 148 * 8), 256, 0, st>>>(src, dst, lo, hi);
}

// ---- DQN_ASYNC: the device generation flag. The comm stream publishes generation k + 1 with
// a release store after its kernels wrote theta_pub[(k + 1) % 3]; a fetch on the compute stream reads the flag
// with an acquire load (one thread, so every block of the copy sees the same generation) and copies that slot.
// Three slots suffice: a push waits until the comm stream has finished round k - 2 (the g_send double buffer),
// so a fetch takes a generation >= k - 1 of the rounds pushed so far and the at most two publications that can
// land during its copy go to the other two slots.
__global__ void async_pick_kernel(AsyncDev* d, long long forced, long long C, long long f) {
  unsigned long long g;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(g) : "l"(&d->pub_gen) : "memory");
  const long long m = forced >= 0 ? forced : (long long)g;
  d->n_local = m;
  d->fetch_gen = m;
  const int refresh = m - d->ell >= C;  // A10: right after the fetch, when n - l >= C
  if (refresh) d->ell = m;
  d->do_refresh = refresh;
  d->fgen_log[f % kDiagSteps] = m;
}

__global__ void async_copy_kernel(const AsyncDev* d, AsyncCopy c) {
  const long long m = *(volatile const long long*)&d->fetch_gen;
  const int slot = (int)((m / c.npr) % 3), refresh = *(volatile const int*)&d->do_refresh;
  const float4* s4 = reinterpret_cast<const float4*>(c.pub[slot]);
  const long long stride = (long long)gridDim.x * blockDim.x, t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (long long i = t0; i < c.n32 / 4; i += stride) {
    const float4 v = s4[i];
    reinterpret_cast<float4*>(c.th)[i] = v;
    if (refresh) reinterpret_cast<float4*>(c.hat)[i] = v;
  }
  if (c.pubb[0]) {
    const uint4* b4 = reinterpret_cast<const uint4*>(c.pubb[slot]);
    for (long long i = t0; i < c.n16 / 8; i += stride) {
      const uint4 v = b4[i];
      reinterpret_cast<uint4*>(c.thb)[i] = v;
      if (refresh) reinterpret_cast<uint4*>(c.hatb)[i] = v;
    }
    for (long long i = c.n16 / 8 * 8 + t0; i < c.n16; i += stride) {
      c.thb[i] = c.pubb[slot][i];
      if (refresh) c.hatb[i] = c.pubb[slot][i];
    }
  }
}

__global__ void async_publish_kernel(AsyncDev* d, long long n0, long long npr, int n_push, int n_fetch,
                                     unsigned delay_ns) {
  const long long k = n0 / npr;  // the round
  if (threadIdx.x == 0) {
    if (delay_ns) {  // DQN_ASYNC_DELAY_US (diagnostic): a slow server, so that fetches see stale generations
      const unsigned long long t0 = gtimer();
      while (gtimer() - t0 < delay_ns) {
      }
    }
    // A25: every replica step t of round k used the generation of its last fetch f = t / n_fetch
    for (long long t = k * n_push; t < (k + 1) * n_push; ++t) {
      const long long base = d->fgen_log[(t / n_fetch) % kDiagSteps];
      const long long st = n0 - base;
      d->hist[st < 31 ? (st < 0 ? 0 : st) : 31] += 1;
    }
    // theta_pub[(k + 1) % 3] was written by this stream's earlier kernels: release generation n0 + npr
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&d->pub_gen), "l"((unsigned long long)(n0 + npr)) : "memory");
  }
}

void launch_async_pick(AsyncDev* d, long long forced, long long C, long long f, cudaStream_t st) {
  async_pick_kernel<<<1, 1, 0, st>>>(d, forced, C, f);
}
void launch_async_copy(const AsyncDev* d, const AsyncCopy& c, cudaStream_t st) {
  const long long n = std::max(c.n32 / 4, c.n16 / 8);
  async_copy_kernel<<<(int)std::min<long long>((n + 255) / 256, 148 * 4), 256, 0, st>>>(d, c);
}
void launch_async_publish(AsyncDev* d, long long n0, long long npr, int n_push, int n_fetch, unsigned delay_ns,
                          cudaStream_t st) {
  async_publish_kernel<<<1, 32, 0, st>>>(d, n0, npr, n_push, n_fetch, delay_ns);
}

// A33 in the asynchronous mode: worker p's gradient slice (the mean of its n_push accumulated gradients, A8) is
// applied to the owned shard as its own RMSProp step, p = 0 .. N-1 in rank order (Alg. 2); the same
// per-element arithmetic as rmsprop_kernel and the fused round's per-gradient branch (A4, A5, A24)
__global__ void rmsprop_per_gradient_kernel(float* __restrict__ theta, float* __restrict__ r,
                                            const float* __restrict__ inbox, int world, long long shard, float inv_np,
                                            float lr, float rho, float omr, float eps, DevCounters* ctr) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= shard / 4) return;
  float4 t4 = reinterpret_cast<const float4*>(theta)[i];
  float4 r4 = reinterpret_cast<const float4*>(r)[i];
  float tv[4] = {t4.x, t4.y, t4.z, t4.w}, rv[4] = {r4.x, r4.y, r4.z, r4.w};
  unsigned bad = 0;
  for (int p = 0; p < world; ++p) {
    const float4 g4 = __ldcg(reinterpret_cast<const float4*>(inbox + (long long)p * shard) + i);
    const float gp[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float gb = gp[q] * inv_np;
      if (isfinite(gb)) {
        const float rr = rho * rv[q] + omr * gb * gb;
        rv[q] = rr;
        tv[q] = tv[q] - lr * gb * rsqrtf(rr + eps);
      } else {
        ++bad;
      }
    }
  }
  reinterpret_cast<float4*>(theta)[i] = make_float4(tv[0], tv[1], tv[2], tv[3]);
  reinterpret_cast<float4*>(r)[i] = make_float4(rv[0], rv[1], rv[2], rv[3]);
  if (bad) atomicAdd(&ctr->nonfinite, bad);
}

void launch_rmsprop_per_gradient(float* theta, float* r, const float* inbox, int world, long long shard, float n_push,
                                 float lr, float rho, float omr, float eps, DevCounters* ctr, cudaStream_t st) {
  const long long n4 = shard / 4;
  rmsprop_per_gradient_kernel<<<(unsigned)std::max<long long>(1, (n4 + 255) / 256), 256, 0, st>>>(
      theta, r, inbox, world, shard, 1.0f / n_push, lr, rho, omr, eps, ctr);
}

DQN_STEP_TRACE_HOST(comm)

}  // namespace dqn
