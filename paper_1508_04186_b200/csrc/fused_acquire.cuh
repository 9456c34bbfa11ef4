// fused_acquire.cuh — system-scope flag helpers of the fused server round (kernels_comm.cu)
// and the acquire half of its second barrier, which the first kernel of the next step runs
// (device code shared by two translation units without relocatable device code).
#pragma once
#include "dqn_internal.h"

namespace dqn {

constexpr long long kSpinLimit = 1LL << 26;  // ~ seconds with the nanosleep back-off

__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// poll until *p >= want (acquire, system scope); bounded: a timeout sets the error bit and returns
__device__ __forceinline__ void spin_acquire_sys(const unsigned long long* p, unsigned long long want,
                                                 DevCounters* ctr) {
  long long spin = 0;
  while (ld_acquire_sys(p) < want) {
    __nanosleep(32);
    if (++spin > kSpinLimit) {
      atomicOr(&ctr->bad_input, 0x80000000u);  // peer barrier timeout (reported as ECUDA by the host)
      return;
    }
  }
}

// If the previous step ran a server round: wait until every rank's last block has released
// its deliveries into this rank's theta_local (done >= rounds * N), then clear this rank's G
// (every peer read its slice before releasing). Call after pdl_wait() and before touching
// theta_local or G (and before pdl_trigger(): the successor reads theta before its own wait).
__device__ __forceinline__ void fused_round_acquire(const FusedAcquire& f) {
  if (f.ctr == nullptr) return;  // no fused round in this context
  const unsigned long long T = f.ctr->T;
  if (T == 0 || T % (unsigned long long)f.n_push != 0) return;  // the previous step did not push
  const unsigned long long rounds = T / (unsigned long long)f.n_push;
  unsigned long long* tr = nullptr;
  if (f.trace && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
    tr = f.trace + (rounds % 64) * 16;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tr[6]));
  }
  if (threadIdx.x == 0) {
    spin_acquire_sys(f.done, rounds * (unsigned long long)f.world, f.ctr);
    if (tr) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(tr[7]));
  }
  __syncthreads();
  const long long g4 = f.grad_elems / 4;
  const long long blk = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  const long long nblk = (long long)gridDim.x * gridDim.y * gridDim.z;
  for (long long i = blk * blockDim.x + threadIdx.x; i < g4; i += nblk * blockDim.x) {
    if (f.g_snap) reinterpret_cast<float4*>(f.g_snap)[i] = reinterpret_cast<const float4*>(f.grad)[i];  // keep_grad
    reinterpret_cast<float4*>(f.grad)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// conv-first delivery: true if the previous step ran a server round (then the caller must not rely
// on griddepcontrol.wait for it); waits until every owner of conv parameters released them
// (done_c >= rounds * n_c). Thread 0 polls; the block synchronises.
__device__ __forceinline__ bool fused_round_acquire_conv(const FusedAcquire& f) {
  if (f.ctr == nullptr || !f.conv_first) return false;
  const unsigned long long T = f.ctr->T;
  if (T == 0 || T % (unsigned long long)f.n_push != 0) return false;
  const unsigned long long rounds = T / (unsigned long long)f.n_push;
  if (threadIdx.x == 0) spin_acquire_sys(f.done_c, rounds * (unsigned long long)f.n_c, f.ctr);
  __syncthreads();
  return true;
}

}  // namespace dqn
