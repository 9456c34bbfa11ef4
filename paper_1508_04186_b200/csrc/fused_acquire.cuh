// fused_acquire.cuh — system-scope flag helpers of the fused server round (kernels_comm.cu)
// and the acquire half of its second barrier, which the first kernel of the next step runs
// (device code shared by two translation units without relocatable device code).
#pragma once
#include "dqn_internal.h"

namespace dqn {

constexpr long long kSpinLimit = 1LL << 26;  // ~ seconds with the nanosleep back-off

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// If the previous step ran a server round: wait until every block of every rank has
// released its deliveries into this rank's theta_local (done >= rounds * N * blocks), then
// clear this rank's G (every peer read its slice before releasing). Call after pdl_wait()
// and before touching theta_local or G. Bounded spin; a timeout is reported, not hung on.
__device__ __forceinline__ void fused_round_acquire(const FusedAcquire& f) {
  if (f.done == nullptr) return;
  const unsigned long long T = f.ctr->T;
  if (T == 0 || T % (unsigned long long)f.n_push != 0) return;  // the previous step did not push
  const unsigned long long expect = (T / (unsigned long long)f.n_push) * f.per_round;
  if (threadIdx.x == 0) {
    long long spin = 0;
    while (ld_acquire_sys(f.done) < expect) {
      __nanosleep(32);
      if (++spin > kSpinLimit) {
        atomicOr(&f.ctr->bad_input, 0x80000000u);
        break;
      }
    }
  }
  __syncthreads();
  const long long g4 = f.grad_elems / 4;
  const long long blk = blockIdx.y * (long long)gridDim.x + blockIdx.x, nblk = (long long)gridDim.x * gridDim.y;
  for (long long i = blk * blockDim.x + threadIdx.x; i < g4; i += nblk * blockDim.x)
    reinterpret_cast<float4*>(f.grad)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

}  // namespace dqn
