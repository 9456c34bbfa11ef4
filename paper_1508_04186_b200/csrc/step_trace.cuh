// step_trace.cuh — DQN_TRACE_STEP=1 diagnostic: globaltimer stamps of CTA 0 of every kernel of a
// step (entry, past its PDL wait, exit), overwritten each step, so a train_steps(k) call leaves
// the last step's timeline. One copy per translation unit (no relocatable device code); the
// runtime merges them (dqn_runtime.cu).
#pragma once
#include <cuda_runtime.h>

namespace dqn {

enum { ST_NONE = 0, ST_FWD, ST_FC_FWD, ST_HEAD, ST_FC_BWD, ST_CONV_BWD, ST_BWD_REDUCE, ST_UPDATE, ST_ROUND, ST_P1, ST_P2, ST_P3, ST_P4, ST_P5, ST_P6, ST_P7, ST_N };
static __device__ unsigned long long g_st[ST_N][3];
static __device__ int g_st_on;

__device__ __forceinline__ void st_stamp(int k, int w) {
  if (k != ST_NONE && g_st_on && (blockIdx.x | blockIdx.y) == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_st[k][w] = t;
  }
}

// same, from whichever CTA calls it (thread 0)
__device__ __forceinline__ void st_stamp_here(int k, int w) {
  if (g_st_on && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_st[k][w] = t;
  }
}

}  // namespace dqn

// host accessor of this translation unit's copy: out == nullptr sets the switch, else reads the stamps
#define DQN_STEP_TRACE_HOST(name)                                                        \
  void step_trace_##name(int on, unsigned long long* out) {                              \
    if (out) cudaMemcpyFromSymbol(out, g_st, sizeof(g_st));                              \
    else cudaMemcpyToSymbol(g_st_on, &on, sizeof(int));                                  \
  }
