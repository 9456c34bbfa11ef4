// stage.cuh — global -> shared staging of UMMA no-swizzle operand tiles with 16-byte cp.async, in a
// thread order that is both bank-conflict free in shared memory and sector-efficient in global memory.
//
// A 16-byte shared store of a warp is served in four phases of eight lanes; a phase is conflict free iff
// its eight stores fill one 128-byte line. The no-swizzle layouts (sm100.cuh) put 8 consecutive ROWS of
// one K chunk (K-major) or 8 consecutive K of one MN group (MN-major) in a 128-byte core matrix, so the
// eight lanes of a phase take 8 consecutive rows (K) of the same chunk (group), and the four phases take
// four consecutive chunks (groups) - each row of the global source then gets 64 contiguous bytes per warp.
// (Lane order "consecutive chunks of one row" puts a phase's stores a whole chunk plane apart: 8-way
// conflicts; "consecutive MN groups of one k" puts them a group plane apart: up to 16-way.)
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

#include "sm100.cuh"

namespace dqn {

// K-major tile: rows [0, R) (R % 8 == 0) x kch chunks of 8 elements -> smem [c][R][8] (16 B units).
// Row r comes from src + r * ld + 8 * c; rows with !row_ok(r) and chunks >= kvalid are zero-filled.
template <typename RowOk>
__device__ __forceinline__ void stage_kmajor(uint8_t* s, const __nv_bfloat16* src, long long ld, int R, int kch,
                                             int kvalid, RowOk row_ok, int tid, int nthreads) {
  const int rb_n = R / 8, cq_n = (kch + 3) / 4;
  for (int e = tid; e < rb_n * cq_n * 32; e += nthreads) {
    const int ri = e & 7, ci = (e >> 3) & 3, rest = e >> 5;
    const int r = (rest % rb_n) * 8 + ri, c = (rest / rb_n) * 4 + ci;
    if (c >= kch) continue;
    uint8_t* d = s + ((long long)c * R + r) * 16;
    if (c < kvalid && row_ok(r)) dqn_sm100::cp_async16(d, src + (long long)r * ld + 8 * c);
    else *reinterpret_cast<uint4*>(d) = make_uint4(0, 0, 0, 0);
  }
}

// MN-major tile: G groups of 8 MN elements x KC rows of k (KC % 8 == 0) -> smem [gi][KC][8] (16 B units).
// Group gi of row k comes from src + k * ld + 8 * gi; groups with !grp_ok(gi) and rows >= kvalid are zero.
template <typename GrpOk>
__device__ __forceinline__ void stage_mnmajor(uint8_t* s, const __nv_bfloat16* src, long long ld, int G, int KC,
                                              int kvalid, GrpOk grp_ok, int tid, int nthreads) {
  const int kb_n = KC / 8, gq_n = (G + 3) / 4;
  for (int e = tid; e < kb_n * gq_n * 32; e += nthreads) {
    const int ki = e & 7, gq = (e >> 3) & 3, rest = e >> 5;
    const int k = (rest % kb_n) * 8 + ki, gi = (rest / kb_n) * 4 + gq;
    if (gi >= G) continue;
    uint8_t* d = s + ((long long)gi * KC + k) * 16;
    if (k < kvalid && grp_ok(gi)) dqn_sm100::cp_async16(d, src + (long long)k * ld + 8 * gi);
    else *reinterpret_cast<uint4*>(d) = make_uint4(0, 0, 0, 0);
  }
}

}  // namespace dqn
