// wimg.cuh — the conv weights of the Mnih bf16 path as the exact shared-memory image the
// forward kernel's MMAs read ("weight image"): conv1 B operand [kchunk 32][n 16][8] then conv2
// [kchunk 32][n 32][8] (bf16), with k = tap*64 + s2d channel. It lives right after the canonical
// P_pad entries of every bf16 theta buffer; whoever writes a new bf16 theta (the update kernels,
// the fetch/refresh paths) writes the image too, so the forward stages its weights with 16-byte
// copies instead of a permuting 2-byte gather on its critical path.
#pragma once

namespace dqn {

constexpr int kW1Elems = 16 * 4 * 8 * 8;    // conv1 W [16][4][8][8]
constexpr int kW2Elems = 32 * 16 * 4 * 4;   // conv2 W [32][16][4][4]
constexpr int kWimgElems = kW1Elems + kW2Elems;

// image element of canonical theta index idx, or -1 outside conv1.W / conv2.W
__host__ __device__ __forceinline__ int wimg_slot(long long idx, long long w1_off, long long w2_off) {
  if (idx >= w1_off && idx < w1_off + kW1Elems) {
    const int r = (int)(idx - w1_off);
    const int kx = r & 7, ky = (r >> 3) & 7, f = (r >> 6) & 3, n = r >> 8;
    const int t = (ky >> 2) * 2 + (kx >> 2), c = f * 16 + (ky & 3) * 4 + (kx & 3);
    const int k = t * 64 + c;
    return ((k >> 3) * 16 + n) * 8 + (k & 7);
  }
  if (idx >= w2_off && idx < w2_off + kW2Elems) {
    const int r = (int)(idx - w2_off);
    const int kx = r & 3, ky = (r >> 2) & 3, c = (r >> 4) & 15, n = r >> 8;
    const int t = (ky >> 1) * 2 + (kx >> 1), q = (ky & 1) * 2 + (kx & 1);
    const int k = t * 64 + q * 16 + c;
    return kW1Elems + ((k >> 3) * 32 + n) * 8 + (k & 7);
  }
  return -1;
}

}  // namespace dqn
