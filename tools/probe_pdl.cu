// probe_pdl.cu — cost of a kernel-to-kernel dependency in a PDL chain: griddepcontrol.wait (the dependent
// waits for the whole primary grid to complete and flush) against a release/acquire counter the primary's
// CTAs bump after their last store (the dependent spins on it instead of waiting for grid completion).
// A chain of `len` launches of one small kernel (grid `ctas` x 128 threads, each CTA does `work` dependent
// global round trips, writes a value, signals); each launch reads what the previous launch wrote.
//   tools/probe_pdl ctas work len       prints us per link for mode 0 (griddepcontrol.wait) and 1 (counter)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/probe_pdl.cu -o tools/probe_pdl
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void link(int mode, unsigned* ctr, unsigned target, float* buf, int ctas, int work, int i) {
  pdl_trigger();
  if (mode == 0) {
    pdl_wait();
  } else if (mode == 1) {
    if (threadIdx.x == 0)
      while (ld_acquire(ctr) < target) {
      }
    __syncthreads();
  }
  // read the previous link's values, some dependent work, write ours
  float v = buf[((i + 1) & 1) * 4096 + (blockIdx.x * 128 + threadIdx.x) % 4096];
  for (int k = 0; k < work; ++k) v = v * 0.999f + buf[(((int)v & 1) + k * 128 + threadIdx.x) % 4096 + 8192];
  buf[(i & 1) * 4096 + (blockIdx.x * 128 + threadIdx.x) % 4096] = v + 1.0f;
  if (mode == 1) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(ctr, 1u);
    }
  }
}

int main(int argc, char** argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 32, work = argc > 2 ? atoi(argv[2]) : 4, len = argc > 3 ? atoi(argv[3]) : 200;
  unsigned* ctr;
  float* buf;
  cudaMalloc(&ctr, 4);
  cudaMalloc(&buf, 3 * 4096 * 4);
  cudaMemset(buf, 0, 3 * 4096 * 4);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  for (int mode = 0; mode < 3; ++mode) {  // 2: no dependency at all (the floor)
    for (int use_graph = 0; use_graph < 2; ++use_graph) {
      cudaMemset(ctr, 0, 4);
      cudaGraphExec_t ge = nullptr;
      auto chain = [&](unsigned base) {
        for (int i = 0; i < len; ++i) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(ctas);
          cfg.blockDim = dim3(128);
          cfg.stream = st;
          cfg.attrs = attr;
          cfg.numAttrs = 1;
          cudaLaunchKernelEx(&cfg, link, mode, ctr, base + (unsigned)(i * ctas), buf, ctas, work, i);
        }
      };
      if (use_graph) {
        // the counter keeps counting across replays: the graph is captured once per replay offset (2 replays)
        cudaGraph_t g;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        chain(0);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphUpload(ge, st);
        cudaMemsetAsync(ctr, 0, 4, st);
        cudaGraphLaunch(ge, st);  // warm
        cudaStreamSynchronize(st);
        cudaMemsetAsync(ctr, 0, 4, st);
      } else {
        chain(0);  // warm
        cudaStreamSynchronize(st);
        cudaMemsetAsync(ctr, 0, 4, st);
      }
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, st);
      if (use_graph) cudaGraphLaunch(ge, st);
      else chain(0);
      cudaEventRecord(e1, st);
      cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("mode %d (%s) graph %d: ctas %d work %d: %.3f us per link\n", mode, mode == 2 ? "none" : mode ? "counter" : "griddepcontrol.wait",
             use_graph, ctas, work, ms * 1e3 / len);
    }
  }
  return 0;
}
