// probe_p2p.cu — two-GPU NVLink signalling / delivery micro-benchmark (one process, peer
// access), to choose the flag semantics of the fused server round (kernels_comm.cu).
//
//   pingpong <mode>: one thread per GPU bounces a counter R times; prints us per round trip.
//   push <sig>     : per round every GPU writes `bytes` into the PEER's buffer (remote stores),
//                    every block signals the peer, waits for the peer's blocks, checks a sample.
//   pull           : per round every GPU writes its own buffer locally, fences at gpu scope,
//                    signals the peer, waits, then reads the PEER's buffer (remote loads).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_p2p tools/probe_p2p.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

typedef unsigned long long u64;

__device__ __forceinline__ u64 ld_relaxed_sys(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 ld_acquire_sys(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(u64* p, u64 v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(u64* p, u64 v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_sys(u64* p, u64 v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys(u64* p, u64 v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_sys() { asm volatile("fence.sc.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acqrel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ bool spin_ge(const u64* p, u64 target, bool acquire) {
  long long n = 0;
  while ((acquire ? ld_acquire_sys(p) : ld_relaxed_sys(p)) < target)
    if (++n > (1LL << 28)) return false;
  return true;
}

// mode 0 relaxed, 1 release/acquire, 2 fence.sc.sys + relaxed, 3 fence.acq_rel.gpu + relaxed
__global__ void pingpong(u64* my_flag, u64* peer_flag, int R, int first, int mode, int* err) {
  for (int r = 1; r <= R; ++r) {
    const u64 want = 2ull * r - (first ? 1 : 0);
    if (!first || r > 1) {
      if (!spin_ge(my_flag, first ? 2ull * (r - 1) : 2ull * r - 1, mode == 1)) { *err = 1; return; }
    }
    if (mode == 2) fence_sys();
    if (mode == 3) fence_gpu();
    if (mode == 1) st_release_sys(peer_flag, want); else st_relaxed_sys(peer_flag, want);
  }
  if (first && !spin_ge(my_flag, 2ull * R, mode == 1)) *err = 1;
}

// push: sig 0 = syncthreads + red.release.sys, 1 = syncthreads + fence.sc.sys + red.relaxed,
//       2 = per-thread fence.acq_rel.sys + syncthreads + red.relaxed, 3 = syncthreads +
//       fence.acq_rel.gpu + red.relaxed (formally insufficient; checked empirically)
__global__ void push_rounds(float4* peer_buf, const float4* my_buf, long long n4, u64* peer_cnt, u64* my_cnt,
                            int R, int sig, int* err) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
  for (int r = 1; r <= R; ++r) {
    const float v = (float)r;
    for (long long i = tid; i < n4; i += nt) peer_buf[i] = make_float4(v, v, v, v);
    if (sig == 2) fence_acqrel_sys();
    __syncthreads();
    if (threadIdx.x == 0) {
      if (sig == 0) red_release_sys(peer_cnt, 1);
      else if (sig == 1) { fence_sys(); red_relaxed_sys(peer_cnt, 1); }
      else if (sig == 2) red_relaxed_sys(peer_cnt, 1);
      else { fence_gpu(); red_relaxed_sys(peer_cnt, 1); }
      if (!spin_ge(my_cnt, (u64)r * gridDim.x, sig != 3)) atomicOr(err, 1);
    }
    __syncthreads();
    // check: the data the PEER wrote into my buffer this round
    for (long long i = tid; i < n4; i += nt * 61) {
      const float4 x = __ldcg(my_buf + i);
      if (x.x != v || x.w != v) atomicAdd(err + 1, 1);
    }
    // second barrier so no peer overwrites my buffer before my check finished
    __syncthreads();
    if (threadIdx.x == 0) {
      red_relaxed_sys(peer_cnt + 1, 1);
      if (!spin_ge(my_cnt + 1, (u64)r * gridDim.x, false)) atomicOr(err, 2);
    }
    __syncthreads();
  }
}

// pull: write own buffer locally, fence gpu, signal the peer; wait; read the peer's buffer
__global__ void pull_rounds(float4* my_buf, const float4* peer_buf, float4* copy, long long n4, u64* peer_cnt,
                            u64* my_cnt, int R, int* err) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
  for (int r = 1; r <= R; ++r) {
    const float v = (float)r;
    for (long long i = tid; i < n4; i += nt) my_buf[i] = make_float4(v, v, v, v);
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_gpu();
      red_relaxed_sys(peer_cnt, 1);
      if (!spin_ge(my_cnt, (u64)r * gridDim.x, false)) atomicOr(err, 1);
    }
    __syncthreads();
    int bad = 0;
    for (long long i = tid; i < n4; i += nt) {
      const float4 x = __ldcg(peer_buf + i);
      copy[i] = x;
      bad += (x.x != v || x.w != v);
    }
    if (bad) atomicAdd(err + 1, bad);
    __syncthreads();
    if (threadIdx.x == 0) {
      red_relaxed_sys(peer_cnt + 1, 1);
      if (!spin_ge(my_cnt + 1, (u64)r * gridDim.x, false)) atomicOr(err, 2);
    }
    __syncthreads();
  }
}

// kernel-boundary latency after a kernel that touched peer memory:
// A: mode 0 local stores, 1 remote stores, 2 remote loads, 3 one remote red only, 4 nothing
// B: launched with programmatic dependent launch; stamps after griddepcontrol.wait
__device__ __forceinline__ u64 gt() {
  u64 t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__global__ void bound_a(float4* local, float4* remote, long long n4, u64* peer_flag, int mode, u64* stamp,
                        float* sink) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x, nt = (long long)gridDim.x * blockDim.x;
  float acc = 0.f;
  for (long long i = tid; i < n4; i += nt) {
    if (mode == 0) local[i] = make_float4(1.f, 2.f, 3.f, (float)i);
    if (mode == 1) remote[i] = make_float4(1.f, 2.f, 3.f, (float)i);
    if (mode == 2) { float4 x = __ldcg(remote + i); acc += x.x + x.w; }
  }
  if (mode == 3 && tid == 0) red_relaxed_sys(peer_flag, 1);
  if (acc == 12345.f) *sink = acc;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(stamp, gt());
}
__global__ void bound_b(u64* stamp) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) stamp[1] = gt();
}

int main(int argc, char** argv) {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("need 2 GPUs\n"); return 1; }
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
  }
  const long long bytes = argc > 1 ? atoll(argv[1]) : 2 << 20;
  const int R = 2000;
  const long long n4 = bytes / 16;
  u64* flag[2]; float4* buf[2]; float4* cpy[2]; int* err[2]; cudaStream_t st[2]; cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&flag[d], 64)); CK(cudaMalloc(&buf[d], bytes)); CK(cudaMalloc(&cpy[d], bytes));
    CK(cudaMalloc(&err[d], 8)); CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d])); CK(cudaEventCreate(&e1[d]));
  }
  auto reset = [&]() {
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMemset(flag[d], 0, 64)); CK(cudaMemset(err[d], 0, 8)); CK(cudaMemset(buf[d], 0, bytes));
      CK(cudaDeviceSynchronize());
    }
  };
  auto report = [&](const char* name, int rounds) {
    float ms[2]; int h[2][2];
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d)); CK(cudaStreamSynchronize(st[d]));
      CK(cudaEventElapsedTime(&ms[d], e0[d], e1[d]));
      CK(cudaMemcpy(h[d], err[d], 8, cudaMemcpyDeviceToHost));
    }
    printf("%-44s %8.3f us/round  (gpu0 %.3f ms, gpu1 %.3f ms)  err %d/%d %d/%d\n", name,
           1000.0 * (ms[0] > ms[1] ? ms[0] : ms[1]) / rounds, ms[0], ms[1], h[0][0], h[0][1], h[1][0], h[1][1]);
  };
  if (argc > 2 && !strcmp(argv[2], "boundary")) {
    CK(cudaSetDevice(0));
    u64* stamp; float* sink;
    CK(cudaMalloc(&stamp, 16)); CK(cudaMalloc(&sink, 4));
    const char* nm[5] = {"local stores", "remote stores", "remote loads", "one remote red", "nothing"};
    for (int mode = 0; mode < 5; ++mode) {
      double tot = 0; int n = 0;
      for (int it = 0; it < 50; ++it) {
        CK(cudaMemset(stamp, 0, 16));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = 1; cfg.stream = st[0];
        cfg.gridDim = dim3(330); cfg.blockDim = dim3(256);
        CK(cudaLaunchKernelEx(&cfg, bound_a, buf[0], buf[1], n4, flag[1], mode, stamp, sink));
        cfg.gridDim = dim3(64); cfg.blockDim = dim3(128);
        CK(cudaLaunchKernelEx(&cfg, bound_b, stamp));
        CK(cudaStreamSynchronize(st[0]));
        u64 h[2];
        CK(cudaMemcpy(h, stamp, 16, cudaMemcpyDeviceToHost));
        if (it >= 10) { tot += (double)(h[1] - h[0]); ++n; }
      }
      printf("boundary after %-16s %8.2f us (A's last block end -> B past griddepcontrol.wait)\n", nm[mode], tot / n / 1e3);
    }
    return 0;
  }
  const char* pp[4] = {"pingpong relaxed.sys", "pingpong release/acquire.sys", "pingpong fence.sc.sys+relaxed",
                       "pingpong fence.acq_rel.gpu+relaxed"};
  for (int mode = 0; mode < 4; ++mode) {
    reset();
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], st[d]));
      pingpong<<<1, 1, 0, st[d]>>>(flag[d], flag[1 - d], R, d == 0, mode, err[d]);
      CK(cudaEventRecord(e1[d], st[d]));
    }
    report(pp[mode], R);
  }
  const char* ps[4] = {"push red.release.sys", "push fence.sc.sys+red.relaxed", "push per-thread fence.acq_rel.sys",
                       "push fence.acq_rel.gpu+red.relaxed (unsafe?)"};
  for (int blocks : {148, 296}) {
    for (int sig = 0; sig < 4; ++sig) {
      reset();
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], st[d]));
        push_rounds<<<blocks, 256, 0, st[d]>>>(buf[1 - d], buf[d], n4, flag[1 - d], flag[d], R / 4, sig, err[d]);
        CK(cudaEventRecord(e1[d], st[d]));
      }
      char name[96];
      snprintf(name, sizeof name, "%s b=%d %lldKB", ps[sig], blocks, bytes >> 10);
      report(name, R / 4);
    }
    reset();
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], st[d]));
      pull_rounds<<<blocks, 256, 0, st[d]>>>(buf[d], buf[1 - d], cpy[d], n4, flag[1 - d], flag[d], R / 4, err[d]);
      CK(cudaEventRecord(e1[d], st[d]));
    }
    char name[96];
    snprintf(name, sizeof name, "pull fence.gpu+red.relaxed b=%d %lldKB", blocks, bytes >> 10);
    report(name, R / 4);
  }
  return 0;
}
