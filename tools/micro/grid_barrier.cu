// Grid-barrier cost on B200: 888 blocks x 128 threads (6 per SM, one
// 100k-agent wave), N barriers per launch, several implementations, against
// the cost of a kernel boundary inside a CUDA graph.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/gb tools/micro/grid_barrier.cu && tools/micro/gb
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// bar[0] = arrival counter, bar[32] = generation (separate lines), bar[64 + 32*g] group counters
template <int MODE>
__global__ void __launch_bounds__(128) k_bar(unsigned* bar, int iters, float* sink) {
  float x = threadIdx.x;
  for (int d = 0; d < iters; ++d) {
    x = x * 1.0001f + 1.f;
    if (MODE == 0) {
      cg::this_grid().sync();
      continue;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (MODE == 1) {           // last arriver bumps the generation
        const unsigned old = atom_add_acqrel(bar, 1u);
        if (old == (unsigned)(d + 1) * gridDim.x - 1) st_release(bar + 32, d + 1);
        else while (ld_acquire(bar + 32) < (unsigned)(d + 1)) {}
      } else if (MODE == 2) {    // two levels: 16 groups, last of each group to the top
        const int G = 16;
        const unsigned grp = blockIdx.x % G;
        const unsigned gsize = (gridDim.x - grp + G - 1) / G;
        const unsigned old = atom_add_acqrel(bar + 64 + 32 * grp, 1u);
        if (old == (unsigned)(d + 1) * gsize - 1) {
          const unsigned o2 = atom_add_acqrel(bar, 1u);
          if (o2 == (unsigned)(d + 1) * G - 1) st_release(bar + 32, d + 1);
        }
        while (ld_acquire(bar + 32) < (unsigned)(d + 1)) {}
      } else if (MODE == 3) {    // counter only, everyone polls it
        atom_add_acqrel(bar, 1u);
        while (ld_acquire(bar) < (unsigned)(d + 1) * gridDim.x) {}
      }
    }
    __syncthreads();
  }
  if (x == -1.f) *sink = x;
}

int main() {
  unsigned* bar;
  float* sink;
  cudaMalloc(&bar, 4096 * 4);
  cudaMalloc(&sink, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 180;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  void (*ks[4])(unsigned*, int, float*) = {k_bar<0>, k_bar<1>, k_bar<2>, k_bar<3>};
  const char* names[4] = {"cg grid.sync", "counter + generation flag", "two-level (16 groups)", "counter polled"};
  for (int per_sm : {1, 6}) {
    const int blocks = sms * per_sm;
    for (int m = 0; m < 4; ++m) {
      float best = 1e9;
      for (int k = 0; k < 5; ++k) {
        cudaMemset(bar, 0, 4096 * 4);
        int it = iters;
        void* args[] = {&bar, &it, &sink};
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)ks[m], dim3(blocks), dim3(128), args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("%4d blocks  %-28s %7.3f us per barrier (%s)\n", blocks, names[m], best * 1000.f / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int d = 0; d < iters; ++d) k_bar<1><<<sms * 6, 128, 0, s>>>(bar, 0, sink);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEventRecord(e0, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("graph of %d empty %d-block kernels: %7.3f us per kernel\n", iters, sms * 6, ms * 1000.f / iters);
  return 0;
}
