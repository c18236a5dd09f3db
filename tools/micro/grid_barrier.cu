// Grid-barrier cost on B200: 782 blocks x 128 threads (one 100k-agent wave),
// N barriers per launch, several implementations.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gb tools/micro/grid_barrier.cu && /tmp/gb
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128) k_bar(unsigned* bar, int iters, float* sink) {
  float x = threadIdx.x;
  for (int d = 0; d < iters; ++d) {
    x = x * 1.0001f + 1.f;
    const unsigned target = (unsigned)(d + 1) * gridDim.x;
    if (MODE == 3) {
      cg::this_grid().sync();
      continue;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (MODE == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire(bar) < target) {}
        __threadfence();
      } else if (MODE == 1) {
        red_release(bar, 1u);
        while (ld_acquire(bar) < target) {}
      } else if (MODE == 2) {
        red_release(bar, 1u);
        while (ld_acquire(bar) < target) __nanosleep(64);
      }
    }
    __syncthreads();
  }
  if (x == -1.f) *sink = x;
}

int main() {
  unsigned* bar;
  float* sink;
  cudaMalloc(&bar, 4);
  cudaMalloc(&sink, 4);
  const int blocks = 782, iters = 180;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  void (*ks[4])(unsigned*, int, float*) = {k_bar<0>, k_bar<1>, k_bar<2>, k_bar<3>};
  const char* names[4] = {"fence+atomic+acquire", "red.release+ld.acquire", "red.release+nanosleep", "cg grid.sync"};
  for (int rep = 0; rep < 2; ++rep)
    for (int m = 0; m < 4; ++m) {
      float best = 1e9;
      for (int k = 0; k < 5; ++k) {
        cudaMemset(bar, 0, 4);
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
      printf("%-26s %7.3f us per barrier (%s)\n", names[m], best * 1000.f / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  // empty kernels back to back (what a kernel boundary costs), plain stream and graph
  for (int m = 0; m < 2; ++m) {
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    int one = 1;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int d = 0; d < iters; ++d) k_bar<1><<<blocks, 128, 0, s>>>(bar + 0, 0, sink);
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
    printf("graph of %d empty 782-block kernels: %7.3f us per kernel\n", iters, ms * 1000.f / iters);
    (void)one;
  }
  return 0;
}
