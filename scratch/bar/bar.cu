// grid-barrier cost micro-benchmark (592x256 vs 148x1024; same-line vs split-line; backoff)
#include <cstdio>
#include <cuda_runtime.h>
template <int SPLIT, int SLEEP>
__device__ void gsync(unsigned* bar) {
  __shared__ unsigned s_last, s_gen;
  unsigned* genp = bar + (SPLIT ? 64 : 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    s_gen = *(volatile unsigned*)genp;
    __threadfence();
    s_last = atomicAdd(bar, 1u) == gridDim.x - 1;
    if (s_last) { atomicExch(bar, 0u); __threadfence(); atomicAdd(genp, 1u); }
    else {
      unsigned g;
      do { if (SLEEP) __nanosleep(SLEEP); asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(genp)); } while (g == s_gen);
    }
  }
  __syncthreads();
}
template <int SPLIT, int SLEEP>
__global__ void kbar(unsigned* bar, int n, float* sink) {
  float acc = 0.f;
  for (int i = 0; i < n; ++i) { gsync<SPLIT, SLEEP>(bar); acc += i; }
  if (acc < 0) sink[0] = acc;
}
template <int SPLIT, int SLEEP>
void run(const char* name, int blocks, int threads) {
  unsigned* bar; float* sink;
  cudaMalloc(&bar, 1024); cudaMemset(bar, 0, 1024); cudaMalloc(&sink, 4);
  void* args[] = {&bar, nullptr, &sink};
  int n = 1; args[1] = &n;
  cudaLaunchCooperativeKernel((void*)kbar<SPLIT, SLEEP>, blocks, threads, args, 0, 0);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  n = 1000;
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)kbar<SPLIT, SLEEP>, blocks, threads, args, 0, 0);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-28s %4d x %4d: %.3f us/barrier (%s)\n", name, blocks, threads, ms * 1000.f / n, cudaGetErrorString(cudaGetLastError()));
  cudaFree(bar); cudaFree(sink);
}
int main() {
  run<0, 32>("sameline sleep32", 592, 256);
  run<1, 32>("splitline sleep32", 592, 256);
  run<1, 0>("splitline nosleep", 592, 256);
  run<1, 100>("splitline sleep100", 592, 256);
  run<1, 32>("splitline sleep32", 148, 1024);
  run<1, 0>("splitline nosleep", 148, 1024);
  run<1, 32>("splitline sleep32", 296, 512);
  return 0;
}
