// Does an event recorded after a PDL kernel (that triggers launch_dependents at
// its start) complete before that kernel finishes?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_prev() { asm volatile("griddepcontrol.wait;" ::: "memory"); asm volatile("griddepcontrol.launch_dependents;"); }
__global__ void k_slow(volatile int* flag) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  long long t0 = clock64();
  while (clock64() - t0 < 200000000LL) {}   // ~100 ms
  *flag = 1;
}
__global__ void k_check(volatile int* flag, int* out) { *out = *flag; }
int main() {
  int *flag, *out; cudaMalloc(&flag, 4); cudaMalloc(&out, 4); cudaMemset(flag, 0, 4); cudaMemset(out, 0, 4);
  cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t ev; cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  cudaLaunchAttribute attr[1]; attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {}; cfg.gridDim = 1; cfg.blockDim = 32; cfg.stream = s1; cfg.attrs = attr; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_prev);
  cudaLaunchKernelEx(&cfg, k_slow, (volatile int*)flag);
  cudaEventRecord(ev, s1);
  cudaStreamWaitEvent(s2, ev, 0);
  k_check<<<1, 1, 0, s2>>>(flag, out);
  cudaDeviceSynchronize();
  int h = -1; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
  printf("side stream saw flag=%d (%s)\n", h, h ? "event waited for completion" : "EVENT FIRED EARLY");
  return 0;
}
