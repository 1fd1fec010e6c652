// hog.cu — TEST ONLY: a kernel that holds SMs (one 200-KB-smem block per SM) for a given time, so a
// product launched next cannot have all of its persistent CTAs resident at once — the situation a
// concurrent NCCL collective or another product creates.  tests/test_gpu_hazards.py.
#include <cuda_runtime.h>
#include <cstdint>

namespace {
__global__ void hog_kernel(unsigned long long duration_ns, unsigned* started) {
  extern __shared__ unsigned char sm[];
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (threadIdx.x == 0) atomicAdd_system(started, 1u);
  unsigned long long t = t0;
  while (t - t0 < duration_ns) {
    __nanosleep(2000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  }
  sm[threadIdx.x] = (unsigned char)t;  // (uses the shared memory)
}
unsigned* g_started = nullptr;  // host-mapped counter
constexpr int kSmem = 200 * 1024;
}  // namespace

extern "C" {
// Launch `blocks` hog blocks on `stream` for duration_ns; returns 0 on success.
int hog_launch(int blocks, long long duration_ns, void* stream) {
  if (!g_started && cudaHostAlloc(&g_started, sizeof(unsigned), cudaHostAllocMapped) != cudaSuccess) return 1;
  *(volatile unsigned*)g_started = 0u;
  unsigned* dev = nullptr;
  if (cudaHostGetDevicePointer(&dev, g_started, 0) != cudaSuccess) return 2;
  if (cudaFuncSetAttribute(hog_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem) != cudaSuccess) return 3;
  hog_kernel<<<blocks, 32, kSmem, static_cast<cudaStream_t>(stream)>>>((unsigned long long)duration_ns, dev);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
// Blocks of the last hog_launch that have started.
unsigned hog_started(void) { return g_started ? *(volatile unsigned*)g_started : 0u; }
}
