// Fixed cost of the kernel shell on sm_100a, timed with CUDA events after a 512-MB memset
// (the state the bench's per-config timings see) and back to back:
//   empty kernel (148 CTAs) | + 2-CTA clusters and 227 KB dynamic smem | + barrier init,
//   TMEM alloc/dealloc and the two cluster barriers of gemm_tc_kernel | + PDL attribute.
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/launch_probe tools/launch_probe.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void k_empty() {}

__global__ void k_shell(int full) {
  extern __shared__ __align__(1024) unsigned char smem[];
  if (!full) return;
  __shared__ unsigned long long bar;
  __shared__ unsigned slot;
  const unsigned sbar = (unsigned)__cvta_generic_to_shared(&bar);
  const unsigned sslot = (unsigned)__cvta_generic_to_shared(&slot);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x / 32 == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sslot));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  const unsigned t = slot;
  smem[threadIdx.x] = (unsigned char)t;
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x / 32 == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

static float median(std::vector<float> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 2];
}

int main() {
  void* flush = nullptr;
  cudaMalloc(&flush, 512u << 20);
  const int smem = 227 * 1024;
  cudaFuncSetAttribute(k_shell, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch = [&](int variant) {
    if (variant == 0) {
      k_empty<<<148, 320, 0, s>>>();
      return;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = variant == 3 ? 2 : 1;
    cudaLaunchKernelEx(&cfg, k_shell, variant >= 2 ? 1 : 0);
  };
  const char* names[4] = {"empty kernel, 148 CTAs, no smem", "2-CTA clusters + 227 KB smem",
                          "+ mbarrier init, TMEM alloc/dealloc, 2 cluster barriers", "same + PDL attribute"};
  for (int v = 0; v < 4; ++v) {
    for (int w = 0; w < 5; ++w) launch(v);
    std::vector<float> cold, warm;
    for (int r = 0; r < 40; ++r) {
      cudaMemsetAsync(flush, r, 512u << 20, s);
      cudaEventRecord(e0, s);
      launch(v);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      cold.push_back(ms * 1e3f);
      launch(v);  // back to back: the previous launch of the same kernel in front
      cudaEventRecord(e0, s);
      launch(v);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      warm.push_back(ms * 1e3f);
    }
    printf("%-60s after memset %6.2f us | back to back %6.2f us\n", names[v], median(cold), median(warm));
  }
  const cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
