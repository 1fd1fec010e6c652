// smid_probe.cu — where do the clusters of a persistent grid land?  Launches one CTA per SM (200 KB
// smem) as clusters of `csize` and records (clusterid, cluster_ctarank, smid) per CTA.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
__global__ void probe(unsigned* out) {
  extern __shared__ unsigned char sm[];
  unsigned smid, cid, crank;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  if (threadIdx.x == 0) { out[3 * blockIdx.x] = cid; out[3 * blockIdx.x + 1] = crank; out[3 * blockIdx.x + 2] = smid; }
  sm[threadIdx.x] = 0;
}
int main(int argc, char** argv) {
  int csize = argc > 1 ? atoi(argv[1]) : 2;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int ctas = sms / csize * csize;
  unsigned* d;
  cudaMalloc(&d, ctas * 3 * sizeof(unsigned));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = csize; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a; cfg.numAttrs = 1;
  int maxcl = 0;
  cudaOccupancyMaxActiveClusters(&maxcl, (void*)probe, &cfg);
  for (int rep = 0; rep < 2; ++rep) {
    cudaError_t e = cudaLaunchKernelEx(&cfg, probe, d);
    cudaDeviceSynchronize();
    std::vector<unsigned> h(ctas * 3);
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    printf("rep %d sms %d csize %d ctas %d max active clusters %d launch %s\ncluster: smids\n", rep, sms, csize, ctas, maxcl,
           cudaGetErrorString(e));
    for (int c = 0; c < ctas / csize; ++c) {
      printf("%d:", c);
      for (int i = 0; i < ctas; ++i) if (h[3 * i] == (unsigned)c) printf(" %u", h[3 * i + 2]);
      printf(c % 8 == 7 ? "\n" : "  |");
    }
    printf("\n");
  }
  return 0;
}
