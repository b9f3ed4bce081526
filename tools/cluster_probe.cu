// Dev probe: how many 2-CTA clusters of a one-CTA-per-SM kernel (256 threads, ~225 KB shared memory) fit on
// this GPU at once (cudaOccupancyMaxActiveClusters), i.e. whether pairing CTAs across TPC partners keeps all SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/cluster_probe tools/cluster_probe.cu && tools/cluster_probe
#include <cuda_runtime.h>

#include <cstdio>

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) pair_kernel(int* out) {
  extern __shared__ int s[];
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if (threadIdx.x == 0) out[blockIdx.x] = static_cast<int>(sm);
  s[threadIdx.x] = 0;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int smem : {120 * 1024, 200 * 1024, 225 * 1024}) {
    cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms, 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&clusters, pair_kernel, &cfg);
    printf("{\"smem_kb\": %d, \"sms\": %d, \"max_active_2cta_clusters\": %d, \"status\": \"%s\"}\n", smem / 1024, sms,
           clusters, cudaGetErrorString(e));
  }
  int* out;
  cudaMalloc(&out, sms * sizeof(int));
  cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  pair_kernel<<<sms, 256, 225 * 1024>>>(out);
  cudaError_t e = cudaDeviceSynchronize();
  int h[256];
  cudaMemcpy(h, out, sms * sizeof(int), cudaMemcpyDeviceToHost);
  int same_tpc = 0;
  for (int c = 0; c < sms / 2; c++) same_tpc += (h[2 * c] / 2 == h[2 * c + 1] / 2);
  printf("{\"launch\": \"%s\", \"clusters_on_one_tpc\": %d, \"of\": %d}\n", cudaGetErrorString(e), same_tpc, sms / 2);
  return 0;
}
