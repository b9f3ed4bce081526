// FP64 instruction throughput / latency on sm_100a (dev tool; profiles/fp64_bench_r2.json).
// Throughput: 4 x 148 CTAs x 512 threads, 8 independent chains per thread.  Latency: one warp, one chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_bench tools/fp64_bench.cu && tools/fp64_bench
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int MODE, int CH>
__global__ void kern(double* out, uint32_t iters, double seed) {
  double f[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) f[c] = seed + threadIdx.x * 1e-3 + c;
  const double k = 0.9999999, m = 1e-9 * seed;
  for (uint32_t i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
#pragma unroll
      for (int c = 0; c < CH; c++) {
        if (MODE == 0) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(f[c]) : "d"(k));
        if (MODE == 1) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[c]) : "d"(k), "d"(m));
        if (MODE == 2) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(f[c]) : "d"(m));
        if (MODE == 3) asm volatile("fma.rn.f64 %0, %0, %1, 0d0000000000000000;" : "+d"(f[c]) : "d"(k));
        if (MODE == 4) {
          asm volatile("{ .reg .pred p; setp.gt.f64 p, %0, %1; selp.f64 %0, %0, %1, p; }" : "+d"(f[c]) : "d"(m));
        }
      }
    }
  }
  double r = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) r += f[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
void run(const char* name) {
  double* out;
  cudaMalloc(&out, 148 * 4 * 512 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint32_t iters = 2048;
  kern<MODE, 8><<<148 * 4, 512>>>(out, iters / 8, 1.0);
  cudaEventRecord(e0);
  kern<MODE, 8><<<148 * 4, 512>>>(out, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warp_instr = 148.0 * 4 * 512 / 32 * iters * 8 * 8;
  const double thr = warp_instr / 148 / (ms * 1e-3 * 1965e6);
  // latency: one warp, one chain
  kern<MODE, 1><<<1, 32>>>(out, iters / 8, 1.0);
  cudaEventRecord(e0);
  kern<MODE, 1><<<1, 32>>>(out, iters * 8, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms2 = 0;
  cudaEventElapsedTime(&ms2, e0, e1);
  const double lat = ms2 * 1e-3 * 1965e6 / (double(iters) * 8 * 8);
  printf("{\"op\": \"%s\", \"warp_instr_per_sm_per_clk_at_1965\": %.3f, \"latency_clk_at_1965\": %.1f}\n", name, thr, lat);
  cudaFree(out);
}

int main() {
  run<0>("DMUL");
  run<1>("DFMA");
  run<2>("DADD");
  run<3>("fma.rn.f64 with 0 addend");
  run<4>("setp.f64 + selp.f64");
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
