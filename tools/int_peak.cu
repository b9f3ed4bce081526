// Integer-pipe peak microbenchmark (the roofline denominator of the ALU-bound blind rotation).
// Each thread runs 8 independent chains of a 1:1 IMAD (fma pipe) / IADD3-LOP3 (alu pipe) mix; the result is
// written out so nothing is dead.  Reports lane-operations per second for the mix and for each pipe alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak tools/int_peak.cu && ./int_peak
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void kern(unsigned* out, unsigned iters, unsigned seed) {
  unsigned a0 = threadIdx.x ^ seed, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, a4 = a0 * 11, a5 = a0 * 13, a6 = a0 * 17,
           a7 = a0 * 19;
  const unsigned k = seed | 1u, m = seed * 0x9E3779B9u;
  for (unsigned i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 4; u++) {
      if (MODE == 0 || MODE == 1) {  // IMAD (fma pipe)
        a0 = a0 * k + m; a1 = a1 * k + m; a2 = a2 * k + m; a3 = a3 * k + m;
      }
      if (MODE == 0 || MODE == 2) {  // IADD3 / LOP3 (alu pipe)
        a4 = a4 + a5 + m; a5 = (a5 ^ a6) & m | a7; a6 = a6 + a7 + k; a7 = (a7 ^ a4) | m;
      }
      if (MODE == 1) { a4 = a4 * k + m; a5 = a5 * k + m; a6 = a6 * k + m; a7 = a7 * k + m; }
      if (MODE == 3) {  // IMAD.HI
        a0 = __umulhi(a0, k) ^ m; a1 = __umulhi(a1, k) ^ m; a2 = __umulhi(a2, k) ^ m; a3 = __umulhi(a3, k) ^ m;
        a4 = __umulhi(a4, k) ^ m; a5 = __umulhi(a5, k) ^ m; a6 = __umulhi(a6, k) ^ m; a7 = __umulhi(a7, k) ^ m;
      }
      if (MODE == 4) {  // IMAD.WIDE (64-bit accumulate)
        unsigned long long w0 = (unsigned long long)a0 * k + a1, w1 = (unsigned long long)a2 * k + a3;
        unsigned long long w2 = (unsigned long long)a4 * k + a5, w3 = (unsigned long long)a6 * k + a7;
        a0 = (unsigned)w0; a1 = (unsigned)(w0 >> 32); a2 = (unsigned)w1; a3 = (unsigned)(w1 >> 32);
        a4 = (unsigned)w2; a5 = (unsigned)(w2 >> 32); a6 = (unsigned)w3; a7 = (unsigned)(w3 >> 32);
      }
      if (MODE == 2) { a0 = a0 + a1 + m; a1 = (a1 ^ a2) & m | a3; a2 = a2 + a3 + k; a3 = (a3 ^ a0) | m; }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
}

__global__ void dkern(double* out, unsigned iters, double seed) {
  double a0 = threadIdx.x * seed, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  const double k = 0.999999, m = 1e-7;
  for (unsigned i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 4; u++) {
      a0 = fma(a0, k, m); a1 = fma(a1, k, m); a2 = fma(a2, k, m); a3 = fma(a3, k, m);
      a4 = fma(a4, k, m); a5 = fma(a5, k, m); a6 = fma(a6, k, m); a7 = fma(a7, k, m);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

double run_d(double* out, int blocks, int threads, unsigned iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dkern<<<blocks, threads>>>(out, iters / 10, 1.0001);
  cudaEventRecord(e0);
  dkern<<<blocks, threads>>>(out, iters, 1.0001);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return double(blocks) * threads * iters * 4 * 8 / (ms * 1e-3) / 1e9;
}

template <int MODE>
double run(unsigned* out, int blocks, int threads, unsigned iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<MODE><<<blocks, threads>>>(out, iters / 10, 1234567u);
  cudaEventRecord(e0);
  kern<MODE><<<blocks, threads>>>(out, iters, 1234567u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = double(blocks) * threads * iters * 4 * 8;
  return ops / (ms * 1e-3) / 1e9;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 512, blocks = sms * 4;
  unsigned* out;
  cudaMalloc(&out, sizeof(unsigned) * blocks * threads);
  const unsigned iters = 20000;
  double mix = run<0>(out, blocks, threads, iters);
  double fma = run<1>(out, blocks, threads, iters);
  double alu = run<2>(out, blocks, threads, iters);
  double hi = run<3>(out, blocks, threads, iters);
  double wide = run<4>(out, blocks, threads, iters) / 2.0;  // 4 IMAD.WIDE per 8 "ops"
  double* dout;
  cudaMalloc(&dout, sizeof(double) * blocks * threads);
  double dfma = run_d(dout, blocks, threads, iters / 4);
  printf("{\"gops\": %.1f, \"imad_only_gops\": %.1f, \"alu_only_gops\": %.1f, \"imad_hi_gops_approx\": %.1f, "
         "\"imad_wide_gops_approx\": %.1f, \"dfma_gops\": %.1f, \"sms\": %d, "
         "\"how\": \"tools/int_peak.cu: 1:1 IMAD/IADD3-LOP3 mix, 8 independent chains/thread, %d x %d threads, CUDA events\"}\n",
         mix, fma, alu, hi, wide, dfma, sms, blocks, threads);
  return 0;
}
