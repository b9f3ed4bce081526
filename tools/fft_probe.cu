// Feasibility probe (dev tool): one warp = one 512-point complex FP64 FFT with 16 points per thread
// (four-step 16 x 32: 16-point DFT in registers, twiddle, transpose through warp-private shared memory,
// 32-point DFTs as 16-point register DFTs + one lane-pair radix-2 stage).  Measures FFTs per second per SM
// on random data (and checks one FFT against a direct DFT on the host).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fft_probe tools/fft_probe.cu && ./fft_probe
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

struct cd { double x, y; };
__device__ __forceinline__ cd cadd(cd a, cd b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ cd csub(cd a, cd b) { return {a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ cd cmul(cd a, cd b) { return {fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)}; }

// in-place 16-point DFT (forward), radix-2 DIF: natural in -> bit-reversed out (v[r] = X[brev4(r)])
__constant__ cd c_w16[16];
__host__ __device__ constexpr int brev4(int r) { return ((r & 1) << 3) | ((r & 2) << 1) | ((r & 4) >> 1) | ((r & 8) >> 3); }
__device__ __forceinline__ void dft16(cd (&v)[16]) {
#pragma unroll
  for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
    for (int k = 0; k < 16; k += 2 * h)
#pragma unroll
      for (int j = 0; j < h; j++) {
        const cd u = v[k + j], x = v[k + j + h];
        v[k + j] = cadd(u, x);
        const cd d = csub(u, x);
        const int e = j * (8 / h);  // twiddle w16^(j * 16 / (2h))
        v[k + j + h] = e == 0 ? d : cmul(d, c_w16[e]);
      }
}

// x[p], p = 32 a + b (register a, lane b) -> X[k], k = k1 + 16 k2 held as (register k1? ...) see below
__global__ void __launch_bounds__(128) fft_kernel(const cd* __restrict__ in, cd* __restrict__ out,
                                                  const cd* __restrict__ tw512, int reps) {
  __shared__ cd xbuf[4][16 * 33];  // warp-private transpose buffers (padded)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int fft = blockIdx.x * 4 + wib;
  cd v[16];
#pragma unroll
  for (int a = 0; a < 16; a++) v[a] = in[(size_t)fft * 512 + 32 * a + lane];
  for (int rep = 0; rep < reps; rep++) {
    // step 1: 16-point DFT over a for this lane b
    dft16(v);
    // step 2: twiddle omega_512^(b k1)
#pragma unroll
    for (int r = 1; r < 16; r++) v[r] = cmul(v[r], tw512[(lane * brev4(r)) & 511]);
    // step 3: transpose: thread b holds Y[b][k1]; we need, per k1, the 32 values over b.  Lane l takes
    // k1 = l & 15 and half h = l >> 4 of b: b = 16 h + i, i in [0,16)
    cd* xb = xbuf[wib];
#pragma unroll
    for (int r = 0; r < 16; r++) xb[brev4(r) * 33 + lane] = v[r];
    __syncwarp();
    const int k1 = lane & 15, hh = lane >> 4;
#pragma unroll
    for (int i = 0; i < 16; i++) v[i] = xb[k1 * 33 + 16 * hh + i];
    __syncwarp();
    // 32-point DFT over b = 16 hh + i: X[k2] = sum_i w32^{i k2} (Y[i] + (-1)^{k2} Y[16+i]) ... radix-2 DIF
    // across the lane pair (l, l ^ 16): partner holds the other half
#pragma unroll
    for (int i = 0; i < 16; i++) {
      cd p;
      p.x = __shfl_xor_sync(0xffffffffu, v[i].x, 16);
      p.y = __shfl_xor_sync(0xffffffffu, v[i].y, 16);
      const cd lo = hh ? p : v[i], hi = hh ? v[i] : p;
      v[i] = hh ? cmul(csub(lo, hi), tw512[(16 * i) & 511]) : cadd(lo, hi);  // w32^i = w512^(16 i)
    }
    dft16(v);  // even (hh = 0) / odd (hh = 1) outputs k2 = 2 brev4(r) + hh in v[r]
  }
#pragma unroll
  for (int i = 0; i < 16; i++) out[(size_t)fft * 512 + lane * 16 + i] = v[i];
}

int main() {
  const int nfft = 148 * 8 * 8, reps = 200;
  std::vector<cd> h(512 * (size_t)nfft), tw(512), w16(16);
  for (int i = 0; i < 512; i++) tw[i] = {cos(-2 * M_PI * i / 512), sin(-2 * M_PI * i / 512)};
  for (int i = 0; i < 16; i++) w16[i] = {cos(-2 * M_PI * i / 16), sin(-2 * M_PI * i / 16)};
  srand(1);
  for (auto& x : h) x = {rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5};
  cd *din, *dout, *dtw;
  cudaMalloc(&din, h.size() * 16); cudaMalloc(&dout, h.size() * 16); cudaMalloc(&dtw, 512 * 16);
  cudaMemcpy(din, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dtw, tw.data(), 512 * 16, cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_w16, w16.data(), 16 * 16);
  fft_kernel<<<nfft / 4, 128>>>(din, dout, dtw, 1);
  std::vector<cd> o(512);
  cudaMemcpy(o.data(), dout, 512 * 16, cudaMemcpyDeviceToHost);
  // reference DFT of FFT 0; output position of X[k], k = k1 + 16 k2, k2 = 2 j + hh: lane l = 16 hh + k1, i = j
  double maxerr = 0;
  for (int lane = 0; lane < 32; lane++)
    for (int i = 0; i < 16; i++) {
      const int k1 = lane & 15, hh = lane >> 4, k = k1 + 16 * (2 * brev4(i) + hh);
      double re = 0, im = 0;
      for (int n = 0; n < 512; n++) {
        const double a = -2 * M_PI * (double)n * k / 512;
        re += h[n].x * cos(a) - h[n].y * sin(a);
        im += h[n].x * sin(a) + h[n].y * cos(a);
      }
      maxerr = fmax(maxerr, fabs(re - o[lane * 16 + i].x) + fabs(im - o[lane * 16 + i].y));
    }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fft_kernel<<<nfft / 4, 128>>>(din, dout, dtw, reps);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double ffts = (double)nfft * reps;
  const double cyc_per_fft_per_sm = 148.0 * 1965e6 * ms * 1e-3 / ffts;
  printf("{\"max_abs_err_fft0\": %.3e, \"ms\": %.3f, \"ffts_per_s\": %.3e, \"sm_cycles_per_fft\": %.1f, \"status\": \"%s\"}\n",
         maxerr, ms, ffts / (ms * 1e-3), cyc_per_fft_per_sm, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
