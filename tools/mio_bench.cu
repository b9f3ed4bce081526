// MIO-side throughput microbenchmark on sm_100a (dev tool): SHFL, LDS.128, and TMEM loads (tcgen05.ld
// 32x32b.x16) per SM per clock.  592 CTAs x 512 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mio_bench tools/mio_bench.cu && ./mio_bench
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

template <int MODE>
__global__ void __launch_bounds__(512, 1) kern(uint32_t* out, uint32_t iters) {
  __shared__ __align__(16) uint32_t sm[512 * 4 + 64];
  __shared__ uint32_t tbase;
  uint32_t v[16];
#pragma unroll
  for (int i = 0; i < 16; i++) v[i] = threadIdx.x * 16 + i;
  for (int i = threadIdx.x; i < 512 * 4; i += 512) sm[i] = i;
  if (MODE == 2) {
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&tbase)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  }
  __syncthreads();
  if (MODE == 2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t ta = (MODE == 2) ? tbase + ((32u * (warp & 3u)) << 16) + (warp >> 2) * 64 : 0;
  uint32_t acc = 0;
  for (uint32_t it = 0; it < iters; it++) {
    if (MODE == 0) {  // 16 SHFL per iteration
#pragma unroll
      for (int i = 0; i < 16; i++) v[i] = __shfl_xor_sync(0xffffffffu, v[i], 1 + (i & 7)) + it;
    }
    if (MODE == 1) {  // 4 LDS.128 per iteration (64 B per thread)
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const uint4 q = reinterpret_cast<const uint4*>(sm)[(threadIdx.x + i * 128 + it) & 511];
        v[4 * i] += q.x; v[4 * i + 1] += q.y; v[4 * i + 2] += q.z; v[4 * i + 3] += q.w;
      }
    }
    if (MODE == 2) {  // one tcgen05.ld 32x32b.x16 (64 B per thread) per iteration
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(ta + (it & 1) * 16)
          : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 16; i++) v[i] += r[i];
    }
  }
#pragma unroll
  for (int i = 0; i < 16; i++) acc ^= v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (MODE == 2) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
}

template <int MODE>
void run(const char* name, double bytes_per_thread_iter, double instr_per_iter, uint32_t* out) {
  const int blocks = 148, threads = 512;
  const uint32_t iters = 1 << 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<MODE><<<blocks, threads>>>(out, iters / 16);
  cudaEventRecord(e0);
  kern<MODE><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double clk = 148.0 * 1965e6 * ms * 1e-3;  // SM-cycles at max clock
  const double warp_instr = double(blocks) * threads / 32 * iters * instr_per_iter;
  const double bytes = double(blocks) * threads * iters * bytes_per_thread_iter;
  printf("{\"mode\": \"%s\", \"warp_instr_per_sm_clk\": %.3f, \"bytes_per_sm_clk\": %.1f, \"ms\": %.3f}\n", name,
         warp_instr / clk, bytes / clk, ms);
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 148 * 512 * 4);
  run<0>("SHFL.BFLY (32-bit)", 16 * 4, 16, out);
  run<1>("LDS.128", 64, 4, out);
  run<2>("tcgen05.ld 32x32b.x16 + wait", 64, 1, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
