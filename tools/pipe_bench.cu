// Per-instruction throughput microbenchmark on sm_100a (dev tool; results go to profiles/).
// Each thread runs 8 independent dependency chains of one instruction kind (or a 1:1 mix of two kinds);
// 4 x 148 CTAs x 512 threads keep every SMSP full.  Reports warp-instructions per SM per cycle at the
// observed clock (computed from the max SM clock: sm_max_mhz), and lane-ops/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench tools/pipe_bench.cu && ./pipe_bench
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CH 8
__device__ __forceinline__ uint32_t umin_(uint32_t a, uint32_t b) { return a < b ? a : b; }

template <int MODE>
__global__ void __launch_bounds__(512) kern(uint32_t* out, uint32_t iters, uint32_t seed) {
  uint32_t a[CH];
  uint64_t w[CH];
  double f[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) {
    a[c] = (threadIdx.x * 2654435761u) ^ (seed + c * 977u);
    w[c] = a[c] * 3ull;
    f[c] = (double)a[c];
  }
  const uint32_t k = seed | 1u, m = seed * 0x9E3779B9u;
  const double dk = 0.9999999, dm = 1e-9 * seed;
  for (uint32_t i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 4; u++) {
#pragma unroll
      for (int c = 0; c < CH; c++) {
        if (MODE == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(k), "r"(m));       // IMAD
        if (MODE == 1) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(k));                    // IMAD.HI
        if (MODE == 2) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[c]) : "r"((uint32_t)(w[c] >> 32)), "r"(k));  // IMAD.WIDE acc
        if (MODE == 3) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[c]) : "d"(dk), "d"(dm));     // DFMA
        if (MODE == 4) asm volatile("add.f64 %0, %0, %1;" : "+d"(f[c]) : "d"(dm));                     // DADD
        if (MODE == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(m));                      // IADD3
        if (MODE == 6) {  // IMAD + DFMA interleaved (separate pipes?)
          asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(k), "r"(m));
          asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[c]) : "d"(dk), "d"(dm));
        }
        if (MODE == 7) {  // IMAD.HI + DFMA
          asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(k));
          asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[c]) : "d"(dk), "d"(dm));
        }
        if (MODE == 8) {  // IMAD + IADD3 (heavy + alu)
          asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(k), "r"(m));
          asm volatile("add.u32 %0, %0, %1;" : "+r"(a[(c + 4) % CH]) : "r"(m));
        }
        if (MODE == 9) asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w[c]) : "r"((uint32_t)(w[c] >> 32)), "r"(k));
        if (MODE == 10) {  // IMAD.HI + IMAD (Shoup product core) -- as a pair
          uint32_t q;
          asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(q) : "r"(a[c]), "r"(k));
          asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(a[c]) : "r"(q), "r"(m));
        }
        if (MODE == 11) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(*reinterpret_cast<float*>(&a[c])) : "f"(0.999f), "f"(1e-7f));
        if (MODE == 12) {  // DFMA + IADD3
          asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(f[c]) : "d"(dk), "d"(dm));
          asm volatile("add.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(m));
        }
        if (MODE == 14) {  // IMAD.WIDE.U32 with 64-bit addend, multiplier refreshed by an IADD3
          a[c] += m;
          asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[c]) : "r"(a[c]), "r"(k));
        }
        if (MODE == 15) {  // IMAD.WIDE.U32 with a 64-bit register addend, multiplier = low word of the chain
          asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[c]) : "r"((uint32_t)w[c]), "r"(k));
        }
        if (MODE == 16) {  // IMAD.WIDE.U32 with RZ addend + LOP3 to refresh the multiplier
          asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w[c]) : "r"((uint32_t)w[c] ^ (uint32_t)(w[c] >> 32)), "r"(k));
        }
        if (MODE == 17) {  // IMAD.WIDE.U32 acc + LOP3 (same ALU op as mode 16, for a fair comparison)
          asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[c]) : "r"((uint32_t)w[c] ^ (uint32_t)(w[c] >> 32)), "r"(k));
        }
        if (MODE == 18) a[c] = umin_(a[c], a[c] - m);  // VIADDMNMX
        if (MODE == 19) {  // VIADDMNMX + IMAD
          a[c] = umin_(a[c], a[c] - m);
          asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(*reinterpret_cast<uint32_t*>(&f[c])) : "r"(k), "r"(m));
        }
        if (MODE == 20) {  // VIADDMNMX + IADD3
          a[c] = umin_(a[c], a[c] - m);
          asm volatile("add.u32 %0, %0, %1;" : "+r"(*reinterpret_cast<uint32_t*>(&f[c])) : "r"(m));
        }
        if (MODE == 21) {  // VIADDMNMX + IMAD.HI
          a[c] = umin_(a[c], a[c] - m);
          asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(*reinterpret_cast<uint32_t*>(&f[c])) : "r"(k));
        }
        if (MODE == 13) {  // IMAD + FFMA
          asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(k), "r"(m));
          asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(*reinterpret_cast<float*>(&w[c])) : "f"(0.999f), "f"(1e-7f));
        }
      }
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) r ^= a[c] ^ (uint32_t)w[c] ^ (uint32_t)(w[c] >> 32) ^ (uint32_t)__double2loint(f[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
void run(const char* name, int per_iter_instr, uint32_t* out, double mhz) {
  const int blocks = 148 * 4, threads = 512;
  const uint32_t iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<MODE><<<blocks, threads>>>(out, iters / 8, 12345u);
  cudaEventRecord(e0);
  kern<MODE><<<blocks, threads>>>(out, iters, 12345u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double instr = double(blocks) * threads * iters * 4 * CH * per_iter_instr;  // lane-instructions
  const double lane_per_s = instr / (ms * 1e-3);
  const double warp_per_sm_clk = lane_per_s / 32 / 148 / (mhz * 1e6);
  printf("{\"mode\": \"%s\", \"lane_instr_per_s_T\": %.2f, \"warp_instr_per_sm_per_clk_at_max\": %.3f, \"ms\": %.3f}\n",
         name, lane_per_s / 1e12, warp_per_sm_clk, ms);
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 148 * 4 * 512 * 4);
  const double mhz = 1965.0;
  run<0>("IMAD", 1, out, mhz);
  run<1>("IMAD.HI", 1, out, mhz);
  run<2>("IMAD.WIDE.U32 acc64", 1, out, mhz);
  run<9>("IMAD.WIDE.U32 no-acc (+LOP3)", 1, out, mhz);
  run<10>("IMAD.HI+IMAD pair (2 instr)", 2, out, mhz);
  run<3>("DFMA", 1, out, mhz);
  run<4>("DADD", 1, out, mhz);
  run<5>("IADD3", 1, out, mhz);
  run<11>("FFMA", 1, out, mhz);
  run<6>("IMAD+DFMA (2 instr)", 2, out, mhz);
  run<7>("IMAD.HI+DFMA (2 instr)", 2, out, mhz);
  run<8>("IMAD+IADD3 (2 instr)", 2, out, mhz);
  run<12>("DFMA+IADD3 (2 instr)", 2, out, mhz);
  run<13>("IMAD+FFMA (2 instr)", 2, out, mhz);
  run<15>("IMAD.WIDE.U32 acc64 chain", 1, out, mhz);
  run<16>("IMAD.WIDE.U32 RZ-addend + LOP3 (2 instr)", 2, out, mhz);
  run<17>("IMAD.WIDE.U32 acc64 + LOP3 (2 instr)", 2, out, mhz);
  run<18>("VIADDMNMX", 1, out, mhz);
  run<19>("VIADDMNMX+IMAD (2 instr)", 2, out, mhz);
  run<20>("VIADDMNMX+IADD3 (2 instr)", 2, out, mhz);
  run<21>("VIADDMNMX+IMAD.HI (2 instr)", 2, out, mhz);
  run<14>("IMAD.WIDE.U32 acc64 + IADD3 (2 instr)", 2, out, mhz);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
