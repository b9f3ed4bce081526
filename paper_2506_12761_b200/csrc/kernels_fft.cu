// kernels_fft.cu -- K2F: the blind rotation (S2-S6 of SURVEY 8(a)) on an exact FP64 negacyclic FFT.
//
// Same job, same bytes as K2 (kernels.cu): gate linear form (S2) + mod-switch (S3) + accumulator init (S4) +
// 630 CMux steps (S5) with the accumulator on chip + SampleExtract (S6).  Only the engine of the external
// product differs ("K2F"):
//
//  * negacyclic product mod X^1024 + 1 through the folded 512-point complex FFT: z_j = (x_j + i x_{j+512}) psi^j,
//    psi = exp(i pi / 1024), A_k = sum_j z_j w^{jk}, w = exp(2 pi i / 512), so A_k = x(psi^{4k+1});
//  * the bootstrapping key split into two signed 16-bit limbs b = lo + 2^16 hi (R_lo, R_hi each bounded by
//    6 * 1024 * 64 * 2^15 = 2^33.6); the FFT-domain key (scaled by 1/512) is computed at setup by a direct DFT
//    (K4F below).  The rounding error of every limb result is far below 1/2 (bound and measured
//    margin, tools/emulate_br_fft.py), so round(R_lo) + 2^16 round(R_hi) mod 2^32 is the exact torus32 external
//    product -- bit-identical to the NTT engine and to the oracle.
//  * one warp = one bootstrap: lane b holds 16 complex points; the 512-point FFT is four-step 16 x 32: a 16-point
//    DFT in registers, per-lane twiddles psi^{b(1 + 4 k1)}, a transpose through warp-private shared memory, one
//    radix-2 stage across the lane pair (L, L ^ 16) by shuffles, a second 16-point DFT in registers.  After the
//    forward transform lane L / register rho holds point k = L + 32 mrev(rho).  No CTA-wide barrier on the step
//    path: the warps of a CTA meet only at the shared key ring (TMA bulk copies, mbarriers).
//  * per digit row, the MAC acc[o][l] += X_r * B_r[o][l] runs right after the row's FFT with the four complex
//    accumulators per point parked in TMEM (tcgen05.ld / st, 256 columns per warp; no MMA).
//  * one kernel launch per wave of 8 x SMs bootstraps (launch_fft_w): all CTAs of a launch walk the 630 steps
//    together, so each key chunk is fetched from DRAM once and served to the other CTAs from L2.
//  * the <W, true> instantiations are the rounding monitor (vlp_debug_fft_error): they also record the largest
//    |V - round(V)| of every limb result (the exactness margin is 1/2).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdint>

#include "devcommon.cuh"
#include "kernels.cuh"

namespace vlp {
namespace {
using namespace dev;

struct cd {
  double x, y;
};
__device__ __forceinline__ cd cadd(cd a, cd b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ cd csub(cd a, cd b) { return {a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ cd cmul(cd a, cd b) { return {fma(a.x, b.x, -(a.y * b.y)), fma(a.x, b.y, a.y * b.x)}; }
__device__ __forceinline__ cd cmulc(cd a, cd b) { return {fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -(a.x * b.y))}; }  // a conj(b)

__constant__ cd c_twist[16];  // psi^(32 a): the uniform part of the fold twist
__constant__ cd c_w16[16];    // w16^k = psi^(128 k)
__constant__ cd c_w32[8];     // w32^r = psi^(64 r)

constexpr int kFSlots = 5;                         // key ring depth (chunks of 16 KB)
#ifndef VLP_DESYNC
#define VLP_DESYNC 3500
#endif
constexpr long long kDesyncCycles = VLP_DESYNC;    // start offset of warps 4-7 (see the step loop)
constexpr int kTrStride = 17;                      // complex per transpose row (one pad: conflict-free LDS.128)
constexpr int kTrBytes = 2 * 16 * kTrStride * 16;  // T[g 2][k1 16][i 16 + 1]: 8704
constexpr int kFWarpBytes = 2 * N * 4 + kTrBytes + 640 * 2;  // accumulator + transpose buffer + abar: 18,176
__host__ __device__ constexpr int fft_smem_bytes(int W) {
  return kFSlots * kFftChunkBytes + W * kFWarpBytes + kFSlots * 8 + kFSlots * 4 + 16;
}
static_assert(fft_smem_bytes(kFftMaxWarps) <= 232448, "shared memory per CTA");
constexpr int kFSmemMin = 120 * 1024;  // every K2F CTA asks for >= this: one CTA per SM (TMEM is allocated whole)

__host__ __device__ constexpr int mrev(int r) { return (r >> 2) | ((r & 3) << 2); }

// 4-point DFT in place, (a, b, c, d) <- (X0, X1, X2, X3), omega_4 = +i (forward) or -i (inverse)
template <bool INV>
__device__ __forceinline__ void bfly4(cd& a, cd& b, cd& c, cd& d) {
  const cd s02 = cadd(a, c), d02 = csub(a, c), s13 = cadd(b, d), d13 = csub(b, d);
  a = cadd(s02, s13);
  c = csub(s02, s13);
  if (!INV) {
    b = {d02.x - d13.y, d02.y + d13.x};
    d = {d02.x + d13.y, d02.y - d13.x};
  } else {
    b = {d02.x + d13.y, d02.y - d13.x};
    d = {d02.x - d13.y, d02.y + d13.x};
  }
}
// multiply by w16^e (e compile-time; e = 0 identity, e = 4 is +i)
template <bool INV>
__device__ __forceinline__ cd tw16(cd v, int e) {
  if (e == 0) return v;
  if (e == 4) return INV ? cd{v.y, -v.x} : cd{-v.y, v.x};
  return INV ? cmulc(v, c_w16[e]) : cmul(v, c_w16[e]);
}
// 16-point DFT, radix 4 x 4.  Forward: natural in -> register rho holds X[mrev(rho)].  Inverse: the exact
// mirror (register rho holds X[mrev(rho)] -> 16 x natural).
__device__ __forceinline__ void dft16_fwd(cd (&v)[16]) {
#pragma unroll
  for (int a0 = 0; a0 < 4; a0++) {
    bfly4<false>(v[a0], v[a0 + 4], v[a0 + 8], v[a0 + 12]);
#pragma unroll
    for (int k0 = 1; k0 < 4; k0++) v[a0 + 4 * k0] = tw16<false>(v[a0 + 4 * k0], a0 * k0);
  }
#pragma unroll
  for (int k0 = 0; k0 < 4; k0++) bfly4<false>(v[4 * k0], v[4 * k0 + 1], v[4 * k0 + 2], v[4 * k0 + 3]);
}
__device__ __forceinline__ void dft16_inv(cd (&v)[16]) {
#pragma unroll
  for (int k0 = 0; k0 < 4; k0++) {
    bfly4<true>(v[4 * k0], v[4 * k0 + 1], v[4 * k0 + 2], v[4 * k0 + 3]);
#pragma unroll
    for (int a0 = 1; a0 < 4; a0++) v[4 * k0 + a0] = tw16<true>(v[4 * k0 + a0], a0 * k0);
  }
#pragma unroll
  for (int a0 = 0; a0 < 4; a0++) bfly4<true>(v[a0], v[a0 + 4], v[a0 + 8], v[a0 + 12]);
}

__device__ __forceinline__ cd shfl16(cd v) {
  return {__shfl_xor_sync(0xffffffffu, v.x, 16), __shfl_xor_sync(0xffffffffu, v.y, 16)};
}

// Gadget digit field f = (w >> s) & 127 (R5: w = D + 0x81020400) enters the FFT as the double f - 64, exactly:
// (2^52 + f) - (2^52 + 64), the first term built by putting f into the low mantissa word of 2^52 (fft_fwd).

// Per-lane constants of the transform (lane b = 16 h + bb).
//  * Lanes with h = 1 negate the odd inputs a of their first 16-point DFT, which shifts its output by 8: register
//    rho then holds k1 = mrev(rho) ^ 8h.  So the registers rho with mrev(rho) < 8 ("A": rho & 2 == 0) hold each
//    lane's own 8 k1 values and the lane-pair partner (b ^ 16) holds the matching values in register rho | 2 --
//    the lane-pair radix-2 stage needs no lane-dependent selects (tools/emulate_br_fft.py --v3).
//  * tw[r] = psi^{b (1 + 4 k1(rho = r))} (the fold twist's psi^b merged in); the 8 with mrev(r) < 8 held in registers.
//  * tau = (h ? -1 : 1) w32^bb, the twiddle of the pair's difference (the sign makes both lanes use own - partner).
struct Lane {
  cd tw[8];  // tw of the registers ra = (q & 1) | (q >> 1) << 2 (mrev(ra) < 8), indexed by q
  cd c32;    // psi^{32 b (h ? -1 : 1)}: tw[ra | 2] = tw[ra] c32 (their k1 differ by 8)
  cd tau;
  double sgn, off;  // sgn = h ? -1 : 1; off = -sgn (2^52 + 64) (odd-a digit conversion)
  uint32_t lane, tbase;  // tbase: this lane's transpose offset (8h * kTrStride + bb) in complex
};
// Half the per-lane twiddles are held (8 complex + c32) and the other half formed by one complex product per
// transform pair: 4 more FP64 instructions per pair, 28 fewer registers held across the step (255-register
// kernel): 16.36 -> 16.06 ms per wave (tools/variant_time.sh; a quarter of them, c16 for odd q: 16.20 ms).
__device__ __forceinline__ cd twid(const Lane& c, int r) {
  const cd t = c.tw[(r & 1) | ((r >> 2) << 1)];
  return (r & 2) ? cmul(t, c.c32) : t;
}

// Forward transform of one digit polynomial of this lane's 32 coefficients (wv[q] = offset D at coefficient
// 32 q + lane, q < 32) -> v[rho] = point lane + 32 mrev(rho).
__device__ __forceinline__ void fft_fwd(cd (&v)[16], const uint32_t (&wv)[32], uint32_t s, const Lane& c, double2* tr) {
#pragma unroll
  for (int a = 0; a < 16; a++) {
    const double rx = __hiloint2double(0x43300000, static_cast<int>((wv[a] >> s) & 127u));
    const double ry = __hiloint2double(0x43300000, static_cast<int>((wv[16 + a] >> s) & 127u));
    // (f - 64), times -1 on odd a of the h = 1 lanes (exact: one rounding of a small integer)
    const cd x = (a & 1) ? cd{fma(c.sgn, rx, c.off), fma(c.sgn, ry, c.off)}
                         : cd{rx - 4503599627370560.0, ry - 4503599627370560.0};
    v[a] = a == 0 ? x : cmul(x, c_twist[a]);
  }
  dft16_fwd(v);
  __syncwarp();  // the previous reader of tr is done
#pragma unroll
  for (int q = 0; q < 8; q++) {
    const int ra = (q & 1) | ((q >> 1) << 2);  // 0, 1, 4, 5, 8, 9, 12, 13
    const cd own = cmul(v[ra], twid(c, ra));
    const cd recv = shfl16(cmul(v[ra | 2], twid(c, ra | 2)));
    const cd sm = cadd(own, recv);
    const cd df = cmul(csub(own, recv), c.tau);
    double2* t = tr + c.tbase + mrev(ra) * kTrStride;
    t[0] = make_double2(sm.x, sm.y);
    t[16 * kTrStride] = make_double2(df.x, df.y);
  }
  __syncwarp();
  const double2* row = tr + (c.lane >> 4) * 16 * kTrStride + (c.lane & 15) * kTrStride;
#pragma unroll
  for (int i = 0; i < 16; i++) {
    const double2 t = row[i];
    v[i] = {t.x, t.y};
  }
  dft16_fwd(v);
}

// Inverse transform: v[rho] at point lane + 32 mrev(rho) -> v[a] = 512 sgn^a (c_{32a+lane} + i c_{32a+lane+512})
// (sgn^a: the h = 1 lanes' odd a come out negated; round_u32s undoes it)
__device__ __forceinline__ void fft_inv(cd (&v)[16], const Lane& c, double2* tr) {
  dft16_inv(v);
  __syncwarp();
  double2* row = tr + (c.lane >> 4) * 16 * kTrStride + (c.lane & 15) * kTrStride;
#pragma unroll
  for (int i = 0; i < 16; i++) row[i] = make_double2(v[i].x, v[i].y);
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 8; q++) {
    const int ra = (q & 1) | ((q >> 1) << 2);
    const double2* t = tr + c.tbase + mrev(ra) * kTrStride;
    const double2 s2 = t[0], d2 = t[16 * kTrStride];
    const cd dd = cmulc(cd{d2.x, d2.y}, c.tau);
    const cd own{s2.x + dd.x, s2.y + dd.y};
    const cd part = shfl16(cd{s2.x - dd.x, s2.y - dd.y});
    v[ra] = cmulc(own, twid(c, ra));
    v[ra | 2] = cmulc(part, twid(c, ra | 2));
  }
  dft16_inv(v);
#pragma unroll
  for (int a = 1; a < 16; a++) v[a] = cmulc(v[a], c_twist[a]);
}
// round(sgn^a v) mod 2^32 (see fft_inv): 1.5 * 2^52 shifts the integer part of |v| < 2^51 into the low mantissa word
template <int A>
__device__ __forceinline__ uint32_t round_u32s(double v, const Lane& c) {
  return static_cast<uint32_t>(__double2loint((A & 1) ? fma(c.sgn, v, 6755399441055744.0) : v + 6755399441055744.0));
}

// TMEM (32x32b: lane = thread): one double <-> 2 consecutive columns (lo, hi word).  Each helper is one asm block
// whose 32-bit temporaries ptxas allocates onto the doubles' own register pairs (no gather moves), with the
// tcgen05.wait::ld inside the block, before the temporaries are read.
__device__ __forceinline__ void tm_ld8d(uint32_t ta, double (&v)[8]) {
  asm volatile(
      "{\n .reg .b32 t<16>;\n"
      " tcgen05.ld.sync.aligned.32x32b.x16.b32 {t0,t1,t2,t3,t4,t5,t6,t7,t8,t9,t10,t11,t12,t13,t14,t15}, [%8];\n"
      " tcgen05.wait::ld.sync.aligned;\n"
      " mov.b64 %0, {t0,t1};\n"
      " mov.b64 %1, {t2,t3};\n"
      " mov.b64 %2, {t4,t5};\n"
      " mov.b64 %3, {t6,t7};\n"
      " mov.b64 %4, {t8,t9};\n"
      " mov.b64 %5, {t10,t11};\n"
      " mov.b64 %6, {t12,t13};\n"
      " mov.b64 %7, {t14,t15};\n"
      "}\n"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]), "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7])
      : "r"(ta)
      : "memory");
}
__device__ __forceinline__ void tm_st8d(uint32_t ta, const double (&v)[8]) {
  asm volatile(
      "{\n .reg .b32 t<16>;\n"
      " mov.b64 {t0,t1}, %1;\n"
      " mov.b64 {t2,t3}, %2;\n"
      " mov.b64 {t4,t5}, %3;\n"
      " mov.b64 {t6,t7}, %4;\n"
      " mov.b64 {t8,t9}, %5;\n"
      " mov.b64 {t10,t11}, %6;\n"
      " mov.b64 {t12,t13}, %7;\n"
      " mov.b64 {t14,t15}, %8;\n"
      " tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {t0,t1,t2,t3,t4,t5,t6,t7,t8,t9,t10,t11,t12,t13,t14,t15};\n"
      "}\n" ::"r"(ta),
      "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]), "d"(v[4]), "d"(v[5]), "d"(v[6]), "d"(v[7])
      : "memory");
}
__device__ __forceinline__ void tm_ld_col16(uint32_t ta, cd (&V)[16]) {
  asm volatile(
      "{\n .reg .b32 t<64>;\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t0,t1,t2,t3}, [%32];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t4,t5,t6,t7}, [%33];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t8,t9,t10,t11}, [%34];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t12,t13,t14,t15}, [%35];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t16,t17,t18,t19}, [%36];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t20,t21,t22,t23}, [%37];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t24,t25,t26,t27}, [%38];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t28,t29,t30,t31}, [%39];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t32,t33,t34,t35}, [%40];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t36,t37,t38,t39}, [%41];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t40,t41,t42,t43}, [%42];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t44,t45,t46,t47}, [%43];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t48,t49,t50,t51}, [%44];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t52,t53,t54,t55}, [%45];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t56,t57,t58,t59}, [%46];\n"
      " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t60,t61,t62,t63}, [%47];\n"
      " tcgen05.wait::ld.sync.aligned;\n"
      " mov.b64 %0, {t0,t1};\n mov.b64 %1, {t2,t3};\n"
      " mov.b64 %2, {t4,t5};\n mov.b64 %3, {t6,t7};\n"
      " mov.b64 %4, {t8,t9};\n mov.b64 %5, {t10,t11};\n"
      " mov.b64 %6, {t12,t13};\n mov.b64 %7, {t14,t15};\n"
      " mov.b64 %8, {t16,t17};\n mov.b64 %9, {t18,t19};\n"
      " mov.b64 %10, {t20,t21};\n mov.b64 %11, {t22,t23};\n"
      " mov.b64 %12, {t24,t25};\n mov.b64 %13, {t26,t27};\n"
      " mov.b64 %14, {t28,t29};\n mov.b64 %15, {t30,t31};\n"
      " mov.b64 %16, {t32,t33};\n mov.b64 %17, {t34,t35};\n"
      " mov.b64 %18, {t36,t37};\n mov.b64 %19, {t38,t39};\n"
      " mov.b64 %20, {t40,t41};\n mov.b64 %21, {t42,t43};\n"
      " mov.b64 %22, {t44,t45};\n mov.b64 %23, {t46,t47};\n"
      " mov.b64 %24, {t48,t49};\n mov.b64 %25, {t50,t51};\n"
      " mov.b64 %26, {t52,t53};\n mov.b64 %27, {t54,t55};\n"
      " mov.b64 %28, {t56,t57};\n mov.b64 %29, {t58,t59};\n"
      " mov.b64 %30, {t60,t61};\n mov.b64 %31, {t62,t63};\n"
      "}\n"
      : "=d"(V[0].x), "=d"(V[0].y), "=d"(V[1].x), "=d"(V[1].y), "=d"(V[2].x), "=d"(V[2].y), "=d"(V[3].x), "=d"(V[3].y), "=d"(V[4].x), "=d"(V[4].y), "=d"(V[5].x), "=d"(V[5].y), "=d"(V[6].x), "=d"(V[6].y), "=d"(V[7].x), "=d"(V[7].y), "=d"(V[8].x), "=d"(V[8].y), "=d"(V[9].x), "=d"(V[9].y), "=d"(V[10].x), "=d"(V[10].y), "=d"(V[11].x), "=d"(V[11].y), "=d"(V[12].x), "=d"(V[12].y), "=d"(V[13].x), "=d"(V[13].y), "=d"(V[14].x), "=d"(V[14].y), "=d"(V[15].x), "=d"(V[15].y)
      : "r"(ta + 0u), "r"(ta + 16u), "r"(ta + 32u), "r"(ta + 48u), "r"(ta + 64u), "r"(ta + 80u), "r"(ta + 96u), "r"(ta + 112u), "r"(ta + 128u), "r"(ta + 144u), "r"(ta + 160u), "r"(ta + 176u), "r"(ta + 192u), "r"(ta + 208u), "r"(ta + 224u), "r"(ta + 240u)
      : "memory");
}
// MAC of one key chunk (digit row r, registers 8h .. 8h + 7): acc[o][l] (+)= X * B_r[o][l] per point, the
// accumulators (doubles, re/im, ol = o * 2 + l) at TMEM columns rho * 16 + ol * 4 + {0: re, 2: im}.
template <bool FIRST>
__device__ __forceinline__ void mac_half(const cd (&X)[16], int h, const double2* kc, uint32_t tm) {
#pragma unroll
  for (int rp = 0; rp < 8; rp++) {
    const int rho = 8 * h + rp;
    const uint32_t ta = tm + rho * 16;
    double ac[8];  // [ol][re, im]
    if (!FIRST) tm_ld8d(ta, ac);
#pragma unroll
    for (int ol = 0; ol < 4; ol++) {
      const double2 k = kc[(rp * 4 + ol) * 32];
      if (FIRST) {
        ac[2 * ol] = fma(X[rho].x, k.x, -(X[rho].y * k.y));
        ac[2 * ol + 1] = fma(X[rho].x, k.y, X[rho].y * k.x);
      } else {
        ac[2 * ol] = fma(X[rho].x, k.x, fma(-X[rho].y, k.y, ac[2 * ol]));
        ac[2 * ol + 1] = fma(X[rho].x, k.y, fma(X[rho].y, k.x, ac[2 * ol + 1]));
      }
    }
    tm_st8d(ta, ac);
  }
}

}  // namespace

// Phase timing (dev builds with -DVLP_PHASE_TIMING, tools/fft_phases.py): clock64 deltas per step phase, summed over
// the warps of a launch (read by vlp_debug_phase_read).  Compiled out of the product library.
#ifdef VLP_PHASE_TIMING
__device__ unsigned long long g_phase[8];
__device__ unsigned long long g_cta[3 * 1024];  // per CTA: start, end (globaltimer ns), SM id
__device__ unsigned long long g_cta_ph[8 * 1024];  // per CTA: phase cycles summed over its warps
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
#define VLP_CTA_START \
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta[3 * blockIdx.x] = gtimer();
#define VLP_CTA_END                                      \
  if (threadIdx.x == 0 && blockIdx.x < 1024) {           \
    g_cta[3 * blockIdx.x + 1] = gtimer();                \
    g_cta[3 * blockIdx.x + 2] = smid();                  \
  }
#define VLP_PHASE_DECL \
  unsigned long long ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; \
  long long ph_t = clock64();
#define VLP_PHASE_MARK(k)                                   \
  {                                                          \
    const long long t_ = clock64();                          \
    ph_acc[k] += static_cast<unsigned long long>(t_ - ph_t); \
    ph_t = t_;                                               \
  }
#define VLP_PHASE_OUT                                                                 \
  if (lane == 0) {                                                                    \
    for (int k_ = 0; k_ < 8; k_++) atomicAdd(&g_phase[k_], ph_acc[k_]);              \
    if (blockIdx.x < 1024)                                                            \
      for (int k_ = 0; k_ < 8; k_++) atomicAdd(&g_cta_ph[8 * blockIdx.x + k_], ph_acc[k_]); \
  }
#else
#define VLP_PHASE_DECL
#define VLP_PHASE_MARK(k)
#define VLP_PHASE_OUT
#define VLP_CTA_START
#define VLP_CTA_END
#endif

// ================================================================================ K2F blind rotation
// W warps per CTA, one bootstrap per warp; persistent over groups of W jobs.  Per CMux step and warp:
//   for u in {0 (mask), 1 (body)}: D = X^abar acc_u - acc_u (offset 0x81020400, R5); for each gadget digit j:
//     forward FFT of digit j, then acc4[o][l] (+)= X * B[3u + j][o][l] over this lane's 16 points (TMEM);
//   for o in {0, 1}: inverse FFT of acc4[o][0], acc4[o][1] -> round -> acc_o += R_lo + 2^16 R_hi (mod 2^32).
// The key of a step is 12 chunks of 16 KB (digit row r, register half h: [rho' 8][o*2 + l][lane 32]) streamed by
// TMA into a ring shared by the CTA's warps; the last warp to release a chunk refills its slot.
template <int W, bool ERR = false>
__global__ void __launch_bounds__(W * 32, 1) vlp_blind_rotate_fft_kernel(const BrArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  double2* ring = reinterpret_cast<double2*>(smem);
  uint8_t* wb = smem + kFSlots * kFftChunkBytes;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  const uint32_t w = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform (lets the TMEM address live in a UR)
  uint32_t* acc = reinterpret_cast<uint32_t*>(wb + w * kFWarpBytes);
  double2* tr = reinterpret_cast<double2*>(wb + w * kFWarpBytes + 2 * N * 4);
  uint16_t* abar = reinterpret_cast<uint16_t*>(wb + w * kFWarpBytes + 2 * N * 4 + kTrBytes);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(wb + W * kFWarpBytes);
  uint32_t* rel = reinterpret_cast<uint32_t*>(mbar + kFSlots);
  uint32_t* tmem_base_sh = rel + kFSlots;
  constexpr int kCols = W <= 4 ? 256 : 512;

  const uint32_t ngroups = (a.njobs + W - 1) / W;
  if (blockIdx.x >= ngroups) return;
  const uint32_t my_groups = (ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const uint32_t steps = static_cast<uint32_t>(a.steps);
  const uint32_t total_chunks = my_groups * steps * kFftChunks;  // < 2^32 (launcher checks)

  if (tid == 0) {
    for (int s = 0; s < kFSlots; s++) {
      mbar_init(&mbar[s], 1);
      rel[s] = 0;
    }
    fence_mbar_init();
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_sh)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  VLP_CTA_START
  // this warp's 256 TMEM columns in its lane quadrant: column rho * 16 + (o * 2 + l) * 4 + {re lo, re hi, im lo, im hi}
  const uint32_t tm = *tmem_base_sh + ((32u * (w & 3u)) << 16) + (w >> 2) * 256u;

  // per-lane constants of the transform (see Lane)
  Lane lc;
  {
    const uint32_t h = lane >> 4;
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const int r = (q & 1) | ((q >> 1) << 2);
      const double2 t = a.psi[(lane * (1u + 4u * (static_cast<uint32_t>(mrev(r)) ^ (8u * h)))) & 2047u];
      lc.tw[q] = {t.x, t.y};
    }
    {
      const double2 t = a.psi[(h ? 2048u - 32u * lane : 32u * lane) & 2047u];
      lc.c32 = {t.x, t.y};
    }
    const double2 w32 = a.psi[(64u * (lane & 15u)) & 2047u];
    lc.sgn = h ? -1.0 : 1.0;
    lc.tau = {lc.sgn * w32.x, lc.sgn * w32.y};
    lc.off = -lc.sgn * 4503599627370560.0;
    lc.lane = lane;
    lc.tbase = 8u * h * kTrStride + (lane & 15u);
  }

  auto issue = [&](uint32_t nseq) {
    const uint32_t step = (nseq / kFftChunks) % steps, c = nseq % kFftChunks, s = nseq % kFSlots;
    bulk_load(ring + s * (kFftChunkBytes / 16),
              a.bskf + (static_cast<size_t>(step) * kFftChunks + c) * (kFftChunkBytes / 16), kFftChunkBytes, &mbar[s]);
  };
  if (tid == 0)
    for (uint32_t q = 0; q < kFSlots && q < total_chunks; q++) issue(q);
  uint32_t nseq = 0, sl = 0, ph = 0;
  auto release = [&]() {  // this warp is done with ring slot sl
    __syncwarp();
    if (lane == 0) {
      // no fence: this warp's reads of the slot are complete (their values fed the MAC before the release)
      if (atomicAdd(&rel[sl], 1u) == W - 1) {
        atomicExch(&rel[sl], 0u);
        if (nseq + kFSlots < total_chunks) {
          fence_proxy_async();
          issue(nseq + kFSlots);
        }
      }
    }
    nseq++;
    if (++sl == kFSlots) {
      sl = 0;
      ph ^= 1u;
    }
  };

  for (uint32_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const uint32_t jb = grp * W + w;
    if (jb >= a.njobs) {  // idle warp of the last group: keep the ring moving
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      for (uint32_t c = 0; c < steps * kFftChunks; c++) {
        mbar_wait(&mbar[sl], ph);
        release();
      }
      continue;
    }
    // ---- S2 gate linear form + S3 mod-switch: abar[0..629], bbar at [630], test-vector select at [631]
    {
      const BrJob job = a.jobs[jb];
      const uint32_t* x = slot_ptr(a.reg, job.x);
      const uint32_t* y = slot_ptr(a.reg, job.y);
      for (uint32_t wd = lane; wd <= static_cast<uint32_t>(n); wd += 32) {
        uint32_t c = static_cast<uint32_t>(static_cast<int32_t>(job.ax)) * x[wd];
        if (job.ay) c += static_cast<uint32_t>(static_cast<int32_t>(job.ay)) * y[wd];
        if (wd == static_cast<uint32_t>(n)) c += job.k0;
        abar[wd] = static_cast<uint16_t>(((c + (1u << 20)) >> 21) & (2 * N - 1));
      }
      if (lane == 0) abar[n + 1] = job.tv;
    }
    __syncwarp();
    // ---- S4 accumulator init: (0, X^{-bbar} testv), testv = 1/8 (R8; 1/4 for R24 jobs)
    {
      const uint32_t bbar = abar[n], mu = abar[n + 1] ? 2u * kMu : kMu;
      for (uint32_t k = lane; k < static_cast<uint32_t>(N); k += 32) {
        acc[k] = 0;
        acc[N + k] = (((k + bbar) & (2 * N - 1)) < static_cast<uint32_t>(N)) ? mu : (0u - mu);
      }
    }
    __syncwarp();

    // The two warps of a scheduler (w, w + 4) run the same step sequence; started together they hit their MAC
    // phases (key LDS bursts, shared by all 8 warps) at the same time.  Starting the second one ~half an
    // FFT + MAC period later interleaves one warp's MAC with the other's FFT: 16.58 -> 16.37 ms per wave
    // (profiles/r2_k2f_phases.txt; 2500-4500 cycles all help, 3500 best).
    if (w >= 4) {
      const long long t0 = clock64();
      while (clock64() - t0 < kDesyncCycles) {
      }
    }
    // ---- S5: CMux steps
    double err = 0.0;  // ERR: this lane's largest rounding distance
    VLP_PHASE_DECL
    for (uint32_t i = 0; i < steps; i++) {
      const uint32_t ab = abar[i];
      if (i == a.pdl_at) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#pragma unroll 1
      for (int u = 0; u < 2; u++) {
        const uint32_t* au = acc + u * N;
        uint32_t wv[32];
#pragma unroll
        for (int q = 0; q < 32; q++) {
          const uint32_t j = 32u * q + lane;
          const uint32_t kk = (j - ab) & (2 * N - 1);
          uint32_t v = au[kk & (N - 1)];
          v = kk >= static_cast<uint32_t>(N) ? 0u - v : v;
          wv[q] = v - au[j] + 0x81020400u;
        }
        VLP_PHASE_MARK(0)
#pragma unroll 1
        for (int dj = 0; dj < 3; dj++) {
          cd X[16];
          fft_fwd(X, wv, 25u - 7u * dj, lc, tr);
          VLP_PHASE_MARK(1)
          if (u == 0 && dj == 0) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
              mbar_wait(&mbar[sl], ph);
              VLP_PHASE_MARK(2)
              mac_half<true>(X, h, ring + sl * (kFftChunkBytes / 16) + lane, tm);
              release();
              VLP_PHASE_MARK(3)
            }
          } else {
#pragma unroll
            for (int h = 0; h < 2; h++) {
              mbar_wait(&mbar[sl], ph);
              VLP_PHASE_MARK(2)
              mac_half<false>(X, h, ring + sl * (kFftChunkBytes / 16) + lane, tm);
              release();
              VLP_PHASE_MARK(3)
            }
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          VLP_PHASE_MARK(3)
        }
      }
      // inverse transforms, rounding: acc_o += R_lo, acc_o += 2^16 R_hi (mod 2^32), one limb at a time
#pragma unroll 1
      for (int ol = 0; ol < 4; ol++) {
        cd V[16];
        tm_ld_col16(tm + ol * 4, V);
        VLP_PHASE_MARK(4)
        fft_inv(V, lc, tr);
        VLP_PHASE_MARK(5)
        uint32_t* ao = acc + (ol >> 1) * N + lane;
        const uint32_t sh = (ol & 1) * 16u;
#pragma unroll
        for (int q = 0; q < 16; q++) {
          const uint32_t rx = (q & 1) ? round_u32s<1>(V[q].x, lc) : round_u32s<0>(V[q].x, lc);
          const uint32_t ry = (q & 1) ? round_u32s<1>(V[q].y, lc) : round_u32s<0>(V[q].y, lc);
          if (ERR) {  // distance of each limb result to the integer it rounds to (exactness margin: < 1/2)
            err = fmax(err, fabs(V[q].x - rint(V[q].x)));
            err = fmax(err, fabs(V[q].y - rint(V[q].y)));
          }
          ao[32 * q] += rx << sh;
          ao[512 + 32 * q] += ry << sh;
        }
        VLP_PHASE_MARK(6)
      }
      __syncwarp();
    }
    VLP_PHASE_OUT
    if (ERR) {
#pragma unroll
      for (int o = 16; o; o >>= 1) err = fmax(err, __shfl_xor_sync(0xffffffffu, err, o));
      if (lane == 0) atomicMax(a.fft_err, static_cast<unsigned long long>(__double_as_longlong(err)));
    }

    // ---- S6 SampleExtract: a'_0 = a_0, a'_k = -a_{N-k}, b' = b_0
    if (a.raw_acc) {
      uint32_t* o = a.raw_acc + static_cast<size_t>(jb) * 2 * N;
      for (uint32_t k = lane; k < 2u * N; k += 32) o[k] = acc[k];
    } else {
      uint32_t* o = a.nlwe + static_cast<size_t>(a.jobs[jb].out) * kNlwe;
      for (uint32_t k = lane; k < static_cast<uint32_t>(N); k += 32) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
      if (lane == 0) o[N] = acc[N];
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  VLP_CTA_END
  if (tid < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_base_sh), "n"(kCols) : "memory");
  // A wave launched early (programmatic dependent launch, launch_fft_wk) completes only after the wave before it:
  // the waves of a level share no data, but the kernel after the level relies on stream order over all of them.
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ================================================================================ K4F key conversion (setup)
// One CTA per (i, digit row r): thread k (< 512) computes the four FFT-domain key values of point k (o in {0, 1}
// output component, l in {lo, hi} limb) by a direct DFT in double: B_k = (1/512) sum_j (p_j + i p_{j+512})
// psi^{j (1 + 4k)}, and stores them where lane L = k & 31, register rho = mrev(k >> 5) reads them.
__global__ void __launch_bounds__(512) vlp_bsk_fft_kernel(const uint32_t* __restrict__ raw, double2* __restrict__ out,
                                                          const double2* __restrict__ psi) {
  __shared__ int32_t limb[4][N];  // [o * 2 + l][j]
  const double2* ps = psi;
  const uint32_t ir = blockIdx.x;  // i * 6 + r
  for (uint32_t t = threadIdx.x; t < 2u * N; t += blockDim.x) {
    const uint32_t o = t / N, j = t % N;
    const int64_t s = static_cast<int32_t>(raw[(static_cast<size_t>(ir) * 2 + o) * N + j]);
    const int64_t lo = ((s + 32768) & 65535) - 32768;
    limb[o * 2 + 0][j] = static_cast<int32_t>(lo);
    limb[o * 2 + 1][j] = static_cast<int32_t>((s - lo) >> 16);
  }
  __syncthreads();
  const uint32_t k = threadIdx.x;
  double re[4] = {0, 0, 0, 0}, im[4] = {0, 0, 0, 0};
  for (uint32_t j = 0; j < 512; j++) {
    const double2 t = __ldg(ps + ((j * (1u + 4u * k)) & 2047u));
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const double x = static_cast<double>(limb[q][j]), y = static_cast<double>(limb[q][j + 512]);
      re[q] = fma(x, t.x, fma(-y, t.y, re[q]));
      im[q] = fma(x, t.y, fma(y, t.x, im[q]));
    }
  }
  const uint32_t L = k & 31, rho = static_cast<uint32_t>(mrev(static_cast<int>(k >> 5)));
  const uint32_t h = rho >> 3, rp = rho & 7;
  double2* dst = out + (static_cast<size_t>(ir) * 2 + h) * (kFftChunkBytes / 16);
#pragma unroll
  for (int q = 0; q < 4; q++) dst[(rp * 4 + q) * 32 + L] = make_double2(re[q] / 512.0, im[q] / 512.0);
}

#ifdef VLP_PHASE_TIMING
extern "C" int vlp_debug_cta_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_cta, sizeof(unsigned long long) * 3 * 1024);
  cudaMemcpyFromSymbol(out + 3 * 1024, g_cta_ph, sizeof(unsigned long long) * 8 * 1024);
  const unsigned long long z[8 * 1024] = {};
  cudaMemcpyToSymbol(g_cta_ph, z, sizeof(z));
  return 0;
}
extern "C" int vlp_debug_phase_read(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_phase, sizeof(unsigned long long) * 8);
  const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyToSymbol(g_phase, z, sizeof(z));
  return 0;
}
#endif

void launch_bsk_fft(const uint32_t* raw, double2* out, const double2* psi, cudaStream_t st) {
  vlp_bsk_fft_kernel<<<n * kRows, 512, 0, st>>>(raw, out, psi);
}

void set_fft_constants(const double2* psi) {
  cd tws[16], w16[16], w32[8];
  for (int a = 0; a < 16; a++) tws[a] = {psi[32 * a].x, psi[32 * a].y};
  for (int k = 0; k < 16; k++) w16[k] = {psi[128 * k].x, psi[128 * k].y};
  for (int r = 0; r < 8; r++) w32[r] = {psi[64 * r].x, psi[64 * r].y};
  cudaMemcpyToSymbol(c_twist, tws, sizeof(tws));
  cudaMemcpyToSymbol(c_w16, w16, sizeof(w16));
  cudaMemcpyToSymbol(c_w32, w32, sizeof(w32));
}

// Programmatic dependent launch between the waves of one level: each CTA of wave k signals at CMux step pdl_at
// (VLP_PDL_AT permille of the steps; 0 = off, the default), and once all have, wave k+1 is launched and its CTAs
// take SMs as wave k's CTAs exit, so SMs that finish early do not idle until the slowest CTA of the wave is done.
// Measured slower at every signal point (221-wave level, 16.07 ms per wave without; 16.22-16.36 ms with the signal
// at 0.1 %, 70 %, 87.5 %, 95 % of the steps; profiles/r2_k2f_pdl.txt): kept as an option, off.
static uint32_t pdl_permille() {
  static const uint32_t v = [] {
    const char* e = getenv("VLP_PDL_AT");
    const int x = e ? atoi(e) : 0;
    return static_cast<uint32_t>(x < 0 ? 0 : (x > 1000 ? 1000 : x));
  }();
  return v;
}

template <int W, bool ERR>
static cudaError_t launch_fft_wk(const BrArgs& a0, int sm_count, cudaStream_t st, bool pdl = false) {
  BrArgs a = a0;
  const uint32_t pm = pdl_permille();
  a.pdl_at = pm ? static_cast<uint32_t>(static_cast<uint64_t>(a.steps) * pm / 1000) : 0xffffffffu;
  static std::atomic<uint64_t> attr_set{0};
  const int smem = fft_smem_bytes(W) > kFSmemMin ? fft_smem_bytes(W) : kFSmemMin;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set.load() & bit)) {
    e = cudaFuncSetAttribute(vlp_blind_rotate_fft_kernel<W, ERR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit);
  }
  if (a.njobs == 0) return cudaSuccess;
  const uint64_t groups = (a.njobs + W - 1) / W;
  const int grid = static_cast<int>(groups < static_cast<uint64_t>(sm_count) ? groups : sm_count);
  if (grid <= 0 || (groups + grid - 1) / grid * static_cast<uint64_t>(a.steps) * kFftChunks >= (1ull << 32))
    return cudaErrorInvalidValue;
  if (pdl && pm) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(W * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, vlp_blind_rotate_fft_kernel<W, ERR>, a);
  }
  vlp_blind_rotate_fft_kernel<W, ERR><<<grid, W * 32, smem, st>>>(a);
  return cudaGetLastError();
}
static int waves_per_launch() {
  // One launch per wave (default; VLP_FFT_WAVES=k: at most k waves per launch, 0: one persistent launch): the CTAs
  // of a persistent multi-wave launch drift apart by whole groups, so the key chunks they stream span many CMux
  // steps and miss in L2; relaunching per wave keeps all CTAs on the same steps (221-wave level: 17.02 -> 16.57 ms
  // per wave, tools/wave_drift.py).
  static const int per_launch = [] {
    const char* e = getenv("VLP_FFT_WAVES");
    return e ? atoi(e) : 1;
  }();
  return per_launch;
}

uint32_t fft_launch_count(uint32_t njobs, int warps, int sm_count) {
  if (njobs == 0) return 0;
  const uint64_t wave = static_cast<uint64_t>(warps) * static_cast<uint64_t>(sm_count);
  const int k = waves_per_launch();
  if (k <= 0 || njobs <= wave * k) return 1;
  const uint64_t span = wave * static_cast<uint64_t>(k);
  return static_cast<uint32_t>((njobs + span - 1) / span);
}

template <int W>
static cudaError_t launch_fft_w(const BrArgs& a, int sm_count, cudaStream_t st) {
  const int per_launch = waves_per_launch();
  const uint64_t wave = static_cast<uint64_t>(W) * static_cast<uint64_t>(sm_count);
  if (per_launch > 0 && a.njobs > wave * per_launch) {
    const uint64_t span = wave * static_cast<uint64_t>(per_launch);
    for (uint64_t off = 0; off < a.njobs; off += span) {
      BrArgs b = a;
      b.jobs = a.jobs + off;
      b.njobs = static_cast<uint32_t>(std::min<uint64_t>(span, a.njobs - off));
      if (a.raw_acc) b.raw_acc = a.raw_acc + off * 2 * N;
      const bool pdl = off > 0;  // the first wave waits for the previous level in full
      const cudaError_t e =
          a.fft_err ? launch_fft_wk<W, true>(b, sm_count, st, pdl) : launch_fft_wk<W, false>(b, sm_count, st, pdl);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  return a.fft_err ? launch_fft_wk<W, true>(a, sm_count, st) : launch_fft_wk<W, false>(a, sm_count, st);
}

cudaError_t launch_blind_rotate_fft(const BrArgs& a, int warps, int sm_count, cudaStream_t st) {
  switch (warps) {
    case 1: return launch_fft_w<1>(a, sm_count, st);
    case 2: return launch_fft_w<2>(a, sm_count, st);
    case 3: return launch_fft_w<3>(a, sm_count, st);
    case 4: return launch_fft_w<4>(a, sm_count, st);
    case 5: return launch_fft_w<5>(a, sm_count, st);
    case 6: return launch_fft_w<6>(a, sm_count, st);
    case 7: return launch_fft_w<7>(a, sm_count, st);
    default: return launch_fft_w<8>(a, sm_count, st);
  }
}

}  // namespace vlp
