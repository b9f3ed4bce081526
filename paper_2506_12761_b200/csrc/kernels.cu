// kernels.cu -- the sm_100a kernels of the hot path.
//
//  K2 vlp_blind_rotate_kernel<B> : gate linear form (S2) + mod-switch (S3) + accumulator init (S4) +
//                               630 CMux steps (S5) with the accumulator on chip + SampleExtract (S6);
//                               B = 5 bootstraps per CTA for whole waves, 1-4 for narrow tails
//  K2 vlp_blind_rotate_lat_kernel : the same for a tail of <= 1 bootstrap per SM, one bootstrap on 6 warp
//                               groups (latency mode)
//  K2 vlp_blind_rotate_clat_kernel : a tail of <= 1 bootstrap per 2 SMs, one bootstrap on a 2-CTA cluster
//                               (one accumulator component per SM, DSMEM exchange of the MAC inputs)
//  K2 vlp_blind_rotate_c6_kernel : a tail of <= 1 bootstrap per resident 6-CTA cluster, one bootstrap on 6
//                               SMs (one digit polynomial and one output limb per SM)
//  K3T (kernels_ks.cu)         : MUX combine (S7) + key switch (S8) as a hand-written tcgen05 int8 GEMM
//  K2F (kernels_fft.cu)        : the blind rotation on an exact FP64 FFT (whole waves)
//  K4 vlp_bsk_convert_kernel  : bsk -> 3-limb NTT domain (setup)
//  K5 vlp_linear_kernel       : R24 linear aggregation (exact ciphertext sums; option outside the paper)
//  vlp_encrypt_db_kernel      : device PubKeyGen + ServerEnc (setup)
//
// Exact arithmetic: NTT prime p = 0x3fff7801 (p = 1 mod 2048, 4p < 2^32); the
// bootstrapping key is split into three signed limbs (11, 11, 10 bits) so every limb product sum is
// below p/2 and lifts back exactly; the torus32 result is R0 + 2^11 R1 + 2^22 R2 mod 2^32.
// Forward transform: Cooley-Tukey, merged psi-twist, natural -> bit-reversed, Harvey lazy butterflies
// (values in [0, 4p)) with Shoup twiddles.  Inverse: Gentleman-Sande, bit-reversed -> natural, values in
// [0, 2p); N^-1 and the Montgomery factor are folded into the stored key.
//
// Thread layout of one bootstrap: see "layouts / swizzle" below (128 threads x 8 coefficients).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"
#include "devcommon.cuh"

namespace vlp {
namespace cg = cooperative_groups;
namespace {
using namespace dev;

constexpr uint32_t P = kP;
constexpr uint32_t P2 = 2u * kP;

constexpr uint32_t inv_mod_2_32(uint32_t p) {
  uint32_t x = p;  // Newton iteration for p^-1 mod 2^32
  for (int i = 0; i < 5; i++) x *= 2u - p * x;
  return x;
}
constexpr uint32_t PINV_NEG = 0u - inv_mod_2_32(P);  // -p^-1 mod 2^32 (Montgomery REDC)
static_assert(static_cast<uint32_t>(P * inv_mod_2_32(P)) == 1u, "inverse");

__constant__ uint2 c_tw[2][8];  // uniform twiddles (k < 8, stages 0-2) of the forward / inverse transforms

// ------------------------------------------------------------------------------ modular helpers
__device__ __forceinline__ uint32_t umin(uint32_t a, uint32_t b) { return a < b ? a : b; }

// Shoup: y * w mod p in [0, 2p) for any y < 2^32, w < p, ws = floor(w 2^32 / p).
__device__ __forceinline__ uint32_t shoup(uint32_t y, uint32_t w, uint32_t ws) {
  const uint32_t q = __umulhi(y, ws);
  return y * w - q * P;
}
// a + b as a three-input add with a runtime zero (BrArgs::zero, always 0): an IADD3 on the ALU pipe, which
// keeps ptxas from turning the add into IMAD.IADD on the heavy FMA pipe -- the binding unit of the blind
// rotation.
__device__ __forceinline__ uint32_t add_alu(uint32_t a, uint32_t b, uint32_t zero) { return a + b + zero; }
// Runtime constants (BrArgs::zero = 0, BrArgs::p2 = 2p): three-register adds cannot become IMAD.IADD.
struct Rc {
  uint32_t z, p2;
};
// Forward CT butterfly, inputs / outputs in [0, 4p).  X_SMALL: x is known to be < 2p already (stage 0 on
// gadget digits, which enter as p + d with |d| <= 64), so its conditional subtraction is skipped.
template <bool X_SMALL = false>
__device__ __forceinline__ void ct_bfly(uint32_t& x, uint32_t& y, uint32_t w, uint32_t ws, Rc z) {
  const uint32_t xr = X_SMALL ? x : umin(x, x - P2);
  const uint32_t t = shoup(y, w, ws);
  x = add_alu(xr, t, z.z);
  y = xr - t + z.p2;
}
// Inverse GS butterfly, inputs / outputs in [0, 2p).
__device__ __forceinline__ void gs_bfly(uint32_t& x, uint32_t& y, uint32_t w, uint32_t ws, Rc z) {
  uint32_t s = add_alu(x, y, z.z);
  s = umin(s, s - P2);
  const uint32_t d = x - y + z.p2;
  x = s;
  y = shoup(d, w, ws);
}

// Per-bootstrap named barrier (ids 1..B; 128 threads): the bootstraps of a CTA only meet at the bsk ring.
__device__ __forceinline__ void bar_boot(uint32_t g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "n"(kBT) : "memory");
}

// ------------------------------------------------------------------------------ layouts / swizzle
// One bootstrap = 128 threads x 8 registers per polynomial (t in [0,128), r in [0,8)):
//   layout A (stages 0-2, uniform twiddles):  j = t | r<<7
//   layout B (stages 3-5):                     j = (t>>4)<<7 | r<<4 | (t&15)
//   layout C (stages 6-8):                     j = (t>>1)<<4 | r<<1 | (t&1)
//   stage 9 pairs lanes t, t^1: a lane-pair register exchange makes them in-register butterflies on
//   (reg[i], reg[4+i]); afterwards slot s of lane t holds NTT position posF(t, s) (tools/emulate_br_v2.py).
// Shared-memory exchanges use phys(j) = j ^ (j5<<1 ^ j6<<2 ^ j7<<3 ^ j7<<4), conflict-free for A, B and C,
// written as base(t) ^ c(r).
__device__ __forceinline__ uint32_t bit(uint32_t x, int b) { return (x >> b) & 1u; }
__device__ __forceinline__ uint32_t baseA(uint32_t t) { return t ^ (bit(t, 5) << 1) ^ (bit(t, 6) << 2); }
__host__ __device__ constexpr uint32_t cA(int r) { return (static_cast<uint32_t>(r) << 7) ^ ((r & 1) * 24u); }
__device__ __forceinline__ uint32_t baseB(uint32_t t) {
  return ((((t >> 4) << 7) | (t & 15u)) ^ (bit(t, 4) * 24u));
}
__host__ __device__ constexpr uint32_t cB(int r) {
  return (static_cast<uint32_t>(r) << 4) ^ (((r >> 1) & 1) << 1) ^ (((r >> 2) & 1) << 2);
}
__device__ __forceinline__ uint32_t baseC(uint32_t t) {
  return ((((t >> 1) << 4) | (t & 1u)) ^ (bit(t, 2) << 1) ^ (bit(t, 3) << 2) ^ (bit(t, 4) * 24u));
}
__host__ __device__ constexpr uint32_t cC(int r) { return static_cast<uint32_t>(r) << 1; }

typedef uint32_t Poly3[3][8];

// Stages 0-2 (layout A): pair (r, r | rb), rb = 4 >> s; twiddle k = 2^s + (r >> (3 - s)), uniform.
template <int S, bool INV, int NP>
__device__ __forceinline__ void stage_A(uint32_t (&d)[NP][8], Rc z) {
  constexpr int rb = 4 >> S;
#pragma unroll
  for (int r = 0; r < 8; r++) {
    if (r & rb) continue;
    const uint2 w = c_tw[INV][(1 << S) + (r >> (3 - S))];
#pragma unroll
    for (int p = 0; p < NP; p++) {
      if (INV) gs_bfly(d[p][r], d[p][r | rb], w.x, w.y, z);
      else ct_bfly<S == 0>(d[p][r], d[p][r | rb], w.x, w.y, z);
    }
  }
}

// Stage 0 of the forward transform on gadget digits: y = p + d with d in [-64, 64) (field f = d + 64), so
// w0 * y mod p = T[f] from a 128-entry shared table (T[f] = w0 (f - 64) mod p) instead of a Shoup product
// (an LDS instead of IMAD.HI + 2 IMAD on the heavy pipe).  x < 2p (digits), outputs < 3p.
template <int NP>
__device__ __forceinline__ void stage0_digits(uint32_t (&d)[NP][8], const uint32_t* __restrict__ t0, Rc z) {
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int p = 0; p < NP; p++) {
      const uint32_t x = d[p][r];
      const uint32_t t = t0[d[p][r + 4] - (P - 64u)];
      d[p][r] = add_alu(x, t, z.z);
      d[p][r + 4] = x - t + z.p2;
    }
}

// Lane-varying stages 3-8: layout B (S = 3..5) or C (S = 6..8); rb = 4 >> (S % 3); twiddle slot
// q = r >> (3 - S % 3) at table row kSlotBase[S] + q, column t.
// SMTW: the twiddle table is in shared memory (cluster kernels: cluster barriers invalidate L1).
template <int S, bool INV, int NP, bool SMTW = false>
__device__ __forceinline__ void stage_BC(uint32_t (&d)[NP][8], const uint2* __restrict__ twl, Rc z) {
  constexpr int rb = 4 >> (S % 3);
  constexpr int base = S == 3 ? 0 : S == 4 ? 1 : S == 5 ? 3 : S == 6 ? 7 : S == 7 ? 8 : 10;
#pragma unroll
  for (int r = 0; r < 8; r++) {
    if (r & rb) continue;
    const uint2 w = SMTW ? twl[(base + (r >> (3 - S % 3))) * kBT] : __ldg(twl + (base + (r >> (3 - S % 3))) * kBT);
#pragma unroll
    for (int p = 0; p < NP; p++) {
      if (INV) gs_bfly(d[p][r], d[p][r | rb], w.x, w.y, z);
      else ct_bfly(d[p][r], d[p][r | rb], w.x, w.y, z);
    }
  }
}

// Stage 9 forward: lane-pair exchange (lower lane keeps pairs r = 0..3, upper lane r = 4..7), then
// butterflies on (d[i], d[4+i]) with twiddle slots 14..17.
template <int NP, bool SMTW = false>
__device__ __forceinline__ void stage9_fwd(uint32_t (&d)[NP][8], uint32_t t, const uint2* __restrict__ twl, Rc z) {
  const bool lo = (t & 1u) == 0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const uint2 w = SMTW ? twl[(14 + i) * kBT] : __ldg(twl + (14 + i) * kBT);
#pragma unroll
    for (int p = 0; p < NP; p++) {
      const uint32_t send = lo ? d[p][4 + i] : d[p][i];
      const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, 1);
      uint32_t x = lo ? d[p][i] : recv;
      uint32_t y = lo ? recv : d[p][4 + i];
      ct_bfly(x, y, w.x, w.y, z);
      d[p][i] = x;
      d[p][4 + i] = y;
    }
  }
}

// Stage 9 inverse: butterflies on (d[i], d[4+i]), then the reverse lane-pair exchange (back to layout C).
template <int NP, bool SMTW = false>
__device__ __forceinline__ void stage9_inv(uint32_t (&d)[NP][8], uint32_t t, const uint2* __restrict__ twl, Rc z) {
  const bool lo = (t & 1u) == 0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const uint2 w = SMTW ? twl[(14 + i) * kBT] : __ldg(twl + (14 + i) * kBT);
#pragma unroll
    for (int p = 0; p < NP; p++) {
      gs_bfly(d[p][i], d[p][4 + i], w.x, w.y, z);
      const uint32_t send = lo ? d[p][4 + i] : d[p][i];
      const uint32_t recv = __shfl_xor_sync(0xffffffffu, send, 1);
      d[p][i] = lo ? d[p][i] : recv;
      d[p][4 + i] = lo ? recv : d[p][4 + i];
    }
  }
}

// Layout change of NP polynomials through shared memory (xb: NP x 1024 words; named barrier g + 1 over the
// 128 threads that own them).
template <int FROM, int TO, int NP>
__device__ __forceinline__ void exchange(uint32_t (&d)[NP][8], uint32_t* xb, uint32_t t, uint32_t g) {
  const uint32_t bs = FROM == 0 ? baseA(t) : (FROM == 1 ? baseB(t) : baseC(t));
  const uint32_t bd = TO == 0 ? baseA(t) : (TO == 1 ? baseB(t) : baseC(t));
  bar_boot(g);
#pragma unroll
  for (int q = 0; q < NP; q++)
#pragma unroll
    for (int r = 0; r < 8; r++) xb[q * N + (bs ^ (FROM == 0 ? cA(r) : (FROM == 1 ? cB(r) : cC(r))))] = d[q][r];
  bar_boot(g);
#pragma unroll
  for (int q = 0; q < NP; q++)
#pragma unroll
    for (int r = 0; r < 8; r++) d[q][r] = xb[q * N + (bd ^ (TO == 0 ? cA(r) : (TO == 1 ? cB(r) : cC(r))))];
}

}  // namespace

// ================================================================================ K2 blind rotation
// Per CMux step and bootstrap: two forward rounds (component u of D = X^abar acc - acc: its 3 gadget digit
// polynomials -> forward NTT -> Montgomery MAC into the 6 output accumulators, bsk chunks streamed by TMA
// into a smem ring shared by the CTA's bootstraps), then two inverse rounds (output component u: its 3
// key limbs -> inverse NTT -> centered lift -> recombine mod 2^32 -> acc_u += ...).  The round loops are
// not unrolled: each round body is ~25 KB of SASS (the instruction cache, not the ALUs, limited the fully
// unrolled form; profiles/).
template <int B>  // bootstraps per CTA (5 = throughput mode; 1-4 for the narrow tail of a level)
__global__ void __launch_bounds__(B * kBT, 1) vlp_blind_rotate_kernel(const BrArgs a) {
  constexpr int kBrBoot = B, kBrThreads = B * kBT, kTmemCols = tmem_cols(B);
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* ring = reinterpret_cast<uint32_t*>(smem);
  uint32_t* acc_all = ring + kSlots * kBT * kChunkWords;
  uint32_t* xb_all = acc_all + kBrBoot * 2 * N;
  uint16_t* abar_all = reinterpret_cast<uint16_t*>(xb_all + kBrBoot * 3 * N);
  uint32_t* t0tab = reinterpret_cast<uint32_t*>(abar_all + kBrBoot * 640);  // [128] stage-0 digit products
  uint64_t* mbar = reinterpret_cast<uint64_t*>(t0tab + 128);
  uint32_t* rel = reinterpret_cast<uint32_t*>(mbar + kSlots);  // per-slot release counters (warps)
  uint32_t* tmem_base_sh = rel + kSlots;

  const uint32_t tid = threadIdx.x, g = tid / kBT, t = tid % kBT;
  uint32_t* acc = acc_all + g * 2 * N;
  uint32_t* xb = xb_all + g * 3 * N;
  uint16_t* abar = abar_all + g * 640;
  const uint2* twf = a.twl_fwd + t;
  const uint2* twi = a.twl_inv + t;
  const Rc zr{a.zero, a.p2};

  const uint32_t ngroups = (a.njobs + kBrBoot - 1) / kBrBoot;
  if (blockIdx.x >= ngroups) return;
  const uint32_t my_groups = (ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const uint32_t total_chunks = my_groups * static_cast<uint32_t>(a.steps) * kChunks;  // < 2^32 (api.cu limits)

  if (tid == 0) {
    for (int s = 0; s < kSlots; s++) {
      mbar_init(&mbar[s], 1);
      rel[s] = 0;
    }
    fence_mbar_init();
  }
  if (tid < 128) {
    const uint64_t w0 = c_tw[0][1].x;  // the stage-0 twiddle
    t0tab[tid] = static_cast<uint32_t>(w0 * ((tid + P - 64u) % P) % P);
  }
  if (tid < 32) {  // warp 0 allocates the CTA's TMEM (one CTA per SM: smem-bound)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_sh)),
                 "n"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // this warp's TMEM: lanes 32 (warp % 4) .. +31, column slot warp / 4
  const uint32_t warp = tid >> 5;
  const uint32_t tm = *tmem_base_sh + ((32u * (warp & 3u)) << 16) + (warp >> 2) * kTmemSlotCols;
  // chunk sequence n -> (step (n / 8) % steps, chunk n % 8) of the bsk; ring slot n % kSlots
  auto issue = [&](uint32_t nseq) {
    const uint32_t step = (nseq / kChunks) % static_cast<uint32_t>(a.steps), c = nseq % kChunks;
    const uint32_t s = nseq % kSlots;
    bulk_load(ring + s * kBT * kChunkWords, a.bsk + (static_cast<size_t>(step) * kChunks + c) * kBT * kChunkWords,
              kChunkBytes, &mbar[s]);
  };
  if (tid == 0)
    for (uint32_t q = 0; q < kSlots && q < total_chunks; q++) issue(q);
  uint32_t nseq = 0, sl = 0, ph = 0;  // chunk sequence number, its ring slot (nseq % kSlots) and phase parity

  for (uint32_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const uint32_t jb = grp * kBrBoot + g;
    const bool active = jb < a.njobs;
    // ---- S2 gate linear form + S3 mod-switch: abar[0..629], bbar at [630]
    if (active) {
      const BrJob job = a.jobs[jb];
      const uint32_t* x = slot_ptr(a.reg, job.x);
      const uint32_t* y = slot_ptr(a.reg, job.y);
      for (uint32_t w = t; w <= static_cast<uint32_t>(n); w += kBT) {
        uint32_t c = static_cast<uint32_t>(static_cast<int32_t>(job.ax)) * x[w];
        if (job.ay) c += static_cast<uint32_t>(static_cast<int32_t>(job.ay)) * y[w];
        if (w == static_cast<uint32_t>(n)) c += job.k0;
        abar[w] = static_cast<uint16_t>(((c + (1u << 20)) >> 21) & (2 * N - 1));
      }
      if (t == 0) abar[n + 1] = job.tv;  // test vector select (R8 / R24)
    } else {
      for (uint32_t w = t; w <= static_cast<uint32_t>(n) + 1u; w += kBT) abar[w] = 0;
    }
    __syncthreads();
    // ---- S4 accumulator init: (0, X^{-bbar} testv), testv = 1/8 everywhere (R8; 1/4 for R24 jobs)
    {
      const uint32_t bbar = abar[n], mu = abar[n + 1] ? 2u * kMu : kMu;
      for (uint32_t k = t; k < static_cast<uint32_t>(N); k += kBT) {
        acc[k] = 0;
        acc[N + k] = (((k + bbar) & (2 * N - 1)) < static_cast<uint32_t>(N)) ? mu : (0u - mu);
      }
    }
    __syncthreads();

    // ---- S5: CMux steps
    for (int i = 0; i < a.steps; i++) {
      const uint32_t ab = abar[i];
#pragma unroll 1
      for (int u = 0; u < 2; u++) {
        Poly3 d;
        // X^abar acc_u - acc_u (layout A: j = t + 128 r), gadget digits (R5, offset 0x81020400),
        // digit + p - 64 in [p-64, p+64)
#pragma unroll
        for (int r = 0; r < 8; r++) {
          const uint32_t j = t + 128u * r;
          const uint32_t kk = (j - ab) & (2 * N - 1);
          uint32_t v = acc[u * N + (kk & (N - 1))];
          v = kk >= static_cast<uint32_t>(N) ? zr.z - v : v;
          const uint32_t w = v - acc[u * N + j] + 0x81020400u;
          d[0][r] = ((w >> 25) & 127u) + (P - 64u);
          d[1][r] = ((w >> 18) & 127u) + (P - 64u);
          d[2][r] = ((w >> 11) & 127u) + (P - 64u);
        }
        stage0_digits(d, t0tab, zr);
        stage_A<1, false>(d, zr);
        stage_A<2, false>(d, zr);
        exchange<0, 1>(d, xb, t, g);
        stage_BC<3, false>(d, twf, zr);
        stage_BC<4, false>(d, twf, zr);
        stage_BC<5, false>(d, twf, zr);
        exchange<1, 2>(d, xb, t, g);
        stage_BC<6, false>(d, twf, zr);
        stage_BC<7, false>(d, twf, zr);
        stage_BC<8, false>(d, twf, zr);
        stage9_fwd(d, t, twf, zr);
        if (u == 0) {  // park component 0's transformed digits in TMEM for the MAC after round 1
#pragma unroll
          for (int j = 0; j < 3; j++) tmem_st8(tm + 64 + 8 * j, d[j]);
          continue;
        }
        Poly3 d0;
        tmem_wait_st();
#pragma unroll
        for (int j = 0; j < 3; j++) tmem_ld8(tm + 64 + 8 * j, d0[j]);
        tmem_wait_ld();
        // MAC: mac[o][s] = sum_{q<6} Dhat_q[s] * B[q][o][s] (Montgomery, one REDC per output; the key holds
        // N^-1 * 2^32).  Inputs in [0, 2p): T < 12p^2 < 2^63.6, T + m p < 2^64, output < (12p/2^32 + 1)p < 4p.
#pragma unroll
        for (int pp = 0; pp < kChunks; pp++) {
          mbar_wait(&mbar[sl], ph);
          const uint32_t* rec = ring + sl * kBT * kChunkWords + t * kChunkWords;
          uint32_t x[2][6];  // the 6 transformed digit polynomials at positions 2pp + e, reduced to [0, 2p)
#pragma unroll
          for (int e = 0; e < 2; e++)
#pragma unroll
            for (int j = 0; j < 3; j++) {
              x[e][j] = umin(d0[j][2 * pp + e], d0[j][2 * pp + e] - P2);
              x[e][3 + j] = umin(d[j][2 * pp + e], d[j][2 * pp + e] - P2);
            }
#pragma unroll
          for (int o = 0; o < 6; o++) {
            const uint4* kp = reinterpret_cast<const uint4*>(rec + o * 12);  // [e 2][q 6]
            const uint4 k0 = kp[0], k1 = kp[1], k2 = kp[2];
            const uint32_t kv[2][6] = {{k0.x, k0.y, k0.z, k0.w, k1.x, k1.y}, {k1.z, k1.w, k2.x, k2.y, k2.z, k2.w}};
            uint32_t res[2];
#pragma unroll
            for (int e = 0; e < 2; e++) {
              uint64_t T = static_cast<uint64_t>(x[e][0]) * kv[e][0];
#pragma unroll
              for (int q = 1; q < 6; q++) T += static_cast<uint64_t>(x[e][q]) * kv[e][q];
              const uint32_t m = static_cast<uint32_t>(T) * PINV_NEG;
              res[e] = static_cast<uint32_t>((T + static_cast<uint64_t>(m) * P) >> 32);
            }
            // MAC output o = 3 u_out + limb at positions 2pp, 2pp+1 -> TMEM column 32 u_out + 8 limb + 2pp
            tmem_st2(tm + 32 * (o / 3) + 8 * (o % 3) + 2 * pp, res[0], res[1]);
          }
          // release slot sl: the last of the CTA's warps to finish with it refills it (no CTA barrier,
          // so the CTA's bootstraps may drift apart by up to the ring depth)
          __syncwarp();
          if ((tid & 31) == 0) {
            __threadfence_block();
            if (atomicAdd(&rel[sl], 1u) == kBrThreads / 32 - 1) {
              atomicExch(&rel[sl], 0u);
              if (nseq + kSlots < total_chunks) {
                fence_proxy_async();
                issue(nseq + kSlots);
              }
            }
          }
          nseq++;
          if (++sl == kSlots) {
            sl = 0;
            ph ^= 1u;
          }
        }
      }
      tmem_wait_st();
#pragma unroll 1
      for (int u = 0; u < 2; u++) {
        Poly3 d;
#pragma unroll
        for (int l = 0; l < 3; l++) tmem_ld8(tm + 32 * u + 8 * l, d[l]);
        tmem_wait_ld();
#pragma unroll
        for (int l = 0; l < 3; l++)
#pragma unroll
          for (int s = 0; s < 8; s++) d[l][s] = umin(d[l][s], d[l][s] - P2);  // [0, 2p) (mac < 4p)
        stage9_inv(d, t, twi, zr);
        stage_BC<8, true>(d, twi, zr);
        stage_BC<7, true>(d, twi, zr);
        stage_BC<6, true>(d, twi, zr);
        exchange<2, 1>(d, xb, t, g);
        stage_BC<5, true>(d, twi, zr);
        stage_BC<4, true>(d, twi, zr);
        stage_BC<3, true>(d, twi, zr);
        exchange<1, 0>(d, xb, t, g);
        stage_A<2, true>(d, zr);
        stage_A<1, true>(d, zr);
        stage_A<0, true>(d, zr);
        // centered lift of the three limbs, recombine mod 2^32, acc_u += (layout A: j = t + 128 r)
#pragma unroll
        for (int r = 0; r < 8; r++) {
          uint32_t sv[3];
#pragma unroll
          for (int l = 0; l < 3; l++) {
            uint32_t v = d[l][r];
            v = umin(v, v - P);                    // [0, p)
            sv[l] = v > (P >> 1) ? v - P : v;      // centered, two's complement
          }
          // sv0 + 2^11 sv1 + 2^22 sv2 + acc (funnel shifts and three-input adds stay on the ALU pipe)
          const uint32_t hi = __funnelshift_l(0u, sv[1], 11) + __funnelshift_l(0u, sv[2], 22) + zr.z;
          uint32_t& av = acc[u * N + t + 128u * r];
          av = add_alu(av, sv[0], hi);
        }
      }
      bar_boot(g);
    }

    // ---- S6 SampleExtract: a'_0 = a_0, a'_k = -a_{N-k}, b' = b_0
    if (active) {
      if (a.raw_acc) {
        uint32_t* o = a.raw_acc + static_cast<size_t>(jb) * 2 * N;
        for (uint32_t k = t; k < 2u * N; k += kBT) o[k] = acc[k];
      } else {
        uint32_t* o = a.nlwe + static_cast<size_t>(a.jobs[jb].out) * kNlwe;
        for (uint32_t k = t; k < static_cast<uint32_t>(N); k += kBT) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
        if (t == 0) o[N] = acc[N];
      }
    }
    __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_base_sh), "n"(kTmemCols) : "memory");
}


// ================================================================================ K2-LAT (latency mode)
// One bootstrap per CTA for the narrow tail of a level (<= one bootstrap per SM): its 6 digit polynomials
// (forward: group G = 3u + j transforms digit j of component u) and its 6 output limbs (MAC + inverse: group
// G = 3 u_out + l) run on 6 warp groups of 128 threads, one polynomial per warp per phase.  The groups meet
// through TMEM: thread t of every group owns TMEM lane t (warp 4G + t/32 sits in quadrant t/32), so the
// transformed digits (columns 8G + s) and the lifted limbs (48 + 8G + r) written by one group are read by
// the others after a CTA barrier.  Same arithmetic, layouts, key and bytes as the throughput kernel.
constexpr int kLatGroups = 6;
constexpr int kLatSlots = 4;  // a whole CMux step of bsk chunks in flight: a lone bootstrap never waits on TMA
constexpr int kLatThreads = kLatGroups * kBT;
constexpr int kLatTmemCols = 128;
__host__ __device__ constexpr int lat_smem_bytes() {
  return kLatSlots * kChunkBytes + (2 * N * 4 + kLatGroups * N * 4 + 640 * 2) + 128 * 4 + kLatSlots * 8 + kLatSlots * 4 + 8;
}

__global__ void __launch_bounds__(kLatThreads, 1) vlp_blind_rotate_lat_kernel(const BrArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* ring = reinterpret_cast<uint32_t*>(smem);
  uint32_t* acc = ring + kLatSlots * kBT * kChunkWords;
  uint32_t* xb_all = acc + 2 * N;  // [group 6][N]
  uint16_t* abar = reinterpret_cast<uint16_t*>(xb_all + kLatGroups * N);
  uint32_t* t0tab = reinterpret_cast<uint32_t*>(abar + 640);  // [128] stage-0 digit products
  uint64_t* mbar = reinterpret_cast<uint64_t*>(t0tab + 128);
  uint32_t* rel = reinterpret_cast<uint32_t*>(mbar + kLatSlots);
  uint32_t* tmem_base_sh = rel + kLatSlots;

  const uint32_t tid = threadIdx.x, G = tid / kBT, t = tid % kBT;
  uint32_t* xb = xb_all + G * N;
  const uint2* twf = a.twl_fwd + t;
  const uint2* twi = a.twl_inv + t;
  const Rc zr{a.zero, a.p2};
  if (blockIdx.x >= a.njobs) return;
  const uint32_t my_jobs = (a.njobs - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const uint32_t total_chunks = my_jobs * static_cast<uint32_t>(a.steps) * kChunks;

  if (tid == 0) {
    for (int s = 0; s < kLatSlots; s++) {
      mbar_init(&mbar[s], 1);
      rel[s] = 0;
    }
    fence_mbar_init();
  }
  if (tid < 128) {
    const uint64_t w0 = c_tw[0][1].x;  // the stage-0 twiddle
    t0tab[tid] = static_cast<uint32_t>(w0 * ((tid + P - 64u) % P) % P);
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_sh)),
                 "n"(kLatTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = *tmem_base_sh + ((32u * ((tid >> 5) & 3u)) << 16);  // lane t of every group

  auto issue = [&](uint32_t nseq) {
    const uint32_t step = (nseq / kChunks) % static_cast<uint32_t>(a.steps), c = nseq % kChunks;
    const uint32_t s = nseq % kLatSlots;
    bulk_load(ring + s * kBT * kChunkWords, a.bsk + (static_cast<size_t>(step) * kChunks + c) * kBT * kChunkWords,
              kChunkBytes, &mbar[s]);
  };
  if (tid == 0)
    for (uint32_t q = 0; q < kLatSlots && q < total_chunks; q++) issue(q);
  uint32_t nseq = 0, sl = 0, ph = 0;
  auto cta_sync_tmem = [&]() {  // TMEM writes of one group -> reads of another
    tmem_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  };

  for (uint32_t jb = blockIdx.x; jb < a.njobs; jb += gridDim.x) {
    // ---- S2 gate linear form + S3 mod-switch
    {
      const BrJob job = a.jobs[jb];
      const uint32_t* x = slot_ptr(a.reg, job.x);
      const uint32_t* y = slot_ptr(a.reg, job.y);
      for (uint32_t w = tid; w <= static_cast<uint32_t>(n); w += kLatThreads) {
        uint32_t c = static_cast<uint32_t>(static_cast<int32_t>(job.ax)) * x[w];
        if (job.ay) c += static_cast<uint32_t>(static_cast<int32_t>(job.ay)) * y[w];
        if (w == static_cast<uint32_t>(n)) c += job.k0;
        abar[w] = static_cast<uint16_t>(((c + (1u << 20)) >> 21) & (2 * N - 1));
      }
      if (tid == 0) abar[n + 1] = job.tv;  // test vector select (R8 / R24)
    }
    __syncthreads();
    // ---- S4 accumulator init (R8)
    {
      const uint32_t bbar = abar[n], mu = abar[n + 1] ? 2u * kMu : kMu;
      for (uint32_t k = tid; k < static_cast<uint32_t>(N); k += kLatThreads) {
        acc[k] = 0;
        acc[N + k] = (((k + bbar) & (2 * N - 1)) < static_cast<uint32_t>(N)) ? mu : (0u - mu);
      }
    }
    __syncthreads();

    // ---- S5: CMux steps
    const uint32_t uc = G / 3, jl = G % 3;          // forward: component uc, digit jl; MAC/inverse: u_out uc, limb jl
    const uint32_t dshift = 25u - 7u * jl;          // gadget digit jl (R5)
    for (int i = 0; i < a.steps; i++) {
      const uint32_t ab = abar[i];
      {  // digit jl of component uc
        uint32_t d[1][8];
#pragma unroll
        for (int r = 0; r < 8; r++) {
          const uint32_t j = t + 128u * r;
          const uint32_t kk = (j - ab) & (2 * N - 1);
          uint32_t v = acc[uc * N + (kk & (N - 1))];
          v = kk >= static_cast<uint32_t>(N) ? zr.z - v : v;
          const uint32_t w = v - acc[uc * N + j] + 0x81020400u;
          d[0][r] = ((w >> dshift) & 127u) + (P - 64u);
        }
        stage0_digits(d, t0tab, zr);
        stage_A<1, false>(d, zr);
        stage_A<2, false>(d, zr);
        exchange<0, 1>(d, xb, t, G);
        stage_BC<3, false>(d, twf, zr);
        stage_BC<4, false>(d, twf, zr);
        stage_BC<5, false>(d, twf, zr);
        exchange<1, 2>(d, xb, t, G);
        stage_BC<6, false>(d, twf, zr);
        stage_BC<7, false>(d, twf, zr);
        stage_BC<8, false>(d, twf, zr);
        stage9_fwd(d, t, twf, zr);
        tmem_st8(tm + 8 * G, d[0]);  // transformed digit (uc, jl) = digit row G
      }
      cta_sync_tmem();
      // MAC for output o = G = 3 u_out + limb
      uint32_t mac[8];
#pragma unroll
      for (int pp = 0; pp < kChunks; pp++) {
        uint32_t xr[6][2];
#pragma unroll
        for (int q = 0; q < 6; q++) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];"
                       : "=r"(xr[q][0]), "=r"(xr[q][1])
                       : "r"(tm + 8 * q + 2 * pp)
                       : "memory");
        }
        tmem_wait_ld();
        uint32_t x[2][6];
#pragma unroll
        for (int e = 0; e < 2; e++)
#pragma unroll
          for (int q = 0; q < 6; q++) {
            uint32_t v = umin(xr[q][e], xr[q][e] - P2);
            x[e][q] = umin(v, v - P);
          }
        mbar_wait(&mbar[sl], ph);
        const uint32_t* rec = ring + sl * kBT * kChunkWords + t * kChunkWords;
        {
          const uint4* kp = reinterpret_cast<const uint4*>(rec + G * 12);  // [e 2][q 6]
          const uint4 k0 = kp[0], k1 = kp[1], k2 = kp[2];
          const uint32_t kv[2][6] = {{k0.x, k0.y, k0.z, k0.w, k1.x, k1.y}, {k1.z, k1.w, k2.x, k2.y, k2.z, k2.w}};
#pragma unroll
          for (int e = 0; e < 2; e++) {
            uint64_t T = static_cast<uint64_t>(x[e][0]) * kv[e][0];
#pragma unroll
            for (int q = 1; q < 6; q++) T += static_cast<uint64_t>(x[e][q]) * kv[e][q];
            const uint32_t m = static_cast<uint32_t>(T) * PINV_NEG;
            mac[2 * pp + e] = static_cast<uint32_t>((T + static_cast<uint64_t>(m) * P) >> 32);
          }
        }
        __syncwarp();
        if ((tid & 31) == 0) {
          __threadfence_block();
          if (atomicAdd(&rel[sl], 1u) == kLatThreads / 32 - 1) {
            atomicExch(&rel[sl], 0u);
            if (nseq + kLatSlots < total_chunks) {
              fence_proxy_async();
              issue(nseq + kLatSlots);
            }
          }
        }
        nseq++;
        if (++sl == kLatSlots) {
          sl = 0;
          ph ^= 1u;
        }
      }
      // inverse NTT of limb G of both components, centered lift, park in TMEM
      {  // inverse NTT of limb jl of component uc, centered lift, park in TMEM
        uint32_t d[1][8];
#pragma unroll
        for (int s = 0; s < 8; s++) d[0][s] = umin(mac[s], mac[s] - P2);
        stage9_inv(d, t, twi, zr);
        stage_BC<8, true>(d, twi, zr);
        stage_BC<7, true>(d, twi, zr);
        stage_BC<6, true>(d, twi, zr);
        exchange<2, 1>(d, xb, t, G);
        stage_BC<5, true>(d, twi, zr);
        stage_BC<4, true>(d, twi, zr);
        stage_BC<3, true>(d, twi, zr);
        exchange<1, 0>(d, xb, t, G);
        stage_A<2, true>(d, zr);
        stage_A<1, true>(d, zr);
        stage_A<0, true>(d, zr);
#pragma unroll
        for (int r = 0; r < 8; r++) {
          const uint32_t v = umin(d[0][r], d[0][r] - P);
          d[0][r] = v > (P >> 1) ? v - P : v;  // centered, two's complement
        }
        tmem_st8(tm + 48 + 8 * G, d[0]);
      }
      cta_sync_tmem();
      // recombine R0 + 2^11 R1 + 2^22 R2 and acc_uc += (layout A: j = t + 128 r); the 3 groups of component
      // uc take r = jl, jl + 3, jl + 6
      {
        uint32_t lv[3][8];
#pragma unroll
        for (int l = 0; l < 3; l++) tmem_ld8(tm + 48 + 8 * (3 * uc + l), lv[l]);
        tmem_wait_ld();
#pragma unroll
        for (int r = 0; r < 8; r++) {
          if (static_cast<uint32_t>(r % 3) != jl) continue;
          const uint32_t hi = __funnelshift_l(0u, lv[1][r], 11) + __funnelshift_l(0u, lv[2][r], 22) + zr.z;
          uint32_t& av = acc[uc * N + t + 128u * r];
          av = add_alu(av, lv[0][r], hi);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();  // acc complete before the next step's digit gather
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }

    // ---- S6 SampleExtract
    if (a.raw_acc) {
      uint32_t* o = a.raw_acc + static_cast<size_t>(jb) * 2 * N;
      for (uint32_t k = tid; k < 2u * N; k += kLatThreads) o[k] = acc[k];
    } else {
      uint32_t* o = a.nlwe + static_cast<size_t>(a.jobs[jb].out) * kNlwe;
      for (uint32_t k = tid; k < static_cast<uint32_t>(N); k += kLatThreads) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
      if (tid == 0) o[N] = acc[N];
    }
    __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_base_sh), "n"(kLatTmemCols) : "memory");
}


// ================================================================================ K2-CLAT (cluster latency mode)
// For the narrowest level tails (<= 74 bootstraps): one bootstrap on a cluster of 2 CTAs (2 SMs).  CTA rank
// r owns accumulator component r: its 3 digit polynomials (forward, one per warp group), the 3 limbs of
// output component r (MAC + inverse, one per group) and the update of acc_r -- so the next step's digits
// need only local data.  The one cross-SM exchange per step is the MAC input: each CTA publishes its 3
// transformed digit polynomials in shared memory (double-buffered, [q][slot][thread]) and reads the peer's
// through distributed shared memory after a cluster barrier.  Same arithmetic, key layout and bytes.
constexpr int kClatGroups = 3;
constexpr int kClatSlots = 3;  // with the twiddles in shared memory a 4th bsk slot no longer fits
constexpr int kClatThreads = kClatGroups * kBT;
constexpr int kClatTmemCols = 32;
__host__ __device__ constexpr int clat_smem_bytes() {
  return 2 * kTwSlots * kBT * 8 + kClatSlots * kChunkBytes + (N * 4 + kClatGroups * N * 4 + 2 * 3 * N * 4 + 640 * 2) + 128 * 4 + kClatSlots * 8 +
         kClatSlots * 4 + 8;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kClatThreads, 1)
    vlp_blind_rotate_clat_kernel(const BrArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint2* tw_s = reinterpret_cast<uint2*>(smem);  // [fwd, inv][kTwSlots][t] twiddles (cluster barriers flush L1)
  uint32_t* ring = reinterpret_cast<uint32_t*>(tw_s + 2 * kTwSlots * kBT);
  uint32_t* acc = ring + kClatSlots * kBT * kChunkWords;  // component r only
  uint32_t* xb_all = acc + N;                            // [group 3][N]
  uint32_t* dig = xb_all + kClatGroups * N;              // [buf 2][q 3][slot 8][thread 128]
  uint16_t* abar = reinterpret_cast<uint16_t*>(dig + 2 * 3 * N);
  uint32_t* t0tab = reinterpret_cast<uint32_t*>(abar + 640);  // [128] stage-0 digit products
  uint64_t* mbar = reinterpret_cast<uint64_t*>(t0tab + 128);
  uint32_t* rel = reinterpret_cast<uint32_t*>(mbar + kClatSlots);
  uint32_t* tmem_base_sh = rel + kClatSlots;

  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rk = cl.block_rank();  // accumulator component owned by this CTA
  const uint32_t* dig_peer = cl.map_shared_rank(dig, rk ^ 1u);
  const uint32_t tid = threadIdx.x, G = tid / kBT, t = tid % kBT;
  uint32_t* xb = xb_all + G * N;
  const uint2* twf = tw_s + t;
  const uint2* twi = tw_s + kTwSlots * kBT + t;
  const Rc zr{a.zero, a.p2};
  const uint32_t nclusters = gridDim.x / 2, cid = blockIdx.x / 2;
  if (cid >= a.njobs) return;  // both CTAs of a cluster take the same branch
  const uint32_t my_jobs = (a.njobs - cid + nclusters - 1) / nclusters;
  const uint32_t total_chunks = my_jobs * static_cast<uint32_t>(a.steps) * kChunks;

  if (tid == 0) {
    for (int s = 0; s < kClatSlots; s++) {
      mbar_init(&mbar[s], 1);
      rel[s] = 0;
    }
    fence_mbar_init();
  }
  if (tid < 128) {
    const uint64_t w0 = c_tw[0][1].x;  // the stage-0 twiddle
    t0tab[tid] = static_cast<uint32_t>(w0 * ((tid + P - 64u) % P) % P);
  }
  for (uint32_t k = tid; k < static_cast<uint32_t>(kTwSlots * kBT); k += kClatThreads) {
    tw_s[k] = a.twl_fwd[k];
    tw_s[kTwSlots * kBT + k] = a.twl_inv[k];
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_sh)),
                 "n"(kClatTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = *tmem_base_sh + ((32u * ((tid >> 5) & 3u)) << 16);

  auto issue = [&](uint32_t nseq) {
    const uint32_t step = (nseq / kChunks) % static_cast<uint32_t>(a.steps), c = nseq % kChunks;
    const uint32_t s = nseq % kClatSlots;
    bulk_load(ring + s * kBT * kChunkWords, a.bsk + (static_cast<size_t>(step) * kChunks + c) * kBT * kChunkWords,
              kChunkBytes, &mbar[s]);
  };
  if (tid == 0)
    for (uint32_t q = 0; q < kClatSlots && q < total_chunks; q++) issue(q);
  uint32_t nseq = 0, sl = 0, ph = 0, buf = 0;
  const uint32_t dshift = 25u - 7u * G;  // forward: gadget digit G of component rk (R5)

  for (uint32_t jb = cid; jb < a.njobs; jb += nclusters) {
    {  // S2 + S3 (both CTAs need every abar)
      const BrJob job = a.jobs[jb];
      const uint32_t* x = slot_ptr(a.reg, job.x);
      const uint32_t* y = slot_ptr(a.reg, job.y);
      for (uint32_t w = tid; w <= static_cast<uint32_t>(n); w += kClatThreads) {
        uint32_t c = static_cast<uint32_t>(static_cast<int32_t>(job.ax)) * x[w];
        if (job.ay) c += static_cast<uint32_t>(static_cast<int32_t>(job.ay)) * y[w];
        if (w == static_cast<uint32_t>(n)) c += job.k0;
        abar[w] = static_cast<uint16_t>(((c + (1u << 20)) >> 21) & (2 * N - 1));
      }
      if (tid == 0) abar[n + 1] = job.tv;  // test vector select (R8 / R24)
    }
    __syncthreads();
    {  // S4 for component rk: acc_0 = 0, acc_1 = X^{-bbar} testv (R8)
      const uint32_t bbar = abar[n], mu = abar[n + 1] ? 2u * kMu : kMu;
      for (uint32_t k = tid; k < static_cast<uint32_t>(N); k += kClatThreads)
        acc[k] = rk == 0 ? 0u : ((((k + bbar) & (2 * N - 1)) < static_cast<uint32_t>(N)) ? mu : (0u - mu));
    }
    __syncthreads();

    for (int i = 0; i < a.steps; i++) {
      const uint32_t ab = abar[i];
      uint32_t* mydig = dig + buf * 3 * N;
      {  // digit G of component rk -> forward NTT -> publish [q][slot][thread]
        uint32_t d[1][8];
#pragma unroll
        for (int r = 0; r < 8; r++) {
          const uint32_t j = t + 128u * r;
          const uint32_t kk = (j - ab) & (2 * N - 1);
          uint32_t v = acc[kk & (N - 1)];
          v = kk >= static_cast<uint32_t>(N) ? zr.z - v : v;
          const uint32_t w = v - acc[j] + 0x81020400u;
          d[0][r] = ((w >> dshift) & 127u) + (P - 64u);
        }
        stage0_digits(d, t0tab, zr);
        stage_A<1, false>(d, zr);
        stage_A<2, false>(d, zr);
        exchange<0, 1>(d, xb, t, G);
        stage_BC<3, false, 1, true>(d, twf, zr);
        stage_BC<4, false, 1, true>(d, twf, zr);
        stage_BC<5, false, 1, true>(d, twf, zr);
        exchange<1, 2>(d, xb, t, G);
        stage_BC<6, false, 1, true>(d, twf, zr);
        stage_BC<7, false, 1, true>(d, twf, zr);
        stage_BC<8, false, 1, true>(d, twf, zr);
        stage9_fwd<1, true>(d, t, twf, zr);
#pragma unroll
        for (int s8 = 0; s8 < 8; s8++) mydig[(G * 8 + s8) * kBT + t] = d[0][s8];
      }
      cl.sync();  // both CTAs' digits published (release / acquire across the cluster)
      const uint32_t* peerdig = dig_peer + buf * 3 * N;
      // MAC for output o = 3 rk + G (component rk, limb G); digit rows q = 3u + j, u = 0 from CTA 0, 1 from CTA 1
      uint32_t mac[8];
#pragma unroll
      for (int pp = 0; pp < kChunks; pp++) {
        uint32_t x[2][6];
#pragma unroll
        for (int q = 0; q < 6; q++) {
          const uint32_t* src = (static_cast<uint32_t>(q / 3) == rk) ? mydig : peerdig;
#pragma unroll
          for (int e = 0; e < 2; e++) {
            uint32_t v = src[((q % 3) * 8 + 2 * pp + e) * kBT + t];
            v = umin(v, v - P2);
            x[e][q] = umin(v, v - P);
          }
        }
        mbar_wait(&mbar[sl], ph);
        const uint32_t* rec = ring + sl * kBT * kChunkWords + t * kChunkWords;
        {
          const uint4* kp = reinterpret_cast<const uint4*>(rec + (3 * rk + G) * 12);  // [e 2][q 6]
          const uint4 k0 = kp[0], k1 = kp[1], k2 = kp[2];
          const uint32_t kv[2][6] = {{k0.x, k0.y, k0.z, k0.w, k1.x, k1.y}, {k1.z, k1.w, k2.x, k2.y, k2.z, k2.w}};
#pragma unroll
          for (int e = 0; e < 2; e++) {
            uint64_t T = static_cast<uint64_t>(x[e][0]) * kv[e][0];
#pragma unroll
            for (int q = 1; q < 6; q++) T += static_cast<uint64_t>(x[e][q]) * kv[e][q];
            const uint32_t m = static_cast<uint32_t>(T) * PINV_NEG;
            mac[2 * pp + e] = static_cast<uint32_t>((T + static_cast<uint64_t>(m) * P) >> 32);
          }
        }
        __syncwarp();
        if ((tid & 31) == 0) {
          __threadfence_block();
          if (atomicAdd(&rel[sl], 1u) == kClatThreads / 32 - 1) {
            atomicExch(&rel[sl], 0u);
            if (nseq + kClatSlots < total_chunks) {
              fence_proxy_async();
              issue(nseq + kClatSlots);
            }
          }
        }
        nseq++;
        if (++sl == kClatSlots) {
          sl = 0;
          ph ^= 1u;
        }
      }
      buf ^= 1u;
      {  // inverse NTT of limb G of component rk, centered lift, park in TMEM
        uint32_t d[1][8];
#pragma unroll
        for (int s8 = 0; s8 < 8; s8++) d[0][s8] = umin(mac[s8], mac[s8] - P2);
        stage9_inv<1, true>(d, t, twi, zr);
        stage_BC<8, true, 1, true>(d, twi, zr);
        stage_BC<7, true, 1, true>(d, twi, zr);
        stage_BC<6, true, 1, true>(d, twi, zr);
        exchange<2, 1>(d, xb, t, G);
        stage_BC<5, true, 1, true>(d, twi, zr);
        stage_BC<4, true, 1, true>(d, twi, zr);
        stage_BC<3, true, 1, true>(d, twi, zr);
        exchange<1, 0>(d, xb, t, G);
        stage_A<2, true>(d, zr);
        stage_A<1, true>(d, zr);
        stage_A<0, true>(d, zr);
#pragma unroll
        for (int r = 0; r < 8; r++) {
          const uint32_t v = umin(d[0][r], d[0][r] - P);
          d[0][r] = v > (P >> 1) ? v - P : v;
        }
        tmem_st8(tm + 8 * G, d[0]);
      }
      tmem_wait_st();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      {  // acc_rk += R0 + 2^11 R1 + 2^22 R2; group G takes r = G, G + 3, G + 6
        uint32_t lv[3][8];
#pragma unroll
        for (int l = 0; l < 3; l++) tmem_ld8(tm + 8 * l, lv[l]);
        tmem_wait_ld();
#pragma unroll
        for (int r = 0; r < 8; r++) {
          if (static_cast<uint32_t>(r % 3) != G) continue;
          const uint32_t hi = __funnelshift_l(0u, lv[1][r], 11) + __funnelshift_l(0u, lv[2][r], 22) + zr.z;
          uint32_t& av = acc[t + 128u * r];
          av = add_alu(av, lv[0][r], hi);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }

    // ---- S6: CTA 0 holds the mask a (a'_0 = a_0, a'_k = -a_{N-k}), CTA 1 the body b (b' = b_0)
    if (a.raw_acc) {
      uint32_t* o = a.raw_acc + static_cast<size_t>(jb) * 2 * N + rk * N;
      for (uint32_t k = tid; k < static_cast<uint32_t>(N); k += kClatThreads) o[k] = acc[k];
    } else {
      uint32_t* o = a.nlwe + static_cast<size_t>(a.jobs[jb].out) * kNlwe;
      if (rk == 0) {
        for (uint32_t k = tid; k < static_cast<uint32_t>(N); k += kClatThreads) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
      } else if (tid == 0) {
        o[N] = acc[0];
      }
    }
    __syncthreads();
  }
  cl.sync();  // the peer may still read this CTA's digits
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_base_sh), "n"(kClatTmemCols) : "memory");
}

// ================================================================================ K2-C6 (6-CTA cluster latency mode)
// For the narrowest level tails (at most one bootstrap per 6 SMs): one bootstrap on a cluster of 6 CTAs of
// one warp group each.  CTA rank c = 3u + j owns digit polynomial j of component u (forward NTT) and output
// o = c, i.e. limb j of component u (MAC + inverse NTT), and keeps a copy of acc_u.  Two exchanges per CMux
// step through distributed shared memory, each after a cluster barrier: the 6 transformed digit polynomials
// (the MAC inputs) and the 3 lifted limbs of each component (the accumulator update, which the 3 CTAs of a
// component apply identically to their copies).  The CTA's 12 key words per thread and chunk (output o of
// the [o 6][e 2][q 6] chunk row) are prefetched one CMux step ahead with cp.async (24 KB per step instead of
// the 156 KB of whole chunks).  One buffer per exchange suffices: a CTA overwrites its digits only after the
// step's second cluster barrier and its limbs only after the next step's first, when every peer has read
// them.  Same arithmetic, key and bytes as the other blind-rotate kernels.
constexpr int kC6 = 6;
constexpr int kC6KeyWords = kChunks * kBT * 12;  // one step of this CTA's key words: [pp 4][t 128][12]
__host__ __device__ constexpr int c6_smem_bytes() {
  return 2 * kTwSlots * kBT * 8 + 2 * kC6KeyWords * 4 + (N * 4 + N * 4 + N * 4 + N * 4) + 640 * 2 + 128 * 4;
}
constexpr int kC6SmemRequest = 120 * 1024;  // > half an SM's shared memory: one CTA per SM
static_assert(c6_smem_bytes() <= kC6SmemRequest, "C6 shared memory");

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(NPEND) : "memory"); }

__global__ void __cluster_dims__(kC6, 1, 1) __launch_bounds__(kBT, 1) vlp_blind_rotate_c6_kernel(const BrArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint2* tw_s = reinterpret_cast<uint2*>(smem);  // [fwd, inv][kTwSlots][t] twiddles (cluster barriers flush L1)
  uint32_t* kbuf = reinterpret_cast<uint32_t*>(tw_s + 2 * kTwSlots * kBT);  // [seq & 1][pp][t][12]
  uint32_t* acc = kbuf + 2 * kC6KeyWords;             // component u only
  uint32_t* xb = acc + N;                             // layout exchanges of this CTA's NTTs
  uint32_t* dig = xb + N;                             // published transformed digit poly [slot 8][t]
  uint32_t* lim = dig + N;                            // published lifted limb [r 8][t]
  uint16_t* abar = reinterpret_cast<uint16_t*>(lim + N);
  uint32_t* t0tab = reinterpret_cast<uint32_t*>(abar + 640);  // [128] stage-0 digit products

  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rk = cl.block_rank(), u = rk / 3u, jl = rk % 3u;
  const uint32_t t = threadIdx.x;
  const uint2* twf = tw_s + t;
  const uint2* twi = tw_s + kTwSlots * kBT + t;
  const Rc zr{a.zero, a.p2};
  const uint32_t nclusters = gridDim.x / kC6, cid = blockIdx.x / kC6;
  if (cid >= a.njobs) return;  // all CTAs of a cluster take the same branch
  const uint32_t dshift = 25u - 7u * jl;  // gadget digit jl (R5)

  if (t < 128) {
    const uint64_t w0 = c_tw[0][1].x;  // the stage-0 twiddle
    t0tab[t] = static_cast<uint32_t>(w0 * ((t + P - 64u) % P) % P);
  }
  for (uint32_t k = t; k < static_cast<uint32_t>(kTwSlots * kBT); k += kBT) {
    tw_s[k] = a.twl_fwd[k];
    tw_s[kTwSlots * kBT + k] = a.twl_inv[k];
  }
  // this thread's 48 key bytes of output rk in chunk pp of bsk step `step` -> kbuf[buf]
  auto prefetch = [&](uint32_t step, uint32_t buf) {
#pragma unroll
    for (int pp = 0; pp < kChunks; pp++) {
      const uint32_t* src = a.bsk + ((static_cast<size_t>(step) * kChunks + pp) * kBT + t) * kChunkWords + rk * 12;
      uint32_t* dst = kbuf + buf * kC6KeyWords + (pp * kBT + t) * 12;
#pragma unroll
      for (int v = 0; v < 3; v++) cp_async16(dst + 4 * v, src + 4 * v);
    }
    cp_async_commit();
  };
  uint32_t seq = 0;  // CMux steps run so far (kbuf[seq & 1] holds step seq's key words)
  prefetch(0, 0);
  __syncthreads();

  for (uint32_t jb = cid; jb < a.njobs; jb += nclusters) {
    {  // S2 + S3 (every CTA needs every abar)
      const BrJob job = a.jobs[jb];
      const uint32_t* x = slot_ptr(a.reg, job.x);
      const uint32_t* y = slot_ptr(a.reg, job.y);
      for (uint32_t w = t; w <= static_cast<uint32_t>(n); w += kBT) {
        uint32_t c = static_cast<uint32_t>(static_cast<int32_t>(job.ax)) * x[w];
        if (job.ay) c += static_cast<uint32_t>(static_cast<int32_t>(job.ay)) * y[w];
        if (w == static_cast<uint32_t>(n)) c += job.k0;
        abar[w] = static_cast<uint16_t>(((c + (1u << 20)) >> 21) & (2 * N - 1));
      }
      if (t == 0) abar[n + 1] = job.tv;  // test vector select (R8 / R24)
    }
    __syncthreads();
    {  // S4 for component u: acc_0 = 0, acc_1 = X^{-bbar} testv (R8)
      const uint32_t bbar = abar[n], mu = abar[n + 1] ? 2u * kMu : kMu;
      for (uint32_t k = t; k < static_cast<uint32_t>(N); k += kBT)
        acc[k] = u == 0 ? 0u : ((((k + bbar) & (2 * N - 1)) < static_cast<uint32_t>(N)) ? mu : (0u - mu));
    }
    __syncthreads();

    for (int i = 0; i < a.steps; i++, seq++) {
      prefetch((static_cast<uint32_t>(i) + 1u) % static_cast<uint32_t>(a.steps), (seq + 1u) & 1u);
      const uint32_t ab = abar[i];
      {  // digit jl of component u -> forward NTT -> publish [slot][t]
        uint32_t d[1][8];
#pragma unroll
        for (int r = 0; r < 8; r++) {
          const uint32_t j = t + 128u * r;
          const uint32_t kk = (j - ab) & (2 * N - 1);
          uint32_t v = acc[kk & (N - 1)];
          v = kk >= static_cast<uint32_t>(N) ? zr.z - v : v;
          const uint32_t w = v - acc[j] + 0x81020400u;
          d[0][r] = ((w >> dshift) & 127u) + (P - 64u);
        }
        stage0_digits(d, t0tab, zr);
        stage_A<1, false>(d, zr);
        stage_A<2, false>(d, zr);
        exchange<0, 1>(d, xb, t, 0);
        stage_BC<3, false, 1, true>(d, twf, zr);
        stage_BC<4, false, 1, true>(d, twf, zr);
        stage_BC<5, false, 1, true>(d, twf, zr);
        exchange<1, 2>(d, xb, t, 0);
        stage_BC<6, false, 1, true>(d, twf, zr);
        stage_BC<7, false, 1, true>(d, twf, zr);
        stage_BC<8, false, 1, true>(d, twf, zr);
        stage9_fwd<1, true>(d, t, twf, zr);
#pragma unroll
        for (int s8 = 0; s8 < 8; s8++) dig[s8 * kBT + t] = d[0][s8];
      }
      cl.sync();  // the 6 transformed digit polynomials are published
      // MAC for output o = rk: digit rows q = 3u' + j' live in CTA q
      uint32_t mac[8];
      {
        uint32_t xq[6][8];
#pragma unroll
        for (int q = 0; q < 6; q++) {
          const uint32_t* src = cl.map_shared_rank(dig, static_cast<unsigned>(q));
#pragma unroll
          for (int s8 = 0; s8 < 8; s8++) {
            const uint32_t v = src[s8 * kBT + t];
            xq[q][s8] = umin(v, v - P2);  // [0, 2p)
          }
        }
        cp_async_wait<1>();  // this step's key words (the newest group is the next step's)
        const uint32_t* kb = kbuf + (seq & 1u) * kC6KeyWords + t * 12;
#pragma unroll
        for (int pp = 0; pp < kChunks; pp++) {
          const uint4* kp = reinterpret_cast<const uint4*>(kb + pp * kBT * 12);  // [e 2][q 6]
          const uint4 k0 = kp[0], k1 = kp[1], k2 = kp[2];
          const uint32_t kv[2][6] = {{k0.x, k0.y, k0.z, k0.w, k1.x, k1.y}, {k1.z, k1.w, k2.x, k2.y, k2.z, k2.w}};
#pragma unroll
          for (int e = 0; e < 2; e++) {
            uint64_t T = static_cast<uint64_t>(xq[0][2 * pp + e]) * kv[e][0];
#pragma unroll
            for (int q = 1; q < 6; q++) T += static_cast<uint64_t>(xq[q][2 * pp + e]) * kv[e][q];
            const uint32_t m = static_cast<uint32_t>(T) * PINV_NEG;
            mac[2 * pp + e] = static_cast<uint32_t>((T + static_cast<uint64_t>(m) * P) >> 32);
          }
        }
      }
      {  // inverse NTT of limb jl of component u, centered lift, publish [r][t]
        uint32_t d[1][8];
#pragma unroll
        for (int s8 = 0; s8 < 8; s8++) d[0][s8] = umin(mac[s8], mac[s8] - P2);
        stage9_inv<1, true>(d, t, twi, zr);
        stage_BC<8, true, 1, true>(d, twi, zr);
        stage_BC<7, true, 1, true>(d, twi, zr);
        stage_BC<6, true, 1, true>(d, twi, zr);
        exchange<2, 1>(d, xb, t, 0);
        stage_BC<5, true, 1, true>(d, twi, zr);
        stage_BC<4, true, 1, true>(d, twi, zr);
        stage_BC<3, true, 1, true>(d, twi, zr);
        exchange<1, 0>(d, xb, t, 0);
        stage_A<2, true>(d, zr);
        stage_A<1, true>(d, zr);
        stage_A<0, true>(d, zr);
#pragma unroll
        for (int r = 0; r < 8; r++) {
          const uint32_t v = umin(d[0][r], d[0][r] - P);
          lim[r * kBT + t] = v > (P >> 1) ? v - P : v;
        }
      }
      cl.sync();  // the 6 lifted limbs are published
      {  // acc_u += R0 + 2^11 R1 + 2^22 R2 (limb l from CTA 3u + l; the same update in all 3 CTAs of u)
        const uint32_t* l0 = cl.map_shared_rank(lim, 3u * u);
        const uint32_t* l1 = cl.map_shared_rank(lim, 3u * u + 1u);
        const uint32_t* l2 = cl.map_shared_rank(lim, 3u * u + 2u);
#pragma unroll
        for (int r = 0; r < 8; r++) {
          const uint32_t hi = __funnelshift_l(0u, l1[r * kBT + t], 11) + __funnelshift_l(0u, l2[r * kBT + t], 22) + zr.z;
          uint32_t& av = acc[t + 128u * r];
          av = add_alu(av, l0[r * kBT + t], hi);
        }
      }
      __syncthreads();  // acc complete before the next step's rotated reads
    }

    // ---- S6: CTA 0 holds the mask a (a'_0 = a_0, a'_k = -a_{N-k}), CTA 3 the body b (b' = b_0)
    if (jl == 0) {
      if (a.raw_acc) {
        uint32_t* o = a.raw_acc + static_cast<size_t>(jb) * 2 * N + u * N;
        for (uint32_t k = t; k < static_cast<uint32_t>(N); k += kBT) o[k] = acc[k];
      } else {
        uint32_t* o = a.nlwe + static_cast<size_t>(a.jobs[jb].out) * kNlwe;
        if (u == 0) {
          for (uint32_t k = t; k < static_cast<uint32_t>(N); k += kBT) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
        } else if (t == 0) {
          o[N] = acc[0];
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  cl.sync();  // peers may still read this CTA's limbs
}

// ================================================================================ device PubKeyGen + ServerEnc
// (setup) one warp per DB ciphertext: the TLWE(0) public-key sample of alg:PubKeyGen
// (mask words from the call's generator -- the seeded counter PRNG of R3 or ChaCha20 under the secure call's
// key --, b = <a, s> + e with e computed on the host by the same libm Box-Muller as vlp_pubkeygen) plus
// (0, Ecd(bit)) of alg:ServerEnc -- byte-identical to the host calls under the same generator.
__device__ __forceinline__ uint64_t prng_mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// ChaCha20 block (RFC 8439 section 2.3) for the secure mask generator: key g.key, block counter `counter`,
// nonce (dom, obj lo, obj hi) -- the words host.cpp's secure Rng draws (mask word w = output 2 (w mod 8) + 1 of block
// w / 8, i.e. the high half of the generator's 64-bit word).
__device__ __forceinline__ void chacha_qr(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  a += b; d = __funnelshift_l(d ^ a, d ^ a, 16);
  c += d; b = __funnelshift_l(b ^ c, b ^ c, 12);
  a += b; d = __funnelshift_l(d ^ a, d ^ a, 8);
  c += d; b = __funnelshift_l(b ^ c, b ^ c, 7);
}
__device__ void chacha20_dev(const MaskGen& g, uint32_t counter, uint64_t obj, uint32_t (&out)[16]) {
  const uint32_t in[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u, g.key[0], g.key[1], g.key[2], g.key[3],
                           g.key[4], g.key[5], g.key[6], g.key[7], counter, g.dom, static_cast<uint32_t>(obj),
                           static_cast<uint32_t>(obj >> 32)};
  uint32_t x[16];
#pragma unroll
  for (int i = 0; i < 16; i++) x[i] = in[i];
#pragma unroll 1
  for (int r = 0; r < 10; r++) {
    chacha_qr(x[0], x[4], x[8], x[12]); chacha_qr(x[1], x[5], x[9], x[13]);
    chacha_qr(x[2], x[6], x[10], x[14]); chacha_qr(x[3], x[7], x[11], x[15]);
    chacha_qr(x[0], x[5], x[10], x[15]); chacha_qr(x[1], x[6], x[11], x[12]);
    chacha_qr(x[2], x[7], x[8], x[13]); chacha_qr(x[3], x[4], x[9], x[14]);
  }
#pragma unroll
  for (int i = 0; i < 16; i++) out[i] = x[i] + in[i];
}

// The n uniform mask words of TLWE sample `obj` by one warp: ct[w] = a_w; returns <a, s> (all lanes).
__device__ uint32_t warp_tlwe_mask(const MaskGen& g, uint64_t obj, const uint32_t* __restrict__ s, uint32_t* ct,
                                   uint32_t lane) {
  uint32_t b = 0;
  if (g.secure) {
    for (uint32_t c = lane; 8 * c < static_cast<uint32_t>(n); c += 32) {
      uint32_t blk[16];
      chacha20_dev(g, c, obj, blk);
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const uint32_t w = 8 * c + i;
        if (w < static_cast<uint32_t>(n)) {
          ct[w] = blk[2 * i + 1];
          b += blk[2 * i + 1] * s[w];
        }
      }
    }
  } else {
    const uint64_t h2 = prng_mix(g.h1 ^ (obj * 0xC2B2AE3D27D4EB4Full));
    for (uint32_t w = lane; w < static_cast<uint32_t>(n); w += 32) {
      const uint32_t a = static_cast<uint32_t>(prng_mix(h2 ^ (w * 0x165667B19E3779F9ull)) >> 32);
      ct[w] = a;
      b += a * s[w];
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
  return b;
}

__global__ void __launch_bounds__(256) vlp_encrypt_db_kernel(const uint32_t* __restrict__ s, const uint32_t* __restrict__ noise,
                                                            const uint8_t* __restrict__ bits, MaskGen g, uint32_t per,
                                                            uint32_t W, uint32_t lI, uint64_t first, uint64_t nsamples,
                                                            uint32_t* __restrict__ out) {
  const uint64_t idx = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  if (idx >= nsamples) return;
  const uint64_t rec = idx / per, row = idx % per;
  const uint64_t local = row < static_cast<uint64_t>(W) * lI ? (row % lI) * W + row / lI : row;  // alg:PubKeyGen order
  const uint64_t obj = (first + rec) * per + local;
  uint32_t* ct = out + idx * kCt;
  const uint32_t b = warp_tlwe_mask(g, obj, s, ct, lane);
  if (lane == 0) {
    ct[n] = b + noise[idx] + (bits ? (bits[idx] ? kMu : 0u - kMu) : 0u);  // bits == nullptr: the pk sample alone
    ct[n + 1] = 0;
  }
}

// Device ServerEnc (alg:ServerEnc P:223-247): out = pk + (0, Ecd(bit)), thread per word (out may alias pk).
__global__ void __launch_bounds__(256) vlp_server_enc_kernel(const uint32_t* pk, const uint8_t* __restrict__ bits,
                                                            uint64_t nsamples, uint32_t* out) {
  const uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= nsamples * kCt) return;
  const uint64_t idx = w / kCt;
  const uint32_t col = static_cast<uint32_t>(w % kCt);
  const uint32_t v = pk[w];
  out[w] = col == static_cast<uint32_t>(n) ? v + (bits[idx] ? kMu : 0u - kMu) : v;
}

// Device KeyGen, bootstrapping key (R4, O7): CTA per row (i, r): a_j = uniform(BSK_A, obj = i*6 + r, word j),
// b = a * z + e (negacyclic, z binary: the sum of the rotations X^k a over supp z), then s_i g_j on component
// r / 3's constant coefficient -- the same words vlp_keygen computes on the host.
__global__ void __launch_bounds__(256) vlp_keygen_bsk_kernel(MaskGen g, const uint32_t* __restrict__ s,
                                                            const uint32_t* __restrict__ z, const uint32_t* __restrict__ e,
                                                            uint32_t* __restrict__ bsk) {
  __shared__ uint32_t a[N];
  __shared__ uint32_t zs[N];
  const uint32_t ir = blockIdx.x;
  if (g.secure) {
    for (uint32_t c = threadIdx.x; c < static_cast<uint32_t>(N) / 8; c += blockDim.x) {
      uint32_t blk[16];
      chacha20_dev(g, c, ir, blk);
#pragma unroll
      for (int q = 0; q < 8; q++) a[8 * c + q] = blk[2 * q + 1];
    }
  } else {
    const uint64_t h2 = prng_mix(g.h1 ^ (static_cast<uint64_t>(ir) * 0xC2B2AE3D27D4EB4Full));
    for (uint32_t j = threadIdx.x; j < static_cast<uint32_t>(N); j += blockDim.x)
      a[j] = static_cast<uint32_t>(prng_mix(h2 ^ (static_cast<uint64_t>(j) * 0x165667B19E3779F9ull)) >> 32);
  }
  for (uint32_t j = threadIdx.x; j < static_cast<uint32_t>(N); j += blockDim.x) zs[j] = z[j];
  __syncthreads();
  uint32_t* ra = bsk + static_cast<size_t>(ir) * 2 * N;
  uint32_t* rb = ra + N;
  const uint32_t i = ir / kRows, r = ir % kRows;
  const uint32_t sg = s[i] ? 1u << (32 - kBgBits * (r % kEll + 1)) : 0u;  // s_i g_j
  for (uint32_t t = threadIdx.x; t < static_cast<uint32_t>(N); t += blockDim.x) {
    uint32_t acc = 0;
    for (uint32_t k = 0; k <= t; k++) acc += zs[k] ? a[t - k] : 0u;
    for (uint32_t k = t + 1; k < static_cast<uint32_t>(N); k++) acc -= zs[k] ? a[t + N - k] : 0u;
    acc += e[static_cast<size_t>(ir) * N + t];
    if (t == 0 && r / kEll == 1) acc += sg;
    rb[t] = acc;
    ra[t] = a[t] + ((t == 0 && r / kEll == 0) ? sg : 0u);
  }
}

// Device KeyGen, key-switching key (O10): warp per row idx = (i*8 + j)*3 + v-1: TLWE_s(v z_i 2^(32-2(j+1))).
__global__ void __launch_bounds__(256) vlp_keygen_ksk_kernel(MaskGen g, const uint32_t* __restrict__ s,
                                                            const uint32_t* __restrict__ z, const uint32_t* __restrict__ e,
                                                            uint32_t* __restrict__ ksk) {
  const uint32_t idx = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31u;
  if (idx >= static_cast<uint32_t>(N * kKsT * 3)) return;
  const uint32_t i = idx / (kKsT * 3), j = (idx / 3) % kKsT, v = idx % 3 + 1;
  uint32_t* ct = ksk + static_cast<size_t>(idx) * kCt;
  const uint32_t b = warp_tlwe_mask(g, idx, s, ct, lane);
  if (lane == 0) {
    ct[n] = b + v * z[i] * (1u << (32 - kKsBaseBits * (j + 1))) + e[idx];
    ct[n + 1] = 0;
  }
}

cudaError_t launch_server_enc(const uint32_t* pk, const uint8_t* bits, uint64_t nsamples, uint32_t* out, cudaStream_t st) {
  const uint64_t words = nsamples * kCt;
  if (words) vlp_server_enc_kernel<<<static_cast<unsigned>((words + 255) / 256), 256, 0, st>>>(pk, bits, nsamples, out);
  return cudaGetLastError();
}

cudaError_t launch_keygen(const MaskGen& g_bsk, const MaskGen& g_ksk, const uint32_t* s, const uint32_t* z, const uint32_t* e_bsk,
                          const uint32_t* e_ksk, uint32_t* bsk, uint32_t* ksk, cudaStream_t st) {
  vlp_keygen_bsk_kernel<<<n * kRows, 256, 0, st>>>(g_bsk, s, z, e_bsk, bsk);
  vlp_keygen_ksk_kernel<<<(N * kKsT * 3 + 7) / 8, 256, 0, st>>>(g_ksk, s, z, e_ksk, ksk);
  return cudaGetLastError();
}

cudaError_t launch_encrypt_db(const uint32_t* s, const uint32_t* noise, const uint8_t* bits, const MaskGen& g, uint32_t per,
                              uint32_t W, uint32_t lI, uint64_t first, uint64_t nsamples, uint32_t* out, cudaStream_t st) {
  if (!nsamples) return cudaSuccess;
  const uint64_t blocks = (nsamples * 32 + 255) / 256;
  vlp_encrypt_db_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(s, noise, bits, g, per, W, lI, first, nsamples, out);
  return cudaGetLastError();
}

// ================================================================================ K4 bsk conversion
// One CTA per (i, key row q, component u): split the 1024 torus32 coefficients into 3 signed limbs, forward
// NTT each limb polynomial mod p (plain, fully reduced; natural twiddle table), multiply by
// N^-1 * 2^32 mod p, and scatter NTT position k to the lane/slot that holds it after the forward
// transform (inverse of posF): chunk slot / 2, word o*12 + (slot & 1)*6 + q, o = u*3 + limb.
__global__ void __launch_bounds__(512) vlp_bsk_convert_kernel(const uint32_t* __restrict__ raw,
                                                              uint32_t* __restrict__ out,
                                                              const uint2* __restrict__ tw, uint32_t c_mont) {
  __shared__ uint32_t poly[3][N];
  const uint32_t bid = blockIdx.x;  // (i*6 + q)*2 + u
  const uint32_t u = bid & 1, q = (bid >> 1) % kRows, i = (bid >> 1) / kRows;
  const uint32_t* src = raw + static_cast<size_t>(bid) * N;
  for (uint32_t k = threadIdx.x; k < static_cast<uint32_t>(N); k += blockDim.x) {
    const int64_t b = static_cast<int64_t>(src[k]);
    const int64_t b0 = ((b + 1024) & 2047) - 1024;
    const int64_t r1 = (b - b0) >> 11;
    const int64_t b1 = ((r1 + 1024) & 2047) - 1024;
    const int64_t r2 = (r1 - b1) >> 11;
    const int64_t b2 = ((r2 + 512) & 1023) - 512;
    poly[0][k] = static_cast<uint32_t>(b0 < 0 ? b0 + P : b0);
    poly[1][k] = static_cast<uint32_t>(b1 < 0 ? b1 + P : b1);
    poly[2][k] = static_cast<uint32_t>(b2 < 0 ? b2 + P : b2);
  }
  __syncthreads();
  for (int s = 0; s < 10; s++) {
    const uint32_t half = 512u >> s;
    const uint32_t bf = threadIdx.x;  // butterfly 0..511
    const uint32_t blk = bf / half, j = 2 * blk * half + (bf % half);
    const uint32_t w = tw[(1u << s) + blk].x;
#pragma unroll
    for (int l = 0; l < 3; l++) {
      const uint32_t x = poly[l][j];
      const uint32_t y = static_cast<uint32_t>(static_cast<uint64_t>(poly[l][j + half]) * w % P);
      poly[l][j] = x + y >= P ? x + y - P : x + y;
      poly[l][j + half] = x >= y ? x - y : x + P - y;
    }
    __syncthreads();
  }
  for (uint32_t k = threadIdx.x; k < static_cast<uint32_t>(N); k += blockDim.x) {
    const uint32_t b0 = k & 1, r = (k >> 1) & 7;
    const uint32_t t = ((k >> 4) << 1) | (r >= 4 ? 1u : 0u);
    const uint32_t slot = (b0 ? 4 : 0) + (r & 3);
    const uint32_t chunk = slot / 2;
    uint32_t* dst = out + ((static_cast<size_t>(i) * kChunks + chunk) * kBT + t) * kChunkWords;
#pragma unroll
    for (int l = 0; l < 3; l++) {
      const uint32_t o = u * 3 + l;
      dst[o * 12 + (slot & 1) * 6 + q] = static_cast<uint32_t>(static_cast<uint64_t>(poly[l][k]) * c_mont % P);
    }
  }
}

__global__ void vlp_init_constants_kernel(uint32_t* mid) {
  // rows 0 / 1 of the intermediate region: trivial (0, -1/8) and (0, +1/8) (R21)
  for (uint32_t k = threadIdx.x; k < 2u * kCt; k += blockDim.x) {
    const uint32_t row = k / kCt, w = k % kCt;
    mid[k] = w == static_cast<uint32_t>(n) ? (row ? kMu : 0u - kMu) : 0u;
  }
}

// R24 linear aggregation: out slot = sum of the job's input slots mod 2^32 (all 632 words; pad words stay 0).
__global__ void __launch_bounds__(128) vlp_linear_kernel(const LinJob* __restrict__ jobs, const uint32_t* __restrict__ ins,
                                                         Regions reg) {
  const LinJob j = jobs[blockIdx.x];
  uint32_t* o = slot_wptr(reg, j.out);
  for (uint32_t w = threadIdx.x; w < static_cast<uint32_t>(kCt); w += blockDim.x) {
    uint32_t acc = 0;
    for (uint32_t i = 0; i < j.count; i++) acc += slot_ptr(reg, ins[j.first + i])[w];
    o[w] = acc;
  }
}

__global__ void vlp_copy_rows_kernel(const uint32_t* __restrict__ slots, Regions reg, uint32_t* out) {
  const uint32_t* src = slot_ptr(reg, slots[blockIdx.x]);
  for (uint32_t k = threadIdx.x; k < static_cast<uint32_t>(kCt); k += blockDim.x)
    out[static_cast<size_t>(blockIdx.x) * kCt + k] = src[k];
}

// ================================================================================ launchers
void set_const_twiddles(const uint2* fwd16, const uint2* inv16) {
  uint2 h[2][8];
  for (int k = 0; k < 8; k++) {
    h[0][k] = fwd16[k];
    h[1][k] = inv16[k];
  }
  cudaMemcpyToSymbol(c_tw, h, sizeof(h));
}

void launch_bsk_convert(const uint32_t* raw, uint32_t* out, const uint2* tw_fwd, uint32_t c_mont, cudaStream_t st) {
  vlp_bsk_convert_kernel<<<n * kRows * 2, 512, 0, st>>>(raw, out, tw_fwd, c_mont);
}

template <int B>
static cudaError_t launch_br_b(const BrArgs& a, int sm_count, cudaStream_t st) {
  // the dynamic shared-memory opt-in is per device: remember it per device ordinal (< 64)
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set.load() & bit)) {
    e = cudaFuncSetAttribute(vlp_blind_rotate_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, br_smem_bytes(B));
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit);
  }
  if (a.njobs == 0) return cudaSuccess;
  const uint64_t groups = (a.njobs + B - 1) / B;
  const int grid = static_cast<int>(groups < static_cast<uint64_t>(sm_count) ? groups : sm_count);
  // the kernel counts bsk chunks in 32 bits: (groups per CTA) x steps x kChunks must stay below 2^32
  if (grid <= 0 || (groups + grid - 1) / grid * static_cast<uint64_t>(a.steps) * kChunks >= (1ull << 32))
    return cudaErrorInvalidValue;
  BrArgs b = a;
  b.zero = 0;
  b.p2 = P2;
  vlp_blind_rotate_kernel<B><<<grid, B * kBT, br_smem_bytes(B), st>>>(b);
  return cudaGetLastError();
}

static cudaError_t launch_br_lat(const BrArgs& a, int sm_count, cudaStream_t st) {
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set.load() & bit)) {
    e = cudaFuncSetAttribute(vlp_blind_rotate_lat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lat_smem_bytes());
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit);
  }
  if (a.njobs == 0) return cudaSuccess;
  const int grid = static_cast<int>(a.njobs < static_cast<uint32_t>(sm_count) ? a.njobs : sm_count);
  if ((static_cast<uint64_t>(a.njobs) + grid - 1) / grid * static_cast<uint64_t>(a.steps) * kChunks >= (1ull << 32))
    return cudaErrorInvalidValue;
  BrArgs b = a;
  b.zero = 0;
  b.p2 = P2;
  vlp_blind_rotate_lat_kernel<<<grid, kLatThreads, lat_smem_bytes(), st>>>(b);
  return cudaGetLastError();
}

static cudaError_t launch_br_clat(const BrArgs& a, int sm_count, cudaStream_t st) {
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set.load() & bit)) {
    e = cudaFuncSetAttribute(vlp_blind_rotate_clat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, clat_smem_bytes());
    if (e != cudaSuccess) return e;
    attr_set.fetch_or(bit);
  }
  if (a.njobs == 0) return cudaSuccess;
  const uint32_t half = static_cast<uint32_t>(sm_count / 2);
  if (half == 0) return launch_br_lat(a, sm_count, st);  // a 2-CTA cluster needs two SMs
  const uint32_t clusters = a.njobs < half ? a.njobs : half;
  if ((static_cast<uint64_t>(a.njobs) + clusters - 1) / clusters * static_cast<uint64_t>(a.steps) * kChunks >= (1ull << 32))
    return cudaErrorInvalidValue;
  BrArgs b = a;
  b.zero = 0;
  b.p2 = P2;
  vlp_blind_rotate_clat_kernel<<<2 * clusters, kClatThreads, clat_smem_bytes(), st>>>(b);
  return cudaGetLastError();
}

// Clusters of 6 CTAs that can be resident at once (GPC packing), per device (queried once).
static uint32_t c6_max_clusters() {
  static std::atomic<int> cached[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  int v = cached[dev & 63].load();
  if (v == 0) {
    if (cudaFuncSetAttribute(vlp_blind_rotate_c6_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kC6SmemRequest) !=
        cudaSuccess)
      return 0;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kC6;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(kC6, 1, 1);
    cfg.blockDim = dim3(kBT, 1, 1);
    cfg.dynamicSmemBytes = kC6SmemRequest;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, vlp_blind_rotate_c6_kernel, &cfg) != cudaSuccess || nc < 1) {
      cudaGetLastError();
      nc = -1;  // not available: never route to it
    }
    cached[dev & 63].store(nc);
    v = nc;
  }
  return v > 0 ? static_cast<uint32_t>(v) : 0u;
}

static cudaError_t launch_br_c6(const BrArgs& a, int sm_count, cudaStream_t st) {
  const uint32_t maxc = c6_max_clusters();
  if (maxc == 0) return launch_br_clat(a, sm_count, st);
  if (a.njobs == 0) return cudaSuccess;
  const uint32_t clusters = a.njobs < maxc ? a.njobs : maxc;
  BrArgs b = a;
  b.zero = 0;
  b.p2 = P2;
  vlp_blind_rotate_c6_kernel<<<kC6 * clusters, kBT, kC6SmemRequest, st>>>(b);
  return cudaGetLastError();
}

static cudaError_t launch_br_width(const BrArgs& a, int B, int sm_count, cudaStream_t st) {
  switch (B) {
    case -2: return launch_br_c6(a, sm_count, st);
    case -1: return launch_br_clat(a, sm_count, st);
    case 0: return launch_br_lat(a, sm_count, st);
    case 1: return launch_br_b<1>(a, sm_count, st);
    case 2: return launch_br_b<2>(a, sm_count, st);
    case 3: return launch_br_b<3>(a, sm_count, st);
    case 4: return launch_br_b<4>(a, sm_count, st);
    default: return launch_br_b<kBrBoot>(a, sm_count, st);
  }
}

// One level of blind rotations.  Engine (VLP_BR_ENGINE, read once): "fft" (default) -- whole waves of
// kFftMaxWarps bootstraps per SM on K2F (kernels_fft.cu), a remainder wider than one bootstrap per SM on a K2F
// wave of ceil(rest / SMs) warps per CTA; "ntt" -- whole waves of kBrBoot bootstraps per SM on K2 and a narrower
// K2 tail.  With either engine a remainder of at most one bootstrap per SM runs on the NTT latency kernels
// (6-CTA cluster / 2-CTA cluster / warp groups per bootstrap).  Both engines are exact: the bytes do not
// depend on the choice.  VLP_BR_BOOT=b (debug) forces one NTT kernel for the whole level (1-5: K2 with b
// bootstraps per CTA, -1 latency, -2 2-CTA cluster, -3 6-CTA cluster); VLP_FFT_WARPS=w forces K2F with w warps.
// Routing state: initialised once from the environment, replaced by vlp_debug_route (set_br_route).
struct Route {
  int engine;     // 0 ntt, 1 fft
  int boot;       // forced NTT kernel (VLP_BR_BOOT meaning) or 0
  int fft_warps;  // forced K2F warps per CTA or 0
};
static Route env_route() {
  Route r{1, 0, 0};
  if (const char* e = getenv("VLP_BR_ENGINE")) r.engine = e[0] == 'n' ? 0 : 1;
  if (const char* e = getenv("VLP_BR_BOOT")) r.boot = atoi(e);
  if (const char* e = getenv("VLP_FFT_WARPS")) {
    const int v = atoi(e);
    r.fft_warps = v >= 1 && v <= kFftMaxWarps ? v : 0;
  }
  return r;
}
static std::atomic<int> g_engine{-1}, g_boot{0}, g_fft_warps{0};
static Route route() {
  if (g_engine.load() < 0) {
    const Route r = env_route();
    g_boot.store(r.boot);
    g_fft_warps.store(r.fft_warps);
    int expect = -1;
    g_engine.compare_exchange_strong(expect, r.engine);
  }
  return Route{g_engine.load(), g_boot.load(), g_fft_warps.load()};
}
int set_br_route(int engine, int param) {
  if (engine == 0) {
    const Route r = env_route();
    g_boot.store(r.boot);
    g_fft_warps.store(r.fft_warps);
    g_engine.store(r.engine);
  } else if (engine == 1) {
    if (!((param >= 0 && param <= kBrBoot) || param == -1 || param == -2 || param == -3)) return -1;
    g_boot.store(param);
    g_fft_warps.store(0);
    g_engine.store(0);
  } else if (engine == 2) {
    if (param < 1 || param > kFftMaxWarps) return -1;
    g_boot.store(0);
    g_fft_warps.store(param);
    g_engine.store(1);
  } else {
    return -1;
  }
  return 0;
}
// vlp_debug_fft_error: every K2F launch records its largest rounding distance (debug; nullptr = off)
static std::atomic<unsigned long long*> g_fft_err{nullptr};
void set_fft_error_monitor(unsigned long long* err_dev) { g_fft_err.store(err_dev); }

static int forced_boot() { return route().boot; }
static int forced_fft_warps() { return route().fft_warps; }
static bool fft_engine() { return route().engine == 1; }
static bool forced_any() {
  const int f = forced_boot();
  return (f >= 1 && f <= kBrBoot) || f == -1 || f == -2 || f == -3 || forced_fft_warps() > 0;
}

int br_launch_count(uint32_t njobs, int sm_count) {
  if (njobs == 0) return 0;
  if (forced_fft_warps()) return static_cast<int>(fft_launch_count(njobs, forced_fft_warps(), sm_count));
  if (forced_any()) return 1;
  const bool fft = fft_engine();
  const uint32_t wave = static_cast<uint32_t>(fft ? kFftMaxWarps : kBrBoot) * static_cast<uint32_t>(sm_count);
  const uint32_t full = njobs / wave * wave;
  const int nfull = full == 0 ? 0 : (fft ? static_cast<int>(fft_launch_count(full, kFftMaxWarps, sm_count)) : 1);
  return nfull + (njobs % wave ? 1 : 0);
}

static cudaError_t launch_blind_rotate_fft_mon(BrArgs a, int warps, int sm_count, cudaStream_t st) {
  a.fft_err = g_fft_err.load();
  return launch_blind_rotate_fft(a, warps, sm_count, st);
}

cudaError_t launch_blind_rotate(const BrArgs& a, int sm_count, cudaStream_t st) {
  if (a.njobs == 0) return cudaSuccess;
  const int forced = forced_boot();
  if (forced_fft_warps()) return launch_blind_rotate_fft_mon(a, forced_fft_warps(), sm_count, st);
  if (forced >= 1 && forced <= kBrBoot) return launch_br_width(a, forced, sm_count, st);
  if (forced == -1) return launch_br_width(a, 0, sm_count, st);   // VLP_BR_BOOT=-1: latency mode
  if (forced == -2) return launch_br_width(a, -1, sm_count, st);  // VLP_BR_BOOT=-2: cluster latency mode
  if (forced == -3) return launch_br_width(a, -2, sm_count, st);  // VLP_BR_BOOT=-3: 6-CTA cluster mode
  const bool fft = fft_engine();
  const uint32_t per_sm = static_cast<uint32_t>(fft ? kFftMaxWarps : kBrBoot);
  const uint32_t wave = per_sm * static_cast<uint32_t>(sm_count);
  const uint32_t full = a.njobs / wave * wave, tail = a.njobs - full;
  cudaError_t e = cudaSuccess;
  if (full) {
    BrArgs f = a;
    f.njobs = full;
    e = fft ? launch_blind_rotate_fft_mon(f, kFftMaxWarps, sm_count, st) : launch_br_width(f, kBrBoot, sm_count, st);
    if (e != cudaSuccess) return e;
  }
  if (tail) {
    BrArgs r = a;
    r.jobs = a.jobs + full;
    r.njobs = tail;
    if (r.raw_acc) r.raw_acc = a.raw_acc + static_cast<size_t>(full) * 2 * N;
    // a tail of at most one bootstrap per SM runs in latency mode (warp groups per bootstrap); at most one per
    // two SMs, on a 2-CTA cluster per bootstrap; at most one per resident 6-CTA cluster, on a 6-CTA cluster
    const uint32_t per = (tail + sm_count - 1) / sm_count;
    // K2F's single-warp bootstraps have a long per-step latency (one bootstrap per SM takes ~11 ms for 630 steps,
    // 2-4 per SM about the same), so tails of at most kBrBoot per SM run on the NTT kernels (K2<b>: 6.1-12.7 ms)
    if (fft && per > static_cast<uint32_t>(kBrBoot)) return launch_blind_rotate_fft_mon(r, static_cast<int>(per), sm_count, st);
    const int b = tail <= c6_max_clusters() ? -2
                  : tail <= static_cast<uint32_t>(sm_count / 2) ? -1
                  : tail <= static_cast<uint32_t>(sm_count) ? 0
                                                             : static_cast<int>(per);
    e = launch_br_width(r, b, sm_count, st);
  }
  return e;
}




cudaError_t launch_init_constants(uint32_t* mid, cudaStream_t st) {
  vlp_init_constants_kernel<<<1, 256, 0, st>>>(mid);
  return cudaGetLastError();
}

cudaError_t launch_linear(const LinJob* jobs, const uint32_t* inputs, uint32_t count, Regions reg, cudaStream_t st) {
  if (!count) return cudaSuccess;
  vlp_linear_kernel<<<count, 128, 0, st>>>(jobs, inputs, reg);
  return cudaGetLastError();
}

cudaError_t launch_copy_rows(const uint32_t* slots, uint32_t count, Regions reg, uint32_t* out, cudaStream_t st) {
  if (!count) return cudaSuccess;
  vlp_copy_rows_kernel<<<count, 128, 0, st>>>(slots, reg, out);
  return cudaGetLastError();
}

}  // namespace vlp
