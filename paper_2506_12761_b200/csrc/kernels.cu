// kernels.cu -- the sm_100a kernels of the hot path.
//
//  K2 vlp_blind_rotate_kernel : gate linear form (S2) + mod-switch (S3) + accumulator init (S4) +
//                               630 CMux steps (S5) with the accumulator on chip + SampleExtract (S6)
//  K3 vlp_keyswitch_kernel    : MUX combine (S7) + key switch (S8)
//  K4 vlp_bsk_convert_kernel  : bsk -> 3-limb NTT domain (setup)
//
// Exact arithmetic: NTT prime p = 0x3fff7801 (p = 1 mod 2048, 4p < 2^32); the
// bootstrapping key is split into three signed limbs (11, 11, 10 bits) so every limb product sum is
// below p/2 and lifts back exactly; the torus32 result is R0 + 2^11 R1 + 2^22 R2 mod 2^32.
// Forward transform: Cooley-Tukey, merged psi-twist, natural -> bit-reversed, Harvey lazy butterflies
// (values in [0, 4p)) with Shoup twiddles.  Inverse: Gentleman-Sande, bit-reversed -> natural, values in
// [0, 2p); N^-1 and the Montgomery factor are folded into the stored key.
//
// Thread layout of one bootstrap (64 threads, 16 coefficients per thread per polynomial):
//   layout A (stages 0-3):  j = t + 64 r                        (twiddles uniform per r)
//   layout B (stages 4-7):  j = (t>>2)<<6 | r<<2 | (t&3)
//   layout C (stages 8-9):  j = t<<4 | r                        (bit-reversed NTT positions 16t..16t+15)
// Layout changes go through shared memory with an XOR swizzle that is bank-conflict free for all three
// layouts (tools/emulate_br_ntt.py checks it).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace vlp {
namespace {

constexpr uint32_t P = kP;
constexpr uint32_t P2 = 2u * kP;

constexpr uint32_t inv_mod_2_32(uint32_t p) {
  uint32_t x = p;  // Newton iteration for p^-1 mod 2^32
  for (int i = 0; i < 5; i++) x *= 2u - p * x;
  return x;
}
constexpr uint32_t PINV_NEG = 0u - inv_mod_2_32(P);  // -p^-1 mod 2^32 (Montgomery REDC)
static_assert(static_cast<uint32_t>(P * inv_mod_2_32(P)) == 1u, "inverse");

__constant__ uint2 c_tw[2][16];  // uniform twiddles (k < 16) of the forward / inverse transforms

// ------------------------------------------------------------------------------ modular helpers
__device__ __forceinline__ uint32_t umin(uint32_t a, uint32_t b) { return a < b ? a : b; }

// Shoup: y * w mod p in [0, 2p) for any y < 2^32, w < p, ws = floor(w 2^32 / p).
__device__ __forceinline__ uint32_t shoup(uint32_t y, uint32_t w, uint32_t ws) {
  const uint32_t q = __umulhi(y, ws);
  return y * w - q * P;
}
// Forward CT butterfly, inputs / outputs in [0, 4p).
__device__ __forceinline__ void ct_bfly(uint32_t& x, uint32_t& y, uint32_t w, uint32_t ws) {
  const uint32_t xr = umin(x, x - P2);
  const uint32_t t = shoup(y, w, ws);
  x = xr + t;
  y = xr - t + P2;
}
// Inverse GS butterfly, inputs / outputs in [0, 2p).
__device__ __forceinline__ void gs_bfly(uint32_t& x, uint32_t& y, uint32_t w, uint32_t ws) {
  uint32_t s = x + y;
  s = umin(s, s - P2);
  const uint32_t d = x - y + P2;
  x = s;
  y = shoup(d, w, ws);
}

// ------------------------------------------------------------------------------ TMA bulk + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint32_t* slot_wptr(const Regions& reg, uint32_t id) {
  const uint32_t r = id >> 28;  // select without dynamic indexing (keeps the params out of local memory)
  uint32_t* b = r == 0 ? reg.base[0] : (r == 1 ? reg.base[1] : (r == 2 ? reg.base[2] : reg.base[3]));
  return b + static_cast<size_t>(id & 0x0FFFFFFFu) * kCt;
}
__device__ __forceinline__ const uint32_t* slot_ptr(const Regions& reg, uint32_t id) { return slot_wptr(reg, id); }

// ------------------------------------------------------------------------------ layouts / swizzle
// phys(j) = j ^ h(j), h = j8 | j5<<1 | j6<<2 | j7<<3 | j8<<4; written as base(t) ^ c(r) per layout.
__device__ __forceinline__ uint32_t bit(uint32_t x, int b) { return (x >> b) & 1u; }
__device__ __forceinline__ uint32_t baseA(uint32_t t) { return t ^ (bit(t, 5) << 1); }
__host__ __device__ constexpr uint32_t cA(int r) {
  return (static_cast<uint32_t>(r) << 6) ^ (((r >> 2) & 1) * 17u) ^ ((r & 1) << 2) ^ (((r >> 1) & 1) << 3);
}
__device__ __forceinline__ uint32_t baseB(uint32_t t) {
  const uint32_t j = ((t >> 2) << 6) | (t & 3u);
  return j ^ (bit(t, 4) * 17u) ^ (bit(t, 2) << 2) ^ (bit(t, 3) << 3);
}
__host__ __device__ constexpr uint32_t cB(int r) {
  return (static_cast<uint32_t>(r) << 2) ^ (((r >> 3) & 1) << 1);
}
__device__ __forceinline__ uint32_t baseC(uint32_t t) {
  return (t << 4) ^ (bit(t, 4) * 17u) ^ (bit(t, 1) << 1) ^ (bit(t, 2) << 2) ^ (bit(t, 3) << 3);
}
__host__ __device__ constexpr uint32_t cC(int r) { return static_cast<uint32_t>(r); }

typedef uint32_t Poly[6][16];

// Uniform stages 0-3 (layout A): pair (r, r | rb), rb = 8 >> s; twiddle k = 2^s + (r >> (4 - s)).
template <int S, bool INV>
__device__ __forceinline__ void stage_uniform(Poly& d) {
  constexpr int rb = 8 >> S;
#pragma unroll
  for (int r = 0; r < 16; r++) {
    if (r & rb) continue;
    const uint2 w = c_tw[INV][(1 << S) + (r >> (4 - S))];
#pragma unroll
    for (int p = 0; p < 6; p++) {
      if (INV)
        gs_bfly(d[p][r], d[p][r | rb], w.x, w.y);
      else
        ct_bfly(d[p][r], d[p][r | rb], w.x, w.y);
    }
  }
}

// Lane-varying stages 4-7 (layout B): rb = 8 >> (S-4); block index j >> (10 - S).
template <int S, bool INV>
__device__ __forceinline__ void stage_B(Poly& d, uint32_t t, const uint2* __restrict__ tw) {
  constexpr int rb = 8 >> (S - 4);
  const uint32_t thi = t >> 2;
#pragma unroll
  for (int r = 0; r < 16; r++) {
    if (r & rb) continue;
    // j = thi<<6 | r<<2 | tlo ; j >> (10 - S) = thi << (S - 4) | r >> (8 - S)
    const uint32_t k = (1u << S) + (thi << (S - 4)) + (static_cast<uint32_t>(r) >> (8 - S));
    const uint2 w = __ldg(tw + k);
#pragma unroll
    for (int p = 0; p < 6; p++) {
      if (INV)
        gs_bfly(d[p][r], d[p][r | rb], w.x, w.y);
      else
        ct_bfly(d[p][r], d[p][r | rb], w.x, w.y);
    }
  }
}

// Lane-varying stages 8-9 (layout C): rb = 2 (S = 8) / 1 (S = 9); j = t<<4 | r.
template <int S, bool INV>
__device__ __forceinline__ void stage_C(Poly& d, uint32_t t, const uint2* __restrict__ tw) {
  constexpr int rb = S == 8 ? 2 : 1;
#pragma unroll
  for (int r = 0; r < 16; r++) {
    if (r & rb) continue;
    const uint32_t k = (1u << S) + (t << (S - 6)) + (static_cast<uint32_t>(r) >> (10 - S));
    const uint2 w = __ldg(tw + k);
#pragma unroll
    for (int p = 0; p < 6; p++) {
      if (INV)
        gs_bfly(d[p][r], d[p][r | rb], w.x, w.y);
      else
        ct_bfly(d[p][r], d[p][r | rb], w.x, w.y);
    }
  }
}

// Layout change through shared memory, 3 polynomials per round (xb holds 3 x 1024 words).
template <int FROM, int TO>
__device__ __forceinline__ void exchange(Poly& d, uint32_t* xb, uint32_t t) {
  const uint32_t bs = FROM == 0 ? baseA(t) : (FROM == 1 ? baseB(t) : baseC(t));
  const uint32_t bd = TO == 0 ? baseA(t) : (TO == 1 ? baseB(t) : baseC(t));
#pragma unroll
  for (int half = 0; half < 2; half++) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 3; q++)
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const uint32_t c = FROM == 0 ? cA(r) : (FROM == 1 ? cB(r) : cC(r));
        xb[q * N + (bs ^ c)] = d[half * 3 + q][r];
      }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 3; q++)
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const uint32_t c = TO == 0 ? cA(r) : (TO == 1 ? cB(r) : cC(r));
        d[half * 3 + q][r] = xb[q * N + (bd ^ c)];
      }
  }
}

}  // namespace

// ================================================================================ K2 blind rotation
__global__ void __launch_bounds__(kBrThreads, 1) vlp_blind_rotate_kernel(const BrArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* ring = reinterpret_cast<uint32_t*>(smem);
  uint32_t* acc_all = ring + kSlots * 64 * kChunkWords;
  uint32_t* xb_all = acc_all + kBrBoot * 2 * N;
  uint16_t* abar_all = reinterpret_cast<uint16_t*>(xb_all + kBrBoot * 3 * N);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(abar_all + kBrBoot * 640);

  const uint32_t tid = threadIdx.x, g = tid >> 6, t = tid & 63;
  uint32_t* acc = acc_all + g * 2 * N;
  uint32_t* xb = xb_all + g * 3 * N;
  uint16_t* abar = abar_all + g * 640;

  const uint32_t ngroups = (a.njobs + kBrBoot - 1) / kBrBoot;
  if (blockIdx.x >= ngroups) return;
  const uint32_t my_groups = (ngroups - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const uint64_t total_chunks = static_cast<uint64_t>(my_groups) * a.steps * kChunks;

  if (tid == 0) {
    for (int s = 0; s < kSlots; s++) mbar_init(&mbar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // chunk sequence n -> (step (n / 8) % steps, chunk n % 8) of the bsk; slot n % kSlots
  auto issue = [&](uint64_t nseq) {
    const uint32_t step = static_cast<uint32_t>((nseq / kChunks) % a.steps), c = nseq % kChunks;
    const uint32_t s = nseq % kSlots;
    bulk_load(ring + s * 64 * kChunkWords, a.bsk + (static_cast<size_t>(step) * kChunks + c) * 64 * kChunkWords,
              kChunkBytes, &mbar[s]);
  };
  if (tid == 0)
    for (uint64_t q = 0; q < kSlots && q < total_chunks; q++) issue(q);
  uint64_t nseq = 0;

  for (uint32_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const uint32_t jb = grp * kBrBoot + g;
    const bool active = jb < a.njobs;
    // ---- S2 gate linear form + S3 mod-switch: abar[0..629], bbar at [630]
    if (active) {
      const BrJob job = a.jobs[jb];
      const uint32_t* x = slot_ptr(a.reg, job.x);
      const uint32_t* y = slot_ptr(a.reg, job.y);
      for (uint32_t w = t; w <= static_cast<uint32_t>(n); w += 64) {
        uint32_t c = static_cast<uint32_t>(static_cast<int32_t>(job.ax)) * x[w];
        if (job.ay) c += static_cast<uint32_t>(static_cast<int32_t>(job.ay)) * y[w];
        if (w == static_cast<uint32_t>(n)) c += job.k0;
        abar[w] = static_cast<uint16_t>(((c + (1u << 20)) >> 21) & (2 * N - 1));
      }
    } else {
      for (uint32_t w = t; w <= static_cast<uint32_t>(n); w += 64) abar[w] = 0;
    }
    __syncthreads();
    // ---- S4 accumulator init: (0, X^{-bbar} testv), testv = 1/8 everywhere (R8)
    {
      const uint32_t bbar = abar[n];
      for (uint32_t k = t; k < static_cast<uint32_t>(N); k += 64) {
        acc[k] = 0;
        acc[N + k] = (((k + bbar) & (2 * N - 1)) < static_cast<uint32_t>(N)) ? kMu : (0u - kMu);
      }
    }
    __syncthreads();

    // ---- S5: CMux steps
    for (int i = 0; i < a.steps; i++) {
      const uint32_t ab = abar[i];
      Poly d;
      // X^{abar} acc - acc, gadget digits (R5, offset 0x81020400), digit + p - 64 in [p-64, p+64)
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const uint32_t j = t + 64u * r;
        const uint32_t kk = (j - ab) & (2 * N - 1);
        const uint32_t src = kk & (N - 1);
        const bool neg = kk >= static_cast<uint32_t>(N);
#pragma unroll
        for (int u = 0; u < 2; u++) {
          uint32_t v = acc[u * N + src];
          v = neg ? 0u - v : v;
          const uint32_t w = v - acc[u * N + j] + 0x81020400u;
          d[u * 3 + 0][r] = ((w >> 25) & 127u) + (P - 64u);
          d[u * 3 + 1][r] = ((w >> 18) & 127u) + (P - 64u);
          d[u * 3 + 2][r] = ((w >> 11) & 127u) + (P - 64u);
        }
      }
      // forward NTT of the 6 digit polynomials
      stage_uniform<0, false>(d);
      stage_uniform<1, false>(d);
      stage_uniform<2, false>(d);
      stage_uniform<3, false>(d);
      exchange<0, 1>(d, xb, t);
      stage_B<4, false>(d, t, a.tw_fwd);
      stage_B<5, false>(d, t, a.tw_fwd);
      stage_B<6, false>(d, t, a.tw_fwd);
      stage_B<7, false>(d, t, a.tw_fwd);
      exchange<1, 2>(d, xb, t);
      stage_C<8, false>(d, t, a.tw_fwd);
      stage_C<9, false>(d, t, a.tw_fwd);

      // pointwise MAC with bsk_i (streamed chunk by chunk through the smem ring, shared by the CTA)
#pragma unroll
      for (int c = 0; c < kChunks; c++) {
        const uint32_t s = nseq % kSlots;
        mbar_wait(&mbar[s], static_cast<uint32_t>((nseq / kSlots) & 1));
        const uint32_t* rec = ring + s * 64 * kChunkWords + t * kChunkWords;
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int r = 2 * c + e;
          uint32_t x[6];
#pragma unroll
          for (int q = 0; q < 6; q++) x[q] = umin(d[q][r], d[q][r] - P2);  // [0, 2p)
          uint32_t kv[36];
#pragma unroll
          for (int v = 0; v < 9; v++) {
            const uint4 b4 = reinterpret_cast<const uint4*>(rec + e * 36)[v];
            kv[4 * v + 0] = b4.x;
            kv[4 * v + 1] = b4.y;
            kv[4 * v + 2] = b4.z;
            kv[4 * v + 3] = b4.w;
          }
#pragma unroll
          for (int o = 0; o < 6; o++) {
            uint64_t T = 0;
#pragma unroll
            for (int q = 0; q < 6; q++) T += static_cast<uint64_t>(x[q]) * kv[o * 6 + q];
            const uint32_t m = static_cast<uint32_t>(T) * PINV_NEG;
            const uint32_t y = static_cast<uint32_t>((T + static_cast<uint64_t>(m) * P) >> 32);  // < 4p
            d[o][r] = umin(y, y - P2);
          }
        }
        __syncthreads();  // every thread is done with slot s
        if (tid == 0 && nseq + kSlots < total_chunks) {
          fence_proxy_async();
          issue(nseq + kSlots);
        }
        nseq++;
      }

      // inverse NTT of the 6 (component, limb) products
      stage_C<9, true>(d, t, a.tw_inv);
      stage_C<8, true>(d, t, a.tw_inv);
      exchange<2, 1>(d, xb, t);
      stage_B<7, true>(d, t, a.tw_inv);
      stage_B<6, true>(d, t, a.tw_inv);
      stage_B<5, true>(d, t, a.tw_inv);
      stage_B<4, true>(d, t, a.tw_inv);
      exchange<1, 0>(d, xb, t);
      stage_uniform<3, true>(d);
      stage_uniform<2, true>(d);
      stage_uniform<1, true>(d);
      stage_uniform<0, true>(d);

      // centered lift of the three limbs, recombine mod 2^32, acc += (layout A: j = t + 64 r)
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const uint32_t j = t + 64u * r;
#pragma unroll
        for (int u = 0; u < 2; u++) {
          uint32_t sum = 0;
#pragma unroll
          for (int l = 0; l < 3; l++) {
            uint32_t v = d[u * 3 + l][r];
            v = umin(v, v - P);                       // [0, p)
            const uint32_t sv = v > (P >> 1) ? v - P : v;  // centered, as a 2's complement u32
            sum += sv << (11 * l);
          }
          acc[u * N + j] += sum;
        }
      }
      __syncthreads();
    }

    // ---- S6 SampleExtract: a'_0 = a_0, a'_k = -a_{N-k}, b' = b_0
    if (active) {
      if (a.raw_acc) {
        uint32_t* o = a.raw_acc + static_cast<size_t>(jb) * 2 * N;
        for (uint32_t k = t; k < 2u * N; k += 64) o[k] = acc[k];
      } else {
        uint32_t* o = a.nlwe + static_cast<size_t>(a.jobs[jb].out) * kNlwe;
        for (uint32_t k = t; k < static_cast<uint32_t>(N); k += 64) o[k] = k == 0 ? acc[0] : 0u - acc[N - k];
        if (t == 0) o[N] = acc[N];
      }
    }
    __syncthreads();
  }
}

// ================================================================================ K3 key switch
// CTA: kKsCt ciphertexts x all 632 columns (160 threads x 4 columns), coefficients [i0, i1).
// The ksk block of one coefficient i (8 x 3 rows, 60,672 B) is streamed into shared memory by TMA
// (double-buffered) and used by all kKsCt ciphertexts.
__global__ void __launch_bounds__(kKsThreads) vlp_keyswitch_kernel(const KsArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* kbuf = reinterpret_cast<uint32_t*>(smem);  // [2][kKsRowWords]
  uint16_t* abar = reinterpret_cast<uint16_t*>(kbuf + 2 * kKsRowWords);  // [kKsCt][N]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(abar + kKsCt * N);

  const uint32_t tid = threadIdx.x;
  const uint32_t c0 = blockIdx.x * kKsCt;
  const uint32_t nct = min(static_cast<uint32_t>(kKsCt), a.njobs - c0);
  const int i0 = static_cast<int>(blockIdx.y) * N / a.parts, i1 = static_cast<int>(blockIdx.y + 1) * N / a.parts;

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    bulk_load(kbuf, a.ksk + static_cast<size_t>(i0) * kKsRowWords, kKsRowWords * 4, &mbar[0]);
    if (i0 + 1 < i1)
      bulk_load(kbuf + kKsRowWords, a.ksk + static_cast<size_t>(i0 + 1) * kKsRowWords, kKsRowWords * 4, &mbar[1]);
  }
  // S7 MUX combine + rounding to 16 bits (R6)
  for (uint32_t idx = tid; idx < nct * (i1 - i0); idx += blockDim.x) {
    const uint32_t c = idx / (i1 - i0), i = i0 + idx % (i1 - i0);
    const KsJob job = a.jobs[c0 + c];
    uint32_t v = a.nlwe[static_cast<size_t>(job.n0) * kNlwe + i];
    if (job.n1 != 0xFFFFFFFFu) v += a.nlwe[static_cast<size_t>(job.n1) * kNlwe + i];
    abar[c * N + i] = static_cast<uint16_t>((v + (1u << 15)) >> 16);
  }
  __syncthreads();

  const uint32_t col = tid * 4;
  const bool live = col < static_cast<uint32_t>(kCt);
  uint32_t acc[kKsCt][4];
#pragma unroll
  for (int c = 0; c < kKsCt; c++) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = 0;

  for (int i = i0; i < i1; i++) {
    const int buf = (i - i0) & 1;
    mbar_wait(&mbar[buf], static_cast<uint32_t>(((i - i0) >> 1) & 1));
    const uint32_t* kb = kbuf + buf * kKsRowWords;
    if (live) {
#pragma unroll
      for (int c = 0; c < kKsCt; c++) {
        if (c >= static_cast<int>(nct)) break;
        const uint32_t ab = abar[c * N + i];
#pragma unroll
        for (int j = 0; j < kKsT; j++) {
          const uint32_t dg = (ab >> (14 - 2 * j)) & 3u;
          if (dg) {
            const uint4 row = *reinterpret_cast<const uint4*>(kb + (j * 3 + (dg - 1)) * kCt + col);
            acc[c][0] += row.x;
            acc[c][1] += row.y;
            acc[c][2] += row.z;
            acc[c][3] += row.w;
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0 && i + 2 < i1) {
      fence_proxy_async();
      bulk_load(kbuf + buf * kKsRowWords, a.ksk + static_cast<size_t>(i + 2) * kKsRowWords, kKsRowWords * 4,
                &mbar[buf]);
    }
  }
  if (!live) return;
  // out = (0, b') - sum (S8); with several coefficient parts the partial sums are reduced atomically
  // into a row pre-set to (0, b') by vlp_ks_init_kernel (u32 adds commute: exact).
#pragma unroll
  for (int c = 0; c < kKsCt; c++) {
    if (c >= static_cast<int>(nct)) break;
    const KsJob job = a.jobs[c0 + c];
    uint32_t* o = slot_wptr(a.reg, job.out);
    if (a.parts == 1) {
      uint32_t bp = a.nlwe[static_cast<size_t>(job.n0) * kNlwe + N];
      if (job.n1 != 0xFFFFFFFFu) bp += a.nlwe[static_cast<size_t>(job.n1) * kNlwe + N];
      bp += job.add;
      uint4 r;
      r.x = (col + 0 == static_cast<uint32_t>(n) ? bp : 0u) - acc[c][0];
      r.y = (col + 1 == static_cast<uint32_t>(n) ? bp : 0u) - acc[c][1];
      r.z = (col + 2 == static_cast<uint32_t>(n) ? bp : 0u) - acc[c][2];
      r.w = col + 3 >= static_cast<uint32_t>(n + 1) ? 0u : ((col + 3 == static_cast<uint32_t>(n) ? bp : 0u) - acc[c][3]);
      *reinterpret_cast<uint4*>(o + col) = r;
    } else {
#pragma unroll
      for (int e = 0; e < 4; e++)
        if (col + e <= static_cast<uint32_t>(n) && acc[c][e]) atomicAdd(o + col + e, 0u - acc[c][e]);
    }
  }
}

__global__ void vlp_ks_init_kernel(const KsArgs a) {
  const uint32_t c = blockIdx.x;
  const KsJob job = a.jobs[c];
  uint32_t* o = slot_wptr(a.reg, job.out);
  for (uint32_t k = threadIdx.x; k < static_cast<uint32_t>(kCt); k += blockDim.x) {
    uint32_t v = 0;
    if (k == static_cast<uint32_t>(n)) {
      v = a.nlwe[static_cast<size_t>(job.n0) * kNlwe + N] + job.add;
      if (job.n1 != 0xFFFFFFFFu) v += a.nlwe[static_cast<size_t>(job.n1) * kNlwe + N];
    }
    o[k] = v;
  }
}

// ================================================================================ K4 bsk conversion
// One CTA per (i, row r, component u): split the 1024 torus32 coefficients into 3 signed limbs, forward
// NTT each limb polynomial mod p (plain, fully reduced), multiply by N^-1 * 2^32 mod p, scatter into
// the chunked layout [i][chunk][t][e*36 + (u*3 + limb)*6 + r] with position 16t + 2*chunk + e.
__global__ void __launch_bounds__(512) vlp_bsk_convert_kernel(const uint32_t* __restrict__ raw,
                                                              uint32_t* __restrict__ out,
                                                              const uint2* __restrict__ tw, uint32_t c_mont) {
  __shared__ uint32_t poly[3][N];
  const uint32_t bid = blockIdx.x;  // (i*6 + r)*2 + u
  const uint32_t u = bid & 1, r = (bid >> 1) % kRows, i = (bid >> 1) / kRows;
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
    const uint32_t q = threadIdx.x;  // butterfly 0..511
    const uint32_t blk = q / half, j = 2 * blk * half + (q % half);
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
    const uint32_t t = k >> 4, pos = k & 15, c = pos >> 1, e = pos & 1;
    uint32_t* dst = out + ((static_cast<size_t>(i) * kChunks + c) * 64 + t) * kChunkWords + e * 36;
#pragma unroll
    for (int l = 0; l < 3; l++) {
      const uint32_t o = u * 3 + l;
      dst[o * 6 + r] = static_cast<uint32_t>(static_cast<uint64_t>(poly[l][k]) * c_mont % P);
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

__global__ void vlp_copy_rows_kernel(const uint32_t* __restrict__ slots, Regions reg, uint32_t* out) {
  const uint32_t* src = slot_ptr(reg, slots[blockIdx.x]);
  for (uint32_t k = threadIdx.x; k < static_cast<uint32_t>(kCt); k += blockDim.x)
    out[static_cast<size_t>(blockIdx.x) * kCt + k] = src[k];
}

// ================================================================================ launchers
void set_const_twiddles(const uint2* fwd16, const uint2* inv16) {
  uint2 h[2][16];
  for (int k = 0; k < 16; k++) {
    h[0][k] = fwd16[k];
    h[1][k] = inv16[k];
  }
  cudaMemcpyToSymbol(c_tw, h, sizeof(h));
}

void launch_bsk_convert(const uint32_t* raw, uint32_t* out, const uint2* tw_fwd, uint32_t c_mont, cudaStream_t st) {
  vlp_bsk_convert_kernel<<<n * kRows * 2, 512, 0, st>>>(raw, out, tw_fwd, c_mont);
}

int br_grid(uint32_t njobs, int sm_count) {
  const uint32_t groups = (njobs + kBrBoot - 1) / kBrBoot;
  return static_cast<int>(groups < static_cast<uint32_t>(sm_count) ? groups : sm_count);
}

cudaError_t launch_blind_rotate(const BrArgs& a, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(vlp_blind_rotate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kBrSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (a.njobs == 0) return cudaSuccess;
  vlp_blind_rotate_kernel<<<grid, kBrThreads, kBrSmemBytes, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_keyswitch(const KsArgs& a0, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(vlp_keyswitch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kKsSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (a0.njobs == 0) return cudaSuccess;
  KsArgs a = a0;
  const uint32_t tiles = (a.njobs + kKsCt - 1) / kKsCt;
  int parts = 1;
  while (parts < 16 && tiles * parts * 2 <= 2 * 148) parts *= 2;  // fill the chip on narrow levels
  a.parts = parts;
  if (parts > 1) vlp_ks_init_kernel<<<a.njobs, 128, 0, st>>>(a);
  vlp_keyswitch_kernel<<<dim3(tiles, parts), kKsThreads, kKsSmemBytes, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_init_constants(uint32_t* mid, cudaStream_t st) {
  vlp_init_constants_kernel<<<1, 256, 0, st>>>(mid);
  return cudaGetLastError();
}

cudaError_t launch_copy_rows(const uint32_t* slots, uint32_t count, Regions reg, uint32_t* out, cudaStream_t st) {
  if (!count) return cudaSuccess;
  vlp_copy_rows_kernel<<<count, 128, 0, st>>>(slots, reg, out);
  return cudaGetLastError();
}

}  // namespace vlp
