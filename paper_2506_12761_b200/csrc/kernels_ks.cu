// kernels_ks.cu -- K3T: the key switch (S8) as a hand-written tcgen05 int8 GEMM, with the MUX
// combine (S7) in its prologue.  Replaces the cuBLASLt call of round 1.
//
// Definition (R6): for each coefficient i < 1024 of the N-LWE a', abar_i = floor((a'_i + 2^15) / 2^16) mod 2^16 and
// its 8 base-4 digits d_ij (field f = 7 - j holds bits 2f, 2f + 1); out = (0, b') - sum_{i,j: d_ij != 0}
// ksk[i][j][d_ij].  Written as a GEMM: D[c][n] = sum_k ind[c][k] * kmat[n][k] with the one-hot digit indicator
// ind[c][k] = [d_ij(c) = v] at k = ((i / 16) * 3 + v - 1) * 128 + (i % 16) * 8 + f (K = 24576) and kmat the ksk split into 4 balanced
// signed byte limbs, n = col * 4 + limb (N = 2528, padded to 2560).  |D| <= 8192 * 128 < 2^31: exact; then
// out[col] = (col == 630 ? b' : 0) - sum_l D[c][4 col + l] 2^(8l) mod 2^32 -- bit-identical to the definition.
//
//  * vlp_ks_prep_kernel: per job, the MUX combine u = (0, add) + n0 (+ n1) (S7), abar[1024] (u16) and b'.
//  * vlp_ks_gemm_kernel: persistent CTAs, tile = 128 jobs x 256 n (64 output columns), K loop of 192 blocks of 128
//    bytes, 4-stage smem ring.  Warp 0: the kmat block by one cp.async.bulk (kmat is pre-laid-out at setup in the
//    UMMA K-major SWIZZLE_128B order, 32 KB per (n tile, K block)); warps 2-5: the indicator block generated in
//    shared memory in the same swizzled layout (one row = one job per thread, 16 coefficients x 8 digit bytes per
//    block), then the epilogue (TMEM -> limb recombination -> the job's output slot); warp 1: one elected thread
//    issues 4 x tcgen05.mma.kind::i8 (M 128, N 256, K 32) per block into a 128 x 256 int32 TMEM accumulator and
//    tcgen05.commit's the ring slot back.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "devcommon.cuh"
#include "kernels.cuh"

namespace vlp {
namespace {
using namespace dev;

constexpr int kKsTileM = 128;
constexpr int kKsTileN = 256;
constexpr int kKsBlockK = 128;                       // bytes (int8) per K block = one SWIZZLE_128B atom row
constexpr int kKsKBlocks = kKsK / kKsBlockK;         // 192
constexpr int kKsStages = 4;
constexpr int kKsABytes = kKsTileM * kKsBlockK;      // 16 KB
constexpr int kKsBBytes = kKsTileN * kKsBlockK;      // 32 KB
constexpr int kKsThreads = 192;
constexpr int kKsSmem = 1024 + kKsStages * (kKsABytes + kKsBBytes) + 256;

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B: rows of 128 B, 8-row groups 1024 B apart (SBO), version 1
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor: kind::i8, D s32, A s8, B s8, both K-major, N = 256, M = 128
constexpr uint32_t kKsIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((kKsTileN >> 3) << 17) | ((kKsTileM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kKsIdesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 4 digit-equality bits (bits 0..3 of m) -> 4 bytes 0/1 (copies 7 bits apart never overlap a 4-bit value)
__device__ __forceinline__ uint32_t spread4(uint32_t m) { return (m * 0x00204081u) & 0x01010101u; }

}  // namespace

// ================================================================================ K3T prologue (S7 + R6)
// One warp per job: u = (0, add) + n0 (+ n1), abar_i = (u_i + 2^15) >> 16 (u16), b' = u_N.
__global__ void __launch_bounds__(256) vlp_ks_prep_kernel(const KsArgs a, uint32_t c0, uint32_t cnt,
                                                          uint16_t* __restrict__ abuf, uint32_t* __restrict__ bbuf) {
  const uint32_t c = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= cnt) return;
  const KsJob job = a.jobs[c0 + c];
  const uint4* x0 = reinterpret_cast<const uint4*>(a.nlwe + static_cast<size_t>(job.n0) * kNlwe);
  const uint4* x1 = job.n1 != 0xFFFFFFFFu ? reinterpret_cast<const uint4*>(a.nlwe + static_cast<size_t>(job.n1) * kNlwe)
                                          : nullptr;
  uint2* dst = reinterpret_cast<uint2*>(abuf + static_cast<size_t>(c) * N);
#pragma unroll
  for (int q = 0; q < 8; q++) {
    const uint32_t idx = q * 32 + lane;  // uint4 index: coefficients 4 idx .. 4 idx + 3
    uint4 v = x0[idx];
    if (x1) {
      const uint4 w = x1[idx];
      v.x += w.x;
      v.y += w.y;
      v.z += w.z;
      v.w += w.w;
    }
    const uint32_t a0 = (v.x + 32768u) >> 16, a1 = (v.y + 32768u) >> 16, a2 = (v.z + 32768u) >> 16,
                   a3 = (v.w + 32768u) >> 16;
    dst[idx] = make_uint2(a0 | (a1 << 16), a2 | (a3 << 16));
  }
  if (lane == 0) {
    uint32_t b = a.nlwe[static_cast<size_t>(job.n0) * kNlwe + N] + job.add;
    if (x1) b += a.nlwe[static_cast<size_t>(job.n1) * kNlwe + N];
    bbuf[c] = b;
  }
}

// ================================================================================ K3T GEMM
__global__ void __launch_bounds__(kKsThreads, 1) vlp_ks_gemm_kernel(const KsArgs a, uint32_t c0, uint32_t cnt,
                                                                    const uint16_t* __restrict__ abuf,
                                                                    const uint32_t* __restrict__ bbuf,
                                                                    const int8_t* __restrict__ kmat_sw) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;                                   // [stage][128 rows][128 B] swizzled
  uint8_t* sB = smem + kKsStages * kKsABytes;           // [stage][256 rows][128 B] swizzled
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kKsStages * kKsBBytes);
  uint64_t* empty = full + kKsStages;
  uint64_t* tfull = empty + kKsStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_sh = reinterpret_cast<uint32_t*>(tempty + 1);

  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
  const uint32_t mtiles = (cnt + kKsTileM - 1) / kKsTileM, ntiles = (kKsNp + kKsTileN - 1) / kKsTileN;
  const uint32_t tiles = mtiles * ntiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kKsStages; s++) {
      mbar_init(&full[s], 1 + 4);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_sh)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_sh;

  if (warp == 0) {
    // ---- kmat producer: one 32 KB bulk copy per K block
    if (lane == 0) {
      uint32_t it = 0;
      for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const uint32_t nt = t % ntiles;
        const int8_t* src = kmat_sw + static_cast<size_t>(nt) * kKsKBlocks * kKsBBytes;
        for (uint32_t kb = 0; kb < static_cast<uint32_t>(kKsKBlocks); kb++, it++) {
          const uint32_t s = it % kKsStages, ph = (it / kKsStages) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          bulk_load(sB + s * kKsBBytes, src + static_cast<size_t>(kb) * kKsBBytes, kKsBBytes, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    uint32_t it = 0, ti = 0;
    for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x, ti++) {
      mbar_wait(tempty, (ti & 1u) ^ 1u);  // the epilogue has drained the accumulator
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (uint32_t kb = 0; kb < static_cast<uint32_t>(kKsKBlocks); kb++, it++) {
        const uint32_t s = it % kKsStages, ph = (it / kKsStages) & 1u;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint32_t a0 = smem_u32(sA + s * kKsABytes), b0 = smem_u32(sB + s * kKsBBytes);
#pragma unroll
          for (int k = 0; k < kKsBlockK / 32; k++)
            mma_i8(tmem, sw128_desc(a0 + 32 * k), sw128_desc(b0 + 32 * k), (kb | k) != 0);
          mma_commit(&empty[s]);  // frees the ring slot once these MMAs have read it
          if (kb == static_cast<uint32_t>(kKsKBlocks) - 1) mma_commit(tfull);
        }
        __syncwarp();
      }
    }
  } else {
    // ---- indicator producers (one job row per thread) + epilogue; TMEM lane quadrant = warp % 4
    const uint32_t q = warp & 3u, r = 32u * q + lane;
    const uint32_t sw = r & 7u;
    uint32_t it = 0, ti = 0;
    for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x, ti++) {
      const uint32_t mt = t / ntiles, nt = t % ntiles;
      const uint32_t c = mt * kKsTileM + r;
      const bool valid = c < cnt;
      const uint4* arow = reinterpret_cast<const uint4*>(abuf + static_cast<size_t>(valid ? c : 0) * N);
      // K blocks are ordered (coefficient block, digit value): kb = (i0 / 16) * 3 + v - 1, so the 16 abar words of
      // a coefficient block serve 3 consecutive blocks; they are loaded one coefficient block ahead.
      uint4 n0 = make_uint4(0, 0, 0, 0), n1 = n0, w0 = n0, w1 = n0;
      if (valid) {
        n0 = __ldg(arow);
        n1 = __ldg(arow + 1);
      }
      for (uint32_t kb = 0; kb < static_cast<uint32_t>(kKsKBlocks); kb++, it++) {
        const uint32_t s = it % kKsStages, ph = (it / kKsStages) & 1u;
        const uint32_t v = kb % 3 + 1, ib = kb / 3;  // digit value, coefficient block (16 coefficients)
        if (v == 1) {
          w0 = n0;
          w1 = n1;
          if (valid && ib + 1 < static_cast<uint32_t>(N / 16)) {
            n0 = __ldg(arow + 2 * (ib + 1));
            n1 = __ldg(arow + 2 * (ib + 1) + 1);
          }
        }
        const uint32_t pat = v * 0x55555555u;  // v in every 2-bit field
        const uint32_t ws[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};  // 2 coefficients each
        mbar_wait(&empty[s], ph ^ 1u);
        uint8_t* dst = sA + s * kKsABytes + r * kKsBlockK;
#pragma unroll
        for (int ch = 0; ch < 8; ch++) {
          // chunk ch = coefficients i0 + 2 ch (bytes 0-7), i0 + 2 ch + 1 (bytes 8-15); byte f = [field f == v]
          const uint32_t x = ws[ch] ^ pat;
          uint32_t e = ~(x | (x >> 1)) & 0x55555555u;  // bit 2f (+16 for the 2nd coefficient): field f == v
          if (!valid) e = 0;
          // gather the even bits: bit 2f -> bit f within each 16-bit half
          e = (e | (e >> 1)) & 0x33333333u;
          e = (e | (e >> 2)) & 0x0F0F0F0Fu;
          e = (e | (e >> 4)) & 0x00FF00FFu;
          const uint4 out = make_uint4(spread4(e & 15u), spread4((e >> 4) & 15u), spread4((e >> 16) & 15u),
                                       spread4((e >> 20) & 15u));
          *reinterpret_cast<uint4*>(dst + ((ch ^ sw) << 4)) = out;
        }
        fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      }
      // ---- epilogue: out[col] = (col == n ? b' : 0) - sum_l D[4 col + l] 2^(8l)
      mbar_wait(tfull, ti & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t* orow = valid ? slot_wptr(a.reg, a.jobs[c0 + c].out) : nullptr;
      const uint32_t bp = valid ? bbuf[c] : 0u;
#pragma unroll 1
      for (int g = 0; g < kKsTileN / 32; g++) {
        uint32_t d[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
            "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
              "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]), "=r"(d[16]),
              "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]), "=r"(d[24]),
              "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
            : "r"(tmem + ((32u * q) << 16) + 32u * g)
            : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (valid) {
          const uint32_t col0 = nt * 64 + g * 8;
          uint32_t o[8];
#pragma unroll
          for (int j = 0; j < 8; j++) {
            const uint32_t sum = d[4 * j] + (d[4 * j + 1] << 8) + (d[4 * j + 2] << 16) + (d[4 * j + 3] << 24);
            o[j] = (col0 + j == static_cast<uint32_t>(n) ? bp : 0u) - sum;
          }
          if (col0 + 8 <= static_cast<uint32_t>(kCt)) {
            reinterpret_cast<uint4*>(orow + col0)[0] = make_uint4(o[0], o[1], o[2], o[3]);
            reinterpret_cast<uint4*>(orow + col0)[1] = make_uint4(o[4], o[5], o[6], o[7]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

// ================================================================================ setup: kmat in UMMA order
// kmat_sw[nt][kb][r][128 B] (SWIZZLE_128B: 16-byte chunk c of row r at (c ^ (r & 7)) * 16); row n = nt * 256 + r =
// col * 4 + limb; K block kb = (coefficient block ib, digit value v): kb = ib * 3 + v - 1, byte b of the block ->
// coefficient i = ib * 16 + b / 8, field f = b % 8 -> ksk[i][j = 7 - f][v - 1][col]'s limb.
__global__ void vlp_kmat_sw_kernel(const uint32_t* __restrict__ ksk, int8_t* __restrict__ out) {
  const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // one 4-byte group per thread
  const size_t total = static_cast<size_t>(kKsNt) * kKsKBlocks * kKsTileN * (kKsBlockK / 4);
  if (idx >= total) return;
  const uint32_t b4 = static_cast<uint32_t>(idx % (kKsBlockK / 4));
  const size_t rowid = idx / (kKsBlockK / 4);
  const uint32_t r = static_cast<uint32_t>(rowid % kKsTileN);
  const uint32_t kb = static_cast<uint32_t>((rowid / kKsTileN) % kKsKBlocks);
  const uint32_t nt = static_cast<uint32_t>(rowid / kKsTileN / kKsKBlocks);
  const uint32_t nrow = nt * kKsTileN + r, col = nrow / 4, l = nrow % 4;
  uint32_t packed = 0;
#pragma unroll
  for (int e = 0; e < 4; e++) {
    const uint32_t b = b4 * 4 + e;  // byte within the block: coefficient ib * 16 + b / 8, field b % 8
    const uint32_t vi = kb % 3, i = (kb / 3) * 16 + b / 8, f = b % 8, j = 7 - f;
    int32_t limb = 0;
    if (col < static_cast<uint32_t>(kCt)) {
      int64_t x = static_cast<int64_t>(ksk[((static_cast<size_t>(i) * kKsT + j) * 3 + vi) * kCt + col]);
      int64_t s = 0;
      for (uint32_t q = 0; q <= l; q++) {
        s = ((x + 128) & 255) - 128;  // balanced byte limb in [-128, 128)
        x = (x - s) >> 8;
      }
      limb = static_cast<int32_t>(s);
    }
    packed |= (static_cast<uint32_t>(limb) & 255u) << (8 * e);
  }
  const uint32_t chunk = (b4 * 4) / 16, within = (b4 * 4) % 16;
  const size_t off = ((static_cast<size_t>(nt) * kKsKBlocks + kb) * kKsTileN + r) * kKsBlockK + ((chunk ^ (r & 7u)) << 4) + within;
  *reinterpret_cast<uint32_t*>(out + off) = packed;
}

void launch_kmat_sw(const uint32_t* ksk, int8_t* kmat_sw, cudaStream_t st) {
  const size_t total = static_cast<size_t>(kKsNt) * kKsKBlocks * kKsTileN * (kKsBlockK / 4);
  vlp_kmat_sw_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(ksk, kmat_sw);
}

size_t ks_stage_bytes_t(uint32_t chunk) {
  return (static_cast<size_t>(chunk) * N * 2 + 255) / 256 * 256 + (static_cast<size_t>(chunk) * 4 + 255) / 256 * 256;
}

cudaError_t launch_keyswitch_t(const KsArgs& a, const int8_t* kmat_sw, uint8_t* stage, uint32_t chunk, int sm_count,
                               cudaStream_t st) {
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set.load() & bit)) {
    if ((e = cudaFuncSetAttribute(vlp_ks_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kKsSmem))) return e;
    attr_set.fetch_or(bit);
  }
  uint16_t* abuf = reinterpret_cast<uint16_t*>(stage);
  uint32_t* bbuf = reinterpret_cast<uint32_t*>(stage + (static_cast<size_t>(chunk) * N * 2 + 255) / 256 * 256);
  for (uint32_t c0 = 0; c0 < a.njobs; c0 += chunk) {
    const uint32_t cnt = a.njobs - c0 < chunk ? a.njobs - c0 : chunk;
    vlp_ks_prep_kernel<<<(cnt + 7) / 8, 256, 0, st>>>(a, c0, cnt, abuf, bbuf);
    const uint32_t tiles = (cnt + kKsTileM - 1) / kKsTileM * kKsNt;
    const uint32_t grid = tiles < static_cast<uint32_t>(sm_count) ? tiles : static_cast<uint32_t>(sm_count);
    vlp_ks_gemm_kernel<<<grid, kKsThreads, kKsSmem, st>>>(a, c0, cnt, abuf, bbuf, kmat_sw);
    if ((e = cudaGetLastError())) return e;
  }
  return cudaSuccess;
}

}  // namespace vlp
