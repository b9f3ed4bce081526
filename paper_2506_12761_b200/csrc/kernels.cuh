// kernels.cuh -- device-side declarations shared by kernels.cu and api.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "vlp_internal.h"

namespace vlp {

// ---- blind rotation (K2): 5 bootstraps per CTA, 128 threads each, 8 coefficients per thread per
// polynomial
constexpr int kBT = 128;                            // threads per bootstrap
constexpr int kBrBoot = 5;                          // bootstraps per CTA
constexpr int kBrThreads = kBT * kBrBoot;           // 512
constexpr int kChunks = 4;                          // bsk chunks per CMux step: slot pairs (positions)
constexpr int kChunkWords = 76;                     // words per thread per chunk: [o 6][e 2][q 6] + 4 pad
constexpr int kChunkBytes = kBT * kChunkWords * 4;  // 38912
constexpr int kSlots = 3;                           // smem ring of bsk chunks
constexpr int kTwSlots = 18;                        // lane-varying twiddle slots (stages 3..9)
constexpr size_t kBskNttWords = static_cast<size_t>(n) * kChunks * kBT * kChunkWords;  // 24,514,560
// shared memory of a blind-rotate CTA with B bootstraps: bsk ring + per bootstrap (accumulator, exchange
// buffer, mod-switched mask) + mbarriers, release counters, TMEM base
__host__ __device__ constexpr int br_smem_bytes(int B) {
  return kSlots * kChunkBytes + B * (2 * N * 4 + 3 * N * 4 + 640 * 2) + 128 * 4 + kSlots * 8 + kSlots * 4 + 8;
}
constexpr int kBrSmemBytes = br_smem_bytes(kBrBoot);
// TMEM (tcgen05.ld/st, no MMA) as per-thread spill space: per warp slot 96 columns -- MAC outputs of
// component u at columns 32u + 8l + s, round-0 transformed digits at 64 + 8j + s.
constexpr int kTmemSlotCols = 96;
__host__ __device__ constexpr int tmem_cols(int B) { return B * kTmemSlotCols <= 128 ? 128 : (B * kTmemSlotCols <= 256 ? 256 : 512); }
static_assert(kBrBoot * kTmemSlotCols <= 512, "TMEM columns");
static_assert(kBrSmemBytes <= 232448, "shared memory per CTA");


// ---- key switch on the tensor cores (K3T, kernels_ks.cu): out = (0, b') - sum_{i,j} ksk[i][j][d_ij] as a
// hand-written tcgen05 int8 GEMM D[c][n] = sum_k ind[c][k] * kmat[n][k] with the one-hot digit indicator
// (generated in shared memory) and kmat = the ksk split into 4 balanced signed byte limbs, n = col * 4 + limb;
// |D| <= 8192 * 128 < 2^31: exact; out[col] = (col == n ? b' : 0) - sum_l D[c][4 col + l] 2^(8l) mod 2^32.
constexpr int kKsK = N * kKsT * 3;               // 24576 GEMM depth
constexpr int kKsNp = 4 * kCt;                   // 2528 GEMM columns (632 columns x 4 limbs)
constexpr int kKsNt = (kKsNp + 255) / 256;       // 10 N tiles of 256
constexpr size_t kKmatSwBytes = static_cast<size_t>(kKsNt) * 256 * kKsK;  // 62,914,560 (UMMA-ordered, zero-padded)
constexpr int kKsChunk = 32768;                  // jobs per key-switch launch pair (staging 2 KB + 4 B per job)

struct Regions {
  uint32_t* base[4];  // kRegIn0, kRegIn1, kRegMid, kRegOut; rows of kCt words
};

struct BrArgs {
  const BrJob* jobs;
  uint32_t njobs;
  int steps;          // CMux steps to run (n normally; fewer for the step-level parity tests)
  Regions reg;
  uint32_t* nlwe;     // [rows][kNlwe] output of extract (unless raw_acc)
  uint32_t* raw_acc;  // debug: [njobs][2][N] accumulators instead of extracting
  const uint32_t* bsk;  // NTT-domain bsk, layout [i][chunk][t][kChunkWords]
  const uint2* twl_fwd;  // [kTwSlots][kBT] (w, floor(w 2^32 / p)) in thread order
  const uint2* twl_inv;
  const double2* bskf;  // FFT-domain bsk (K2F engine), layout [i][chunk 12][rho' 8][o*2 + l][lane 32] complex
  const double2* psi;   // psi^e = exp(i pi e / 1024), e < 2048 (K2F per-lane twiddles)
  unsigned long long* fft_err;  // debug (vlp_debug_fft_error): max |V - round(V)| of K2F's roundings, double bits
  uint32_t zero;  // always 0 (a runtime zero; see add_alu in kernels.cu)
  uint32_t p2;    // always 2p, set by launch_blind_rotate (a runtime constant; see ct_bfly in kernels.cu)
  uint32_t pdl_at;  // K2F: CMux step at which a CTA lets the next wave's launch start (kernels_fft.cu; set there)
};

struct KsArgs {
  const KsJob* jobs;
  uint32_t njobs;
  Regions reg;
  const uint32_t* nlwe;  // [rows][kNlwe]
  const uint32_t* ksk;   // [N][8][3][kCt] (torus32 key-switching key; the GEMM uses its byte limbs)
};

// ---- K2F: the blind rotation on an exact FP64 negacyclic FFT (kernels_fft.cu).
// One warp = one bootstrap (32 lanes x 16 complex points of the folded 512-point transform), up to 8 per CTA;
// the FFT-domain key holds 2 signed 16-bit limbs per coefficient, scaled by 1/512.
constexpr int kFftMaxWarps = 8;
constexpr int kFftChunks = 12;                         // ring chunks per CMux step: 6 digit rows x 2 halves
constexpr int kFftChunkBytes = 8 * 4 * 32 * 16;        // 16384: [rho' 8][o*2 + l 4][lane 32] complex double
constexpr size_t kBskFftBytes = static_cast<size_t>(n) * kFftChunks * kFftChunkBytes;  // 123,863,040
constexpr size_t kPsiBytes = 2048 * sizeof(double2);
void launch_bsk_fft(const uint32_t* raw, double2* out, const double2* psi, cudaStream_t st);
void set_fft_constants(const double2* psi_host);
cudaError_t launch_blind_rotate_fft(const BrArgs& a, int warps, int sm_count, cudaStream_t st);
uint32_t fft_launch_count(uint32_t njobs, int warps, int sm_count);  // kernel launches of one K2F level

void launch_bsk_convert(const uint32_t* raw, uint32_t* out, const uint2* tw_fwd, uint32_t c_mont,
                        cudaStream_t st);
void set_const_twiddles(const uint2* fwd16, const uint2* inv16);
// one level: whole waves of kBrBoot bootstraps per CTA + a narrower tail wave (1 or 2 kernel launches)
cudaError_t launch_blind_rotate(const BrArgs& a, int sm_count, cudaStream_t st);
int set_br_route(int engine, int param);  // vlp_debug_route
void set_fft_error_monitor(unsigned long long* err_dev);  // vlp_debug_fft_error
int br_launch_count(uint32_t njobs, int sm_count);
// The mask generator a device kernel continues (host.cpp's Rng of the call): seeded, h1 = mix(seed ^ dom * C1)
// (R3); secure, ChaCha20 under `key` with nonce (dom, obj lo, obj hi) and block counter word / 8.
struct MaskGen {
  uint64_t h1;
  uint32_t key[8];
  uint32_t dom;
  uint32_t secure;
};
cudaError_t launch_encrypt_db(const uint32_t* s, const uint32_t* noise, const uint8_t* bits, const MaskGen& g, uint32_t per,
                              uint32_t W, uint32_t lI, uint64_t first, uint64_t nsamples, uint32_t* out, cudaStream_t st);
cudaError_t launch_server_enc(const uint32_t* pk, const uint8_t* bits, uint64_t nsamples, uint32_t* out, cudaStream_t st);
cudaError_t launch_keygen(const MaskGen& g_bsk, const MaskGen& g_ksk, const uint32_t* s, const uint32_t* z, const uint32_t* e_bsk,
                          const uint32_t* e_ksk, uint32_t* bsk, uint32_t* ksk, cudaStream_t st);
void launch_kmat_sw(const uint32_t* ksk, int8_t* kmat_sw, cudaStream_t st);
size_t ks_stage_bytes_t(uint32_t chunk);
// K3T over all jobs of a level in chunks of `chunk`: prologue (S7 + R6) + tcgen05 GEMM with fused epilogue
cudaError_t launch_keyswitch_t(const KsArgs& a, const int8_t* kmat_sw, uint8_t* stage, uint32_t chunk, int sm_count,
                               cudaStream_t st);
cudaError_t launch_init_constants(uint32_t* mid, cudaStream_t st);
cudaError_t launch_copy_rows(const uint32_t* slots, uint32_t count, Regions reg, uint32_t* out, cudaStream_t st);
cudaError_t launch_linear(const LinJob* jobs, const uint32_t* inputs, uint32_t count, Regions reg, cudaStream_t st);

}  // namespace vlp
