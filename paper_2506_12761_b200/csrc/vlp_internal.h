// Internal definitions shared by the host C++ (host.cpp, sched.cpp) and the CUDA side (kernels.cu,
// api.cu).  Not part of the ABI (include/vlp.h is).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/vlp.h"

namespace vlp {

constexpr int n = VLP_N_LWE;     // 630
constexpr int N = VLP_N_RING;    // 1024
constexpr int kRows = 6;         // (k+1) * ell TRGSW rows
constexpr int kEll = 3;
constexpr int kBgBits = 7;
constexpr int kKsT = 8;
constexpr int kKsBaseBits = 2;
constexpr int kCt = VLP_CT_STRIDE;     // 632
constexpr int kNlwe = VLP_NLWE_STRIDE; // 1028
constexpr uint32_t kMu = 0x20000000u;  // 1/8

// ---- error handling (thread-local message, no exceptions across the ABI)
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

// ---- PRNG domains (R3)
enum : uint64_t {
  kSkLwe = 1, kSkRing = 2, kBskA = 3, kBskE = 4, kKskA = 5, kKskE = 6,
  kPkA = 7, kPkE = 8, kQryA = 9, kQryE = 10, kFreshA = 12, kFreshE = 13
};
uint64_t prng(uint64_t seed, uint64_t dom, uint64_t obj, uint64_t word);
uint64_t prng_prefix(uint64_t seed, uint64_t dom);
void chacha20_block(const uint32_t key[8], uint32_t counter, const uint32_t nonce[3], uint32_t out[16]);

// The randomness of one call: the seeded counter PRNG (R3; reproducible, 64-bit seed: tests and benchmarks), or
// ChaCha20 under a 256-bit key drawn from the OS (getrandom) for the *_secure calls.  Either way a random-access
// generator u64(dom, obj, word); the secure one uses nonce (dom, obj), block counter word / 8.
struct Rng {
  uint64_t seed = 0;
  bool secure = false;
  uint32_t key[8] = {};
  uint64_t u64(uint64_t dom, uint64_t obj, uint64_t word) const;
  ~Rng();
};
Rng seeded(uint64_t seed);
int os_random(Rng* r);  // secure generator: getrandom key (or the key of vlp_debug_next_secure_key)
uint32_t noise(const Rng& g, uint64_t dom, uint64_t obj, uint64_t t, double sigma);  // Box-Muller (R2, R3)

int resolve_params(const vlp_params* params, vlp_params* out);
void secret_keys(const Rng& g, vlp_sk* sk);
void keygen_noise(const Rng& g, const vlp_params& p, uint32_t* bsk_noise, uint32_t* ksk_noise);
int prepare_db_bits(const vlp_meta* meta, size_t count, const uint64_t* words, const uint64_t* payloads,
                    std::vector<uint8_t>& bits);
int prepare_pk_noise(const vlp_sk* sk, const vlp_meta* meta, const Rng& g, size_t first, size_t count,
                     std::vector<uint32_t>& nz);
int prepare_encrypt_db(const vlp_sk* sk, const vlp_meta* meta, const Rng& g, size_t first, size_t count,
                       const uint64_t* words, const uint64_t* payloads, std::vector<uint32_t>& nz,
                       std::vector<uint8_t>& bits);

int check_meta(const vlp_meta* m);
// Bound words per record (R17) and query words.
inline size_t record_words(const vlp_meta& m) {
  return m.mode == VLP_MODE_INTV ? 2 * m.d : (m.mode == VLP_MODE_COV ? m.d : 1);
}
inline size_t query_words(const vlp_meta& m) { return m.mode == VLP_MODE_IDM ? 1 : m.d; }

}  // namespace vlp

struct vlp_sk {
  uint32_t s[vlp::n];
  uint32_t z[vlp::N];
  vlp_params params;
};

struct vlp_evk {
  std::vector<uint32_t> bsk;  // [n][6][2][N] torus32
  std::vector<uint32_t> ksk;  // [N][8][3][632] torus32 (631 used, pad 0)
  vlp_params params;
};

struct vlp_pk {
  vlp_meta meta;
  size_t first = 0, count = 0;
  std::vector<uint32_t> samples;  // [count][W*l_I + l_S][632] TLWE(0) samples (alg:PubKeyGen)
  bool used = false;              // single-use (ServerEnc consumes them)
};

namespace vlp {

// Per-program job descriptors (device layout; see kernels.cu)
struct BrJob {       // one blind rotation: input c = k0 + ax*x + ay*y (linear form, S2)
  uint32_t x, y;     // slot ids (region << 28 | row)
  uint32_t k0;       // constant added to b
  int8_t ax, ay;     // coefficients
  uint16_t tv;       // test vector: 0 -> mu = 1/8 (R8); 1 -> mu = 1/4 (R24 linear aggregation)
  uint32_t out;      // N-LWE row
};
struct KsJob {       // one key switch of nlwe[n0] (+ nlwe[n1] + (0, add) for MUX, S7)
  uint32_t n0, n1;   // n1 = 0xFFFFFFFF if none
  uint32_t add;      // added to b' before switching
  uint32_t out;      // slot id
};
static_assert(sizeof(BrJob) == 20, "BrJob layout");
static_assert(sizeof(KsJob) == 16, "KsJob layout");

enum Region : uint32_t { kRegIn0 = 0, kRegIn1 = 1, kRegMid = 2, kRegOut = 3 };
inline uint32_t slot(uint32_t region, uint32_t row) { return (region << 28) | row; }

struct LinJob {      // R24: out slot = sum of `count` input slots (mod 2^32, no bootstrap), after the level's KS
  uint32_t out, first, count, pad;  // first: index into the level's lin_in
};
static_assert(sizeof(LinJob) == 16, "LinJob layout");

struct Level {
  std::vector<BrJob> br;
  std::vector<KsJob> ks;
  std::vector<LinJob> lin;
  std::vector<uint32_t> lin_in;  // input slot ids of the level's linear jobs
};

// Circuit compiler output (sched.cpp)
struct Schedule {
  std::vector<Level> levels;
  uint64_t mid_rows = 0;      // intermediate TLWE rows (region kRegMid), rows 0,1 = trivial 0 / 1
  uint64_t nlwe_rows = 0;     // N-LWE staging rows
  uint64_t in0_cts = 0, in1_cts = 0, out_cts = 0;
  uint64_t gates = 0, br = 0, ks = 0;
  std::vector<uint32_t> out_slots;  // final results copied to out (if not already in kRegOut)
  std::vector<uint64_t> v_rows;     // per record: validation bit row (kRegMid), for parity dumps
  std::vector<uint64_t> mask_rows;  // per record * l_S: masked payload rows
  uint32_t l_S = 0;
};

int compile_velopir(const vlp_meta& meta, size_t first, size_t count, Schedule* out, uint32_t nq = 1);
int compile_gates(int op, size_t count, Schedule* out);
int compile_combine(const vlp_meta& meta, uint32_t G, Schedule* out);

// Host-side twiddle tables and constants for the device NTT (kernels.cu).
constexpr uint32_t kP = 0x3fff7801u;  // NTT prime, p = 1 mod 2048, 4p < 2^32

}  // namespace vlp
