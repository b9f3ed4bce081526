/*
 * oracle/tfhe_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the TFHE gate bootstrapping that VeLoPIR
 * (arXiv 2506.12761) evaluates its circuits with.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` leg may load it.  It shares no code, header, table or constant
 * generator with the CUDA product path (paper_2506_12761_b200/); neither side imports the other.
 *
 * Citation key: P:n = /root/reference/PAPER.md line n (LaTeX section / algorithm named beside it);
 * S:n = SPEC.md line n; Rk = reading k in DESIGN.md section 3 (where the paper is silent).
 *
 * Everything here is exact integer arithmetic: torus values are uint32_t (mod 2^32, R1); polynomial
 * products in Z[X]/(X^N+1) are computed exactly (a textbook negacyclic NTT over the 62-bit prime Q, whose
 * result is lifted back to Z and reduced mod 2^32 -- the "library primitive" step; pinned against
 * the schoolbook definition in tests/test_oracle_pins.py).  The only floating point is the Box-Muller
 * Gaussian used at key generation / encryption time (R3).
 *
 * Parity pins: see tests/test_oracle_pins.py.  Ciphertext bytes themselves are "parity unpinned" by the
 * paper (no printed ciphertexts, P9 in DESIGN.md): they are pinned by closed forms (trivial-input
 * bootstrap), truth tables, noise statistics and decrypted predicates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------------
 * Parameters: tab:tfhe_params: n = 630, N = 1024, k = 1, log2 Bg = 7, l = 3,
 * KS base 2^2, t = 8, sigma_KS = 2^-15, sigma_BK = 2^-25.
 * ------------------------------------------------------------------------------------------------ */
#define ON 630  /* TLWE dimension n */
#define ONR 1024 /* ring dimension N */
#define OBG_BITS 7 /* log2 Bg */
#define OELL 3   /* decomposition length l */
#define OKS_BITS 2 /* log2 KS base */
#define OKS_T 8  /* KS length t */
#define OROWS 6  /* (k+1) * l TRGSW rows */

typedef uint32_t torus32;

int oracle_dims(int* n, int* N) {
  *n = ON;
  *N = ONR;
  return 0;
}

/* ------------------------------------------------------------------------------------------------
 * Counter-based PRNG (R3; DESIGN.md section 3 "PRNG").  H(seed, domain, object, word) -> u64.
 * ------------------------------------------------------------------------------------------------ */
static uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t oracle_prng(uint64_t seed, uint64_t domain, uint64_t object, uint64_t word) {
  uint64_t x = mix64(seed ^ (domain * 0x9E3779B97F4A7C15ull));
  x = mix64(x ^ (object * 0xC2B2AE3D27D4EB4Full));
  x = mix64(x ^ (word * 0x165667B19E3779F9ull));
  return x;
}

/* Domains. */
enum {
  D_SK_LWE = 1, D_SK_RING = 2, D_BSK_A = 3, D_BSK_E = 4, D_KSK_A = 5, D_KSK_E = 6,
  D_PK_A = 7, D_PK_E = 8, D_QRY_A = 9, D_QRY_E = 10, D_FRESH_A = 12, D_FRESH_E = 13
};

/* Uniform torus element: the high 32 bits of one PRNG word. */
static torus32 uniform_torus(uint64_t seed, uint64_t dom, uint64_t obj, uint64_t word) {
  return (torus32)(oracle_prng(seed, dom, obj, word) >> 32);
}

/* Gaussian N(0, sigma) on the torus, P:128 ("e is a noise term drawn from a Gaussian distribution
 * N(0, sigma)"), R2/R3: one Box-Muller sample from words (2t, 2t+1), scaled by sigma*2^32 and rounded
 * half away from zero (llround), reduced mod 2^32. */
int32_t oracle_gaussian(uint64_t seed, uint64_t dom, uint64_t obj, uint64_t t, double sigma) {
  uint64_t w1 = oracle_prng(seed, dom, obj, 2 * t);
  uint64_t w2 = oracle_prng(seed, dom, obj, 2 * t + 1);
  double u1 = ((double)(w1 >> 11) + 1.0) * 0x1p-53; /* (0, 1] */
  double u2 = (double)(w2 >> 11) * 0x1p-53;         /* [0, 1) */
  double z = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
  long long e = llround(z * (sigma * 4294967296.0));
  return (int32_t)(uint32_t)(uint64_t)e;
}

/* Ecd: m -> m/4 - 1/8: 1 -> +1/8 = 0x20000000, 0 -> -1/8 = 0xE0000000. */
torus32 oracle_ecd(int m) { return m ? 0x20000000u : 0xE0000000u; }

/* ------------------------------------------------------------------------------------------------
 * Exact negacyclic polynomial products in Z[X]/(X^N + 1).
 * Definition (schoolbook): c_k = sum_{i+j=k} a_i b_j - sum_{i+j=k+N} a_i b_j.
 * ------------------------------------------------------------------------------------------------ */

/* Schoolbook product mod 2^32, any N (used by the pins, and as the definition). */
void oracle_negacyclic_schoolbook(const uint32_t* a, const uint32_t* b, uint32_t* c, int n) {
  for (int k = 0; k < n; k++) c[k] = 0;
  for (int i = 0; i < n; i++)
    for (int j = 0; j < n; j++) {
      uint32_t prod = a[i] * b[j];
      if (i + j < n)
        c[i + j] += prod;
      else
        c[i + j - n] -= prod;
    }
}

/* Textbook NTT over Q = 0x3fffffffffffa801 (prime, Q = 1 mod 2048), N = 1024.  Exact as long as the
 * true integer coefficients lie in (-Q/2, Q/2); every use below stays below 2^50. */
static const uint64_t Q = 0x3fffffffffffa801ull;
static uint64_t g_psi, g_psi_inv, g_n_inv;
static uint64_t g_psi_pow[ONR], g_psi_inv_pow[ONR];
static int g_ntt_ready = 0;

/* a*b mod Q by Barrett reduction (Handbook of Applied Cryptography, Alg. 14.42, base 2, k = 62):
 * q = floor(floor(x / 2^60) * floor(2^124 / Q) / 2^64), r = x - q*Q < 3Q, then at most two subtractions.
 * Identical to ((unsigned __int128)a*b) % Q, only faster (a library-primitive speed-up; pinned by
 * tests/test_oracle_pins.py::test_mulq_matches_modulo). */
static const unsigned __int128 BARRETT_MU = (((unsigned __int128)1) << 124) / 0x3fffffffffffa801ull;
static uint64_t mulq(uint64_t a, uint64_t b) {
  unsigned __int128 x = (unsigned __int128)a * b;
  uint64_t q1 = (uint64_t)(x >> 60);
  uint64_t q3 = (uint64_t)(((unsigned __int128)q1 * (uint64_t)BARRETT_MU) >> 64);
  uint64_t r = (uint64_t)(x - (unsigned __int128)q3 * Q);
  while (r >= Q) r -= Q;
  return r;
}

uint64_t oracle_mulq(uint64_t a, uint64_t b) { return mulq(a, b); }
uint64_t oracle_modulus(void) { return Q; }
static uint64_t addq(uint64_t a, uint64_t b) { uint64_t s = a + b; return s >= Q ? s - Q : s; }
static uint64_t subq(uint64_t a, uint64_t b) { return a >= b ? a - b : a + Q - b; }
static uint64_t powq(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r = mulq(r, b);
    b = mulq(b, b);
    e >>= 1;
  }
  return r;
}

static void ntt_init(void) {
  if (g_ntt_ready) return;
  /* psi: a primitive 2N-th root of unity (psi^N = -1). */
  for (uint64_t g = 2;; g++) {
    uint64_t x = powq(g, (Q - 1) / (2 * ONR));
    if (powq(x, ONR) == Q - 1) {
      g_psi = x;
      break;
    }
  }
  g_psi_inv = powq(g_psi, Q - 2);
  g_n_inv = powq(ONR, Q - 2);
  g_psi_pow[0] = 1;
  g_psi_inv_pow[0] = 1;
  for (int j = 1; j < ONR; j++) {
    g_psi_pow[j] = mulq(g_psi_pow[j - 1], g_psi);
    g_psi_inv_pow[j] = mulq(g_psi_inv_pow[j - 1], g_psi_inv);
  }
  g_ntt_ready = 1;
}

/* Cyclic length-N NTT (bit-reversal permutation, then iterative radix-2 butterflies), root omega. */
static void ntt_cyclic(uint64_t* a, uint64_t omega) {
  for (int i = 1, j = 0; i < ONR; i++) {
    int bit = ONR >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      uint64_t t = a[i];
      a[i] = a[j];
      a[j] = t;
    }
  }
  for (int len = 2; len <= ONR; len <<= 1) {
    uint64_t wlen = powq(omega, ONR / len);
    for (int i = 0; i < ONR; i += len) {
      uint64_t w = 1;
      for (int k = 0; k < len / 2; k++) {
        uint64_t u = a[i + k], v = mulq(a[i + k + len / 2], w);
        a[i + k] = addq(u, v);
        a[i + k + len / 2] = subq(u, v);
        w = mulq(w, wlen);
      }
    }
  }
}

/* Negacyclic forward transform of a signed integer polynomial: twist by psi^j, cyclic NTT with psi^2. */
static void nega_forward(const int64_t* a, uint64_t* out) {
  ntt_init();
  for (int j = 0; j < ONR; j++) {
    int64_t v = a[j];
    uint64_t r = v >= 0 ? (uint64_t)v % Q : Q - ((uint64_t)(-v) % Q);
    if (r == Q) r = 0;
    out[j] = mulq(r, g_psi_pow[j]);
  }
  ntt_cyclic(out, mulq(g_psi, g_psi));
}

/* Inverse: cyclic NTT with psi^-2, times N^-1 psi^-j; centered lift to (-Q/2, Q/2]; reduce mod 2^32. */
static void nega_inverse_to_torus(uint64_t* A, uint32_t* out) {
  ntt_cyclic(A, mulq(g_psi_inv, g_psi_inv));
  for (int j = 0; j < ONR; j++) {
    uint64_t v = mulq(mulq(A[j], g_n_inv), g_psi_inv_pow[j]);
    int64_t s = v > Q / 2 ? -(int64_t)(Q - v) : (int64_t)v;
    out[j] = (uint32_t)(uint64_t)s;
  }
}

/* Signed lift of a torus32 value to [-2^31, 2^31). */
static int64_t lift32(uint32_t x) { return (int64_t)(int32_t)x; }

/* sum_t a_t * b_t in Z[X]/(X^N+1), reduced mod 2^32, N = 1024; a_t, b_t signed integer polynomials
 * (torus32 inputs lifted to [-2^31, 2^31)).  Exact for sum |a||b| N < Q/2. */
void oracle_negacyclic_dot(int terms, const int64_t* a, const int64_t* b, uint32_t* out) {
  uint64_t* fa = malloc(sizeof(uint64_t) * ONR);
  uint64_t* fb = malloc(sizeof(uint64_t) * ONR);
  uint64_t* acc = calloc(ONR, sizeof(uint64_t));
  for (int t = 0; t < terms; t++) {
    nega_forward(a + (size_t)t * ONR, fa);
    nega_forward(b + (size_t)t * ONR, fb);
    for (int j = 0; j < ONR; j++) acc[j] = addq(acc[j], mulq(fa[j], fb[j]));
  }
  nega_inverse_to_torus(acc, out);
  free(fa);
  free(fb);
  free(acc);
}

/* Product of a torus32 polynomial a (lifted to [-2^31, 2^31)) with a small polynomial b (lifted the same
 * way), mod 2^32.  Exact when sum |a_i||b_j| < Q/2, e.g. b binary (the ring key z: a*z, |.| < 2^41). */
void oracle_negacyclic_mul(const uint32_t* a, const uint32_t* b, uint32_t* c) {
  int64_t* la = malloc(sizeof(int64_t) * ONR);
  int64_t* lb = malloc(sizeof(int64_t) * ONR);
  for (int j = 0; j < ONR; j++) {
    la[j] = lift32(a[j]);
    lb[j] = lift32(b[j]);
  }
  oracle_negacyclic_dot(1, la, lb, c);
  free(la);
  free(lb);
}

/* X^e * p in T[X]/(X^N+1), e in [0, 2N): coefficient k moves to k+e, negated when it wraps past N. */
static void poly_mul_monomial(const uint32_t* p, int e, uint32_t* out) {
  for (int k = 0; k < ONR; k++) {
    int pos = (k + e) % (2 * ONR);
    uint32_t v = p[k];
    if (pos >= ONR) {
      pos -= ONR;
      v = (uint32_t)(0u - v);
    }
    out[pos] = v;
  }
}

/* ------------------------------------------------------------------------------------------------
 * Decompositions and roundings (R5, R6, R7).
 * ------------------------------------------------------------------------------------------------ */

/* Gadget decomposition (R5): x ~ sum_{j=1..3} d_j 2^(32-7j), d_j in [-64, 64), rounding x to the nearest
 * multiple of 2^11 (half up).  Written as the definition: round, then balanced base-2^7 digits from the
 * least significant up, carrying when a digit is >= 64. */
void oracle_gadget_digits(uint32_t x, int32_t* d /* [3], d[0] <-> 2^25 */) {
  uint32_t r = (x + (1u << 10)) >> 11; /* x / 2^11 rounded half up, 21 bits (mod 2^21) */
  r &= (1u << 21) - 1;
  int carry = 0;
  for (int j = OELL - 1; j >= 0; j--) { /* j = 2 <-> 2^11 (least significant) */
    int v = (int)((r >> (7 * (OELL - 1 - j))) & 127) + carry;
    if (v >= 64) {
      v -= 128;
      carry = 1;
    } else {
      carry = 0;
    }
    d[j] = v;
  }
  /* A carry out of the top digit is a multiple of 2^32: dropped (torus). */
}

/* KS digits (R6): abar = floor((a + 2^15) / 2^16) mod 2^16, 8 unsigned base-4 digits, most significant
 * first: d_j = (abar >> (14 - 2j)) & 3, so that a ~ sum_j d_j 4^-(j+1). */
void oracle_ks_digits(uint32_t x, int32_t* d /* [8] */) {
  uint32_t abar = ((x + (1u << 15)) >> 16) & 0xFFFF;
  for (int j = 0; j < OKS_T; j++) d[j] = (int32_t)((abar >> (14 - 2 * j)) & 3);
}

/* Mod-switch (R7): round(x * 2N / 2^32) mod 2N, half up. */
int oracle_modswitch(uint32_t x) { return (int)(((x + (1u << 20)) >> 21) & (2 * ONR - 1)); }

/* ------------------------------------------------------------------------------------------------
 * Keys.  P:127 (KeyGen); TRGSW / ksk layout R4, O7, O10 in DESIGN.md.
 * ------------------------------------------------------------------------------------------------ */
typedef struct {
  uint32_t s[ON];                  /* LWE key s in B^n */
  uint32_t z[ONR];                 /* ring key z in B[X] (R4) */
  uint32_t* bsk;                   /* [ON][OROWS][2][ONR] torus32 TRGSW rows */
  uint64_t* bsk_hat;               /* same rows lifted to signed and transformed (nega_forward): a
                                      memo of the exact product's transform of each fixed key row */
  uint32_t* ksk;                   /* [ONR][OKS_T][3][ON+1] TLWE samples (v = 1..3) */
  uint64_t seed;
} oracle_keys;

static size_t bsk_index(int i, int r, int c) { return (((size_t)i * OROWS + r) * 2 + c) * ONR; }
static size_t ksk_index(int i, int j, int v /* 1..3 */) {
  return (((size_t)i * OKS_T + j) * 3 + (v - 1)) * (ON + 1);
}

/* TLWE encryption: a uniform (domain dom_a, object obj, words 0..n-1), e Gaussian (dom_e, obj,
 * pair 0), b = <a, s> + mu + e. */
static void tlwe_encrypt_raw(const uint32_t* s, torus32 mu, double sigma, uint64_t seed, uint64_t dom_a,
                             uint64_t dom_e, uint64_t obj, uint32_t* ct) {
  uint32_t b = 0;
  for (int i = 0; i < ON; i++) {
    ct[i] = uniform_torus(seed, dom_a, obj, i);
    b += ct[i] * s[i];
  }
  b += mu;
  b += (uint32_t)oracle_gaussian(seed, dom_e, obj, 0, sigma);
  ct[ON] = b;
}

/* KeyGen with explicit sigmas (the pins use sigma = 0 keys). */
oracle_keys* oracle_keygen(uint64_t seed, double sigma_bk, double sigma_ks) {
  oracle_keys* k = calloc(1, sizeof(oracle_keys));
  k->seed = seed;
  for (int i = 0; i < ON; i++) k->s[i] = (uint32_t)(oracle_prng(seed, D_SK_LWE, 0, i) >> 63);
  for (int j = 0; j < ONR; j++) k->z[j] = (uint32_t)(oracle_prng(seed, D_SK_RING, 0, j) >> 63);

  /* bsk_i, row r = u*3 + j (O7): TRLWE_z(0) + s_i * g_j on component u's constant coefficient,
   * g_j = 2^(32 - 7(j+1)). TRLWE_z(0) = (a, a*z + e), a uniform, e ~ N(0, sigma_bk). */
  k->bsk = malloc(sizeof(uint32_t) * (size_t)ON * OROWS * 2 * ONR);
  uint32_t* az = malloc(sizeof(uint32_t) * ONR);
  for (int i = 0; i < ON; i++) {
    for (int r = 0; r < OROWS; r++) {
      uint64_t obj = (uint64_t)i * OROWS + r;
      uint32_t* a = k->bsk + bsk_index(i, r, 0);
      uint32_t* b = k->bsk + bsk_index(i, r, 1);
      for (int j = 0; j < ONR; j++) a[j] = uniform_torus(seed, D_BSK_A, obj, j);
      oracle_negacyclic_mul(a, k->z, az);
      for (int j = 0; j < ONR; j++) b[j] = az[j] + (uint32_t)oracle_gaussian(seed, D_BSK_E, obj, j, sigma_bk);
      int u = r / OELL, jj = r % OELL;
      if (k->s[i]) (u == 0 ? a : b)[0] += 1u << (32 - OBG_BITS * (jj + 1));
    }
  }
  free(az);
  k->bsk_hat = malloc(sizeof(uint64_t) * (size_t)ON * OROWS * 2 * ONR);
  int64_t* lifted = malloc(sizeof(int64_t) * ONR);
  for (size_t row = 0; row < (size_t)ON * OROWS * 2; row++) {
    for (int j = 0; j < ONR; j++) lifted[j] = lift32(k->bsk[row * ONR + j]);
    nega_forward(lifted, k->bsk_hat + row * ONR);
  }
  free(lifted);

  /* ksk[i][j][v] = TLWE_s(v * z_i * 2^(32 - 2(j+1))), sigma_ks (O10). */
  k->ksk = malloc(sizeof(uint32_t) * (size_t)ONR * OKS_T * 3 * (ON + 1));
  for (int i = 0; i < ONR; i++)
    for (int j = 0; j < OKS_T; j++)
      for (int v = 1; v <= 3; v++) {
        uint64_t obj = ((uint64_t)i * OKS_T + j) * 3 + (v - 1);
        torus32 mu = (uint32_t)v * k->z[i] * (1u << (32 - OKS_BITS * (j + 1)));
        tlwe_encrypt_raw(k->s, mu, sigma_ks, seed, D_KSK_A, D_KSK_E, obj, k->ksk + ksk_index(i, j, v));
      }
  return k;
}

void oracle_free_keys(oracle_keys* k) {
  if (!k) return;
  free(k->bsk);
  free(k->bsk_hat);
  free(k->ksk);
  free(k);
}

void oracle_export_keys(const oracle_keys* k, uint32_t* s, uint32_t* z, uint32_t* bsk, uint32_t* ksk) {
  if (s) memcpy(s, k->s, sizeof(k->s));
  if (z) memcpy(z, k->z, sizeof(k->z));
  if (bsk) memcpy(bsk, k->bsk, sizeof(uint32_t) * (size_t)ON * OROWS * 2 * ONR);
  if (ksk) memcpy(ksk, k->ksk, sizeof(uint32_t) * (size_t)ONR * OKS_T * 3 * (ON + 1));
}

/* ------------------------------------------------------------------------------------------------
 * TLWE encrypt / phase / decrypt.
 * ------------------------------------------------------------------------------------------------ */
/* Domain pairs: 0 = fresh (tests / NAND sweep), 1 = query, 2 = public key (alg:PubKeyGen). */
void oracle_encrypt(const oracle_keys* k, int m, uint64_t seed, int kind, uint64_t obj, double sigma,
                    uint32_t* ct) {
  uint64_t da = kind == 1 ? D_QRY_A : kind == 2 ? D_PK_A : D_FRESH_A;
  uint64_t de = kind == 1 ? D_QRY_E : kind == 2 ? D_PK_E : D_FRESH_E;
  tlwe_encrypt_raw(k->s, kind == 2 ? 0u : oracle_ecd(m), sigma, seed, da, de, obj, ct);
}

uint32_t oracle_phase(const oracle_keys* k, const uint32_t* ct) {
  uint32_t d = 0;
  for (int i = 0; i < ON; i++) d += ct[i] * k->s[i];
  return ct[ON] - d;
}

/* Dec: nearest of {-1/8, +1/8}; ties (phase 0 or 1/2) -> 0 (R18): bit = [int32(phase) > 0]. */
int oracle_decrypt(const oracle_keys* k, const uint32_t* ct) { return (int32_t)oracle_phase(k, ct) > 0; }

/* TRLWE phase b - a*z (O6), for the external-product pin. */
void oracle_trlwe_phase(const oracle_keys* k, const uint32_t* trlwe /* [2][N] */, uint32_t* out) {
  uint32_t* az = malloc(sizeof(uint32_t) * ONR);
  oracle_negacyclic_mul(trlwe, k->z, az);
  for (int j = 0; j < ONR; j++) out[j] = trlwe[ONR + j] - az[j];
  free(az);
}

/* ------------------------------------------------------------------------------------------------
 * Bootstrapping: BlindRotate -> SampleExtract -> KeySwitch.
 * ------------------------------------------------------------------------------------------------ */

/* External product (O8): D = (D_a, D_b); decompose each component into 3 digit polynomials (u-major,
 * j ascending: row r = u*3 + j); result component c = sum_r dec_r * row_r[c] exactly, mod 2^32. */
void oracle_external_product(const oracle_keys* k, int i, const uint32_t* D /* [2][N] */,
                             uint32_t* out /* [2][N] */) {
  int64_t* dec = malloc(sizeof(int64_t) * ONR);
  uint64_t* dec_hat = malloc(sizeof(uint64_t) * OROWS * ONR);
  uint64_t* acc = malloc(sizeof(uint64_t) * ONR);
  for (int u = 0; u < 2; u++)
    for (int j = 0; j < OELL; j++) {
      for (int x = 0; x < ONR; x++) {
        int32_t d[OELL];
        oracle_gadget_digits(D[u * ONR + x], d);
        dec[x] = d[j];
      }
      nega_forward(dec, dec_hat + (size_t)(u * OELL + j) * ONR); /* row r = u*3 + j */
    }
  /* component c: sum_r dec_r * row_r[c], the sum taken in the transform domain (linearity), one inverse:
   * |coefficients| <= 6 * 1024 * 64 * 2^31 < 2^50 < Q/2, so the result is exact. */
  for (int c = 0; c < 2; c++) {
    for (int x = 0; x < ONR; x++) acc[x] = 0;
    for (int r = 0; r < OROWS; r++) {
      const uint64_t* row_hat = k->bsk_hat + bsk_index(i, r, c);
      for (int x = 0; x < ONR; x++) acc[x] = addq(acc[x], mulq(dec_hat[(size_t)r * ONR + x], row_hat[x]));
    }
    nega_inverse_to_torus(acc, out + c * ONR);
  }
  free(dec);
  free(dec_hat);
  free(acc);
}

/* BlindRotate (O9): acc = (0, X^{-bbar} testv), testv = mu in every coefficient -- mu = 1/8 for
 * every gate of the paper (R8); mu = 1/4 only for the R24 linear-aggregation bootstraps (not in the paper);
 * for i = 0..n-1: if abar_i != 0: acc += ExtProd(bsk_i, X^{abar_i} acc - acc).  Works on an
 * already-formed TLWE input c (gate linear form applied by the caller). Output: the TRLWE acc. */
void oracle_blind_rotate_mu(const oracle_keys* k, const uint32_t* c /* [n+1] */, int steps, uint32_t mu,
                            uint32_t* acc /* [2][N] */) {
  uint32_t* testv = malloc(sizeof(uint32_t) * ONR);
  uint32_t* rot = malloc(sizeof(uint32_t) * 2 * ONR);
  uint32_t* ep = malloc(sizeof(uint32_t) * 2 * ONR);
  for (int j = 0; j < ONR; j++) testv[j] = mu;
  int bbar = oracle_modswitch(c[ON]);
  memset(acc, 0, sizeof(uint32_t) * ONR);
  poly_mul_monomial(testv, (2 * ONR - bbar) % (2 * ONR), acc + ONR);
  for (int i = 0; i < steps; i++) {
    int abar = oracle_modswitch(c[i]);
    if (abar == 0) continue;
    for (int u = 0; u < 2; u++) {
      poly_mul_monomial(acc + u * ONR, abar, rot + u * ONR);
      for (int j = 0; j < ONR; j++) rot[u * ONR + j] -= acc[u * ONR + j];
    }
    oracle_external_product(k, i, rot, ep);
    for (int j = 0; j < 2 * ONR; j++) acc[j] += ep[j];
  }
  free(testv);
  free(rot);
  free(ep);
}

void oracle_blind_rotate(const oracle_keys* k, const uint32_t* c, int steps, uint32_t* acc) {
  oracle_blind_rotate_mu(k, c, steps, 0x20000000u, acc);
}

/* SampleExtract (S6): a'_0 = a_0, a'_j = -a_{N-j} (j >= 1), b' = b_0. */
void oracle_sample_extract(const uint32_t* acc, uint32_t* nlwe /* [N+1] */) {
  nlwe[0] = acc[0];
  for (int j = 1; j < ONR; j++) nlwe[j] = (uint32_t)(0u - acc[ONR - j]);
  nlwe[ONR] = acc[ONR];
}

/* KeySwitch (S8, O10): out = (0, b') - sum_{i,j: d_ij != 0} ksk[i][j][d_ij]. */
void oracle_keyswitch(const oracle_keys* k, const uint32_t* nlwe, uint32_t* out /* [n+1] */) {
  memset(out, 0, sizeof(uint32_t) * (ON + 1));
  out[ON] = nlwe[ONR];
  for (int i = 0; i < ONR; i++) {
    int32_t d[OKS_T];
    oracle_ks_digits(nlwe[i], d);
    for (int j = 0; j < OKS_T; j++) {
      if (d[j] == 0) continue;
      const uint32_t* row = k->ksk + ksk_index(i, j, d[j]);
      for (int x = 0; x <= ON; x++) out[x] -= row[x];
    }
  }
}

/* Blind rotate the full n steps and extract: the N-dimensional "BR" output (used by MUX). */
void oracle_bootstrap_nlwe(const oracle_keys* k, const uint32_t* c, uint32_t* nlwe) {
  uint32_t* acc = malloc(sizeof(uint32_t) * 2 * ONR);
  oracle_blind_rotate(k, c, ON, acc);
  oracle_sample_extract(acc, nlwe);
  free(acc);
}

/* R24: BlindRotate with test vector mu -> SampleExtract -> KeySwitch. */
void oracle_bootstrap_mu(const oracle_keys* k, const uint32_t* c, uint32_t mu, uint32_t* out) {
  uint32_t* acc = malloc(sizeof(uint32_t) * 2 * ONR);
  uint32_t* nlwe = malloc(sizeof(uint32_t) * (ONR + 1));
  oracle_blind_rotate_mu(k, c, ON, mu, acc);
  oracle_sample_extract(acc, nlwe);
  oracle_keyswitch(k, nlwe, out);
  free(acc);
  free(nlwe);
}

/* Bootstrap = BlindRotate -> SampleExtract -> KeySwitch. */
void oracle_bootstrap(const oracle_keys* k, const uint32_t* c, uint32_t* out) {
  uint32_t* nlwe = malloc(sizeof(uint32_t) * (ONR + 1));
  oracle_bootstrap_nlwe(k, c, nlwe);
  oracle_keyswitch(k, nlwe, out);
  free(nlwe);
}

/* ------------------------------------------------------------------------------------------------
 * Gates.  HomAND = Bootstrap((0, -1/8) + ct1 + ct2); the others per R10 / S2:
 *   op 0 AND  (-1/8,  1,  1)   op 1 NAND ( 1/8, -1, -1)   op 2 OR  ( 1/8, 1, 1)
 *   op 3 XOR  ( 1/4,  2,  2)   op 4 XNOR (-1/4, -2, -2)
 * ------------------------------------------------------------------------------------------------ */
static void linear_form(int op, const uint32_t* x, const uint32_t* y, uint32_t* c) {
  uint32_t k0;
  int32_t ax, ay;
  switch (op) {
    case 0: k0 = 0xE0000000u; ax = 1; ay = 1; break;
    case 1: k0 = 0x20000000u; ax = -1; ay = -1; break;
    case 2: k0 = 0x20000000u; ax = 1; ay = 1; break;
    case 3: k0 = 0x40000000u; ax = 2; ay = 2; break;
    default: k0 = 0xC0000000u; ax = -2; ay = -2; break;
  }
  for (int i = 0; i <= ON; i++) c[i] = (uint32_t)ax * x[i] + (uint32_t)ay * y[i];
  c[ON] += k0;
}

void oracle_gate(const oracle_keys* k, int op, const uint32_t* x, const uint32_t* y, uint32_t* out) {
  uint32_t c[ON + 1];
  linear_form(op, x, y, c);
  oracle_bootstrap(k, c, out);
}

/* HomMUX(c, a, b) = c ? a : b, R10:
 * KS( (0, 1/8) + BR_N((0,-1/8) + c + a) + BR_N((0,-1/8) - c + b) ). */
void oracle_mux(const oracle_keys* k, const uint32_t* c, const uint32_t* a, const uint32_t* b, uint32_t* out) {
  uint32_t t[ON + 1];
  uint32_t* u1 = malloc(sizeof(uint32_t) * (ONR + 1));
  uint32_t* u2 = malloc(sizeof(uint32_t) * (ONR + 1));
  for (int i = 0; i <= ON; i++) t[i] = c[i] + a[i];
  t[ON] += 0xE0000000u;
  oracle_bootstrap_nlwe(k, t, u1);
  for (int i = 0; i <= ON; i++) t[i] = b[i] - c[i];
  t[ON] += 0xE0000000u;
  oracle_bootstrap_nlwe(k, t, u2);
  for (int i = 0; i <= ONR; i++) u1[i] += u2[i];
  u1[ONR] += 0x20000000u;
  oracle_keyswitch(k, u1, out);
  free(u1);
  free(u2);
}
