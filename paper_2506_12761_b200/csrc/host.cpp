// host.cpp -- client-side and preprocessing calls of the C ABI (include/vlp.h): parameters, KeyGen,
// TLWE encryption / decryption, PubKeyGen, ServerEnc.  Host C++.  The seeded calls are deterministic in their
// 64-bit seed (R3: reproducible test / benchmark mode, not secret); the *_secure calls draw a fresh 256-bit key
// from the OS (getrandom) and use ChaCha20 as the counter generator.
//
// Independent of the test oracle (oracle/): same published conventions, separate
// code.  The ring products a*z of KeyGen are computed here as sums of rotations X^j * a over the
// support of the binary key z (the oracle uses an NTT), and are exact mod 2^32.
#include <sys/random.h>

#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <thread>

#include "vlp_internal.h"

namespace vlp {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

// splitmix64 finalizer of (x + golden gamma); H = mix(mix(mix(seed ^ dom*C1) ^ obj*C2) ^ word*C3)
static inline uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
uint64_t prng(uint64_t seed, uint64_t dom, uint64_t obj, uint64_t word) {
  uint64_t h = mix(seed ^ (dom * 0x9E3779B97F4A7C15ull));
  h = mix(h ^ (obj * 0xC2B2AE3D27D4EB4Full));
  return mix(h ^ (word * 0x165667B19E3779F9ull));
}

// ---- ChaCha20 block function (RFC 8439 section 2.3): the keyed counter generator of the secure calls.
static inline uint32_t rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }
static inline void quarter(uint32_t* x, int a, int b, int c, int d) {
  x[a] += x[b]; x[d] = rotl32(x[d] ^ x[a], 16);
  x[c] += x[d]; x[b] = rotl32(x[b] ^ x[c], 12);
  x[a] += x[b]; x[d] = rotl32(x[d] ^ x[a], 8);
  x[c] += x[d]; x[b] = rotl32(x[b] ^ x[c], 7);
}
void chacha20_block(const uint32_t key[8], uint32_t counter, const uint32_t nonce[3], uint32_t out[16]) {
  uint32_t in[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u, key[0], key[1], key[2], key[3],
                     key[4], key[5], key[6], key[7], counter, nonce[0], nonce[1], nonce[2]};
  uint32_t x[16];
  std::memcpy(x, in, sizeof(x));
  for (int i = 0; i < 10; i++) {
    quarter(x, 0, 4, 8, 12); quarter(x, 1, 5, 9, 13); quarter(x, 2, 6, 10, 14); quarter(x, 3, 7, 11, 15);
    quarter(x, 0, 5, 10, 15); quarter(x, 1, 6, 11, 12); quarter(x, 2, 7, 8, 13); quarter(x, 3, 4, 9, 14);
  }
  for (int i = 0; i < 16; i++) out[i] = x[i] + in[i];
}

Rng seeded(uint64_t seed) {
  Rng r;
  r.seed = seed;
  return r;
}

uint64_t Rng::u64(uint64_t dom, uint64_t obj, uint64_t word) const {
  if (!secure) return prng(seed, dom, obj, word);
  const uint32_t nonce[3] = {static_cast<uint32_t>(dom), static_cast<uint32_t>(obj), static_cast<uint32_t>(obj >> 32)};
  uint32_t blk[16];
  chacha20_block(key, static_cast<uint32_t>(word >> 3), nonce, blk);
  const int w = static_cast<int>(word & 7);
  return static_cast<uint64_t>(blk[2 * w]) | (static_cast<uint64_t>(blk[2 * w + 1]) << 32);
}

Rng::~Rng() {  // the key does not outlive the call
  volatile uint32_t* k = key;
  for (int i = 0; i < 8; i++) k[i] = 0;
}

// vlp_debug_next_secure_key: a key the calling thread's next secure call takes instead of getrandom (tests only)
static thread_local bool g_next_key_set = false;
static thread_local uint32_t g_next_key[8];

int os_random(Rng* r) {
  r->secure = true;
  if (g_next_key_set) {
    std::memcpy(r->key, g_next_key, sizeof(r->key));
    volatile uint32_t* k = g_next_key;
    for (int i = 0; i < 8; i++) k[i] = 0;
    g_next_key_set = false;
    return VLP_OK;
  }
  size_t got = 0;
  uint8_t* dst = reinterpret_cast<uint8_t*>(r->key);
  while (got < sizeof(r->key)) {
    const ssize_t k = getrandom(dst + got, sizeof(r->key) - got, 0);
    if (k < 0) {
      if (errno == EINTR) continue;
      return fail(VLP_EINVAL, "getrandom failed: no OS randomness for a secure call");
    }
    got += static_cast<size_t>(k);
  }
  return VLP_OK;
}

// Box-Muller Gaussian, "N(0, sigma)" (R2, R3); scalar glibc libm, no FMA contraction.
uint32_t noise(const Rng& g, uint64_t dom, uint64_t obj, uint64_t t, double sigma) {
  const uint64_t w1 = g.u64(dom, obj, 2 * t), w2 = g.u64(dom, obj, 2 * t + 1);
  const double u1 = (static_cast<double>(w1 >> 11) + 1.0) * 0x1p-53;
  const double u2 = static_cast<double>(w2 >> 11) * 0x1p-53;
  const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  const long long e = std::llround(z * (sigma * 4294967296.0));
  return static_cast<uint32_t>(static_cast<uint64_t>(e));
}

static inline uint32_t uniform(const Rng& g, uint64_t dom, uint64_t obj, uint64_t word) {
  return static_cast<uint32_t>(g.u64(dom, obj, word) >> 32);
}

// TLWE sample: a_i uniform (dom_a, obj, word i), b = <a, s> + mu + e (dom_e, obj, pair 0).
static void tlwe_sample(const uint32_t* s, uint32_t mu, double sigma, const Rng& g, uint64_t dom_a,
                        uint64_t dom_e, uint64_t obj, uint32_t* ct) {
  uint32_t b = 0;
  for (int i = 0; i < n; i++) {
    ct[i] = uniform(g, dom_a, obj, i);
    b += ct[i] * s[i];
  }
  ct[n] = b + mu + noise(g, dom_e, obj, 0, sigma);
  ct[n + 1] = 0;
}

template <class F>
static void parallel_for(size_t count, F&& fn) {
  unsigned hw = std::thread::hardware_concurrency();
  size_t nt = std::max<size_t>(1, std::min<size_t>(hw ? hw : 4, (count + 63) / 64));
  if (nt == 1) {
    for (size_t i = 0; i < count; i++) fn(i);
    return;
  }
  std::vector<std::thread> th;
  for (size_t t = 0; t < nt; t++)
    th.emplace_back([&, t] {
      for (size_t i = t; i < count; i += nt) fn(i);
    });
  for (auto& x : th) x.join();
}

int check_meta(const vlp_meta* m) {
  if (!m) return fail(VLP_EINVAL, "meta is NULL");
  if (m->mode > VLP_MODE_IDM) return fail(VLP_EMODE, "unknown mode");
  if (m->l_I < 2 || m->l_I > 32 || m->l_S < 1 || m->l_S > 128)
    return fail(VLP_EWIDTH, "l_I must be in [2, 32] and l_S in [1, 128]");
  if (m->mode == VLP_MODE_IDM ? m->d != 1 : (m->d < 1 || m->d > 2)) return fail(VLP_EMODE, "bad d for mode");
  if (m->M < 1) return fail(VLP_EINVAL, "M must be >= 1");
  return VLP_OK;
}

int resolve_params(const vlp_params* params, vlp_params* p) {
  *p = vlp_params{630, 1024, 1, 7, 3, 2, 8, 0x1p-15, 0x1p-25, 0x1p-15};
  if (params) {
    if (params->n != 630 || params->N != 1024 || params->k != 1 || params->bg_bits != 7 || params->ell != 3 ||
        params->ks_base_bits != 2 || params->ks_t != 8)
      return fail(VLP_EINVAL, "only the 128-bit parameter set of tab:tfhe_params is supported");
    *p = *params;
  }
  return VLP_OK;
}

// Binary LWE key s and ring key z (O4): bit 63 of the generator.
void secret_keys(const Rng& g, vlp_sk* sk) {
  for (int i = 0; i < n; i++) sk->s[i] = static_cast<uint32_t>(g.u64(kSkLwe, 0, i) >> 63);
  for (int j = 0; j < N; j++) sk->z[j] = static_cast<uint32_t>(g.u64(kSkRing, 0, j) >> 63);
}

// Host half of vlp_keygen_device: every Gaussian noise word of the evaluation key, exactly the values vlp_keygen
// draws -- bsk row (i, r) coefficient j at [(i*6 + r)*N + j] (sigma_bk), ksk row idx at [idx] (sigma_ks).
void keygen_noise(const Rng& g, const vlp_params& p, uint32_t* bsk_noise, uint32_t* ksk_noise) {
  parallel_for(static_cast<size_t>(n) * kRows, [&](size_t ir) {
    for (int j = 0; j < N; j++) bsk_noise[ir * N + j] = noise(g, kBskE, ir, j, p.sigma_bk);
  });
  parallel_for(static_cast<size_t>(N) * kKsT * 3, [&](size_t idx) { ksk_noise[idx] = noise(g, kKskE, idx, 0, p.sigma_ks); });
}

uint64_t prng_prefix(uint64_t seed, uint64_t dom) { return mix(seed ^ (dom * 0x9E3779B97F4A7C15ull)); }

}  // namespace vlp

using namespace vlp;

extern "C" {

const char* vlp_last_error(void) { return g_err.c_str(); }

int vlp_params_tfhe128(vlp_params* p) {
  if (!p) return fail(VLP_EINVAL, "params is NULL");
  *p = vlp_params{630, 1024, 1, 7, 3, 2, 8, 0x1p-15, 0x1p-25, 0x1p-15};
  return VLP_OK;
}

static int keygen_impl(const Rng& g, const vlp_params* params, vlp_sk** sk_out, vlp_evk** evk_out) {
  if (!sk_out || !evk_out) return fail(VLP_EINVAL, "null output");
  vlp_params p;
  if (int rc = resolve_params(params, &p)) return rc;
  std::unique_ptr<vlp_sk> skp(new (std::nothrow) vlp_sk);
  std::unique_ptr<vlp_evk> evkp(new (std::nothrow) vlp_evk);
  if (!skp || !evkp) return fail(VLP_ENOMEM, "out of memory");
  vlp_sk* sk = skp.get();
  vlp_evk* evk = evkp.get();
  try {  // the key vectors (124 MB): no exception crosses the C ABI
    evk->bsk.assign(static_cast<size_t>(n) * kRows * 2 * N, 0);
    evk->ksk.assign(static_cast<size_t>(N) * kKsT * 3 * kCt, 0);
  } catch (const std::bad_alloc&) {
    return fail(VLP_ENOMEM, "out of memory for the evaluation key");
  }
  sk->params = p;
  evk->params = p;
  secret_keys(g, sk);
  std::vector<int> support;
  support.reserve(N);
  for (int j = 0; j < N; j++)
    if (sk->z[j]) support.push_back(j);

  // bsk_i row r = u*3 + j: (a, a*z + e) + s_i * g_j on component u's constant term (R4, O7).
  parallel_for(static_cast<size_t>(n) * kRows, [&](size_t ir) {
    const uint64_t obj = ir;
    uint32_t* a = evk->bsk.data() + ir * 2 * N;
    uint32_t* b = a + N;
    for (int j = 0; j < N; j++) a[j] = uniform(g, kBskA, obj, j);
    // a*z = sum_{k in supp z} X^k * a  (negacyclic: coefficient i moves to i+k, negated past N)
    for (int j = 0; j < N; j++) b[j] = 0;
    for (int k : support) {
      for (int i = 0; i < N - k; i++) b[i + k] += a[i];
      for (int i = N - k; i < N; i++) b[i + k - N] -= a[i];
    }
    for (int j = 0; j < N; j++) b[j] += noise(g, kBskE, obj, j, p.sigma_bk);
    const int i = static_cast<int>(ir / kRows), r = static_cast<int>(ir % kRows);
    if (sk->s[i]) (r / kEll == 0 ? a : b)[0] += 1u << (32 - kBgBits * (r % kEll + 1));
  });

  // ksk[i][j][v] = TLWE_s(v z_i 2^(32-2(j+1))), sigma_ks (R6, O10).
  parallel_for(static_cast<size_t>(N) * kKsT * 3, [&](size_t idx) {
    const int i = static_cast<int>(idx / (kKsT * 3)), j = static_cast<int>((idx / 3) % kKsT);
    const uint32_t v = static_cast<uint32_t>(idx % 3) + 1;
    const uint32_t mu = v * sk->z[i] * (1u << (32 - kKsBaseBits * (j + 1)));
    tlwe_sample(sk->s, mu, p.sigma_ks, g, kKskA, kKskE, idx, evk->ksk.data() + idx * kCt);
  });
  *sk_out = skp.release();
  *evk_out = evkp.release();
  return VLP_OK;
}

int vlp_keygen(uint64_t seed, const vlp_params* params, vlp_sk** sk_out, vlp_evk** evk_out) {
  return keygen_impl(seeded(seed), params, sk_out, evk_out);
}

int vlp_keygen_secure(const vlp_params* params, vlp_sk** sk_out, vlp_evk** evk_out) {
  Rng g;
  if (int rc = os_random(&g)) return rc;
  return keygen_impl(g, params, sk_out, evk_out);
}

int vlp_sk_export(const vlp_sk* sk, uint32_t* s, uint32_t* z) {
  if (!sk) return fail(VLP_EINVAL, "sk is NULL");
  if (s) std::memcpy(s, sk->s, sizeof(sk->s));
  if (z) std::memcpy(z, sk->z, sizeof(sk->z));
  return VLP_OK;
}

int vlp_evk_export(const vlp_evk* evk, uint32_t* bsk, uint32_t* ksk) {
  if (!evk) return fail(VLP_EINVAL, "evk is NULL");
  if (bsk) std::memcpy(bsk, evk->bsk.data(), evk->bsk.size() * 4);
  if (ksk)
    for (size_t r = 0; r < static_cast<size_t>(N) * kKsT * 3; r++)
      std::memcpy(ksk + r * (n + 1), evk->ksk.data() + r * kCt, (n + 1) * 4);
  return VLP_OK;
}

static int encrypt_bits_impl(const vlp_sk* sk, const uint8_t* bits, size_t count, const Rng& g, uint64_t obj0,
                             uint32_t* out) {
  if (!sk || (!bits && count) || (!out && count)) return fail(VLP_EINVAL, "null argument");
  parallel_for(count, [&](size_t i) {
    tlwe_sample(sk->s, bits[i] ? kMu : 0u - kMu, sk->params.sigma_lwe, g, kFreshA, kFreshE, obj0 + i,
                out + i * kCt);
  });
  return VLP_OK;
}
int vlp_encrypt_bits(const vlp_sk* sk, const uint8_t* bits, size_t count, uint64_t seed, uint64_t obj0,
                     uint32_t* out) {
  return encrypt_bits_impl(sk, bits, count, seeded(seed), obj0, out);
}
int vlp_encrypt_bits_secure(const vlp_sk* sk, const uint8_t* bits, size_t count, uint32_t* out) {
  Rng g;
  if (int rc = os_random(&g)) return rc;
  return encrypt_bits_impl(sk, bits, count, g, 0, out);
}

static int encrypt_query_impl(const vlp_sk* sk, const vlp_meta* meta, const uint64_t* values, const Rng& g,
                              uint32_t* out) {
  if (!sk || !values || !out) return fail(VLP_EINVAL, "null argument");
  if (int rc = check_meta(meta)) return rc;
  const size_t W = query_words(*meta), l = meta->l_I;
  for (size_t w = 0; w < W; w++)
    if (l < 64 && values[w] >> l) return fail(VLP_ERANGE, "query value >= 2^l_I");
  parallel_for(W * l, [&](size_t idx) {
    const size_t w = idx / l, j = idx % l;
    const uint32_t bit = static_cast<uint32_t>((values[w] >> j) & 1);
    tlwe_sample(sk->s, bit ? kMu : 0u - kMu, sk->params.sigma_lwe, g, kQryA, kQryE, idx, out + idx * kCt);
  });
  return VLP_OK;
}
int vlp_encrypt_query(const vlp_sk* sk, const vlp_meta* meta, const uint64_t* values, uint64_t seed,
                      uint32_t* out) {
  return encrypt_query_impl(sk, meta, values, seeded(seed), out);
}
int vlp_encrypt_query_secure(const vlp_sk* sk, const vlp_meta* meta, const uint64_t* values, uint32_t* out) {
  Rng g;
  if (int rc = os_random(&g)) return rc;
  return encrypt_query_impl(sk, meta, values, g, out);
}

int vlp_decrypt_bits(const vlp_sk* sk, const uint32_t* ct, size_t count, uint8_t* bits) {
  if (!sk || (count && (!ct || !bits))) return fail(VLP_EINVAL, "null argument");
  for (size_t c = 0; c < count; c++) {
    const uint32_t* x = ct + c * kCt;
    uint32_t dot = 0;
    for (int i = 0; i < n; i++) dot += x[i] * sk->s[i];
    bits[c] = static_cast<int32_t>(x[n] - dot) > 0 ? 1 : 0;
  }
  return VLP_OK;
}

int vlp_decrypt_result(const vlp_sk* sk, const uint32_t* ct, uint32_t l_S, uint8_t* bits, uint64_t* value) {
  if (!sk || (l_S && (!ct || !bits))) return fail(VLP_EINVAL, "null argument");
  if (value && l_S > 64) return fail(VLP_EWIDTH, "value_out needs l_S <= 64");
  if (int rc = vlp_decrypt_bits(sk, ct, l_S, bits)) return rc;
  if (value) {
    uint64_t v = 0;
    for (uint32_t j = 0; j < l_S; j++) v |= static_cast<uint64_t>(bits[j]) << j;
    *value = v;
  }
  return VLP_OK;
}

int vlp_db_record_cts(const vlp_meta* meta, size_t* per_record) {
  if (int rc = check_meta(meta)) return rc;
  if (!per_record) return fail(VLP_EINVAL, "null output");
  *per_record = record_words(*meta) * meta->l_I + meta->l_S;
  return VLP_OK;
}

static int pubkeygen_impl(const vlp_sk* sk, const vlp_meta* meta, const Rng& g, size_t first, size_t count,
                          vlp_pk** out) {
  if (!sk || !out) return fail(VLP_EINVAL, "null argument");
  if (int rc = check_meta(meta)) return rc;
  if (first + count > meta->M) return fail(VLP_EINVAL, "record range exceeds M");
  vlp_pk* pk = new (std::nothrow) vlp_pk;
  if (!pk) return fail(VLP_ENOMEM, "out of memory");
  pk->meta = *meta;
  pk->first = first;
  pk->count = count;
  const size_t W = record_words(*meta), lI = meta->l_I, lS = meta->l_S, per = W * lI + lS;
  try {
    pk->samples.assign(count * per * kCt, 0);
  } catch (...) {
    delete pk;
    return fail(VLP_ENOMEM, "out of memory for pk samples");
  }
  // Row order of a record: word k bit j at k*l_I + j, then payload bit j.  PRNG object of each sample:
  // record i, local index j*W + k (pk^I, bit j outer / word k inner as alg:PubKeyGen P:200-209) or
  // W*l_I + j (pk^S); obj = i*per + local.
  parallel_for(count * per, [&](size_t idx) {
    const size_t rec = idx / per, row = idx % per, i = first + rec;
    size_t local;
    if (row < W * lI) {
      const size_t k = row / lI, j = row % lI;
      local = j * W + k;
    } else {
      local = row;  // W*l_I + j
    }
    tlwe_sample(sk->s, 0u, sk->params.sigma_lwe, g, kPkA, kPkE, i * per + local,
                pk->samples.data() + idx * kCt);
  });
  *out = pk;
  return VLP_OK;
}
int vlp_pubkeygen(const vlp_sk* sk, const vlp_meta* meta, uint64_t seed, size_t first, size_t count,
                  vlp_pk** out) {
  return pubkeygen_impl(sk, meta, seeded(seed), first, count, out);
}
int vlp_pubkeygen_secure(const vlp_sk* sk, const vlp_meta* meta, size_t first, size_t count, vlp_pk** out) {
  Rng g;
  if (int rc = os_random(&g)) return rc;
  return pubkeygen_impl(sk, meta, g, first, count, out);
}

int vlp_debug_next_secure_key(const uint32_t* key) {
  if (!key) return fail(VLP_EINVAL, "null argument");
  const char* on = getenv("VLP_TEST_HOOKS");
  if (!on || std::strcmp(on, "1") != 0)
    return fail(VLP_EINVAL, "vlp_debug_next_secure_key is a test hook: set VLP_TEST_HOOKS=1 to enable it");
  std::memcpy(g_next_key, key, sizeof(g_next_key));
  g_next_key_set = true;
  return VLP_OK;
}

int vlp_debug_chacha20_block(const uint32_t* key, uint32_t counter, const uint32_t* nonce, uint32_t* out) {
  if (!key || !nonce || !out) return fail(VLP_EINVAL, "null argument");
  chacha20_block(key, counter, nonce, out);
  return VLP_OK;
}

}  // extern "C"

namespace vlp {
// Host half of vlp_encrypt_db_device (api.cu): range checks, the per-sample Gaussian noise of alg:PubKeyGen
// (exactly the values vlp_pubkeygen draws), the plaintext bit of every DB row, and the PRNG prefix
// h1 = mix(seed ^ PK_A * C1) the device continues from.
// ServerEnc's plaintext: range checks and the bit of every DB row (words then payload bits, see
// vlp_server_encrypt_db).
int prepare_db_bits(const vlp_meta* meta, size_t count, const uint64_t* words, const uint64_t* payloads,
                    std::vector<uint8_t>& bits) {
  if (int rc = check_meta(meta)) return rc;
  if (count && (!words || !payloads)) return fail(VLP_EINVAL, "null argument");
  const size_t W = record_words(*meta), lI = meta->l_I, lS = meta->l_S, per = W * lI + lS;
  const size_t PW = (lS + 63) / 64, top = lS - 64 * (PW - 1);
  for (size_t r = 0; r < count; r++) {
    for (size_t k = 0; k < W; k++)
      if (lI < 64 && words[r * W + k] >> lI) return fail(VLP_ERANGE, "record word >= 2^l_I");
    if (top < 64 && payloads[r * PW + PW - 1] >> top) return fail(VLP_ERANGE, "payload >= 2^l_S");
  }
  try {
    bits.resize(count * per);
  } catch (...) {
    return fail(VLP_ENOMEM, "out of host memory");
  }
  parallel_for(count * per, [&](size_t idx) {
    const size_t rec = idx / per, row = idx % per;
    if (row < W * lI) {
      bits[idx] = static_cast<uint8_t>((words[rec * W + row / lI] >> (row % lI)) & 1);
    } else {
      const size_t j = row - W * lI;
      bits[idx] = static_cast<uint8_t>((payloads[rec * PW + j / 64] >> (j % 64)) & 1);
    }
  });
  return VLP_OK;
}

// PubKeyGen's host half: the per-sample Gaussian noise of alg:PubKeyGen (exactly the values vlp_pubkeygen /
// vlp_pubkeygen_secure draw under the same generator); the device continues the mask words.
int prepare_pk_noise(const vlp_sk* sk, const vlp_meta* meta, const Rng& g, size_t first, size_t count,
                     std::vector<uint32_t>& nz) {
  if (!sk) return fail(VLP_EINVAL, "null argument");
  if (int rc = check_meta(meta)) return rc;
  if (count == 0 || first + count > meta->M) return fail(VLP_EINVAL, "bad record range");
  const size_t W = record_words(*meta), lI = meta->l_I, lS = meta->l_S, per = W * lI + lS;
  try {
    nz.resize(count * per);
  } catch (...) {
    return fail(VLP_ENOMEM, "out of host memory");
  }
  parallel_for(count * per, [&](size_t idx) {
    const size_t rec = idx / per, row = idx % per;
    const size_t local = row < W * lI ? (row % lI) * W + row / lI : row;
    nz[idx] = noise(g, kPkE, (first + rec) * per + local, 0, sk->params.sigma_lwe);
  });
  return VLP_OK;
}

// Host half of vlp_encrypt_db_device (api.cu): PubKeyGen's noise plus ServerEnc's row bits.
int prepare_encrypt_db(const vlp_sk* sk, const vlp_meta* meta, const Rng& g, size_t first, size_t count,
                       const uint64_t* words, const uint64_t* payloads, std::vector<uint32_t>& nz,
                       std::vector<uint8_t>& bits) {
  if (!sk) return fail(VLP_EINVAL, "null argument");
  if (int rc = check_meta(meta)) return rc;
  if (count == 0 || first + count > meta->M) return fail(VLP_EINVAL, "bad record range");
  if (!words || !payloads) return fail(VLP_EINVAL, "null argument");
  if (int rc = prepare_db_bits(meta, count, words, payloads, bits)) return rc;
  return prepare_pk_noise(sk, meta, g, first, count, nz);
}
}  // namespace vlp

extern "C" {

int vlp_server_encrypt_db(vlp_pk* pk, const uint64_t* words, const uint64_t* payloads, uint32_t* out) {
  if (!pk || !out || (pk->count && (!words || !payloads))) return fail(VLP_EINVAL, "null argument");
  if (pk->used) return fail(VLP_EPKUSED, "public-key samples already used (single-use, alg:PubKeyGen)");
  const vlp_meta& m = pk->meta;
  const size_t W = record_words(m), lI = m.l_I, lS = m.l_S, per = W * lI + lS;
  const size_t PW = (lS + 63) / 64, top = lS - 64 * (PW - 1);  // payload words per record, bits in the last
  for (size_t r = 0; r < pk->count; r++) {
    for (size_t k = 0; k < W; k++)
      if (lI < 64 && words[r * W + k] >> lI) return fail(VLP_ERANGE, "record word >= 2^l_I");
    if (top < 64 && payloads[r * PW + PW - 1] >> top) return fail(VLP_ERANGE, "payload >= 2^l_S");
  }
  parallel_for(pk->count * per, [&](size_t idx) {
    const size_t rec = idx / per, row = idx % per;
    uint32_t bit;
    if (row < W * lI) {
      bit = static_cast<uint32_t>((words[rec * W + row / lI] >> (row % lI)) & 1);
    } else {
      const size_t j = row - W * lI;
      bit = static_cast<uint32_t>((payloads[rec * PW + j / 64] >> (j % 64)) & 1);
    }
    const uint32_t* s = pk->samples.data() + idx * kCt;
    uint32_t* d = out + idx * kCt;
    std::memcpy(d, s, kCt * 4);
    d[n] += bit ? kMu : 0u - kMu;  // (0, Ecd(bit)) + pk
  });
  pk->used = true;
  pk->samples.clear();
  pk->samples.shrink_to_fit();
  return VLP_OK;
}

void vlp_free_sk(vlp_sk* sk) { delete sk; }
void vlp_free_evk(vlp_evk* evk) { delete evk; }
void vlp_free_pk(vlp_pk* pk) { delete pk; }

}  // extern "C"
