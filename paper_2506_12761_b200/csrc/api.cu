// api.cu -- the device half of the C ABI (include/vlp.h): server creation (evk upload + NTT conversion),
// program compilation / binding / evaluation (one BR launch + one KS launch per circuit level),
// and the debug entry points used by the parity tests.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "kernels.cuh"

struct vlp_server {
  int device = 0;
  int sm_count = 148;
  uint8_t* evk_dev = nullptr;
  uint32_t* bsk_ntt = nullptr;
  uint32_t* ksk = nullptr;
  uint2* tw_fwd = nullptr;   // natural order (bsk conversion)
  uint2* twl_fwd = nullptr;  // thread-layout tables of the blind-rotate kernel
  uint2* twl_inv = nullptr;
  int8_t* kmat = nullptr;  // ksk as 4 signed byte limbs in UMMA order (K3T key switch, kernels_ks.cu)
  double2* bsk_fft = nullptr;  // FFT-domain bsk of the K2F engine (2 x 16-bit limbs, scaled 1/512)
  double2* psi = nullptr;      // psi^e, e < 2048
  // programs compiled by the problem-statement calls (vlp_server_eval, vlp_server_combine, vlp_gate_batch)
  std::mutex mu;
  // LRU-bounded (kMaxCachedPrograms): an evicted program (and its pinned job tables) is freed once the last call
  // using it has returned (shared ownership)
  struct Cached {
    std::shared_ptr<vlp_program> prog;
    uint64_t last_use = 0;
  };
  std::map<std::string, Cached> cache;
  uint64_t use_clock = 0;
};

struct vlp_program {
  vlp_server* server = nullptr;
  vlp::Schedule sched;
  // scratch layout (byte offsets)
  size_t off_br = 0, off_ks = 0, off_lin = 0, off_lin_in = 0, off_outslots = 0, off_mid = 0, off_nlwe = 0, bytes = 0;
  size_t off_ks_ws = 0;  // key-switch staging (abar + b' per job of a chunk, ks_stage_bytes)
  uint32_t ks_chunk = 0;
  std::vector<size_t> br_first, ks_first;  // per level, index of the level's first job
  std::vector<size_t> lin_first, lin_in_first;  // per level (R24 linear jobs and their input slots)
  std::vector<uint32_t> copy_slots;        // outputs that are not written in place
  // host image of the scratch's job-table region [0, off_mid) in pinned memory (allocated on the first
  // evaluation), copied into the caller's scratch by every evaluation: nothing is assumed about what a
  // scratch buffer held before, so one buffer may serve several programs in turn
  std::mutex tables_mu;
  uint8_t* tables = nullptr;
  uint32_t launches = 0;
  // optional per-kernel timing with CUDA events recorded on the launch stream (vlp_program_profile)
  bool profile = false;
  struct Ev { cudaEvent_t a, b; int kind; };
  std::vector<Ev> pending, pool;
  double br_ms = 0, ks_ms = 0;
  uint64_t br_launches = 0, ks_launches = 0;
  ~vlp_program() {
    if (tables) cudaFreeHost(tables);
    for (auto& e : pending) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
    for (auto& e : pool) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
  }
  Ev* begin(int kind, cudaStream_t st) {
    if (!profile) return nullptr;
    Ev e;
    if (!pool.empty()) { e = pool.back(); pool.pop_back(); }
    else { cudaEventCreate(&e.a); cudaEventCreate(&e.b); }
    e.kind = kind;
    cudaEventRecord(e.a, st);
    pending.push_back(e);
    return &pending.back();
  }
  void end(int kind, cudaStream_t st) {
    if (profile) cudaEventRecord(pending.back().b, st);
  }
};

namespace vlp {
namespace {

constexpr size_t kBskNttBytes = kBskNttWords * 4;
constexpr size_t kKskBytes = static_cast<size_t>(N) * kKsT * 3 * kCt * 4;
constexpr size_t kTwBytes = static_cast<size_t>(N) * sizeof(uint2);
constexpr size_t kTwlBytes = static_cast<size_t>(kTwSlots) * kBT * sizeof(uint2);
constexpr size_t kRawBskBytes = static_cast<size_t>(n) * kRows * 2 * N * 4;
constexpr size_t kEvkBytes =
    kBskNttBytes + kKskBytes + kTwBytes + 2 * kTwlBytes + kRawBskBytes + kKmatSwBytes + kBskFftBytes + kPsiBytes;

size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

// Makes `device` current for one C call and restores the caller's current device on return (the library never
// leaves a changed current device behind).
struct DeviceGuard {
  int prev = -1;
  cudaError_t set(int device) {
    cudaError_t e = cudaGetDevice(&prev);
    if (e != cudaSuccess) return e;
    return prev == device ? cudaSuccess : cudaSetDevice(device);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

int cuda_fail(cudaError_t e, const char* what) {
  return fail(VLP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

uint64_t mulmod(uint64_t a, uint64_t b) { return a * b % kP; }
uint64_t powmod(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  b %= kP;
  while (e) {
    if (e & 1) r = mulmod(r, b);
    b = mulmod(b, b);
    e >>= 1;
  }
  return r;
}
uint32_t bitrev10(uint32_t x) {
  uint32_t r = 0;
  for (int b = 0; b < 10; b++) r |= ((x >> b) & 1u) << (9 - b);
  return r;
}

// Twiddles of the negacyclic transform mod p: psi a primitive 2N-th root of unity;
// fwd[k] = psi^brv(k), inv[k] = psi^-brv(k), each with its Shoup companion floor(w 2^32 / p).
void make_twiddles(std::vector<uint2>& fwd, std::vector<uint2>& inv) {
  uint64_t psi = 0;
  for (uint64_t g = 2; g < 1000; g++) {
    const uint64_t x = powmod(g, (kP - 1) / (2 * N));
    if (powmod(x, N) == kP - 1) {
      psi = x;
      break;
    }
  }
  const uint64_t psi_inv = powmod(psi, kP - 2);
  fwd.resize(N);
  inv.resize(N);
  for (uint32_t k = 0; k < static_cast<uint32_t>(N); k++) {
    const uint64_t w = powmod(psi, bitrev10(k)), wi = powmod(psi_inv, bitrev10(k));
    fwd[k] = make_uint2(static_cast<uint32_t>(w), static_cast<uint32_t>((w << 32) / kP));
    inv[k] = make_uint2(static_cast<uint32_t>(wi), static_cast<uint32_t>((wi << 32) / kP));
  }
}

// Thread-layout twiddle tables of the blind-rotate kernel: slot q (stage 3..9 lane-varying twiddles) x
// thread t; k(stage, t, qq) is the twiddle index the butterflies of thread t use (kernels.cu layouts).
void make_layout_twiddles(const std::vector<uint2>& nat, std::vector<uint2>& lay) {
  lay.resize(static_cast<size_t>(kTwSlots) * kBT);
  const int st[kTwSlots] = {3, 4, 4, 5, 5, 5, 5, 6, 7, 7, 8, 8, 8, 8, 9, 9, 9, 9};
  const int qq[kTwSlots] = {0, 0, 1, 0, 1, 2, 3, 0, 0, 1, 0, 1, 2, 3, 0, 1, 2, 3};
  for (int q = 0; q < kTwSlots; q++)
    for (uint32_t t = 0; t < static_cast<uint32_t>(kBT); t++) {
      const uint32_t th = t >> 4, tc = t >> 1;
      uint32_t k = 0;
      switch (st[q]) {
        case 3: k = 8 + th; break;
        case 4: k = 16 + 2 * th + qq[q]; break;
        case 5: k = 32 + 4 * th + qq[q]; break;
        case 6: k = 64 + tc; break;
        case 7: k = 128 + 2 * tc + qq[q]; break;
        case 8: k = 256 + 4 * tc + qq[q]; break;
        default: k = 512 + 8 * tc + ((t & 1) ? 4 + qq[q] : qq[q]); break;
      }
      lay[static_cast<size_t>(q) * kBT + t] = nat[k];
    }
}

int run_keyswitch(vlp_server* s, const KsArgs& ka, uint8_t* stage, uint32_t chunk, cudaStream_t st) {
  if (cudaError_t e = launch_keyswitch_t(ka, s->kmat, stage, chunk, s->sm_count, st)) return cuda_fail(e, "key switch");
  return VLP_OK;
}

size_t ks_stage_bytes(uint32_t chunk) { return ks_stage_bytes_t(chunk); }

Regions regions(const vlp_program* p, void* scratch, const uint32_t* in0, const uint32_t* in1, uint32_t* out) {
  Regions r;
  r.base[kRegIn0] = const_cast<uint32_t*>(in0);
  r.base[kRegIn1] = const_cast<uint32_t*>(in1);
  r.base[kRegMid] = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + p->off_mid);
  r.base[kRegOut] = out;
  return r;
}

int build_program(vlp_server* server, std::unique_ptr<vlp_program>& p) {
  Schedule& s = p->sched;
  size_t nbr = 0, nks = 0, nlin = 0, nlin_in = 0;
  for (auto& L : s.levels) {
    p->br_first.push_back(nbr);
    p->ks_first.push_back(nks);
    p->lin_first.push_back(nlin);
    p->lin_in_first.push_back(nlin_in);
    nbr += L.br.size();
    nks += L.ks.size();
    nlin += L.lin.size();
    nlin_in += L.lin_in.size();
  }
  for (uint32_t sl : s.out_slots)
    if ((sl >> 28) != kRegOut) p->copy_slots.push_back(sl);
  p->off_br = 0;
  p->off_ks = align256(p->off_br + nbr * sizeof(BrJob));
  p->off_lin = align256(p->off_ks + nks * sizeof(KsJob));
  p->off_lin_in = align256(p->off_lin + nlin * sizeof(LinJob));
  p->off_outslots = align256(p->off_lin_in + nlin_in * 4);
  p->off_mid = align256(p->off_outslots + p->copy_slots.size() * 4 + 4);
  p->off_nlwe = align256(p->off_mid + s.mid_rows * kCt * 4);
  size_t max_ks = 0;
  for (auto& L : s.levels) max_ks = std::max(max_ks, L.ks.size());
  p->ks_chunk = static_cast<uint32_t>(std::min<size_t>(std::max<size_t>(max_ks, 1), kKsChunk));
  p->off_ks_ws = align256(p->off_nlwe + s.nlwe_rows * kNlwe * 4);
  p->bytes = p->off_ks_ws + ks_stage_bytes(p->ks_chunk);
  p->server = server;
  p->launches = 1 + (p->copy_slots.empty() ? 0 : 1);
  for (auto& L : s.levels) {  // our kernels: BR waves + (prologue, tcgen05 GEMM) per key-switch chunk
    p->launches += br_launch_count(static_cast<uint32_t>(L.br.size()), server ? server->sm_count : 148) +
                   2 * static_cast<uint32_t>((L.ks.size() + p->ks_chunk - 1) / p->ks_chunk) + (L.lin.empty() ? 0 : 1);
  }
  return VLP_OK;
}

}  // namespace
}  // namespace vlp

using namespace vlp;

// No C++ exception crosses the C ABI: allocation failures while compiling become VLP_ENOMEM.
extern "C++" {
template <class F>
static int no_throw(F&& f) {
  try {
    return f();
  } catch (const std::bad_alloc&) {
    return fail(VLP_ENOMEM, "out of host memory");
  } catch (const std::exception& e) {
    return fail(VLP_EINVAL, e.what());
  }
}
}  // extern "C++"

extern "C++" {
// The device half of a call's generator (host.cpp Rng): the mask words of domain `dom`.
static MaskGen mask_gen(const Rng& g, uint64_t dom) {
  MaskGen m{};
  m.secure = g.secure ? 1u : 0u;
  m.dom = static_cast<uint32_t>(dom);
  if (g.secure)
    std::memcpy(m.key, g.key, sizeof(m.key));
  else
    m.h1 = prng_prefix(g.seed, dom);
  return m;
}
}  // extern "C++"

extern "C" {

int vlp_encrypt_db_device_scratch_bytes(const vlp_meta* meta, size_t count, size_t* scratch_bytes) {
  size_t per = 0;
  if (int rc = vlp_db_record_cts(meta, &per)) return rc;
  if (!scratch_bytes) return fail(VLP_EINVAL, "null argument");
  *scratch_bytes = align256(n * 4) + align256(count * per * 4) + align256(count * per);
  return VLP_OK;
}

int vlp_encrypt_db_device(const vlp_sk* sk, const vlp_meta* meta, uint64_t pk_seed, size_t first, size_t count,
                          const uint64_t* words, const uint64_t* payloads, uint32_t* out_dev, void* scratch,
                          size_t scratch_bytes, uint64_t stream) {
  if (!out_dev || !scratch) return fail(VLP_EINVAL, "null argument");
  return no_throw([&] {
    std::vector<uint32_t> nz;
    std::vector<uint8_t> bits;
    const Rng g = seeded(pk_seed);
    if (int rc = prepare_encrypt_db(sk, meta, g, first, count, words, payloads, nz, bits)) return rc;
    size_t need = 0;
    vlp_encrypt_db_device_scratch_bytes(meta, count, &need);
    if (scratch_bytes < need) return fail(VLP_ENOMEM, "scratch too small");
    const size_t per = nz.size() / count, W = record_words(*meta);
    uint8_t* sc = static_cast<uint8_t*>(scratch);
    uint32_t* s_dev = reinterpret_cast<uint32_t*>(sc);
    uint32_t* nz_dev = reinterpret_cast<uint32_t*>(sc + align256(n * 4));
    uint8_t* bits_dev = sc + align256(n * 4) + align256(nz.size() * 4);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e;
    if ((e = cudaMemcpyAsync(s_dev, sk->s, n * 4, cudaMemcpyHostToDevice, st)) ||
        (e = cudaMemcpyAsync(nz_dev, nz.data(), nz.size() * 4, cudaMemcpyHostToDevice, st)) ||
        (e = cudaMemcpyAsync(bits_dev, bits.data(), bits.size(), cudaMemcpyHostToDevice, st)))
      return cuda_fail(e, "upload");
    if ((e = launch_encrypt_db(s_dev, nz_dev, bits_dev, mask_gen(g, kPkA), static_cast<uint32_t>(per), static_cast<uint32_t>(W),
                               meta->l_I, first, nz.size(), out_dev, st)))
      return cuda_fail(e, "encrypt db");
    if ((e = cudaMemsetAsync(s_dev, 0, n * 4, st))) return cuda_fail(e, "scrub");  // s does not outlive the call
    if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "encrypt db sync");
    return static_cast<int>(VLP_OK);
  });
}

size_t vlp_keygen_device_scratch_bytes(void) {
  return align256(kRawBskBytes) + align256(kKskBytes) + align256(kRawBskBytes / 2) + align256(static_cast<size_t>(N) * kKsT * 3 * 4) +
         align256(n * 4) + align256(N * 4);
}

static int keygen_device_impl(const Rng& g, const vlp_params* params, void* scratch, size_t scratch_bytes,
                              uint64_t stream, vlp_sk** sk_out, vlp_evk** evk_out) {
  if (!sk_out || !evk_out || !scratch) return fail(VLP_EINVAL, "null argument");
  if (scratch_bytes < vlp_keygen_device_scratch_bytes()) return fail(VLP_ENOMEM, "scratch too small");
  vlp_params p;
  if (int rc = resolve_params(params, &p)) return rc;
  return no_throw([&] {
    auto sk = std::make_unique<vlp_sk>();
    auto evk = std::make_unique<vlp_evk>();
    sk->params = p;
    evk->params = p;
    secret_keys(g, sk.get());
    evk->bsk.assign(static_cast<size_t>(n) * kRows * 2 * N, 0);
    evk->ksk.assign(static_cast<size_t>(N) * kKsT * 3 * kCt, 0);
    std::vector<uint32_t> e_bsk(static_cast<size_t>(n) * kRows * N), e_ksk(static_cast<size_t>(N) * kKsT * 3);
    keygen_noise(g, p, e_bsk.data(), e_ksk.data());  // host libm Box-Muller (byte-identical noise)
    uint8_t* sc = static_cast<uint8_t*>(scratch);
    uint32_t* bsk = reinterpret_cast<uint32_t*>(sc);
    uint32_t* ksk = reinterpret_cast<uint32_t*>(sc + align256(kRawBskBytes));
    uint32_t* eb = reinterpret_cast<uint32_t*>(sc + align256(kRawBskBytes) + align256(kKskBytes));
    uint32_t* ek = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(eb) + align256(kRawBskBytes / 2));
    uint32_t* s_dev = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(ek) + align256(e_ksk.size() * 4));
    uint32_t* z_dev = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(s_dev) + align256(n * 4));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e;
    if ((e = cudaMemcpyAsync(s_dev, sk->s, n * 4, cudaMemcpyHostToDevice, st)) ||
        (e = cudaMemcpyAsync(z_dev, sk->z, N * 4, cudaMemcpyHostToDevice, st)) ||
        (e = cudaMemcpyAsync(eb, e_bsk.data(), e_bsk.size() * 4, cudaMemcpyHostToDevice, st)) ||
        (e = cudaMemcpyAsync(ek, e_ksk.data(), e_ksk.size() * 4, cudaMemcpyHostToDevice, st)))
      return cuda_fail(e, "keygen upload");
    if ((e = launch_keygen(mask_gen(g, kBskA), mask_gen(g, kKskA), s_dev, z_dev, eb, ek, bsk, ksk, st)))
      return cuda_fail(e, "keygen kernels");
    if ((e = cudaMemcpyAsync(evk->bsk.data(), bsk, kRawBskBytes, cudaMemcpyDeviceToHost, st)) ||
        (e = cudaMemcpyAsync(evk->ksk.data(), ksk, kKskBytes, cudaMemcpyDeviceToHost, st)) ||
        (e = cudaMemsetAsync(s_dev, 0, align256(n * 4) + N * 4, st)))  // the secret keys do not outlive the call
      return cuda_fail(e, "keygen download");
    if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "keygen sync");
    *sk_out = sk.release();
    *evk_out = evk.release();
    return static_cast<int>(VLP_OK);
  });
}

int vlp_keygen_device(uint64_t seed, const vlp_params* params, void* scratch, size_t scratch_bytes, uint64_t stream,
                      vlp_sk** sk_out, vlp_evk** evk_out) {
  return keygen_device_impl(seeded(seed), params, scratch, scratch_bytes, stream, sk_out, evk_out);
}

int vlp_keygen_device_secure(const vlp_params* params, void* scratch, size_t scratch_bytes, uint64_t stream,
                             vlp_sk** sk_out, vlp_evk** evk_out) {
  Rng g;
  if (int rc = os_random(&g)) return rc;
  return keygen_device_impl(g, params, scratch, scratch_bytes, stream, sk_out, evk_out);
}

int vlp_pubkeygen_device_scratch_bytes(const vlp_meta* meta, size_t count, size_t* scratch_bytes) {
  size_t per = 0;
  if (int rc = vlp_db_record_cts(meta, &per)) return rc;
  if (!scratch_bytes) return fail(VLP_EINVAL, "null argument");
  *scratch_bytes = align256(n * 4) + align256(count * per * 4);
  return VLP_OK;
}

static int pubkeygen_device_impl(const vlp_sk* sk, const vlp_meta* meta, const Rng& g, size_t first, size_t count,
                                 uint32_t* pk_dev, void* scratch, size_t scratch_bytes, uint64_t stream) {
  if (!pk_dev || !scratch) return fail(VLP_EINVAL, "null argument");
  return no_throw([&] {
    std::vector<uint32_t> nz;
    if (int rc = prepare_pk_noise(sk, meta, g, first, count, nz)) return rc;
    size_t need = 0;
    vlp_pubkeygen_device_scratch_bytes(meta, count, &need);
    if (scratch_bytes < need) return fail(VLP_ENOMEM, "scratch too small");
    const size_t per = nz.size() / count, W = record_words(*meta);
    uint8_t* sc = static_cast<uint8_t*>(scratch);
    uint32_t* s_dev = reinterpret_cast<uint32_t*>(sc);
    uint32_t* nz_dev = reinterpret_cast<uint32_t*>(sc + align256(n * 4));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e;
    if ((e = cudaMemcpyAsync(s_dev, sk->s, n * 4, cudaMemcpyHostToDevice, st)) ||
        (e = cudaMemcpyAsync(nz_dev, nz.data(), nz.size() * 4, cudaMemcpyHostToDevice, st)))
      return cuda_fail(e, "upload");
    if ((e = launch_encrypt_db(s_dev, nz_dev, nullptr, mask_gen(g, kPkA), static_cast<uint32_t>(per), static_cast<uint32_t>(W),
                               meta->l_I, first, nz.size(), pk_dev, st)))
      return cuda_fail(e, "pubkeygen");
    if ((e = cudaMemsetAsync(s_dev, 0, n * 4, st))) return cuda_fail(e, "scrub");  // s does not outlive the call
    if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "pubkeygen sync");
    return static_cast<int>(VLP_OK);
  });
}

int vlp_pubkeygen_device(const vlp_sk* sk, const vlp_meta* meta, uint64_t seed, size_t first, size_t count,
                         uint32_t* pk_dev, void* scratch, size_t scratch_bytes, uint64_t stream) {
  return pubkeygen_device_impl(sk, meta, seeded(seed), first, count, pk_dev, scratch, scratch_bytes, stream);
}

int vlp_pubkeygen_device_secure(const vlp_sk* sk, const vlp_meta* meta, size_t first, size_t count, uint32_t* pk_dev,
                                void* scratch, size_t scratch_bytes, uint64_t stream) {
  Rng g;
  if (int rc = os_random(&g)) return rc;
  return pubkeygen_device_impl(sk, meta, g, first, count, pk_dev, scratch, scratch_bytes, stream);
}

int vlp_server_encrypt_db_device_scratch_bytes(const vlp_meta* meta, size_t count, size_t* scratch_bytes) {
  size_t per = 0;
  if (int rc = vlp_db_record_cts(meta, &per)) return rc;
  if (!scratch_bytes) return fail(VLP_EINVAL, "null argument");
  *scratch_bytes = align256(count * per);
  return VLP_OK;
}

int vlp_server_encrypt_db_device(const vlp_meta* meta, size_t count, const uint32_t* pk_dev, const uint64_t* words,
                                 const uint64_t* payloads, uint32_t* out_dev, void* scratch, size_t scratch_bytes,
                                 uint64_t stream) {
  if (!pk_dev || !out_dev || !scratch) return fail(VLP_EINVAL, "null argument");
  return no_throw([&] {
    std::vector<uint8_t> bits;
    if (int rc = prepare_db_bits(meta, count, words, payloads, bits)) return rc;
    if (scratch_bytes < align256(bits.size())) return fail(VLP_ENOMEM, "scratch too small");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e;
    if ((e = cudaMemcpyAsync(scratch, bits.data(), bits.size(), cudaMemcpyHostToDevice, st))) return cuda_fail(e, "upload");
    if ((e = launch_server_enc(pk_dev, static_cast<const uint8_t*>(scratch), bits.size(), out_dev, st)))
      return cuda_fail(e, "server enc");
    if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "server enc sync");
    return static_cast<int>(VLP_OK);
  });
}

int vlp_server_load_records(vlp_pk* pk, const uint64_t* words, const uint64_t* payloads, uint32_t* db_dev,
                            void* scratch, size_t scratch_bytes, uint64_t stream) {
  if (!pk || !db_dev || !scratch) return fail(VLP_EINVAL, "null argument");
  if (pk->used) return fail(VLP_EPKUSED, "public-key samples already used (single-use, alg:PubKeyGen)");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if ((e = cudaMemcpyAsync(db_dev, pk->samples.data(), pk->samples.size() * 4, cudaMemcpyHostToDevice, st)))
    return cuda_fail(e, "upload pk");
  if (int rc = vlp_server_encrypt_db_device(&pk->meta, pk->count, db_dev, words, payloads, db_dev, scratch,
                                            scratch_bytes, stream))
    return rc;  // synchronous: the pk upload is complete
  pk->used = true;
  pk->samples.clear();
  pk->samples.shrink_to_fit();
  return VLP_OK;
}

size_t vlp_server_evk_bytes(void) { return kEvkBytes; }

int vlp_server_create(int device, const vlp_evk* evk, void* evk_dev, size_t evk_bytes, uint64_t stream,
                      vlp_server** out) {
  if (!evk || !evk_dev || !out) return fail(VLP_EINVAL, "null argument");
  if (evk_bytes < kEvkBytes) return fail(VLP_ENOMEM, "evk buffer too small");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(VLP_ENODEV, "no CUDA device");
  DeviceGuard dg;
  if (cudaError_t e = dg.set(device)) return cuda_fail(e, "cudaSetDevice");
  return no_throw([&] {
    auto srv = std::make_unique<vlp_server>();
    srv->device = device;
    cudaDeviceGetAttribute(&srv->sm_count, cudaDevAttrMultiProcessorCount, device);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    uint8_t* base = static_cast<uint8_t*>(evk_dev);
    srv->evk_dev = base;
    srv->bsk_ntt = reinterpret_cast<uint32_t*>(base);
    srv->ksk = reinterpret_cast<uint32_t*>(base + kBskNttBytes);
    srv->tw_fwd = reinterpret_cast<uint2*>(base + kBskNttBytes + kKskBytes);
    srv->twl_fwd = reinterpret_cast<uint2*>(base + kBskNttBytes + kKskBytes + kTwBytes);
    srv->twl_inv = reinterpret_cast<uint2*>(base + kBskNttBytes + kKskBytes + kTwBytes + kTwlBytes);
    uint32_t* raw = reinterpret_cast<uint32_t*>(base + kBskNttBytes + kKskBytes + kTwBytes + 2 * kTwlBytes);
    srv->kmat = reinterpret_cast<int8_t*>(base + kBskNttBytes + kKskBytes + kTwBytes + 2 * kTwlBytes + kRawBskBytes);
    srv->bsk_fft = reinterpret_cast<double2*>(reinterpret_cast<uint8_t*>(srv->kmat) + kKmatSwBytes);
    srv->psi = reinterpret_cast<double2*>(reinterpret_cast<uint8_t*>(srv->bsk_fft) + kBskFftBytes);

    std::vector<uint2> fwd, inv, lf, li;
    make_twiddles(fwd, inv);
    make_layout_twiddles(fwd, lf);
    make_layout_twiddles(inv, li);
    set_const_twiddles(fwd.data(), inv.data());
    cudaError_t e;
    if ((e = cudaMemsetAsync(srv->bsk_ntt, 0, kBskNttBytes, st))) return cuda_fail(e, "memset");
    if ((e = cudaMemcpyAsync(srv->tw_fwd, fwd.data(), kTwBytes, cudaMemcpyHostToDevice, st))) return cuda_fail(e, "tw");
    if ((e = cudaMemcpyAsync(srv->twl_fwd, lf.data(), kTwlBytes, cudaMemcpyHostToDevice, st))) return cuda_fail(e, "twl");
    if ((e = cudaMemcpyAsync(srv->twl_inv, li.data(), kTwlBytes, cudaMemcpyHostToDevice, st))) return cuda_fail(e, "twl");
    if ((e = cudaMemcpyAsync(srv->ksk, evk->ksk.data(), kKskBytes, cudaMemcpyHostToDevice, st))) return cuda_fail(e, "ksk");
    if ((e = cudaMemcpyAsync(raw, evk->bsk.data(), kRawBskBytes, cudaMemcpyHostToDevice, st))) return cuda_fail(e, "bsk");
    // Montgomery factor with N^-1 folded in: c = N^-1 * 2^32 mod p
    const uint32_t c_mont = static_cast<uint32_t>(mulmod(powmod(N, kP - 2), (1ull << 32) % kP));
    launch_bsk_convert(raw, srv->bsk_ntt, srv->tw_fwd, c_mont, st);
    // K2F: psi^e = exp(i pi e / 1024) in double (host libm), the FFT-domain key by a direct DFT on the device
    std::vector<double2> psi(2048);
    for (int k = 0; k < 2048; k++) psi[k] = make_double2(cos(M_PI * k / 1024.0), sin(M_PI * k / 1024.0));
    set_fft_constants(psi.data());
    if ((e = cudaMemcpyAsync(srv->psi, psi.data(), kPsiBytes, cudaMemcpyHostToDevice, st))) return cuda_fail(e, "psi");
    launch_bsk_fft(raw, srv->bsk_fft, srv->psi, st);
    launch_kmat_sw(srv->ksk, srv->kmat, st);
    if ((e = cudaGetLastError())) return cuda_fail(e, "bsk convert launch");
    if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "server create");
    *out = srv.release();
    return static_cast<int>(VLP_OK);
  });
}

static int finish_program(vlp_server* server, std::unique_ptr<vlp_program>& p, vlp_program** out) {
  if (int rc = build_program(server, p)) return rc;
  *out = p.release();
  return VLP_OK;
}


int vlp_program_create(vlp_server* server, const vlp_meta* meta, size_t first, size_t count, vlp_program** out) {
  if (!meta || !out) return fail(VLP_EINVAL, "null argument");  // server may be NULL: compile only
  return no_throw([&] {
    auto p = std::make_unique<vlp_program>();
    if (int rc = compile_velopir(*meta, first, count, &p->sched)) return rc;
    return finish_program(server, p, out);
  });
}

int vlp_program_create_queries(vlp_server* server, const vlp_meta* meta, size_t first, size_t count, uint32_t nq,
                               vlp_program** out) {
  if (!meta || !out) return fail(VLP_EINVAL, "null argument");
  return no_throw([&] {
    auto p = std::make_unique<vlp_program>();
    if (int rc = compile_velopir(*meta, first, count, &p->sched, nq)) return rc;
    return finish_program(server, p, out);
  });
}

int vlp_program_create_gates(vlp_server* server, int op, size_t count, vlp_program** out) {
  if (!out) return fail(VLP_EINVAL, "null argument");
  return no_throw([&] {
    auto p = std::make_unique<vlp_program>();
    if (int rc = compile_gates(op, count, &p->sched)) return rc;
    return finish_program(server, p, out);
  });
}

int vlp_program_create_combine(vlp_server* server, const vlp_meta* meta, uint32_t G, vlp_program** out) {
  if (!meta || !out) return fail(VLP_EINVAL, "null argument");
  return no_throw([&] {
    auto p = std::make_unique<vlp_program>();
    if (int rc = compile_combine(*meta, G, &p->sched)) return rc;
    return finish_program(server, p, out);
  });
}

int vlp_program_get_info(const vlp_program* p, vlp_program_info* info) {
  if (!p || !info) return fail(VLP_EINVAL, "null argument");
  std::memset(info, 0, sizeof(*info));
  info->levels = static_cast<uint32_t>(p->sched.levels.size());
  info->br = p->sched.br;
  info->ks = p->sched.ks;
  info->gates = p->sched.gates;
  info->in0_cts = p->sched.in0_cts;
  info->in1_cts = p->sched.in1_cts;
  info->out_cts = p->sched.out_cts;
  info->scratch_bytes = p->bytes;
  for (auto& L : p->sched.levels) info->max_level_br = std::max<uint64_t>(info->max_level_br, L.br.size());
  info->kernel_launches = p->launches;
  info->table_bytes = p->off_mid;
  return VLP_OK;
}

int vlp_program_node_row(const vlp_program* p, int kind, size_t record, uint32_t bit, uint64_t* row) {
  if (!p || !row) return fail(VLP_EINVAL, "null argument");
  uint32_t sl;
  if (kind == 0 && record < p->sched.v_rows.size())
    sl = static_cast<uint32_t>(p->sched.v_rows[record]);
  else if (kind == 1 && p->sched.l_S && record * p->sched.l_S + bit < p->sched.mask_rows.size() && bit < p->sched.l_S)
    sl = static_cast<uint32_t>(p->sched.mask_rows[record * p->sched.l_S + bit]);
  else
    return fail(VLP_EINVAL, "no such node");
  if ((sl >> 28) != kRegMid) return fail(VLP_EINVAL, "node is not in the intermediate region");
  *row = sl & 0x0FFFFFFFu;
  return VLP_OK;
}

int vlp_program_level_jobs(const vlp_program* p, uint32_t level, vlp_br_job* br, uint64_t* nbr, vlp_ks_job* ks,
                           uint64_t* nks) {
  static_assert(sizeof(vlp_br_job) == sizeof(BrJob) && sizeof(vlp_ks_job) == sizeof(KsJob), "job layout");
  if (!p || !nbr || !nks) return fail(VLP_EINVAL, "null argument");
  if (level >= p->sched.levels.size()) return fail(VLP_EINVAL, "no such level");
  const Level& lv = p->sched.levels[level];
  *nbr = lv.br.size();
  *nks = lv.ks.size();
  if (br) std::memcpy(br, lv.br.data(), lv.br.size() * sizeof(BrJob));
  if (ks) std::memcpy(ks, lv.ks.data(), lv.ks.size() * sizeof(KsJob));
  return VLP_OK;
}

int vlp_program_level_linear(const vlp_program* p, uint32_t level, uint32_t* jobs, uint64_t* njobs, uint32_t* inputs,
                             uint64_t* ninputs) {
  if (!p || !njobs || !ninputs) return fail(VLP_EINVAL, "null argument");
  if (level >= p->sched.levels.size()) return fail(VLP_EINVAL, "no such level");
  const Level& lv = p->sched.levels[level];
  *njobs = lv.lin.size();
  *ninputs = lv.lin_in.size();
  if (jobs) std::memcpy(jobs, lv.lin.data(), lv.lin.size() * sizeof(LinJob));
  if (inputs) std::memcpy(inputs, lv.lin_in.data(), lv.lin_in.size() * 4);
  return VLP_OK;
}

int vlp_program_intermediate_offset(const vlp_program* p, uint64_t* off) {
  if (!p || !off) return fail(VLP_EINVAL, "null argument");
  *off = p->off_mid;
  return VLP_OK;
}

extern "C++" {
// Build the pinned host image of the job tables once per program (thread-safe).
static int stage_tables(vlp_program* p) {
  std::lock_guard<std::mutex> lock(p->tables_mu);
  if (p->tables) return VLP_OK;
  uint8_t* h = nullptr;
  if (cudaError_t e = cudaMallocHost(&h, std::max<size_t>(p->off_mid, 1))) return cuda_fail(e, "pinned job tables");
  std::memset(h, 0, p->off_mid);
  for (size_t L = 0; L < p->sched.levels.size(); L++) {
    const Level& lv = p->sched.levels[L];
    if (!lv.br.empty()) std::memcpy(h + p->off_br + p->br_first[L] * sizeof(BrJob), lv.br.data(), lv.br.size() * sizeof(BrJob));
    if (!lv.ks.empty()) std::memcpy(h + p->off_ks + p->ks_first[L] * sizeof(KsJob), lv.ks.data(), lv.ks.size() * sizeof(KsJob));
    if (!lv.lin.empty()) {
      std::memcpy(h + p->off_lin + p->lin_first[L] * sizeof(LinJob), lv.lin.data(), lv.lin.size() * sizeof(LinJob));
      std::memcpy(h + p->off_lin_in + p->lin_in_first[L] * 4, lv.lin_in.data(), lv.lin_in.size() * 4);
    }
  }
  if (!p->copy_slots.empty()) std::memcpy(h + p->off_outslots, p->copy_slots.data(), p->copy_slots.size() * 4);
  p->tables = h;
  return VLP_OK;
}
}  // extern "C++"

int vlp_program_eval(vlp_program* p, void* scratch, size_t scratch_bytes, const uint32_t* in0,
                     const uint32_t* in1, uint32_t* out, uint64_t stream) {
  if (!p || !scratch) return fail(VLP_EINVAL, "null argument");
  if (!p->server) return fail(VLP_EINVAL, "program was compiled without a server (compile-only)");
  if (scratch_bytes < p->bytes) return fail(VLP_ENOMEM, "scratch too small");
  if ((p->sched.in0_cts && !in0) || (p->sched.in1_cts && !in1) || (p->sched.out_cts && !out))
    return fail(VLP_EINVAL, "missing input / output buffer");
  vlp_server* s = p->server;
  cudaError_t e;
  DeviceGuard dg;
  if ((e = dg.set(s->device))) return cuda_fail(e, "cudaSetDevice");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* sc = static_cast<uint8_t*>(scratch);
  if (int rc = stage_tables(p)) return rc;
  // the job tables into this scratch, every evaluation (asynchronous, from pinned memory, stream-ordered
  // before the kernels that read them; 20 B per BR + 16 B per KS)
  if ((e = cudaMemcpyAsync(sc, p->tables, p->off_mid, cudaMemcpyHostToDevice, st))) return cuda_fail(e, "upload jobs");
  const Regions reg = regions(p, scratch, in0, in1, out);
  if ((e = launch_init_constants(reg.base[kRegMid], st))) return cuda_fail(e, "init constants");
  uint32_t* nlwe = reinterpret_cast<uint32_t*>(sc + p->off_nlwe);
  struct NvtxLevel {  // one NVTX range per circuit level (host-side launch span; nsys / ncu show it)
    explicit NvtxLevel(size_t L, size_t br, size_t ks) {
      char name[96];
      snprintf(name, sizeof(name), "vlp level %zu: %zu BR, %zu KS", L, br, ks);
      nvtxRangePushA(name);
    }
    ~NvtxLevel() { nvtxRangePop(); }
  };
  for (size_t L = 0; L < p->sched.levels.size(); L++) {
    const Level& lv = p->sched.levels[L];
    const NvtxLevel range(L, lv.br.size(), lv.ks.size());
    BrArgs ba{};
    ba.jobs = reinterpret_cast<const BrJob*>(sc + p->off_br) + p->br_first[L];
    ba.njobs = static_cast<uint32_t>(lv.br.size());
    ba.steps = n;
    ba.reg = reg;
    ba.nlwe = nlwe;
    ba.raw_acc = nullptr;
    ba.bsk = s->bsk_ntt;
    ba.twl_fwd = s->twl_fwd;
    ba.twl_inv = s->twl_inv;
    ba.bskf = s->bsk_fft;
    ba.psi = s->psi;
    if (ba.njobs) {
      p->begin(0, st);
      if ((e = launch_blind_rotate(ba, s->sm_count, st))) return cuda_fail(e, "blind rotate");
      p->end(0, st);
    }
    KsArgs ka{};
    ka.jobs = reinterpret_cast<const KsJob*>(sc + p->off_ks) + p->ks_first[L];
    ka.njobs = static_cast<uint32_t>(lv.ks.size());
    ka.reg = reg;
    ka.nlwe = nlwe;
    ka.ksk = s->ksk;
    if (ka.njobs) {
      p->begin(1, st);
      if (int rc = run_keyswitch(s, ka, sc + p->off_ks_ws, p->ks_chunk, st)) return rc;
      p->end(1, st);
    }
    if (!lv.lin.empty() &&
        (e = launch_linear(reinterpret_cast<const LinJob*>(sc + p->off_lin) + p->lin_first[L],
                           reinterpret_cast<const uint32_t*>(sc + p->off_lin_in) + p->lin_in_first[L],
                           static_cast<uint32_t>(lv.lin.size()), reg, st)))
      return cuda_fail(e, "linear sums");
  }
  if (!p->copy_slots.empty() &&
      (e = launch_copy_rows(reinterpret_cast<const uint32_t*>(sc + p->off_outslots),
                            static_cast<uint32_t>(p->copy_slots.size()), reg, out, st)))
    return cuda_fail(e, "copy out");
  return VLP_OK;
}

int vlp_program_profile(vlp_program* p, int enable) {
  if (!p) return fail(VLP_EINVAL, "null argument");
  p->profile = enable != 0;
  return VLP_OK;
}

int vlp_program_profile_read(vlp_program* p, double* br_ms, double* ks_ms, uint64_t* br_launches,
                             uint64_t* ks_launches, int reset) {
  if (!p) return fail(VLP_EINVAL, "null argument");
  for (auto& ev : p->pending) {
    float ms = 0;
    if (cudaError_t e = cudaEventSynchronize(ev.b)) return cuda_fail(e, "profile event");
    cudaEventElapsedTime(&ms, ev.a, ev.b);
    (ev.kind == 0 ? p->br_ms : p->ks_ms) += ms;
    (ev.kind == 0 ? p->br_launches : p->ks_launches) += 1;
    p->pool.push_back(ev);
  }
  p->pending.clear();
  if (br_ms) *br_ms = p->br_ms;
  if (ks_ms) *ks_ms = p->ks_ms;
  if (br_launches) *br_launches = p->br_launches;
  if (ks_launches) *ks_launches = p->ks_launches;
  if (reset) {
    p->br_ms = p->ks_ms = 0;
    p->br_launches = p->ks_launches = 0;
  }
  return VLP_OK;
}

int vlp_debug_fft_error(uint64_t* err_dev) {
  set_fft_error_monitor(reinterpret_cast<unsigned long long*>(err_dev));
  return VLP_OK;
}

int vlp_debug_route(int engine, int param) {
  return set_br_route(engine, param) == 0 ? VLP_OK : fail(VLP_EINVAL, "vlp_debug_route: bad engine / param");
}

size_t vlp_debug_scratch_bytes(size_t count) {
  const uint32_t chunk = static_cast<uint32_t>(std::min<size_t>(std::max<size_t>(count, 1), kKsChunk));
  return std::max(align256(count * sizeof(BrJob)), align256(count * sizeof(KsJob)) + ks_stage_bytes(chunk));
}

int vlp_debug_blind_rotate(vlp_server* s, const uint32_t* in_dev, size_t count, int steps, uint32_t* acc_dev,
                           void* scratch, uint64_t stream) {
  if (!s || !scratch || (count && (!in_dev || !acc_dev))) return fail(VLP_EINVAL, "null argument");
  if (count == 0) return VLP_OK;
  if (steps < 0 || steps > n) return fail(VLP_EINVAL, "steps out of range");
  cudaError_t e;
  DeviceGuard dg;
  if ((e = dg.set(s->device))) return cuda_fail(e, "cudaSetDevice");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  std::vector<BrJob> jobs(count);
  for (size_t i = 0; i < count; i++) jobs[i] = BrJob{slot(kRegIn0, static_cast<uint32_t>(i)), 0, 0, 1, 0, 0, static_cast<uint32_t>(i)};
  if ((e = cudaMemcpyAsync(scratch, jobs.data(), count * sizeof(BrJob), cudaMemcpyHostToDevice, st)))
    return cuda_fail(e, "upload");
  BrArgs ba{};
  ba.jobs = static_cast<const BrJob*>(scratch);
  ba.njobs = static_cast<uint32_t>(count);
  ba.steps = steps;
  ba.reg.base[kRegIn0] = const_cast<uint32_t*>(in_dev);
  ba.raw_acc = acc_dev;
  ba.bsk = s->bsk_ntt;
  ba.twl_fwd = s->twl_fwd;
  ba.twl_inv = s->twl_inv;
  ba.bskf = s->bsk_fft;
  ba.psi = s->psi;
  if ((e = launch_blind_rotate(ba, s->sm_count, st))) return cuda_fail(e, "blind rotate");
  if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "debug sync");
  return VLP_OK;
}

int vlp_debug_keyswitch(vlp_server* s, const uint32_t* nlwe_dev, size_t count, uint32_t* out_dev, void* scratch,
                        uint64_t stream) {
  if (!s || !scratch || (count && (!nlwe_dev || !out_dev))) return fail(VLP_EINVAL, "null argument");
  if (count == 0) return VLP_OK;
  cudaError_t e;
  DeviceGuard dg;
  if ((e = dg.set(s->device))) return cuda_fail(e, "cudaSetDevice");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  std::vector<KsJob> jobs(count);
  for (size_t i = 0; i < count; i++)
    jobs[i] = KsJob{static_cast<uint32_t>(i), 0xFFFFFFFFu, 0u, slot(kRegOut, static_cast<uint32_t>(i))};
  if ((e = cudaMemcpyAsync(scratch, jobs.data(), count * sizeof(KsJob), cudaMemcpyHostToDevice, st)))
    return cuda_fail(e, "upload");
  KsArgs ka{};
  ka.jobs = static_cast<const KsJob*>(scratch);
  ka.njobs = static_cast<uint32_t>(count);
  ka.reg.base[kRegOut] = out_dev;
  ka.nlwe = nlwe_dev;
  ka.ksk = s->ksk;
  const uint32_t chunk = static_cast<uint32_t>(std::min<size_t>(std::max<size_t>(count, 1), kKsChunk));
  if (int rc = run_keyswitch(s, ka, static_cast<uint8_t*>(scratch) + align256(count * sizeof(KsJob)), chunk, st))
    return rc;
  if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "debug sync");
  return VLP_OK;
}

// ------------------------------------------------------------------------- problem-statement calls
extern "C++" {
static std::string meta_key(const char* kind, const vlp_meta& m, size_t a, size_t b) {
  return std::string(kind) + ":" + std::to_string(m.mode) + "," + std::to_string(m.M) + "," +
         std::to_string(m.l_I) + "," + std::to_string(m.l_S) + "," + std::to_string(m.d) + "," +
         std::to_string(m.flags) + "," + std::to_string(a) + "," + std::to_string(b);
}

constexpr size_t kMaxCachedPrograms = 16;
template <class Make>
static int cached_program(vlp_server* s, const std::string& key, Make make, std::shared_ptr<vlp_program>* out) {
  return no_throw([&] {
    std::lock_guard<std::mutex> lock(s->mu);
    auto it = s->cache.find(key);
    if (it == s->cache.end()) {
      vlp_program* p = nullptr;
      if (int rc = make(&p)) return rc;
      if (s->cache.size() >= kMaxCachedPrograms) {  // evict the least recently used schedule
        auto lru = s->cache.begin();
        for (auto c = s->cache.begin(); c != s->cache.end(); ++c)
          if (c->second.last_use < lru->second.last_use) lru = c;
        s->cache.erase(lru);
      }
      it = s->cache.emplace(key, vlp_server::Cached{std::shared_ptr<vlp_program>(p), 0}).first;
    }
    it->second.last_use = ++s->use_clock;
    *out = it->second.prog;
    return static_cast<int>(VLP_OK);
  });
}
static size_t gate_stage_bytes(int op, size_t count) { return op == VLP_MUX ? 2 * count * kCt * 4 : 0; }
}  // extern "C++"

int vlp_server_workspace_bytes(const vlp_meta* meta, size_t count, size_t* evk_bytes, size_t* db_bytes,
                               size_t* scratch_bytes) {
  if (!meta) return fail(VLP_EINVAL, "null argument");
  size_t per = 0;
  if (int rc = vlp_db_record_cts(meta, &per)) return rc;
  vlp_program* p = nullptr;
  if (int rc = vlp_program_create(nullptr, meta, 0, count, &p)) return rc;
  if (evk_bytes) *evk_bytes = kEvkBytes;
  if (db_bytes) *db_bytes = count * per * kCt * 4;
  if (scratch_bytes) *scratch_bytes = p->bytes;
  delete p;
  return VLP_OK;
}

int vlp_server_eval(vlp_server* s, const vlp_meta* meta, size_t first, size_t count, const uint32_t* query_dev,
                    const uint32_t* db_dev, uint32_t* out_dev, void* scratch, size_t scratch_bytes,
                    uint64_t stream) {
  if (!s || !meta) return fail(VLP_EINVAL, "null argument");
  std::shared_ptr<vlp_program> p;
  if (int rc = cached_program(s, meta_key("eval", *meta, first, count),
                              [&](vlp_program** o) { return vlp_program_create(s, meta, first, count, o); }, &p))
    return rc;
  return vlp_program_eval(p.get(), scratch, scratch_bytes, query_dev, db_dev, out_dev, stream);
}

int vlp_server_eval_host_workspace_bytes(const vlp_meta* meta, size_t count, size_t* scratch_bytes) {
  if (!meta || !scratch_bytes) return fail(VLP_EINVAL, "null argument");
  size_t prog = 0;
  if (int rc = vlp_server_workspace_bytes(meta, count, nullptr, nullptr, &prog)) return rc;
  *scratch_bytes = align256(prog) + align256(query_words(*meta) * meta->l_I * kCt * 4) +
                   align256(static_cast<size_t>(meta->l_S) * kCt * 4);
  return VLP_OK;
}

int vlp_server_eval_host(vlp_server* s, const vlp_meta* meta, size_t first, size_t count, const uint32_t* query_host,
                         const uint32_t* db_dev, uint32_t* out_host, void* scratch, size_t scratch_bytes,
                         uint64_t stream) {
  if (!s || !meta || !query_host || !out_host || !scratch) return fail(VLP_EINVAL, "null argument");
  if (int rc = check_meta(meta)) return rc;
  std::shared_ptr<vlp_program> p;
  if (int rc = cached_program(s, meta_key("eval", *meta, first, count),
                              [&](vlp_program** o) { return vlp_program_create(s, meta, first, count, o); }, &p))
    return rc;
  const size_t qbytes = query_words(*meta) * meta->l_I * kCt * 4, obytes = static_cast<size_t>(meta->l_S) * kCt * 4;
  const size_t prog = align256(p->bytes);
  if (scratch_bytes < prog + align256(qbytes) + align256(obytes)) return fail(VLP_ENOMEM, "scratch too small");
  uint8_t* sc = static_cast<uint8_t*>(scratch);
  uint32_t* qd = reinterpret_cast<uint32_t*>(sc + prog);
  uint32_t* od = reinterpret_cast<uint32_t*>(sc + prog + align256(qbytes));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DeviceGuard dg;
  cudaError_t e;
  if ((e = dg.set(s->device))) return cuda_fail(e, "cudaSetDevice");
  if ((e = cudaMemcpyAsync(qd, query_host, qbytes, cudaMemcpyHostToDevice, st))) return cuda_fail(e, "query upload");
  if (int rc = vlp_program_eval(p.get(), scratch, prog, qd, db_dev, od, stream)) return rc;
  if ((e = cudaMemcpyAsync(out_host, od, obytes, cudaMemcpyDeviceToHost, st))) return cuda_fail(e, "result download");
  if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "server eval sync");
  return VLP_OK;
}

int vlp_server_batch_workspace_bytes(const vlp_meta* meta, size_t count, uint32_t nq, size_t* scratch_bytes) {
  if (!meta || !scratch_bytes) return fail(VLP_EINVAL, "null argument");
  vlp_program* p = nullptr;
  if (int rc = vlp_program_create_queries(nullptr, meta, 0, count, nq, &p)) return rc;
  *scratch_bytes = p->bytes;
  delete p;
  return VLP_OK;
}

int vlp_server_eval_batch(vlp_server* s, const vlp_meta* meta, uint32_t nq, size_t first, size_t count,
                          const uint32_t* queries_dev, const uint32_t* db_dev, uint32_t* out_dev, void* scratch,
                          size_t scratch_bytes, uint64_t stream) {
  if (!s || !meta) return fail(VLP_EINVAL, "null argument");
  std::shared_ptr<vlp_program> p;
  if (int rc = cached_program(s, meta_key("batch", *meta, first, count) + "," + std::to_string(nq),
                              [&](vlp_program** o) { return vlp_program_create_queries(s, meta, first, count, nq, o); },
                              &p))
    return rc;
  return vlp_program_eval(p.get(), scratch, scratch_bytes, queries_dev, db_dev, out_dev, stream);
}

int vlp_server_combine_workspace_bytes(const vlp_meta* meta, uint32_t G, size_t* scratch_bytes) {
  if (!meta || !scratch_bytes) return fail(VLP_EINVAL, "null argument");
  vlp_program* p = nullptr;
  if (int rc = vlp_program_create_combine(nullptr, meta, G, &p)) return rc;
  *scratch_bytes = p->bytes;
  delete p;
  return VLP_OK;
}

int vlp_server_combine(vlp_server* s, const vlp_meta* meta, uint32_t G, const uint32_t* partials_dev,
                       uint32_t* out_dev, void* scratch, size_t scratch_bytes, uint64_t stream) {
  if (!s || !meta) return fail(VLP_EINVAL, "null argument");
  std::shared_ptr<vlp_program> p;
  if (int rc = cached_program(s, meta_key("combine", *meta, G, 0),
                              [&](vlp_program** o) { return vlp_program_create_combine(s, meta, G, o); }, &p))
    return rc;
  return vlp_program_eval(p.get(), scratch, scratch_bytes, partials_dev, nullptr, out_dev, stream);
}

int vlp_gate_batch_workspace_bytes(int op, size_t count, size_t* scratch_bytes) {
  if (!scratch_bytes) return fail(VLP_EINVAL, "null argument");
  if (count == 0) {  // an empty batch needs no scratch (vlp_gate_batch is a no-op)
    *scratch_bytes = 0;
    return VLP_OK;
  }
  vlp_program* p = nullptr;
  if (int rc = vlp_program_create_gates(nullptr, op, count, &p)) return rc;
  *scratch_bytes = align256(p->bytes) + gate_stage_bytes(op, count);
  delete p;
  return VLP_OK;
}

int vlp_gate_batch(vlp_server* s, int op, const uint32_t* a_dev, const uint32_t* b_dev, const uint32_t* c_dev,
                   uint32_t* out_dev, size_t count, void* scratch, size_t scratch_bytes, uint64_t stream) {
  if (!s || !scratch || (count && (!a_dev || !b_dev || !out_dev || (op == VLP_MUX && !c_dev))))
    return fail(VLP_EINVAL, "null argument");
  if (count == 0) return VLP_OK;
  std::shared_ptr<vlp_program> p;
  if (int rc = cached_program(s, "gates:" + std::to_string(op) + "," + std::to_string(count),
                              [&](vlp_program** o) { return vlp_program_create_gates(s, op, count, o); }, &p))
    return rc;
  const size_t prog_bytes = align256(p->bytes);
  if (scratch_bytes < prog_bytes + gate_stage_bytes(op, count)) return fail(VLP_ENOMEM, "scratch too small");
  const uint32_t* in1 = b_dev;
  if (op == VLP_MUX) {  // the program reads c right after b: stage both behind the program's scratch
    uint32_t* st_bc = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + prog_bytes);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e;
    DeviceGuard dg;
  if ((e = dg.set(s->device))) return cuda_fail(e, "cudaSetDevice");
    if ((e = cudaMemcpyAsync(st_bc, b_dev, count * kCt * 4, cudaMemcpyDeviceToDevice, st)) ||
        (e = cudaMemcpyAsync(st_bc + count * kCt, c_dev, count * kCt * 4, cudaMemcpyDeviceToDevice, st)))
      return cuda_fail(e, "stage mux operands");
    in1 = st_bc;
  }
  return vlp_program_eval(p.get(), scratch, scratch_bytes, a_dev, in1, out_dev, stream);
}

void vlp_free_server(vlp_server* s) { delete s; }
void vlp_free_program(vlp_program* p) { delete p; }

}  // extern "C"
