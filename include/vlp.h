/*
 * vlp.h -- C ABI of the B200 VeLoPIR gate-bootstrapping engine (libvlp.so).
 *
 * Citation key: P:n = /root/reference/PAPER.md line n; Rk = DESIGN.md section 3 reading k.
 * The calls follow the paper's problem statement: keygen, encrypt query, server
 * evaluation (alg:VeLoPIR P:307-329), decrypt; plus the preprocessing the paper's
 * server performs (alg:PubKeyGen P:194-219, alg:ServerEnc P:223-247) and the raw gate batch of
 * BASELINE.json config 5.
 *
 * Conventions
 *  - Every call returns an int status: VLP_OK (0) or a negative VLP_E* code; no exceptions cross the
 *    ABI.  vlp_last_error() returns a thread-local description of the last failure.
 *  - Handles (vlp_sk, vlp_evk, vlp_pk, vlp_server, vlp_program) are opaque and library-owned; free them
 *    with the matching vlp_free_* call.
 *  - Ciphertext buffers are caller-owned arrays uint32_t[count][VLP_CT_STRIDE] (632 words: a[0..629],
 *    b at word 630, one zero pad word), little-endian.  Arguments ending in _dev are device pointers
 *    (CUDA, on the given stream, passed as plain pointers); all others are host pointers.
 *  - Device memory belongs to the caller (PyTorch tensors): the library asks for sizes
 *    (vlp_server_evk_bytes, vlp_program_info) and never allocates device memory itself.
 *  - Streams are passed as uint64_t (a cudaStream_t value; 0 = legacy default stream).  Device calls
 *    are asynchronous on that stream unless stated.
 *  - Everything is deterministic in its seeds (R3).  The library's keys and encryptions are
 *    byte-identical to the test oracle's for the same seeds (tested, not shared code).
 */
#ifndef VLP_H
#define VLP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VLP_N_LWE 630       /* TLWE dimension n, tab:tfhe_params P:1236 */
#define VLP_N_RING 1024     /* ring dimension N */
#define VLP_CT_STRIDE 632   /* words per TLWE ciphertext buffer row (631 + pad) */
#define VLP_NLWE_STRIDE 1028 /* words per N-LWE row (1025 + pad) */

enum {
  VLP_OK = 0,
  VLP_EINVAL = -1,   /* bad argument (null pointer, size out of range) */
  VLP_EMODE = -2,    /* mode / meta mismatch */
  VLP_EWIDTH = -3,   /* width mismatch or l < 2 */
  VLP_ERANGE = -4,   /* plaintext value >= 2^l */
  VLP_EPKUSED = -5,  /* public-key samples already consumed (alg:PubKeyGen samples are single-use) */
  VLP_ECUDA = -6,    /* CUDA runtime error (see vlp_last_error) */
  VLP_ENOMEM = -7,   /* host allocation failed or caller buffer too small */
  VLP_ENODEV = -8    /* no CUDA device / kernel image for this device */
};

/* Modes and flags (readings R11, R12, R14, R15, R19; R23 / R24 are options outside the paper). */
enum { VLP_MODE_INTV = 0, VLP_MODE_COV = 1, VLP_MODE_IDM = 2 };
enum {
  VLP_F_CLOSED_UPPER = 1, /* R12: lo <= x <= hi (CompLE on the right bound) instead of x < hi */
  VLP_F_UNSIGNED = 2,     /* R11: unsigned comparators (final MUX selects ct2[l-1]) */
  VLP_F_EQ_TREE = 4,      /* R14: alg:HomEqOPT pairwise AND tree instead of the serial HomEQ */
  VLP_F_SUM_TREE = 8,     /* R15: outermost XOR tree instead of the serial HomSum */
  VLP_F_OR_REDUCE = 16,   /* R19: OR instead of XOR in the aggregation */
  VLP_F_PREFIX_COMP = 32, /* R23 (NOT in the paper): log-depth parallel-prefix unsigned
                             comparators (depth 1 + ceil(log2 l) instead of l + 1; more gates; needs UNSIGNED) */
  VLP_F_LINEAR_SUM = 64,  /* R24 (NOT in the paper): linear XOR aggregation -- masked bits
                             in the {0, 1/2} encoding summed without bootstrapping in groups of 64, one refresh
                             bootstrap per group and bit (XOR only: not with OR_REDUCE) */
  VLP_F_KEEP_ALL = 128    /* debug: every intermediate keeps its own scratch row for the whole evaluation (for
                             pure-function parity dumps); by default rows are recycled by liveness, and only
                             the validation bits and masked payloads (vlp_program_node_row) are kept */
};
#define VLP_CONFIG_FLAGS (VLP_F_CLOSED_UPPER | VLP_F_UNSIGNED | VLP_F_EQ_TREE | VLP_F_SUM_TREE)

/* Gate opcodes (R10). */
enum { VLP_AND = 0, VLP_NAND = 1, VLP_OR = 2, VLP_XOR = 3, VLP_XNOR = 4, VLP_MUX = 5 };

/* tab:tfhe_params plus R2's fresh-encryption sigma. */
typedef struct {
  uint32_t n, N, k, bg_bits, ell, ks_base_bits, ks_t;
  double sigma_lwe, sigma_bk, sigma_ks;
} vlp_params;

/* Session meta: M records, l_I location bits (2..32), l_S payload bits (1..128), d coordinates. */
typedef struct {
  uint32_t mode, M, l_I, l_S, d, flags;
} vlp_meta;

typedef struct vlp_sk vlp_sk;
typedef struct vlp_evk vlp_evk;
typedef struct vlp_pk vlp_pk;
typedef struct vlp_server vlp_server;
typedef struct vlp_program vlp_program;

/* Program description (sizes the caller allocates; counts of the compiled level schedule). */
typedef struct {
  uint32_t levels;          /* circuit levels (one BR launch + one KS launch each) */
  uint64_t br, ks;          /* blind rotations (MUX = 2) and key switches per evaluation */
  uint64_t gates;           /* gates (MUX = 1) */
  uint64_t in0_cts, in1_cts; /* ciphertexts read from in0 (query / a) and in1 (DB / b) */
  uint64_t out_cts;         /* ciphertexts written to out */
  uint64_t scratch_bytes;   /* device scratch the caller must provide */
  uint64_t max_level_br;    /* widest level */
  uint32_t kernel_launches; /* kernels launched per evaluation */
  uint64_t table_bytes;     /* job tables every evaluation copies host -> device into scratch */
} vlp_program_info;

const char* vlp_last_error(void);

/* Fills the 128-bit parameter set of tab:tfhe_params; sigma_lwe = 2^-15 (R2). */
int vlp_params_tfhe128(vlp_params* out);

/* Randomness.  Every seeded call (a `seed` argument) is byte-reproducible from its 64-bit seed through the counter
 * PRNG of R3: the test / benchmark mode, whose keys and noise are only as secret as the
 * seed -- do NOT use it to protect data.  The *_secure calls draw a fresh 256-bit key from the OS (getrandom) per
 * call and generate every mask, noise and key bit with ChaCha20 (RFC 8439) under it; the algorithms and layouts are
 * the same.  VLP_EINVAL if the OS has no randomness to give. */

/* KeyGen.  Host.  s in B^630, ring key z in B^1024 (R4), bsk (630 TRGSW,
 * rows r = u*3 + j, R4) and ksk ([1024][8][3] TLWE samples, R6), all from `seed` (R3).
 * Only the default parameter set is supported (VLP_EINVAL otherwise). */
int vlp_keygen(uint64_t seed, const vlp_params* params, vlp_sk** sk, vlp_evk** evk);
/* KeyGen from OS randomness (see "Randomness"). */
int vlp_keygen_secure(const vlp_params* params, vlp_sk** sk, vlp_evk** evk);
/* Copies of the key material for the byte-equality tests: s[630], z[1024] as 0/1 words;
 * bsk[630][6][2][1024] torus32; ksk[1024][8][3][631] torus32.  Any pointer may be NULL. */
int vlp_sk_export(const vlp_sk* sk, uint32_t* s, uint32_t* z);
int vlp_evk_export(const vlp_evk* evk, uint32_t* bsk, uint32_t* ksk);

/* TLWE encryption of `count` bits under s with the fresh-encryption domains (R3), objects
 * obj0 .. obj0+count-1; out: host [count][632]. */
int vlp_encrypt_bits(const vlp_sk* sk, const uint8_t* bits, size_t count, uint64_t seed, uint64_t obj0,
                     uint32_t* out);
/* Query encryption: values[w] for w < query words (IntV: d coordinates; CoV: d; IdM: 1),
 * l_I bits each, LSB first (R20); object w*l_I + j of the query domains.  out: host [words*l_I][632].
 * VLP_ERANGE if a value >= 2^l_I. */
int vlp_encrypt_query(const vlp_sk* sk, const vlp_meta* meta, const uint64_t* values, uint64_t seed,
                      uint32_t* out);
/* The same encryptions from OS randomness (see "Randomness"). */
int vlp_encrypt_query_secure(const vlp_sk* sk, const vlp_meta* meta, const uint64_t* values, uint32_t* out);
int vlp_encrypt_bits_secure(const vlp_sk* sk, const uint8_t* bits, size_t count, uint32_t* out);
/* Dec: bit = [int32(b - <a, s>) > 0] (ties -> 0, R18).  Host. */
int vlp_decrypt_bits(const vlp_sk* sk, const uint32_t* ct, size_t count, uint8_t* bits_out);

/* alg:PubKeyGen for records [first, first+count): single-use TLWE(0) samples, pk^I
 * (R17 counts: words W = 2d interval, d CoV, 1 IdM; bit j outer, word k inner as in the listing)
 * then pk^S, materialised on the host (the client sends them to the server).  Multi-threaded. */
int vlp_pubkeygen(const vlp_sk* sk, const vlp_meta* meta, uint64_t seed, size_t first, size_t count,
                  vlp_pk** pk);
/* PubKeyGen from OS randomness (see "Randomness"). */
int vlp_pubkeygen_secure(const vlp_sk* sk, const vlp_meta* meta, size_t first, size_t count, vlp_pk** pk);
/* Test hook: one ChaCha20 block (RFC 8439 section 2.3) -- key[8], counter, nonce[3] -> out[16] (words, little
 * endian), to pin the secure generator against an independent implementation. */
int vlp_debug_chacha20_block(const uint32_t* key, uint32_t counter, const uint32_t* nonce, uint32_t* out);
/* Test hook: the calling thread's NEXT *_secure call (host or device) uses key[8] instead of a getrandom key, then
 * the hook is cleared.  Lets a test compare a device secure call with the host secure call under one key; never
 * use it to protect data (the key is whatever the caller passed).  Disabled (VLP_EINVAL) unless the environment
 * variable VLP_TEST_HOOKS is "1". */
int vlp_debug_next_secure_key(const uint32_t* key);
/* Ciphertexts per record in the encrypted DB: W * l_I + l_S. */
int vlp_db_record_cts(const vlp_meta* meta, size_t* per_record);
/* alg:ServerEnc for the pk's records: ct = (0, Ecd(bit)) + pk sample.
 * words: [count][W] plaintext bound words (IntV: lo,hi per axis; CoV: loc per axis; IdM: id);
 * payloads: [count][ceil(l_S / 64)] little-endian 64-bit words (value < 2^l_S; one word for l_S <= 64).
 * out: host [count][per_record][632] in the order word-major
 * location bits (word k bit j at row k*l_I + j) then payload bits (row W*l_I + j).  Consumes the pk:
 * a second call returns VLP_EPKUSED.  Server side: needs no secret key. */
int vlp_server_encrypt_db(vlp_pk* pk, const uint64_t* words, const uint64_t* payloads, uint32_t* out);

/* ---- GPU preprocessing, role-separated like P:192: the client's KeyGen and PubKeyGen take
 * the secret key, the server's ServerEnc takes only public-key samples.  Each is byte-identical to its host call;
 * the Gaussian noise is drawn on the host (the same libm Box-Muller: device libm may round differently), the
 * counter-PRNG mask words, ring products and inner products run on `stream`'s device.  Synchronous. */

/* Device KeyGen (client): the same sk / evk as vlp_keygen(seed, params), byte for byte -- the
 * bootstrapping key's masks and ring products a*z (R4, O7) and the key-switching key's masks and <a, s> (O10) are
 * computed on the device and copied back into the host evk.  scratch_dev >= vlp_keygen_device_scratch_bytes(). */
size_t vlp_keygen_device_scratch_bytes(void);
int vlp_keygen_device(uint64_t seed, const vlp_params* params, void* scratch_dev, size_t scratch_bytes,
                      uint64_t stream, vlp_sk** sk, vlp_evk** evk);
/* The same from OS randomness (see "Randomness"): equal, byte for byte, to vlp_keygen_secure under the same
 * ChaCha20 key (the device draws the masks from ChaCha20 blocks, the host the secret keys and the noise). */
int vlp_keygen_device_secure(const vlp_params* params, void* scratch_dev, size_t scratch_bytes, uint64_t stream,
                             vlp_sk** sk, vlp_evk** evk);
/* Device PubKeyGen (client; alg:PubKeyGen P:194-219): the single-use TLWE(0) samples of records
 * [first, first+count) written to pk_dev ([count][per_record][632], the row order of vlp_server_encrypt_db),
 * byte-identical to vlp_pubkeygen(sk, meta, seed, first, count)'s samples.  The copy of s placed in scratch_dev
 * is zeroed before the call returns.  scratch_dev >= vlp_pubkeygen_device_scratch_bytes(meta, count). */
int vlp_pubkeygen_device_scratch_bytes(const vlp_meta* meta, size_t count, size_t* scratch_bytes);
int vlp_pubkeygen_device(const vlp_sk* sk, const vlp_meta* meta, uint64_t seed, size_t first, size_t count,
                         uint32_t* pk_dev, void* scratch_dev, size_t scratch_bytes, uint64_t stream);
/* The same from OS randomness: equal to vlp_pubkeygen_secure's samples under the same ChaCha20 key. */
int vlp_pubkeygen_device_secure(const vlp_sk* sk, const vlp_meta* meta, size_t first, size_t count, uint32_t* pk_dev,
                                void* scratch_dev, size_t scratch_bytes, uint64_t stream);
/* Device ServerEnc (server; alg:ServerEnc P:223-247): out_dev = pk_dev + (0, Ecd(bit)) for every row of records
 * [0, count) of the public-key samples (out_dev may equal pk_dev).  Needs no secret key.  words / payloads as in
 * vlp_server_encrypt_db (host, range-checked: VLP_ERANGE).  scratch_dev >=
 * vlp_server_encrypt_db_device_scratch_bytes(meta, count). */
int vlp_server_encrypt_db_device_scratch_bytes(const vlp_meta* meta, size_t count, size_t* scratch_bytes);
int vlp_server_encrypt_db_device(const vlp_meta* meta, size_t count, const uint32_t* pk_dev, const uint64_t* words,
                                 const uint64_t* payloads, uint32_t* out_dev, void* scratch_dev, size_t scratch_bytes,
                                 uint64_t stream);

/* load records: the server's ServerEnc of a received host pk (vlp_pubkeygen / _secure) straight into
 * device memory -- the pk's samples are uploaded into db_dev ([pk count][per_record][632], record pk->first at row
 * 0) and (0, Ecd(bit)) is added on the device; marks the pk used (a second call: VLP_EPKUSED) and frees its host
 * samples.  words / payloads as in vlp_server_encrypt_db.  scratch_dev as vlp_server_encrypt_db_device.
 * Synchronous.  Needs no secret key. */
int vlp_server_load_records(vlp_pk* pk, const uint64_t* words, const uint64_t* payloads, uint32_t* db_dev,
                            void* scratch_dev, size_t scratch_bytes, uint64_t stream);

/* Device PubKeyGen + ServerEnc fused (both roles on one machine, e.g. to build benchmark DBs): the encrypted DB of records [first, first+count) written straight to out_dev ([count][per_record]
 * [632], the vlp_server_encrypt_db layout), byte-identical to vlp_pubkeygen(sk, meta, pk_seed, first, count)
 * followed by vlp_server_encrypt_db.  The Gaussian noise is drawn on the host (the same libm Box-Muller),
 * the PRNG mask words and inner products on the device.  words / payloads as in vlp_server_encrypt_db.
 * scratch_dev >= vlp_encrypt_db_device_scratch_bytes(meta, count); the copy of s in it is zeroed before
 * returning.  Synchronous. */
int vlp_encrypt_db_device_scratch_bytes(const vlp_meta* meta, size_t count, size_t* scratch_bytes);
int vlp_encrypt_db_device(const vlp_sk* sk, const vlp_meta* meta, uint64_t pk_seed, size_t first, size_t count,
                          const uint64_t* words, const uint64_t* payloads, uint32_t* out_dev, void* scratch_dev,
                          size_t scratch_bytes, uint64_t stream);

/* Server: the evaluation key on one device.  evk_dev must hold vlp_server_evk_bytes() bytes (device
 * memory on `device`); the bootstrapping key is uploaded and converted to the NTT domain in place
 * (kernel vlp_bsk_convert_kernel), the key-switching key uploaded.  Synchronous. */
size_t vlp_server_evk_bytes(void);
int vlp_server_create(int device, const vlp_evk* evk, void* evk_dev, size_t evk_bytes, uint64_t stream,
                      vlp_server** out);

/* Compile VeLoPIR (alg:VeLoPIR with the readings of `meta->flags`) for records [first, first+count)
 * into a level schedule (one BR launch + one KS launch per level, every independent gate of a level
 * across all records in one batch; MUX halves hoisted).  The shard's XOR tree stops at its root; the
 * l_S root ciphertexts are written to `out`.  in0 = query ciphertexts (vlp_encrypt_query layout),
 * in1 = the shard's encrypted DB (vlp_server_encrypt_db layout, record `first` at row 0).
 * `server` may be NULL to compile only (vlp_program_get_info works; vlp_program_eval fails). */
int vlp_program_create(vlp_server* server, const vlp_meta* meta, size_t first, size_t count,
                       vlp_program** out);
/* Multi-query packing: nq queries against the same shard in one schedule, so every
 * level launch carries the gates of all nq queries.  in0 = nq query sets back to back ([nq][query cts]),
 * out = [nq][l_S] result ciphertexts; each query's result is byte-identical to its single-query evaluation
 * (ciphertexts do not depend on the schedule).  nq in [1, 4096]. */
int vlp_program_create_queries(vlp_server* server, const vlp_meta* meta, size_t first, size_t count, uint32_t nq,
                               vlp_program** out);
/* A single level of `count` independent gates `op` (config 5): out[i] = op(in0[i], in1[i]); for
 * VLP_MUX, out[i] = MUX(in0[i], in1[i], in2[i]) where in2 = in1 + count rows. */
int vlp_program_create_gates(vlp_server* server, int op, size_t count, vlp_program** out);
/* The top log2(G) levels of the aggregation tree over G shard roots (in0: [G][l_S][632], shards in
 * rank order; G a power of two); writes the l_S result ciphertexts to out (R15). */
int vlp_program_create_combine(vlp_server* server, const vlp_meta* meta, uint32_t G, vlp_program** out);
int vlp_program_get_info(const vlp_program* prog, vlp_program_info* info);
/* Device slot (row index in the scratch intermediate region) holding a named node of a circuit
 * program, for sampled parity dumps: kind 0 = validation bit v of record r (bit ignored), kind 1 =
 * masked payload bit (r, bit).  Returns VLP_EINVAL if absent. */
int vlp_program_node_row(const vlp_program* prog, int kind, size_t record, uint32_t bit, uint64_t* row);
/* The compiled schedule, for pure-function parity checks (SURVEY 4 layer 3): level `level`'s gate
 * bootstraps and key switches.  vlp_br_job: output c = (0, k0) + ax*in[x] + ay*in[y] is bootstrapped into
 * N-LWE row `row`; vlp_ks_job: out slot = KS((0, add) + nlwe[n0] (+ nlwe[n1] if n1 != 0xFFFFFFFF)).  Slot ids
 * are region << 28 | row with regions 0 = in0, 1 = in1, 2 = intermediates (vlp_program_intermediate_offset),
 * 3 = out.  Pass NULL arrays to get the counts. */
typedef struct {
  uint32_t x, y, k0;
  int8_t ax, ay;
  uint16_t tv; /* test vector of the bootstrap: 0 -> 1/8 (R8), 1 -> 1/4 (R24 linear aggregation) */
  uint32_t row;
} vlp_br_job;
typedef struct {
  uint32_t n0, n1, add, out;
} vlp_ks_job;
int vlp_program_level_jobs(const vlp_program* prog, uint32_t level, vlp_br_job* br, uint64_t* nbr, vlp_ks_job* ks,
                           uint64_t* nks);
/* R24 linear jobs of level `level` (run after its key switches): jobs [n][4] = (out slot, first, count, 0),
 * out = sum of the input slots inputs[first .. first + count) mod 2^32.  NULL arrays: counts only. */
int vlp_program_level_linear(const vlp_program* prog, uint32_t level, uint32_t* jobs, uint64_t* njobs,
                             uint32_t* inputs, uint64_t* ninputs);
/* Pointer to the intermediate region inside `scratch_dev` (rows of 632 words). */
int vlp_program_intermediate_offset(const vlp_program* prog, uint64_t* byte_offset);

/* Evaluate the program on `stream` (asynchronous).  scratch_dev: >= info.scratch_bytes of device
 * memory.  Every call first copies the program's job tables (info.table_bytes, from a pinned host image the
 * library keeps) into the scratch on `stream`, so no state carries over between calls and one buffer may
 * serve several programs in turn; the scratch also holds the intermediates, the N-LWE staging and the
 * key-switch GEMM staging, so two evaluations in flight at the same time need two scratch buffers. */
int vlp_program_eval(vlp_program* prog, void* scratch_dev, size_t scratch_bytes, const uint32_t* in0_dev,
                     const uint32_t* in1_dev, uint32_t* out_dev, uint64_t stream);

/* Per-kernel timing: when enabled, vlp_program_eval records CUDA events on its stream around every
 * blind-rotate launch and every key-switch launch (init + switch); vlp_program_profile_read waits for
 * them and returns the accumulated milliseconds and launch counts (reset != 0 clears the totals). */
int vlp_program_profile(vlp_program* prog, int enable);
int vlp_program_profile_read(vlp_program* prog, double* br_ms, double* ks_ms, uint64_t* br_launches,
                             uint64_t* ks_launches, int reset);

/* Debug / parity entry points (device, asynchronous): blind rotation of `count` TLWE inputs
 * (in_dev [count][632], used as is: no gate linear form) for the first `steps` CMux steps, writing the
 * raw TRLWE accumulators acc_dev [count][2][1024]; and the key switch of N-LWE rows
 * (nlwe_dev [count][1028]) into out_dev [count][632].  scratch_dev: >= vlp_debug_scratch_bytes(count). */
size_t vlp_debug_scratch_bytes(size_t count);
int vlp_debug_blind_rotate(vlp_server* server, const uint32_t* in_dev, size_t count, int steps,
                           uint32_t* acc_dev, void* scratch_dev, uint64_t stream);
int vlp_debug_keyswitch(vlp_server* server, const uint32_t* nlwe_dev, size_t count, uint32_t* out_dev,
                        void* scratch_dev, uint64_t stream);
/* Blind-rotation routing for every later launch in this process (debug / parity tests).
 * Both engines are exact, so the bytes never depend on the route -- the parity tests use this to run every
 * kernel against the oracle.  engine: 0 = default (VLP_BR_ENGINE / VLP_BR_BOOT / VLP_FFT_WARPS from the
 * environment, else the FP64-FFT engine K2F for waves with the NTT latency kernels for narrow tails);
 * 1 = NTT engine only (K2 waves + NTT tails; param != 0 forces one NTT kernel for whole levels, with the
 * VLP_BR_BOOT meaning: 1-5 bootstraps per CTA, -1 latency, -2 2-CTA cluster, -3 6-CTA cluster);
 * 2 = K2F with param warps (1-8) per CTA for whole levels.  Returns VLP_EINVAL on other values. */
int vlp_debug_route(int engine, int param);
/* Test hook (process-wide): while err_dev != NULL, every K2F launch (the FP64 FFT engine)
 * runs its monitoring build and atomically raises *err_dev to the largest distance |V - round(V)| between a limb
 * result and the integer it rounds to, as the bit pattern of a non-negative double (the exactness margin is 1/2).
 * err_dev: caller-owned device memory (8 bytes, zero it first).  NULL turns the monitor off. */
int vlp_debug_fft_error(uint64_t* err_dev);

/* ---- The problem-statement calls (the north star's keygen / encrypt_query / server_eval /
 * decrypt_result).  They wrap the program calls above: the schedule for a (meta, first, count) shard, a
 * gate batch or a combine is compiled on first use and cached in the server (thread-safe); device buffers
 * stay caller-owned. */

/* Sizes of the caller-owned device buffers for vlp_server_eval on a shard of `count` records:
 * evaluation key (vlp_server_evk_bytes), encrypted DB rows (count * per_record * 632 * 4) and scratch
 * (job arrays, intermediates, N-LWE staging).  Host only (compiles the schedule). */
int vlp_server_workspace_bytes(const vlp_meta* meta, size_t count, size_t* evk_bytes, size_t* db_bytes,
                               size_t* scratch_bytes);
/* server_eval (alg:VeLoPIR P:307-329): evaluate the encrypted query (query_dev, vlp_encrypt_query
 * layout) against records [first, first+count) of the encrypted DB (db_dev, record `first` at row 0),
 * writing the shard's l_S aggregate ciphertexts to out_dev.  Asynchronous on `stream`. */
int vlp_server_eval(vlp_server* server, const vlp_meta* meta, size_t first, size_t count,
                    const uint32_t* query_dev, const uint32_t* db_dev, uint32_t* out_dev, void* scratch_dev,
                    size_t scratch_bytes, uint64_t stream);
/* server_eval with HOST query and result buffers (the end-to-end call of one query): copies query_host
 * ([query cts][632] u32, vlp_encrypt_query layout; pinned memory recommended) into scratch, runs vlp_server_eval
 * against the device-resident DB, and copies the l_S result ciphertexts to out_host ([l_S][632]); returns after the
 * result is on the host.  scratch_dev >= vlp_server_eval_host_workspace_bytes(meta, count). */
int vlp_server_eval_host_workspace_bytes(const vlp_meta* meta, size_t count, size_t* scratch_bytes);
int vlp_server_eval_host(vlp_server* server, const vlp_meta* meta, size_t first, size_t count,
                         const uint32_t* query_host, const uint32_t* db_dev, uint32_t* out_host, void* scratch_dev,
                         size_t scratch_bytes, uint64_t stream);
/* server_eval for nq queries at once (multi-query packing): queries_dev [nq][query cts][632],
 * out_dev [nq][l_S][632]; scratch from vlp_server_batch_workspace_bytes. */
int vlp_server_batch_workspace_bytes(const vlp_meta* meta, size_t count, uint32_t nq, size_t* scratch_bytes);
int vlp_server_eval_batch(vlp_server* server, const vlp_meta* meta, uint32_t nq, size_t first, size_t count,
                          const uint32_t* queries_dev, const uint32_t* db_dev, uint32_t* out_dev, void* scratch_dev,
                          size_t scratch_bytes, uint64_t stream);
/* Scratch bytes of vlp_server_combine for G shard roots. */
int vlp_server_combine_workspace_bytes(const vlp_meta* meta, uint32_t G, size_t* scratch_bytes);
/* The top log2(G) XOR-tree levels over the G shard roots partials_dev [G][l_S][632] (rank order, G a power
 * of two): the query's l_S result ciphertexts to out_dev (R15). */
int vlp_server_combine(vlp_server* server, const vlp_meta* meta, uint32_t G, const uint32_t* partials_dev,
                       uint32_t* out_dev, void* scratch_dev, size_t scratch_bytes, uint64_t stream);
/* Scratch bytes of vlp_gate_batch (includes room to stage b and c contiguously for VLP_MUX); 0 for an empty
 * batch, which vlp_gate_batch accepts as a no-op. */
int vlp_gate_batch_workspace_bytes(int op, size_t count, size_t* scratch_bytes);
/* A batch of `count` independent gates (BASELINE config 5): out[i] = op(a[i], b[i]), or for VLP_MUX
 * out[i] = MUX(a[i], b[i], c[i]) = a ? b : c (R10).  c_dev is ignored unless op == VLP_MUX. */
int vlp_gate_batch(vlp_server* server, int op, const uint32_t* a_dev, const uint32_t* b_dev,
                   const uint32_t* c_dev, uint32_t* out_dev, size_t count, void* scratch_dev,
                   size_t scratch_bytes, uint64_t stream);
/* decrypt_result: bit j = [int32(phase of ct[j]) > 0] (R18), LSB first (R20); *value_out (may
 * be NULL) = sum bit_j 2^j for l_S <= 64. */
int vlp_decrypt_result(const vlp_sk* sk, const uint32_t* ct, uint32_t l_S, uint8_t* bits_out, uint64_t* value_out);

void vlp_free_sk(vlp_sk* sk);
void vlp_free_evk(vlp_evk* evk);
void vlp_free_pk(vlp_pk* pk);
void vlp_free_server(vlp_server* server);
void vlp_free_program(vlp_program* prog);

#ifdef __cplusplus
}
#endif
#endif /* VLP_H */
