/* Plain-C user of the server half of the C ABI (include/vlp.h) on a GPU: device memory from the CUDA runtime
 * (the library never allocates it), vlp_server_create, vlp_gate_batch (8 NAND gates), vlp_server_eval on two
 * record shards + vlp_server_combine (G = 2) versus one vlp_server_eval over all records: the two
 * results are byte-identical (R15) and decrypt to the plain predicate (R = XOR of the matching payloads); and
 * vlp_server_eval_host (host query in, host result out) gives the same bytes.
 * Built and run by tests/test_c_abi.py (-m gpu) against libvlp.so. */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "vlp.h"

#define CHECK(x)                                                         \
  do {                                                                   \
    int rc_ = (x);                                                       \
    if (rc_ != VLP_OK) {                                                 \
      fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, vlp_last_error()); \
      return 1;                                                          \
    }                                                                    \
  } while (0)
#define CUDA(x)                                                              \
  do {                                                                       \
    cudaError_t e_ = (x);                                                    \
    if (e_ != cudaSuccess) {                                                 \
      fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));        \
      return 1;                                                              \
    }                                                                        \
  } while (0)

static void* dev_alloc(size_t bytes) {
  void* p = NULL;
  if (cudaMalloc(&p, bytes ? bytes : 256) != cudaSuccess) return NULL;
  cudaMemset(p, 0, bytes ? bytes : 256);
  return p;
}

int main(void) {
  const size_t ct_bytes = VLP_CT_STRIDE * 4;
  vlp_sk* sk = NULL;
  vlp_evk* evk = NULL;
  CHECK(vlp_keygen(11, NULL, &sk, &evk));
  const size_t evk_bytes = vlp_server_evk_bytes();
  void* evk_dev = dev_alloc(evk_bytes);
  if (!evk_dev) return 2;
  vlp_server* srv = NULL;
  CHECK(vlp_server_create(0, evk, evk_dev, evk_bytes, 0, &srv));

  /* ---- 8 NAND gates on fresh encryptions */
  enum { G = 8 };
  uint8_t xa[G], xb[G], got[G];
  for (int i = 0; i < G; i++) {
    xa[i] = (uint8_t)(i & 1);
    xb[i] = (uint8_t)((i >> 1) & 1);
  }
  uint32_t* ha = (uint32_t*)calloc(G, ct_bytes);
  uint32_t* hb = (uint32_t*)calloc(G, ct_bytes);
  uint32_t* ho = (uint32_t*)calloc(G, ct_bytes);
  CHECK(vlp_encrypt_bits(sk, xa, G, 5, 0, ha));
  CHECK(vlp_encrypt_bits(sk, xb, G, 5, G, hb));
  uint32_t *da = (uint32_t*)dev_alloc(G * ct_bytes), *db = (uint32_t*)dev_alloc(G * ct_bytes),
           *dout = (uint32_t*)dev_alloc(G * ct_bytes);
  CUDA(cudaMemcpy(da, ha, G * ct_bytes, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(db, hb, G * ct_bytes, cudaMemcpyHostToDevice));
  size_t gsb = 0;
  CHECK(vlp_gate_batch_workspace_bytes(VLP_NAND, G, &gsb));
  void* gs = dev_alloc(gsb);
  CHECK(vlp_gate_batch(srv, VLP_NAND, da, db, NULL, dout, G, gs, gsb, 0));
  CUDA(cudaMemcpy(ho, dout, G * ct_bytes, cudaMemcpyDeviceToHost));
  CHECK(vlp_decrypt_bits(sk, ho, G, got));
  for (int i = 0; i < G; i++)
    if (got[i] != (uint8_t)(1 - (xa[i] & xb[i]))) {
      fprintf(stderr, "NAND %d wrong\n", i);
      return 3;
    }

  /* ---- a 4-record IntV instance: two shards + combine == one evaluation */
  vlp_meta m = {VLP_MODE_INTV, 4, 4, 3, 1, VLP_CONFIG_FLAGS};
  const uint64_t words[8] = {2, 9, 0, 5, 4, 4, 3, 15}; /* [lo, hi] per record */
  const uint64_t pays[4] = {5, 3, 6, 1};
  const uint64_t x = 4; /* lo <= 4 <= hi for all four records -> R = 5 ^ 3 ^ 6 ^ 1 */
  size_t per = 0;
  CHECK(vlp_db_record_cts(&m, &per));
  vlp_pk* pk = NULL;
  CHECK(vlp_pubkeygen(sk, &m, 99, 0, 4, &pk));
  uint32_t* hdb = (uint32_t*)calloc(4 * per, ct_bytes);
  CHECK(vlp_server_encrypt_db(pk, words, pays, hdb));
  vlp_free_pk(pk);
  uint32_t* hq = (uint32_t*)calloc(m.l_I, ct_bytes);
  CHECK(vlp_encrypt_query(sk, &m, &x, 7, hq));
  uint32_t *ddb = (uint32_t*)dev_alloc(4 * per * ct_bytes), *dq = (uint32_t*)dev_alloc(m.l_I * ct_bytes);
  CUDA(cudaMemcpy(ddb, hdb, 4 * per * ct_bytes, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(dq, hq, m.l_I * ct_bytes, cudaMemcpyHostToDevice));
  size_t sb_all = 0, sb_half = 0, sb_comb = 0;
  CHECK(vlp_server_workspace_bytes(&m, 4, NULL, NULL, &sb_all));
  CHECK(vlp_server_workspace_bytes(&m, 2, NULL, NULL, &sb_half));
  CHECK(vlp_server_combine_workspace_bytes(&m, 2, &sb_comb));
  void* s_all = dev_alloc(sb_all);
  void* s_half = dev_alloc(sb_half);
  void* s_comb = dev_alloc(sb_comb);
  uint32_t *dall = (uint32_t*)dev_alloc(m.l_S * ct_bytes), *dpart = (uint32_t*)dev_alloc(2 * m.l_S * ct_bytes),
           *dcomb = (uint32_t*)dev_alloc(m.l_S * ct_bytes);
  CHECK(vlp_server_eval(srv, &m, 0, 4, dq, ddb, dall, s_all, sb_all, 0));
  /* each shard reads its own records: the DB pointer of shard 1 starts at record 2 */
  CHECK(vlp_server_eval(srv, &m, 0, 2, dq, ddb, dpart, s_half, sb_half, 0));
  CHECK(vlp_server_eval(srv, &m, 2, 2, dq, ddb + 2 * per * VLP_CT_STRIDE, dpart + m.l_S * VLP_CT_STRIDE, s_half,
                        sb_half, 0));
  CHECK(vlp_server_combine(srv, &m, 2, dpart, dcomb, s_comb, sb_comb, 0));
  CUDA(cudaDeviceSynchronize());
  uint32_t* hall = (uint32_t*)calloc(m.l_S, ct_bytes);
  uint32_t* hcomb = (uint32_t*)calloc(m.l_S, ct_bytes);
  CUDA(cudaMemcpy(hall, dall, m.l_S * ct_bytes, cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(hcomb, dcomb, m.l_S * ct_bytes, cudaMemcpyDeviceToHost));
  if (memcmp(hall, hcomb, m.l_S * ct_bytes) != 0) {
    fprintf(stderr, "sharded + combine != single evaluation\n");
    return 4;
  }
  /* the same query through the host-buffer call: query from host memory, result to host memory */
  size_t sb_host = 0;
  CHECK(vlp_server_eval_host_workspace_bytes(&m, 4, &sb_host));
  void* s_host = dev_alloc(sb_host);
  uint32_t* hhost = (uint32_t*)calloc(m.l_S, ct_bytes);
  CHECK(vlp_server_eval_host(srv, &m, 0, 4, hq, ddb, hhost, s_host, sb_host, 0));
  if (memcmp(hall, hhost, m.l_S * ct_bytes) != 0) {
    fprintf(stderr, "vlp_server_eval_host != vlp_server_eval\n");
    return 6;
  }
  uint8_t rbits[3];
  uint64_t value = 0;
  CHECK(vlp_decrypt_result(sk, hall, m.l_S, rbits, &value));
  uint64_t want = 0; /* the plain predicate: XOR of the payloads of the records with lo <= x <= hi */
  for (int i = 0; i < 4; i++)
    if (words[2 * i] <= x && x <= words[2 * i + 1]) want ^= pays[i];
  if (value != want) {
    fprintf(stderr, "R = %llu, want %llu\n", (unsigned long long)value, (unsigned long long)want);
    return 5;
  }
  vlp_free_server(srv);
  vlp_free_sk(sk);
  vlp_free_evk(evk);
  printf("c abi server ok: NAND x%d, IntV M=4 sharded x2 + combine == single == host-buffer call, R=%llu\n", G,
         (unsigned long long)value);
  return 0;
}
