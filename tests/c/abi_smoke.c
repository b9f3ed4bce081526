/* Plain-C user of the C ABI (include/vlp.h): client-side calls that need no GPU -- parameters, keygen,
 * query encryption, PubKeyGen + ServerEnc, decryption of fresh encryptions, error codes.  Built and run by
 * tests/test_c_abi.py against libvlp.so. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "vlp.h"

#define CHECK(x)                                                       \
  do {                                                                 \
    int rc_ = (x);                                                     \
    if (rc_ != VLP_OK) {                                               \
      fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, vlp_last_error()); \
      return 1;                                                        \
    }                                                                  \
  } while (0)

int main(void) {
  vlp_params p;
  CHECK(vlp_params_tfhe128(&p));
  if (p.n != VLP_N_LWE || p.N != VLP_N_RING) return 2;
  vlp_sk* sk = NULL;
  vlp_evk* evk = NULL;
  CHECK(vlp_keygen(7, &p, &sk, &evk));

  /* fresh encryptions decrypt back */
  uint8_t bits[64], back[64];
  for (int i = 0; i < 64; i++) bits[i] = (uint8_t)((i * 37 + 11) % 3 == 0);
  uint32_t* ct = (uint32_t*)calloc(64 * VLP_CT_STRIDE, 4);
  CHECK(vlp_encrypt_bits(sk, bits, 64, 99, 0, ct));
  CHECK(vlp_decrypt_bits(sk, ct, 64, back));
  for (int i = 0; i < 64; i++)
    if (back[i] != bits[i]) return 3;

  /* an encrypted IntV query and a 3-record DB (PubKeyGen + ServerEnc) */
  vlp_meta m = {VLP_MODE_INTV, 3, 8, 8, 1, VLP_F_CLOSED_UPPER | VLP_F_UNSIGNED | VLP_F_EQ_TREE | VLP_F_SUM_TREE};
  uint64_t x = 77;
  uint32_t* q = (uint32_t*)calloc(8 * VLP_CT_STRIDE, 4);
  CHECK(vlp_encrypt_query(sk, &m, &x, 5, q));
  uint8_t qb[8];
  CHECK(vlp_decrypt_bits(sk, q, 8, qb));
  for (int j = 0; j < 8; j++)
    if (qb[j] != ((x >> j) & 1)) return 4;
  size_t per = 0;
  CHECK(vlp_db_record_cts(&m, &per));
  if (per != 2 * 8 + 8) return 5;
  vlp_pk* pk = NULL;
  CHECK(vlp_pubkeygen(sk, &m, 11, 0, 3, &pk));
  uint64_t words[6] = {10, 90, 100, 200, 70, 77}, pays[3] = {0x5a, 0x11, 0xc3};
  uint32_t* db = (uint32_t*)calloc(3 * per * VLP_CT_STRIDE, 4);
  CHECK(vlp_server_encrypt_db(pk, words, pays, db));
  if (vlp_server_encrypt_db(pk, words, pays, db) != VLP_EPKUSED) return 6; /* single-use samples */
  uint8_t rb[24];
  CHECK(vlp_decrypt_bits(sk, db + (2 * per) * VLP_CT_STRIDE, per, rb)); /* record 2: lo 70, hi 77, 0xc3 */
  for (int j = 0; j < 8; j++)
    if (rb[j] != ((70 >> j) & 1) || rb[8 + j] != ((77 >> j) & 1) || rb[16 + j] != ((0xc3 >> j) & 1)) return 7;

  /* decrypt_result assembles the value LSB first */
  uint8_t rbits[8];
  uint64_t value = 0;
  CHECK(vlp_decrypt_result(sk, db + (2 * per + 16) * VLP_CT_STRIDE, 8, rbits, &value));
  if (value != 0xc3) return 8;

  /* errors: bad width, out-of-range value */
  vlp_meta bad = m;
  bad.l_I = 1;
  if (vlp_encrypt_query(sk, &bad, &x, 5, q) != VLP_EWIDTH) return 9;
  uint64_t big = 256;
  if (vlp_encrypt_query(sk, &m, &big, 5, q) != VLP_ERANGE) return 10;

  vlp_free_pk(pk);
  vlp_free_sk(sk);
  vlp_free_evk(evk);
  free(ct);
  free(q);
  free(db);
  printf("c abi ok\n");
  return 0;
}
