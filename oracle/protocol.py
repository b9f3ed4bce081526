"""oracle/protocol.py -- TEST INFRASTRUCTURE ONLY.

Client/server preprocessing of the VeLoPIR protocol, plainly:
* alg:PubKeyGen: fresh TLWE(0) per record bit, pk^I then pk^S per record, in the listing's
  loop order (bit j outer, coordinate word k inner), object numbering per DESIGN.md section 3 (R17).
* alg:ServerEnc: ct = (0, Ecd(bit)) + pk sample.
* query encryption and decryption of the l_S result bits.
"""
from __future__ import annotations

import numpy as np

from . import KIND_PK, KIND_QUERY, MU, SIGMA_LWE, OracleKeys, n
from .circuits import MODE_COV, MODE_IDM, MODE_INTV


def record_words(mode: int, d: int) -> int:
    """Bound words per record (R17): interval 2d, CoV d, IdM 1."""
    return 2 * d if mode == MODE_INTV else (d if mode == MODE_COV else 1)


def query_words(mode: int, d: int) -> int:
    return 1 if mode == MODE_IDM else d


def bits_of(v: int, l: int):
    """LSB first (R20)."""
    return [(int(v) >> j) & 1 for j in range(l)]


def pk_object(i: int, local: int, W: int, l_I: int, l_S: int) -> int:
    return i * (W * l_I + l_S) + local


def pubkeygen_record(keys: OracleKeys, seed: int, i: int, W: int, l_I: int, l_S: int):
    """alg:PubKeyGen body for record i: pk^I[j][k] (j < l_I, k < W), then pk^S[j] (j < l_S)."""
    pkI = [[None] * W for _ in range(l_I)]
    for j in range(l_I):
        for k in range(W):
            pkI[j][k] = keys.encrypt(0, seed, pk_object(i, j * W + k, W, l_I, l_S), KIND_PK, SIGMA_LWE)
    pkS = [keys.encrypt(0, seed, pk_object(i, W * l_I + j, W, l_I, l_S), KIND_PK, SIGMA_LWE)
           for j in range(l_S)]
    return pkI, pkS


def ecd_add(pk: np.ndarray, bit: int) -> np.ndarray:
    ct = pk.copy()
    ct[n] = np.uint32((int(ct[n]) + (MU if bit else (0x100000000 - MU))) & 0xFFFFFFFF)
    return ct


def server_enc_record(keys: OracleKeys, seed: int, i: int, words, payload: int, l_I: int, l_S: int):
    """alg:ServerEnc body for record i: returns (record word ciphertexts [W][l_I], payload [l_S])."""
    W = len(words)
    pkI, pkS = pubkeygen_record(keys, seed, i, W, l_I, l_S)
    rec = [[ecd_add(pkI[j][k], bits_of(words[k], l_I)[j]) for j in range(l_I)] for k in range(W)]
    pay = [ecd_add(pkS[j], bits_of(payload, l_S)[j]) for j in range(l_S)]
    return rec, pay


def encrypt_query(keys: OracleKeys, values, l_I: int, seed: int):
    """Enc_s(x), Enc_s(y): word w bit j is object w*l_I + j of the query domain."""
    return [[keys.encrypt(b, seed, w * l_I + j, KIND_QUERY, SIGMA_LWE) for j, b in enumerate(bits_of(v, l_I))]
            for w, v in enumerate(values)]


def decrypt_bits(keys: OracleKeys, cts) -> int:
    v = 0
    for j, ct in enumerate(cts):
        v |= keys.decrypt(ct) << j
    return v
