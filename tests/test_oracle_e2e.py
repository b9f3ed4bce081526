"""P8: the oracle end to end on config 1 (IntV 1D tiny): keygen -> PubKeyGen/ServerEnc -> query encryption
-> alg:VeLoPIR on TFHE ciphertexts -> decryption equals the plain predicate (thm:VeLoPIR),
and every per-record validation bit v_i decrypts to that record's predicate (thm:bb1)."""
import numpy as np

import oracle as O
from oracle import circuits as C
from oracle import protocol as P
from synth import make_workload


def run_oracle_config(wl, keys, query_seed=7):
    q = P.encrypt_query(keys, wl.query, wl.l_I, query_seed)
    recs, pays = [], []
    for i in range(wl.M):
        r, p = P.server_enc_record(keys, wl.key_seed + 1, i, [int(v) for v in wl.records[i]], int(wl.payloads[i]),
                                   wl.l_I, wl.l_S)
        recs.append(r)
        pays.append(p)
    B = C.TfheBackend(keys)
    R, vs, masked = C.velopir(B, wl.mode, q, recs, pays, wl.l_I, wl.d, wl.l_S, wl.flags)
    return R, vs, masked


def test_config1_end_to_end():
    wl = make_workload(1)
    keys = O.OracleKeys(wl.key_seed)
    R, vs, masked = run_oracle_config(wl, keys)
    got = P.decrypt_bits(keys, R)
    want = C.plain_result(wl.mode, wl.query, [list(map(int, r)) for r in wl.records], wl.payloads, wl.d, wl.flags)
    assert got == want
    for i in range(wl.M):
        m = C.plain_match(wl.mode, wl.query, list(map(int, wl.records[i])), wl.d, wl.flags)
        assert keys.decrypt(vs[i]) == int(m)
        assert P.decrypt_bits(keys, masked[i]) == (int(wl.payloads[i]) if m else 0)


def test_config1_linear_aggregation_end_to_end():
    """R24 (not in the paper) on TFHE ciphertexts: config 1 with linear XOR aggregation (masks in the {0, 1/2}
    encoding, one sum and one refresh bootstrap per payload bit) decrypts to the plain predicate; every masked
    bit decrypts to v_i AND s_ij in the {0, 1/2} encoding (phase near 1/2 for 1)."""
    wl = make_workload(1, flags=C.CONFIG_FLAGS | C.F_LINEAR_SUM)
    keys = O.OracleKeys(wl.key_seed)
    R, vs, masked = run_oracle_config(wl, keys)
    want = C.plain_result(wl.mode, wl.query, [list(map(int, r)) for r in wl.records], wl.payloads, wl.d, wl.flags)
    assert P.decrypt_bits(keys, R) == want
    for i in range(wl.M):
        m = C.plain_match(wl.mode, wl.query, list(map(int, wl.records[i])), wl.d, wl.flags)
        for j in range(wl.l_S):
            bit = (int(wl.payloads[i]) >> j) & 1 if m else 0
            ph = int(keys.phase(masked[i][j]))  # bit * 1/2 + noise
            assert abs(((ph - bit * 2 ** 31 + 2 ** 31) % 2 ** 32) - 2 ** 31) < 2 ** 28, (i, j, hex(ph))
