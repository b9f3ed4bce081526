"""CPU tests of the C-ABI library (no GPU needed): it loads and exports every symbol include/vlp.h declares;
its host-side KeyGen / encryption / PubKeyGen / ServerEnc bytes equal the oracle's (P10, R3); the level
scheduler's gate counts and depths equal the closed forms of SURVEY 8(d) / Appendix A."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
from oracle import protocol as OP
from paper_2506_12761_b200 import _lib as L
from paper_2506_12761_b200 import api as A
from synth import make_workload

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "vlp.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"\b(vlp_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(L.SIGNATURES), declared ^ set(L.SIGNATURES)
    lib = L.lib()
    for name in declared:
        assert getattr(lib, name) is not None
    p = L.VlpParams()
    assert L.lib().vlp_params_tfhe128(ctypes.byref(p)) == 0
    assert (p.n, p.N, p.k, p.bg_bits, p.ell, p.ks_base_bits, p.ks_t) == (630, 1024, 1, 7, 3, 2, 8)
    assert (p.sigma_lwe, p.sigma_bk, p.sigma_ks) == (2.0 ** -15, 2.0 ** -25, 2.0 ** -15)


@pytest.fixture(scope="module")
def lkeys():
    return A.Keys(123)


def test_keygen_bytes_equal_oracle(lkeys, okeys):
    """P10: the library's keys are byte-identical to the oracle's for the same seed (independent code)."""
    s1, z1, b1, k1 = lkeys.export()
    s2, z2, b2, k2 = okeys.export()
    assert np.array_equal(s1, s2) and np.array_equal(z1, z2)
    assert np.array_equal(b1, b2)
    assert np.array_equal(k1, k2)


def test_encryptions_equal_oracle(lkeys, okeys):
    bits = np.array([1, 0, 1, 1, 0], np.uint8)
    got = lkeys.encrypt_bits(bits, 77, obj0=10)
    for i, b in enumerate(bits):
        want = okeys.encrypt(int(b), 77, 10 + i)
        assert np.array_equal(got[i, :631], want) and got[i, 631] == 0
    m = A.meta(L.MODE_INTV, 4, 8, 8, 2)
    q = lkeys.encrypt_query(m, [200, 13], 9)
    oq = OP.encrypt_query(okeys, [200, 13], 8, 9)
    assert np.array_equal(q[:, :631], np.array([c for w in oq for c in w]))
    assert list(lkeys.decrypt_bits(q)) == OP.bits_of(200, 8) + OP.bits_of(13, 8)


@pytest.mark.parametrize("cfg", [1, 3, 4])
def test_server_enc_equals_oracle(lkeys, okeys, cfg):
    """alg:PubKeyGen + alg:ServerEnc bytes (two records) equal the oracle's protocol module."""
    wl = make_workload(cfg, M=2)
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    db = lkeys.encrypt_db(m, wl.records, wl.payloads, pk_seed=555)
    per = A.record_cts(m)
    W = wl.records.shape[1]
    assert per == W * wl.l_I + wl.l_S
    for i in range(wl.M):
        rec, pay = OP.server_enc_record(okeys, 555, i, [int(v) for v in wl.records[i]], int(wl.payloads[i]),
                                        wl.l_I, wl.l_S)
        want = [c for word in rec for c in word] + pay
        assert np.array_equal(db[i * per:(i + 1) * per, :631], np.array(want))


def test_pk_single_use(lkeys):
    m = A.meta(L.MODE_IDM, 2, 4, 2, 1)
    pk = ctypes.c_void_p()
    L.check(L.lib().vlp_pubkeygen(lkeys.sk, ctypes.byref(m), 1, 0, 2, ctypes.byref(pk)))
    w = np.array([3, 5], np.uint64)
    p = np.array([1, 2], np.uint64)
    out = np.zeros((2 * 6, 632), np.uint32)
    assert L.lib().vlp_server_encrypt_db(pk, A._u64p(w), A._u64p(p), A._u32p(out)) == 0
    assert L.lib().vlp_server_encrypt_db(pk, A._u64p(w), A._u64p(p), A._u32p(out)) == L.VLP_EPKUSED
    L.lib().vlp_free_pk(pk)


def test_error_codes(lkeys):
    bad = A.meta(L.MODE_INTV, 4, 1, 8, 1)
    out = np.zeros((8, 632), np.uint32)
    v = np.array([1], np.uint64)
    assert L.lib().vlp_encrypt_query(lkeys.sk, ctypes.byref(bad), A._u64p(v), 0, A._u32p(out)) == L.VLP_EWIDTH
    m = A.meta(L.MODE_INTV, 4, 8, 8, 1)
    v = np.array([256], np.uint64)
    assert L.lib().vlp_encrypt_query(lkeys.sk, ctypes.byref(m), A._u64p(v), 0, A._u32p(out)) == L.VLP_ERANGE
    assert L.lib().vlp_last_error()


def _info(m, first=0, count=None):
    h = ctypes.c_void_p()
    L.check(L.lib().vlp_program_create(None, ctypes.byref(m), first, m.M if count is None else count, ctypes.byref(h)))
    info = L.VlpProgramInfo()
    L.check(L.lib().vlp_program_get_info(h, ctypes.byref(info)))
    L.lib().vlp_free_program(h)
    return info


@pytest.mark.parametrize("cfg,br,ks,levels", [(1, 252, 188, 13), (2, 132080, 99312, 29), (3, 1060832, 798688, 32),
                                              (4, 6750176, 6750176, 23)])
def test_schedule_closed_forms(cfg, br, ks, levels):
    """Gate model of Appendix A (comparator 3l BR / 2l KS, EQ tree 2l-1, mask l_S, tree (M-1) l_S) and the
    hoisted depths 13 / 29 / 32 / 23 of SURVEY 8(d)."""
    wl = make_workload(cfg, M=None) if cfg != 4 else None
    c = {1: (0, 4, 8, 8, 1), 2: (0, 1024, 16, 16, 1), 3: (0, 4096, 16, 32, 2), 4: (2, 65536, 20, 32, 1)}[cfg]
    info = _info(A.meta(*c))
    assert (info.br, info.ks, info.levels) == (br, ks, levels)


@pytest.mark.parametrize("c,levels", [((0, 4, 8, 8, 1), 8), ((0, 1024, 16, 16, 1), 17), ((0, 4096, 16, 32, 2), 20)])
def test_prefix_schedule_depth(c, levels):
    """R23 prefix comparators (VLP_F_PREFIX_COMP): comparator depth 1 + log2 l instead of l + 1, so config 1
    needs 8 levels (13 ripple), config 2 17 (29), config 3 20 (32); more gates than the ripple form."""
    m = A.meta(c[0], c[1], c[2], c[3], c[4], L.CONFIG_FLAGS | L.F_PREFIX_COMP)
    info = _info(m)
    ripple = _info(A.meta(*c))
    assert info.levels == levels and info.br > ripple.br
    bad = A.meta(c[0], c[1], c[2], c[3], c[4], L.F_PREFIX_COMP)  # signed comparators: not supported
    h = ctypes.c_void_p()
    assert L.lib().vlp_program_create(None, ctypes.byref(bad), 0, c[1], ctypes.byref(h)) == L.VLP_EINVAL


def test_linear_aggregation_schedule():
    """R24 (VLP_F_LINEAR_SUM): config 2's (M-1) l_S = 16,368 tree bootstraps become 16 x 16 group refreshes +
    16 final ones (levels 29 -> 21); XOR only (OR_REDUCE refused)."""
    m = A.meta(0, 1024, 16, 16, 1, L.CONFIG_FLAGS | L.F_LINEAR_SUM)
    info = _info(m)
    assert (info.br, info.ks, info.levels) == (132080 - 16368 + 272, 99312 - 16368 + 272, 21)
    small = _info(A.meta(0, 4, 8, 8, 1, L.CONFIG_FLAGS | L.F_LINEAR_SUM))
    assert (small.br, small.levels) == (252 - 24 + 8, 12)
    bad = A.meta(0, 4, 8, 8, 1, L.CONFIG_FLAGS | L.F_LINEAR_SUM | L.F_OR_REDUCE)
    h = ctypes.c_void_p()
    assert L.lib().vlp_program_create(None, ctypes.byref(bad), 0, 4, ctypes.byref(h)) == L.VLP_EINVAL


@pytest.mark.parametrize("c", [(2, 65536, 20, 32, 1), (0, 4096, 16, 32, 2), (0, 1024, 16, 16, 1)])
def test_liveness_recycles_scratch_rows(c):
    """Intermediate and N-LWE rows are recycled by liveness (default) instead of one row per gate
    (VLP_F_KEEP_ALL): the same schedule in well under half the scratch for configs 2-4 (config 4: 45 -> 19 GB)."""
    a, b = _info(A.meta(*c)), _info(A.meta(*c, L.CONFIG_FLAGS | L.F_KEEP_ALL))
    assert (a.br, a.ks, a.levels) == (b.br, b.ks, b.levels)
    assert a.scratch_bytes < 0.55 * b.scratch_bytes


def test_schedule_level_widths_config2():
    """SURVEY 8(d) config 2 widths: L1 32,768; L2 34,816; L3-L17 2,048; L18 1,024; L19 16,384; tree 8,192 -> 16."""
    h = ctypes.c_void_p()
    m = A.meta(0, 1024, 16, 16, 1)
    L.check(L.lib().vlp_program_create(None, ctypes.byref(m), 0, 1024, ctypes.byref(h)))
    info = L.VlpProgramInfo()
    L.check(L.lib().vlp_program_get_info(h, ctypes.byref(info)))
    assert info.max_level_br == 34816
    L.lib().vlp_free_program(h)


def test_shard_schedules_sum_to_whole():
    """Contiguous power-of-two shards + combine (R15) need exactly the single-shot gate count."""
    m = A.meta(0, 1024, 16, 16, 1)
    whole = _info(m)
    G = 8
    shards = [_info(m, g * 128, 128) for g in range(G)]
    h = ctypes.c_void_p()
    L.check(L.lib().vlp_program_create_combine(None, ctypes.byref(m), G, ctypes.byref(h)))
    ci = L.VlpProgramInfo()
    L.check(L.lib().vlp_program_get_info(h, ctypes.byref(ci)))
    L.lib().vlp_free_program(h)
    assert sum(s.br for s in shards) + ci.br == whole.br
    assert ci.br == (G - 1) * 16 and ci.levels == 3


def test_multi_query_schedule():
    """Multi-query packing: nq queries against one shard -> nq x the gates of one query in the same number of
    levels (every level launch carries all queries' gates)."""
    m = A.meta(L.MODE_INTV, 58, 16, 22, 2)
    one = _info(m)
    h = ctypes.c_void_p()
    L.check(L.lib().vlp_program_create_queries(None, ctypes.byref(m), 0, 58, 5, ctypes.byref(h)))
    info = L.VlpProgramInfo()
    L.check(L.lib().vlp_program_get_info(h, ctypes.byref(info)))
    L.lib().vlp_free_program(h)
    assert (info.br, info.ks, info.levels) == (5 * one.br, 5 * one.ks, one.levels)
    assert info.in0_cts == 5 * one.in0_cts and info.out_cts == 5 * one.out_cts and info.in1_cts == one.in1_cts
    assert L.lib().vlp_program_create_queries(None, ctypes.byref(m), 0, 58, 0, ctypes.byref(h)) == L.VLP_EINVAL


def test_oversized_schedules_are_refused():
    """Slot ids address 2^28 rows per region: a shard with more input ciphertexts (or a combine over too many
    shards) is refused with VLP_EINVAL instead of wrapping row indices."""
    h = ctypes.c_void_p()
    m = A.meta(L.MODE_INTV, 1 << 23, 16, 16, 1)  # 2^23 records x 48 ciphertexts > 2^28
    assert L.lib().vlp_program_create(None, ctypes.byref(m), 0, 1 << 23, ctypes.byref(h)) == L.VLP_EINVAL
    assert "too large" in L.lib().vlp_last_error().decode()
    assert L.lib().vlp_program_create_combine(None, ctypes.byref(m), 1 << 20, ctypes.byref(h)) == L.VLP_EINVAL


# ----------------------------------------------------------------------------------- secure randomness (ADVICE)
def test_chacha20_block_matches_independent_implementation():
    """The secure calls' generator is ChaCha20 (RFC 8439 2.3): vlp_debug_chacha20_block equals the keystream of
    the `cryptography` package's ChaCha20 (an independent implementation) for random keys, nonces and counters,
    and the RFC's own block-function example."""
    import ctypes
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms
    lib = L.lib()
    rng = np.random.default_rng(8439)
    cases = [(np.arange(32, dtype=np.uint8).view(np.uint32), 1,
              np.frombuffer(bytes.fromhex("000000090000004a00000000"), dtype=np.uint32))]
    for _ in range(8):
        cases.append((rng.integers(0, 2 ** 32, 8, dtype=np.uint64).astype(np.uint32), int(rng.integers(0, 2 ** 32)),
                      rng.integers(0, 2 ** 32, 3, dtype=np.uint64).astype(np.uint32)))
    for key, ctr, nonce in cases:
        key, nonce = np.ascontiguousarray(key), np.ascontiguousarray(nonce)
        out = np.zeros(16, np.uint32)
        p = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))  # noqa: E731
        assert lib.vlp_debug_chacha20_block(p(key), ctr, p(nonce), p(out)) == 0
        full_nonce = np.uint32(ctr).tobytes() + nonce.tobytes()  # cryptography: 4-byte LE counter || 12-byte nonce
        ks = Cipher(algorithms.ChaCha20(key.tobytes(), full_nonce), mode=None).encryptor().update(bytes(64))
        assert out.tobytes() == ks
    # RFC 8439 2.3.2 test vector, first serialized bytes
    key, ctr, nonce = cases[0]
    out = np.zeros(16, np.uint32)
    lib.vlp_debug_chacha20_block(key.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), ctr,
                                 nonce.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
    assert out.tobytes()[:16].hex() == "10f1e7e4d13b5915500fdd1fa32071c4"


def test_secure_calls_are_fresh_and_correct():
    """ADVICE (secure randomness): two OS-random KeyGens give different keys; OS-random query encryptions of the
    same value differ yet decrypt to it; secure encryptions of random bits decrypt correctly; the secure pk
    encrypts a DB that decrypts to its plaintext bits."""
    k1, k2 = A.Keys(), A.Keys()
    s1, z1, _, _ = k1.export()
    s2, z2, _, _ = k2.export()
    assert not np.array_equal(s1, s2) and not np.array_equal(z1, z2)
    assert 200 < int(s1.sum()) < 430 and 400 < int(z1.sum()) < 624  # binary keys, about half ones
    m = A.meta(L.MODE_INTV, 2, 8, 4, 1)
    q1, q2 = k1.encrypt_query(m, [173]), k1.encrypt_query(m, [173])
    assert not np.array_equal(q1, q2)
    for q in (q1, q2):
        assert int(sum(int(b) << j for j, b in enumerate(k1.decrypt_bits(q)))) == 173
    bits = np.random.default_rng(1).integers(0, 2, 64, dtype=np.uint8)
    assert np.array_equal(k1.decrypt_bits(k1.encrypt_bits(bits)), bits)
    db = k1.encrypt_db(m, np.array([[3, 9], [0, 200]], np.uint64), np.array([5, 10], np.uint64))
    want = [(3 >> j) & 1 for j in range(8)] + [(9 >> j) & 1 for j in range(8)] + [(5 >> j) & 1 for j in range(4)]
    assert list(k1.decrypt_bits(db[:20])) == want


def _next_key(key):
    os.environ["VLP_TEST_HOOKS"] = "1"  # the hook is disabled without it
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32))
    A.check(A.lib().vlp_debug_next_secure_key(A._u32p(k)))


def test_secure_key_hook_needs_the_test_switch(monkeypatch):
    """vlp_debug_next_secure_key is refused (VLP_EINVAL) unless VLP_TEST_HOOKS=1: a production process cannot have
    its secure calls' keys injected."""
    monkeypatch.delenv("VLP_TEST_HOOKS", raising=False)
    k = np.zeros(8, np.uint32)
    assert A.lib().vlp_debug_next_secure_key(A._u32p(k)) == L.VLP_EINVAL
    k1, k2 = A.Keys(), A.Keys()  # still fresh OS randomness
    assert not np.array_equal(k1.export()[0], k2.export()[0])


def test_secure_key_hook_is_single_use():
    """vlp_debug_next_secure_key (test hook): the next secure call of this thread takes the given ChaCha20 key --
    the same key gives the same keys and pk bytes --, and the call after it is back on getrandom."""
    key = np.arange(1, 9, dtype=np.uint32) * 0x01010101
    _next_key(key)
    k1 = A.Keys()
    _next_key(key)
    k2 = A.Keys()
    k3 = A.Keys()
    for x, y in zip(k1.export(), k2.export()):
        assert np.array_equal(x, y)
    assert not np.array_equal(k1.export()[0], k3.export()[0])
    m = A.meta(L.MODE_INTV, 2, 8, 4, 1)
    words, pays = np.array([[3, 9], [0, 200]], np.uint64), np.array([5, 10], np.uint64)
    _next_key(key)
    db1 = k1.encrypt_db(m, words, pays)
    _next_key(key)
    db2 = k1.encrypt_db(m, words, pays)
    db3 = k1.encrypt_db(m, words, pays)
    assert np.array_equal(db1, db2) and not np.array_equal(db1, db3)
    assert list(k1.decrypt_bits(db1[:20])) == list(k1.decrypt_bits(db3[:20]))
