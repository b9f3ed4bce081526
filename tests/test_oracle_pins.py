"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test names the plausible oracle mistake it would catch.  None of them compares the oracle with
itself: schoolbook vs NTT are two different algorithms; closed forms are computed by hand in the test;
truth tables / predicates come from the paper's statements (thm:comple, cor:compl, lem:EQ, ...).
"""
import ctypes
import itertools
import json
import math
import os
import random
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle as O
from oracle import circuits as C
from oracle import protocol as P

HERE = os.path.dirname(os.path.abspath(__file__))
RNG = np.random.default_rng(99)
POOL = ThreadPoolExecutor(max_workers=os.cpu_count() or 4)


def _u32(x):
    return np.uint32(x & 0xFFFFFFFF)


# ----------------------------------------------------------------------------------- P2: products
def test_mulq_matches_modulo():
    """Barrett modmul == exact (a*b) % Q (catches a wrong Barrett constant / shift)."""
    L = O.lib()
    L.oracle_mulq.restype = ctypes.c_uint64
    L.oracle_mulq.argtypes = [ctypes.c_uint64] * 2
    L.oracle_modulus.restype = ctypes.c_uint64
    Q = L.oracle_modulus()
    rnd = random.Random(5)
    for _ in range(20000):
        a, b = rnd.randrange(Q), rnd.randrange(Q)
        assert L.oracle_mulq(a, b) == a * b % Q
    for a, b in [(Q - 1, Q - 1), (0, Q - 1), (1, Q - 1), (Q - 1, 2)]:
        assert L.oracle_mulq(a, b) == a * b % Q


@pytest.mark.parametrize("n", [4, 8, 16, 32, 64])
def test_schoolbook_ring_axioms(n):
    """X^N = -1 (catches a cyclic instead of negacyclic wrap), commutativity, distributivity,
    associativity of the schoolbook definition at small N."""
    x = np.zeros(n, np.uint32); x[1] = 1
    xn1 = np.zeros(n, np.uint32); xn1[n - 1] = 1
    minus_one = np.zeros(n, np.uint32); minus_one[0] = 0xFFFFFFFF
    assert np.array_equal(O.negacyclic_schoolbook(x, xn1), minus_one)
    for _ in range(5):
        a, b, c = (RNG.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32) for _ in range(3))
        ab = O.negacyclic_schoolbook(a, b)
        assert np.array_equal(ab, O.negacyclic_schoolbook(b, a))
        assert np.array_equal(O.negacyclic_schoolbook(ab, c), O.negacyclic_schoolbook(a, O.negacyclic_schoolbook(b, c)))
        assert np.array_equal(O.negacyclic_schoolbook(a, (b + c).astype(np.uint32)), (ab + O.negacyclic_schoolbook(a, c)).astype(np.uint32))


def test_monomial_closed_form():
    """X^k * a shifts coefficients with sign flips (closed form, written out here independently)."""
    n = 64
    a = RNG.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
    for k in [0, 1, 5, 63]:
        m = np.zeros(n, np.uint32); m[k] = 1
        want = np.array([a[j - k] if j >= k else (0 - int(a[j - k + n])) & 0xFFFFFFFF for j in range(n)], dtype=np.uint32)
        assert np.array_equal(O.negacyclic_schoolbook(m, a), want)


@pytest.mark.parametrize("terms", [1, 6])
def test_ntt_product_equals_schoolbook_1024(terms):
    """The exact NTT path (Q = 0x3fffffffffffa801) equals the schoolbook definition mod 2^32 at N = 1024
    for the operand sizes the external product uses: digits in [-64, 64) times torus32 rows."""
    a = RNG.integers(-64, 64, (terms, O.N)).astype(np.int64)
    b = RNG.integers(-(2 ** 31), 2 ** 31, (terms, O.N)).astype(np.int64)
    got = O.negacyclic_dot(a, b)
    want = np.zeros(O.N, np.uint32)
    for t in range(terms):
        want = (want + O.negacyclic_schoolbook(a[t].astype(np.uint32), b[t].astype(np.uint32))).astype(np.uint32)
    assert np.array_equal(got, want)


# ----------------------------------------------------------------------------------- R5-R8 vectors
def _golden():
    with open(os.path.join(HERE, "golden", "derived_vectors.json")) as f:
        return json.load(f)["vectors"]


def test_derived_vectors():
    for v in _golden():
        x = int(v["x"], 16)
        if "gadget" in v:
            assert O.gadget_digits(x) == v["gadget"], v
        if "ks" in v:
            assert O.ks_digits(x) == v["ks"], v
        assert O.modswitch(x) == v["modswitch"], v


def test_gadget_reconstruction_property():
    """R5: digits in [-64, 64) and sum_j d_j 2^(32-7j) = x rounded (half up) to a multiple of 2^11."""
    rnd = random.Random(3)
    for _ in range(20000):
        x = rnd.randrange(2 ** 32)
        d = O.gadget_digits(x)
        assert all(-64 <= t < 64 for t in d)
        rec = (d[0] * 2 ** 25 + d[1] * 2 ** 18 + d[2] * 2 ** 11) % 2 ** 32
        want = (((x + 2 ** 10) >> 11) << 11) % 2 ** 32
        assert rec == want


def test_ks_digit_reconstruction_property():
    """R6: sum_j d_j 4^(7-j) = round(x / 2^16) mod 2^16, digits in {0,1,2,3}, MSB first."""
    rnd = random.Random(4)
    for _ in range(20000):
        x = rnd.randrange(2 ** 32)
        d = O.ks_digits(x)
        assert sum(t * 4 ** (7 - j) for j, t in enumerate(d)) == ((x + 2 ** 15) >> 16) % 2 ** 16


# ----------------------------------------------------------------------------------- P3 / P11
def test_trivial_bootstrap_closed_form(okeys):
    """P3: for a trivial input (0, b) every abar_i = 0, so BlindRotate leaves (0, X^{-bbar} testv);
    extract gives (0, +-1/8) and KS of a zero mask subtracts nothing: output (0, +2^29) iff
    floor((b + 2^20) / 2^21) mod 2048 < 1024.  Catches rotation direction, extract sign, KS wiring."""
    bs = [int(v["x"], 16) for v in _golden() if "trivial_bootstrap" in v]
    want = [int(v["trivial_bootstrap"], 16) for v in _golden() if "trivial_bootstrap" in v]
    bs += [random.Random(8).randrange(2 ** 32) for _ in range(6)]
    want += [0x20000000 if (((b + 2 ** 20) >> 21) % 2048) < 1024 else 0xE0000000 for b in bs[len(want):]]

    outs = list(POOL.map(lambda b: okeys.bootstrap(O.trivial_mu(b)), bs))
    for b, w, out in zip(bs, want, outs):
        assert not out[:O.n].any(), hex(b)
        assert int(out[O.n]) == w, (hex(b), hex(int(out[O.n])), hex(w))


def test_trivial_bootstrap_mu_closed_form(okeys):
    """R24 (not in the paper): the same closed form with test vector 1/4 -- output (0, +-2^30) exactly, with
    the sign of P3; so the R24 mask (+ 1/4) lands on (0, 1/2) or (0, 0) and the refresh of x - 1/4 reads it."""
    bs = [0, 0x20000000, 0xE0000000, 0x80000000, 0xFFF00000, 0xFFEFFFFF, 0x7FEFFFFF, 0x7FF00000]
    bs += [random.Random(9).randrange(2 ** 32) for _ in range(4)]
    outs = list(POOL.map(lambda b: okeys.bootstrap_mu(O.trivial_mu(b), 0x40000000), bs))
    for b, out in zip(bs, outs):
        want = 0x40000000 if (((b + 2 ** 20) >> 21) % 2048) < 1024 else 0xC0000000
        assert not out[:O.n].any(), hex(b)
        assert int(out[O.n]) == want, (hex(b), hex(int(out[O.n])))
    # mu = 1/8 through the same entry point is the P3 bootstrap itself
    assert np.array_equal(okeys.bootstrap_mu(O.trivial_mu(0x12345678), 0x20000000), okeys.bootstrap(O.trivial_mu(0x12345678)))


# ----------------------------------------------------------------------------------- P4: external product
def test_external_product_invariant(okeys_noiseless):
    """P4, sigma = 0 keys: phase(ExtProd(bsk_i, D)) = 0 exactly if s_i = 0, and phase(D) + eps with
    |eps_j| <= (1 + N) 2^10 (the R5 rounding only) if s_i = 1.  Catches TRGSW row order, a transposed
    component, a wrong g_j, or a decomposition that does not reconstruct."""
    k = okeys_noiseless
    s, z, _, _ = k.export()
    D = RNG.integers(0, 2 ** 32, 2 * O.N, dtype=np.uint64).astype(np.uint32)
    ph_D = k.trlwe_phase(D)
    i1 = int(np.flatnonzero(s == 1)[0])
    i0 = int(np.flatnonzero(s == 0)[0])
    out1 = k.external_product(i1, D)
    out0 = k.external_product(i0, D)
    assert not k.trlwe_phase(out0).any()
    err = (k.trlwe_phase(out1).astype(np.int64) - ph_D.astype(np.int64) + 2 ** 31) % 2 ** 32 - 2 ** 31
    assert np.abs(err).max() <= (1 + O.N) * 2 ** 10


# ----------------------------------------------------------------------------------- P5 / P6: gates
def _and_chain(k, length=100):
    x = k.encrypt(1, 55, 0)
    out = []
    for i in range(length):
        x = k.gate(O.AND, x, k.encrypt(1, 55, i + 1))
        out.append((k.decrypt(x), ((k.phase(x) - 0x20000000 + 2 ** 31) % 2 ** 32 - 2 ** 31) / 2 ** 32))
    return out


@pytest.fixture(scope="module")
def and_chain(okeys):
    """P6's 100-gate chain is sequential: start it on its own thread so it overlaps P5's threaded trials."""
    ex = ThreadPoolExecutor(max_workers=1)
    fut = ex.submit(_and_chain, okeys)
    yield fut
    ex.shutdown(wait=True)


def test_gate_truth_tables(okeys, and_chain):
    """P5 (R10): AND/NAND/OR/XOR/XNOR on all 4 input pairs and MUX on all 8 triples,
    100 trials of fresh encryptions per row (2,800 gates, threaded), 0 errors.  Catches a wrong linear-form
    constant or coefficient, and any noise failure rate above ~1e-3 per gate."""
    k = okeys
    ops = {O.AND: lambda a, b: a & b, O.NAND: lambda a, b: 1 - (a & b), O.OR: lambda a, b: a | b,
           O.XOR: lambda a, b: a ^ b, O.XNOR: lambda a, b: 1 - (a ^ b)}
    jobs = []
    obj = 0
    for trial in range(100):
        for op, f in ops.items():
            for a, b in itertools.product((0, 1), repeat=2):
                jobs.append(("g", op, (a, b), f(a, b), obj)); obj += 2
        for c, a, b in itertools.product((0, 1), repeat=3):
            jobs.append(("m", None, (c, a, b), a if c else b, obj)); obj += 3

    def run(job):
        kind, op, bits, want, o = job
        cts = [k.encrypt(bit, 77, o + t) for t, bit in enumerate(bits)]
        out = k.gate(op, *cts) if kind == "g" else k.mux(*cts)
        return k.decrypt(out), want, k.phase(out)

    res = list(POOL.map(run, jobs))
    assert all(got == want for got, want, _ in res)
    # gate outputs are +-1/8 plus bootstrapping noise (Appendix A of SURVEY: sigma ~ 3.5e-3)
    errs = [((ph - (0x20000000 if want else 0xE0000000) + 2 ** 31) % 2 ** 32 - 2 ** 31) / 2 ** 32 for _, want, ph in res]
    assert max(abs(e) for e in errs) < 1 / 32


def test_and_chain_noise_refresh(and_chain):
    """P6: a 100-gate AND chain with a fresh Enc(1) each time keeps decrypting correctly; the
    output noise stays at the bootstrapped level (does not grow with depth): its standard deviation is within
    a factor of ~2 of the predicted 3.5e-3, first half vs second half alike."""
    res = and_chain.result()
    assert len(res) == 100 and all(bit == 1 for bit, _ in res)
    errs = [e for _, e in res]
    sd = float(np.sqrt(np.mean(np.square(errs))))
    assert 1.75e-3 < sd < 7.0e-3, sd
    sd1, sd2 = (float(np.sqrt(np.mean(np.square(h)))) for h in (errs[:50], errs[50:]))
    assert sd2 < 2 * sd1 and sd1 < 2 * sd2, (sd1, sd2)  # no growth with depth


# ----------------------------------------------------------------------------------- P10: keys
def test_key_statistics(okeys):
    """P10 (S:53-62 style): secret bits ~ Bernoulli(1/2); bsk / ksk / fresh noise sigma within 5-10%."""
    s, z, bsk, ksk = okeys.export()
    assert abs(int(s.sum()) - 315) < 4 * math.sqrt(630) / 2 * 2
    assert abs(int(z.sum()) - 512) < 4 * math.sqrt(1024) / 2 * 2
    # bsk rows: phase(row) = s_i g_j (on component u at coefficient 0) + e, sigma_BK * 2^32 = 128
    ph = []
    for i in range(6):
        for r in range(6):
            u, j = divmod(r, 3)
            if u == 0 and s[i]:
                continue  # s_i g_j sits in the mask: phase(b - a z) picks up -g_j z; not pure noise
            p = okeys.trlwe_phase(bsk[i, r].reshape(-1))
            if u == 1 and s[i]:
                p[0] = (int(p[0]) - 2 ** (32 - 7 * (j + 1))) % 2 ** 32
            ph.append(((p.astype(np.int64) + 2 ** 31) % 2 ** 32) - 2 ** 31)
    ph = np.concatenate(ph)
    assert np.abs(ph).max() < 128 * 8
    assert abs(np.std(ph) / 128.0 - 1.0) < 0.05
    # ksk: phase = v z_i 2^(32-2(j+1)) + e, sigma_KS * 2^32 = 131072
    e = []
    for i in range(0, 1024, 8):
        for j in range(8):
            for v in range(1, 4):
                row = ksk[i, j, v - 1]
                mu = (v * int(z[i]) * 2 ** (32 - 2 * (j + 1))) % 2 ** 32
                e.append(((okeys.phase(row) - mu + 2 ** 31) % 2 ** 32) - 2 ** 31)
    assert abs(np.std(e) / 131072.0 - 1.0) < 0.05
    # fresh TLWE (R2): sigma_LWE * 2^32
    f = [((okeys.phase(okeys.encrypt(1, 9, o)) - 0x20000000 + 2 ** 31) % 2 ** 32) - 2 ** 31 for o in range(3000)]
    assert abs(np.std(f) / 131072.0 - 1.0) < 0.05


def test_encrypt_decrypt_roundtrip(okeys):
    """2000 fresh encryptions of each bit decrypt correctly; trivial +-1/8 decrypt to 1/0;
    phase ties (0, 1/2) decrypt to 0 (R18)."""
    for bit in (0, 1):
        for o in range(1000):
            assert okeys.decrypt(okeys.encrypt(bit, 11, o + 5000 * bit)) == bit
    assert okeys.decrypt(O.trivial(1)) == 1 and okeys.decrypt(O.trivial(0)) == 0
    assert okeys.decrypt(O.trivial_mu(0)) == 0 and okeys.decrypt(O.trivial_mu(0x80000000)) == 0


# ----------------------------------------------------------------------------------- P7: topology
@pytest.mark.parametrize("l", [2, 3, 4, 5, 6])
def test_comparators_exhaustive_plain(l):
    """thm:comple / cor:compl on the PlainOracle, every pair at width l: the paper-literal
    form is signed two's complement; the R11 UNSIGNED form is unsigned order.  Gate model 3l BR,
    2l KS, depth l+1 (S9 hoisting)."""
    B = C.PlainBackend()
    for z1, z2 in itertools.product(range(2 ** l), repeat=2):
        a = [B.const(b) for b in P.bits_of(z1, l)]
        b = [B.const(bb) for bb in P.bits_of(z2, l)]
        s1 = z1 - 2 ** l if z1 >> (l - 1) else z1
        s2 = z2 - 2 ** l if z2 >> (l - 1) else z2
        assert C.hom_comp_le(B, a, b, l, unsigned=False)[0] == (s1 <= s2)
        assert C.hom_comp_l(B, a, b, l, unsigned=False)[0] == (s1 < s2)
        assert C.hom_comp_le(B, a, b, l, unsigned=True)[0] == (z1 <= z2)
        assert C.hom_comp_l(B, a, b, l, unsigned=True)[0] == (z1 < z2)
    B = C.PlainBackend()
    a = [B.const(0)] * l
    r = C.hom_comp_le(B, a, a, l)
    assert (B.br, B.ks, r[1]) == (3 * l, 2 * l, l + 1)


@pytest.mark.parametrize("l", [1, 2, 3, 4, 5, 6, 7])
def test_prefix_comparators_exhaustive_plain(l):
    """R23 (NOT in the paper): the log-depth prefix comparator on the PlainOracle, every
    pair at width l: [z1 > z2], [z1 <= z2], [z1 < z2] in unsigned order, depth 1 + ceil(log2 l)."""
    depth = 1 + (math.ceil(math.log2(l)) if l > 1 else 0)
    for z1, z2 in itertools.product(range(2 ** l), repeat=2):
        B = C.PlainBackend()
        a = [B.const(b) for b in P.bits_of(z1, l)]
        b = [B.const(bb) for bb in P.bits_of(z2, l)]
        g = C.hom_comp_gt_prefix(B, a, b, l)
        assert g == (z1 > z2, depth), (z1, z2)
        assert C.hom_comp_le_prefix(B, a, b, l)[0] == (z1 <= z2)
        assert C.hom_comp_l_prefix(B, a, b, l)[0] == (z1 < z2)


@pytest.mark.parametrize("l", [1, 2, 3, 5, 8, 16, 20])
def test_equality_plain(l):
    """lem:EQ for the serial and the OPT tree; tree gate count l XNOR +
    (l-1) AND, depth ceil(log2 l) + 1."""
    rnd = random.Random(l)
    pairs = [(rnd.randrange(2 ** l), rnd.randrange(2 ** l)) for _ in range(50)] + [(v, v) for v in range(min(2 ** l, 40))]
    for z1, z2 in pairs:
        B = C.PlainBackend()
        a = [B.const(b) for b in P.bits_of(z1, l)]
        b = [B.const(bb) for bb in P.bits_of(z2, l)]
        assert C.hom_eq_serial(B, a, b, l)[0] == (z1 == z2)
        B2 = C.PlainBackend()
        r = C.hom_eq_tree(B2, a, b, l)
        assert r[0] == (z1 == z2)
        assert B2.br == 2 * l - 1 and r[1] == math.ceil(math.log2(l)) + 1


@pytest.mark.parametrize("M", [1, 2, 63, 64, 65, 200, 4100])
def test_linear_aggregation_plain(M):
    """R24 on the PlainOracle: XOR of the matching records' payloads for record counts around the group size
    (64) and past two group levels (4100); depth = mask level + one refresh level per group level."""
    rnd = random.Random(M)
    l, l_S = 4, 3
    recs = [sorted((rnd.randrange(16), rnd.randrange(16))) for _ in range(M)]
    q = [rnd.randrange(16)]
    pays = [rnd.randrange(8) for _ in range(M)]
    B = C.PlainBackend()
    qc = [[B.const(b) for b in P.bits_of(v, l)] for v in q]
    rc = [[[B.const(b) for b in P.bits_of(v, l)] for v in r] for r in recs]
    pc = [[B.const(b) for b in P.bits_of(v, l_S)] for v in pays]
    R, vs, _ = C.velopir(B, C.MODE_INTV, qc, rc, pc, l, 1, l_S, C.CONFIG_FLAGS | C.F_LINEAR_SUM, threads=1)
    assert sum(int(b[0]) << j for j, b in enumerate(R)) == C.plain_result(C.MODE_INTV, q, recs, pays, 1, C.CONFIG_FLAGS)
    groups = 1 + (M > 64) + (M > 4096)
    assert max(b[1] for b in R) == max(v[1] for v in vs) + 1 + groups


def test_velopir_plain_configs():
    """thm:VeLoPIR on the PlainOracle for small instances of every mode/flag combination:
    R = XOR (or OR, R19) of the matching records' payloads, 0 if none."""
    rnd = random.Random(17)
    for mode, d, l in [(C.MODE_INTV, 1, 6), (C.MODE_INTV, 2, 4), (C.MODE_COV, 2, 4), (C.MODE_IDM, 1, 5)]:
        for flags in [C.CONFIG_FLAGS, C.CONFIG_FLAGS | C.F_OR_REDUCE, C.F_UNSIGNED,
                      C.F_CLOSED_UPPER | C.F_UNSIGNED, C.CONFIG_FLAGS | C.F_PREFIX_COMP, C.F_UNSIGNED | C.F_PREFIX_COMP]:
            for M in [1, 3, 4, 7]:
                W = P.record_words(mode, d)
                recs = []
                for _ in range(M):
                    w = [rnd.randrange(2 ** l) for _ in range(W)]
                    if mode == C.MODE_INTV:
                        for a in range(d):
                            w[2 * a], w[2 * a + 1] = sorted((w[2 * a], w[2 * a + 1]))
                    recs.append(w)
                q = [rnd.randrange(2 ** l) for _ in range(P.query_words(mode, d))]
                if mode != C.MODE_INTV and rnd.random() < 0.5:
                    q = list(recs[0][:len(q)])
                pays = [rnd.randrange(2 ** 5) for _ in range(M)]
                B = C.PlainBackend()
                qc = [[B.const(b) for b in P.bits_of(v, l)] for v in q]
                rc = [[[B.const(b) for b in P.bits_of(v, l)] for v in r] for r in recs]
                pc = [[B.const(b) for b in P.bits_of(v, 5)] for v in pays]
                R, _, _ = C.velopir(B, mode, qc, rc, pc, l, d, 5, flags, threads=1)
                got = sum(int(b[0]) << j for j, b in enumerate(R))
                assert got == C.plain_result(mode, q, recs, pays, d, flags, l), (mode, d, flags, M)


# ----------------------------------------------------------------------------------- P8 on TFHE
def test_tfhe_comparator_small(okeys):
    """thm:comple on real ciphertexts at l = 3 (9 BR each) for a few pairs, threaded."""
    k = okeys
    B = C.TfheBackend(k)
    pairs = [(0, 0), (3, 5), (5, 3), (7, 6), (2, 2), (6, 7)]

    def run(pq):
        z1, z2 = pq
        a = [k.encrypt(b, 31, 10 * z1 + 100 * z2 + j) for j, b in enumerate(P.bits_of(z1, 3))]
        b = [k.encrypt(bb, 32, 10 * z1 + 100 * z2 + j) for j, bb in enumerate(P.bits_of(z2, 3))]
        return k.decrypt(C.hom_comp_le(B, a, b, 3)), int(z1 <= z2)

    for got, want in POOL.map(run, pairs):
        assert got == want


def test_tfhe_prefix_comparator_small(okeys):
    """R23 on real ciphertexts at l = 3 (AND-with-NOT leaves, XNORs, MUX / AND merges; the result negated
    for <=): decrypts to the unsigned predicate for a few pairs, threaded."""
    k = okeys
    B = C.TfheBackend(k)
    pairs = [(0, 0), (3, 5), (5, 3), (7, 6), (6, 7), (4, 4)]

    def run(pq):
        z1, z2 = pq
        a = [k.encrypt(b, 33, 10 * z1 + 100 * z2 + j) for j, b in enumerate(P.bits_of(z1, 3))]
        b = [k.encrypt(bb, 34, 10 * z1 + 100 * z2 + j) for j, bb in enumerate(P.bits_of(z2, 3))]
        return (k.decrypt(C.hom_comp_le_prefix(B, a, b, 3)), k.decrypt(C.hom_comp_l_prefix(B, a, b, 3))), \
            (int(z1 <= z2), int(z1 < z2))

    for got, want in POOL.map(run, pairs):
        assert got == want
