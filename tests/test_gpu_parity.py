"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bit-exact everywhere: torus32 integer arithmetic, with the external product computed exactly by either engine --
K2F (FP64 negacyclic FFT, 2 x 16-bit key limbs, rounding error far below 1/2: DESIGN.md section 4) for whole
waves of 8 bootstraps per SM, the NTT kernels (K2, latency / cluster kernels) for narrow tails and on request
(vlp_debug_route).  Sizes span several CTAs and tiles with ragged tails; full-size configs are checked on sampled
outputs the oracle recomputes one by one plus properties that hold at any size (decrypted predicate,
all-trivial closed form P11)."""
import ctypes
import os
import random
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from oracle import circuits as OC  # noqa: E402
from oracle import protocol as OP  # noqa: E402
from paper_2506_12761_b200 import _lib as L  # noqa: E402
from paper_2506_12761_b200 import api as A  # noqa: E402
from synth import make_workload, nand_inputs  # noqa: E402
from synth.workloads import expected_result  # noqa: E402

POOL = ThreadPoolExecutor(max_workers=max(4, os.cpu_count() or 4))
SEED = 123


@pytest.fixture(scope="module")
def gkeys():
    return A.Keys(SEED)


@pytest.fixture(scope="module")
def server(gkeys):
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return A.Server(gkeys, 0)


def rand_tlwe(rng, count):
    return rng.integers(0, 2 ** 32, (count, 632), dtype=np.uint64).astype(np.uint32)


@pytest.fixture
def route():
    """Force a blind-rotation route for one test (vlp_debug_route), restore the default afterwards."""
    def set_route(engine, param=0):
        assert L.lib().vlp_debug_route(engine, param) == 0
    yield set_route
    L.lib().vlp_debug_route(0, 0)


@pytest.mark.parametrize("warps", [1, 3, 8])
def test_fft_engine_steps_bit_exact(server, okeys, route, warps):
    """K2F (FP64 FFT engine) with 1 / 3 / 8 warps (bootstraps) per CTA after 1, 2 and 7 CMux steps == oracle
    BlindRotate: 19 inputs (ragged groups; idle warps in the last CTA), uniformly random masks plus one trivial
    input."""
    route(2, warps)
    rng = np.random.default_rng(10 + warps)
    cts = rand_tlwe(rng, 19)
    cts[:, 631] = 0
    cts[6, :630] = 0
    dev = A.to_device(cts)
    for steps in (1, 2, 7):
        got = A.to_host(server.debug_blind_rotate(dev, steps))
        want = list(POOL.map(lambda c: okeys.blind_rotate(c[:631], steps), cts))
        for i in range(len(cts)):
            assert np.array_equal(got[i], want[i]), (warps, steps, i, np.flatnonzero(got[i] != want[i])[:8])


def test_fft_engine_full_630_and_extreme_digits(server, okeys, route):
    """K2F over all 630 steps on fresh encryptions and on inputs whose first steps see extreme gadget digits
    (accumulator words near +-2^31 give digits of magnitude 64: the largest FFT inputs), byte-equal to the
    oracle; and the same level run by the NTT engine gives the same bytes."""
    k = server.keys
    cts = np.concatenate([k.encrypt_bits([1, 0, 1, 1, 0], 93),
                          rand_tlwe(np.random.default_rng(4), 4)])
    cts[5:, 631] = 0x80000000  # b = 1/2: the test vector rotates by 1024 -> acc = +-mu everywhere, D = +-2 mu
    route(2, 8)
    got = A.to_host(server.debug_blind_rotate(A.to_device(cts), 630))
    want = list(POOL.map(lambda c: okeys.blind_rotate(c[:631], 630), cts))
    for i in range(len(cts)):
        assert np.array_equal(got[i], want[i]), i
    route(1, 5)
    assert np.array_equal(A.to_host(server.debug_blind_rotate(A.to_device(cts), 630)), got)


@pytest.mark.parametrize("extra", [0, 1, 150, 900, 1183])
def test_default_route_wave_and_tail_bit_exact(server, okeys, extra):
    """The default routing of a level (K2F whole waves of 8 x SMs, then the tail: <= 1 per SM on the NTT latency /
    cluster kernels, 2-5 per SM on NTT K2<b>, 6-8 per SM on K2F with that many warps): 2 CMux steps on 8 x 148 +
    extra inputs; sampled rows on both sides of the split and the ragged end byte-equal to the oracle."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    count = 8 * sms + extra
    rng = np.random.default_rng(100 + extra)
    cts = rand_tlwe(rng, count)
    cts[:, 631] = 0
    got = A.to_host(server.debug_blind_rotate(A.to_device(cts), 2))
    idx = sorted(set([i for i in (0, 7, 8, 8 * sms - 1, 8 * sms, 8 * sms + 1) if i < count] + [count - 2, count - 1] +
                     random.Random(extra).sample(range(count), 8)))
    want = list(POOL.map(lambda i: okeys.blind_rotate(cts[i, :631], 2), idx))
    for i, w in zip(idx, want):
        assert np.array_equal(got[i], w), (extra, i)


def test_multi_wave_level_one_launch_per_wave(server, okeys, route):
    """A level of 3 whole K2F waves + 100 (one kernel launch per wave, then the tail): every row byte-equal to the
    same level on the NTT engine (K2 waves + K2 tail) after 3 CMux steps, and sampled rows (first / last of each
    wave, the ragged end) byte-equal to the oracle."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    count = 3 * 8 * sms + 100
    rng = np.random.default_rng(77)
    cts = rand_tlwe(rng, count)
    cts[:, 631] = 0
    dev = A.to_device(cts)
    got = A.to_host(server.debug_blind_rotate(dev, 3))
    route(1, 0)
    ntt = A.to_host(server.debug_blind_rotate(dev, 3))
    assert np.array_equal(got, ntt)
    w = 8 * sms
    idx = sorted(set([0, w - 1, w, 2 * w - 1, 2 * w, 3 * w - 1, 3 * w, count - 1]))
    want = list(POOL.map(lambda i: okeys.blind_rotate(cts[i, :631], 3), idx))
    for i, x in zip(idx, want):
        assert np.array_equal(got[i], x), i


def test_blind_rotate_steps_bit_exact(server, okeys, route):
    """K2 (NTT engine, forced) after 1, 2 and 7 CMux steps (raw TRLWE accumulator) == oracle BlindRotate, 9 inputs (3 CTAs,
    ragged), uniformly random masks (every abar_i != 0 path) plus one trivial input."""
    route(1, 0)
    rng = np.random.default_rng(1)
    cts = rand_tlwe(rng, 9)
    cts[:, 631] = 0
    cts[4, :630] = 0
    dev = A.to_device(cts)
    for steps in (1, 2, 7):
        got = A.to_host(server.debug_blind_rotate(dev, steps))
        want = list(POOL.map(lambda c: okeys.blind_rotate(c[:631], steps), cts))
        for i in range(len(cts)):
            assert np.array_equal(got[i], want[i]), (steps, i, np.flatnonzero(got[i] != want[i])[:8])


@pytest.mark.parametrize("tail", [1, 50, 100, 150, 300, 600])
def test_blind_rotate_wave_split_bit_exact(server, okeys, route, tail):
    """NTT engine (forced): a level of 5 x 148 + tail blind rotations runs as one whole wave (5 bootstraps per
    CTA) plus a tail wave (kernels.cu launch_blind_rotate): tail 1 on the 6-CTA cluster kernel, 50 on the 2-CTA
    cluster kernel, 100 on the 6-group latency kernel, 150 / 300 / 600 on 2 / 3 / 5 bootstraps per CTA.  2 CMux
    steps; sampled rows on both sides of the split and the ragged end byte-equal to the oracle."""
    route(1, 0)
    count = 740 + tail
    rng = np.random.default_rng(tail)
    cts = rand_tlwe(rng, count)
    cts[:, 631] = 0
    got = A.to_host(server.debug_blind_rotate(A.to_device(cts), 2))
    idx = sorted(set([i for i in (0, 4, 5, 738, 739, 740, 741) if i < count] + [count - 2, count - 1] +
                     random.Random(tail).sample(range(count), 8)))
    want = list(POOL.map(lambda i: okeys.blind_rotate(cts[i, :631], 2), idx))
    for i, w in zip(idx, want):
        assert np.array_equal(got[i], w), (tail, i)


def test_blind_rotate_full_bit_exact(server, okeys):
    """All 630 steps on 5 fresh encryptions (a ragged group of 4 + 1)."""
    cts = server.keys.encrypt_bits([1, 0, 1, 1, 0], 91)
    got = A.to_host(server.debug_blind_rotate(A.to_device(cts), 630))
    want = list(POOL.map(lambda c: okeys.blind_rotate(c[:631], 630), cts))
    for i in range(5):
        assert np.array_equal(got[i], want[i]), i


@pytest.mark.parametrize("count", [1, 17, 130, 300])
def test_keyswitch_bit_exact(server, okeys, count):
    """K3T (tcgen05 int8 GEMM key switch) on random N-LWE rows: 1 job (one M tile, 127 idle rows), 17, 130 (two
    M tiles, ragged) and 300 (three M tiles; 30 tiles over the 10 N tiles, persistent CTAs): every output word
    byte-equal to the oracle's KeySwitch (R6), pad word 0."""
    rng = np.random.default_rng(count)
    nl = rng.integers(0, 2 ** 32, (count, 1028), dtype=np.uint64).astype(np.uint32)
    nl[:, 1025:] = 0
    got = A.to_host(server.debug_keyswitch(A.to_device(nl)))
    want = list(POOL.map(lambda r: okeys.keyswitch(r[:1025]), nl))
    for i in range(count):
        assert np.array_equal(got[i, :631], want[i]), i
        assert got[i, 631] == 0


def _gate_program(server, op, a, b, c=None):
    count = a.shape[0]
    prog = A.Program.gates(server, op, count)
    in1 = b if c is None else np.concatenate([b, c])
    out = torch.zeros((count, 632), dtype=torch.int32, device="cuda:0")
    prog.eval(A.to_device(a), A.to_device(in1), out)
    torch.cuda.synchronize()
    return A.to_host(out)


@pytest.mark.parametrize("op", [L.AND, L.NAND, L.OR, L.XOR, L.XNOR, L.MUX])
def test_gate_batches_bit_exact(server, okeys, op):
    """Every gate type on 13 fresh input pairs (4 CTAs, ragged): ciphertexts byte-equal to the oracle's
    gates, decrypting to the truth table (R10)."""
    count = 13
    rng = np.random.default_rng(op)
    bits = rng.integers(0, 2, (3, count), dtype=np.uint8)
    k = server.keys
    a = k.encrypt_bits(bits[0], 500 + op, 0)
    b = k.encrypt_bits(bits[1], 600 + op, 0)
    c = k.encrypt_bits(bits[2], 700 + op, 0) if op == L.MUX else None
    got = _gate_program(server, op, a, b, c)
    if op == L.MUX:
        want = list(POOL.map(lambda i: okeys.mux(a[i, :631], b[i, :631], c[i, :631]), range(count)))
        truth = np.where(bits[0] == 1, bits[1], bits[2])
    else:
        want = list(POOL.map(lambda i: okeys.gate(op, a[i, :631], b[i, :631]), range(count)))
        f = {L.AND: lambda x, y: x & y, L.NAND: lambda x, y: 1 - (x & y), L.OR: lambda x, y: x | y,
             L.XOR: lambda x, y: x ^ y, L.XNOR: lambda x, y: 1 - (x ^ y)}[op]
        truth = f(bits[0], bits[1])
    for i in range(count):
        assert np.array_equal(got[i, :631], want[i]), i
    assert np.array_equal(k.decrypt_bits(got), truth)


def test_nand_batch_sampled(server, okeys):
    """Config 5 shape at 2^12 + 37 gates (ragged): every output decrypts to NAND; 24 sampled outputs are
    recomputed by the oracle and byte-equal."""
    count = 4096 + 37
    a_bits, b_bits = nand_inputs(count, 77)
    k = server.keys
    a = k.encrypt_bits(a_bits, 2005, 0)
    b = k.encrypt_bits(b_bits, 2005, count)
    got = _gate_program(server, L.NAND, a, b)
    assert np.array_equal(k.decrypt_bits(got), 1 - (a_bits & b_bits))
    idx = sorted(random.Random(5).sample(range(count), 23)) + [count - 1]
    want = list(POOL.map(lambda i: okeys.gate(O.NAND, a[i, :631], b[i, :631]), idx))
    for i, w in zip(idx, want):
        assert np.array_equal(got[i, :631], w), i


def _run_config(server, wl, query_seed=7, pk_seed=None):
    k = server.keys
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    q = k.encrypt_query(m, wl.query, query_seed)
    db = k.encrypt_db(m, wl.records, wl.payloads, pk_seed=wl.key_seed + 1 if pk_seed is None else pk_seed)
    prog = A.Program.velopir(server, m)
    out = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
    prog.eval(A.to_device(q), A.to_device(db), out)
    torch.cuda.synchronize()
    return prog, q, db, A.to_host(out)


_VARIANT_FLAGS = {"paper": 0, "prefix": OC.F_PREFIX_COMP, "linear": OC.F_LINEAR_SUM,
                  "prefix+linear": OC.F_PREFIX_COMP | OC.F_LINEAR_SUM}


@pytest.mark.parametrize("variant", list(_VARIANT_FLAGS))
def test_config1_full_parity(server, variant):
    """Config 1 (IntV 1D tiny): the final aggregate, every record's validation bit and masked payload are
    byte-equal to the oracle's alg:VeLoPIR, and decrypt to the plain predicate; also with the R23 prefix
    comparators (8 levels instead of 13) and / or the R24 linear aggregation (masks in the {0, 1/2} encoding)."""
    wl = make_workload(1, key_seed=SEED, flags=OC.CONFIG_FLAGS | _VARIANT_FLAGS[variant])
    okeys = O.OracleKeys(SEED)
    prog, q, db, out = _run_config(server, wl)
    per = A.record_cts(A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags))
    # oracle from the same inputs it generates itself (same seeds; byte-equality of the inputs is pinned
    # by test_library_host.py)
    oq = OP.encrypt_query(okeys, wl.query, wl.l_I, 7)
    recs, pays = [], []
    for i in range(wl.M):
        r, p = OP.server_enc_record(okeys, wl.key_seed + 1, i, [int(v) for v in wl.records[i]], int(wl.payloads[i]),
                                    wl.l_I, wl.l_S)
        recs.append(r)
        pays.append(p)
        assert np.array_equal(db[i * per:(i + 1) * per, :631], np.array([c for w in r for c in w] + p))
    R, vs, masked = OC.velopir(OC.TfheBackend(okeys), wl.mode, oq, recs, pays, wl.l_I, wl.d, wl.l_S, wl.flags)
    mid = A.to_host(prog.intermediate())
    for i in range(wl.M):
        assert np.array_equal(mid[prog.node_row(0, i), :631], vs[i]), ("v", i)
        for j in range(wl.l_S):
            assert np.array_equal(mid[prog.node_row(1, i, j), :631], masked[i][j]), ("mask", i, j)
    for j in range(wl.l_S):
        assert np.array_equal(out[j, :631], R[j]), ("R", j)
    want = OC.plain_result(wl.mode, wl.query, [list(map(int, r)) for r in wl.records], wl.payloads, wl.d, wl.flags)
    assert server.keys.decrypt_value(out) == want


def _trivial_db(wl, per):
    """All-trivial inputs (P11): (0, Ecd(bit)) for every record bit."""
    W = wl.records.shape[1]
    db = np.zeros((wl.M * per, 632), np.uint32)
    for i in range(wl.M):
        bits = [(int(wl.records[i, k]) >> j) & 1 for k in range(W) for j in range(wl.l_I)]
        bits += [(int(wl.payloads[i]) >> j) & 1 for j in range(wl.l_S)]
        db[i * per:(i + 1) * per, 630] = np.where(np.array(bits) == 1, 0x20000000, 0xE0000000)
    return db


@pytest.mark.parametrize("cfg", [2, 3])
def test_all_trivial_closed_form_full_size(server, cfg):
    """P11 at full size: with trivial (noiseless, zero-mask) inputs every bootstrap reduces to the P3
    closed form and every key switch to the identity, so the aggregate must be exactly (0, Ecd(bit)) of
    the plain result, byte for byte (exercises the scheduler, linear forms, MUX combine, tree, layout)."""
    wl = make_workload(cfg, key_seed=SEED)
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    per = A.record_cts(m)
    db = _trivial_db(wl, per)
    q = np.zeros((len(wl.query) * wl.l_I, 632), np.uint32)
    for w, v in enumerate(wl.query):
        for j in range(wl.l_I):
            q[w * wl.l_I + j, 630] = 0x20000000 if (v >> j) & 1 else 0xE0000000
    prog = A.Program.velopir(server, m)
    out = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
    prog.eval(A.to_device(q), A.to_device(db), out)
    torch.cuda.synchronize()
    out = A.to_host(out)
    want = OC.plain_result(wl.mode, wl.query, [list(map(int, r)) for r in wl.records], wl.payloads, wl.d, wl.flags)
    assert not out[:, :630].any()
    assert [int(x) for x in out[:, 630]] == [0x20000000 if (want >> j) & 1 else 0xE0000000 for j in range(wl.l_S)]


def _full_size_sampled(server, cfg, sample, keep_all=True, per_level=4):
    """A config at full size: decrypted result == plain predicate; the sampled records' validation bits and
    masked payloads are recomputed by the oracle (from the same seeded inputs) and byte-equal.  keep_all:
    every intermediate keeps its row (VLP_F_KEEP_ALL), so 4 random gates of every level are rechecked too;
    otherwise rows are recycled by liveness (the production layout) and only the kept rows are compared."""
    wl = make_workload(cfg, key_seed=SEED)
    if keep_all:
        wl = make_workload(cfg, key_seed=SEED, flags=wl.flags | L.F_KEEP_ALL)
    prog, q, db, out = _run_config(server, wl)
    want = OC.plain_result(wl.mode, wl.query, [list(map(int, r)) for r in wl.records], wl.payloads, wl.d, wl.flags)
    assert server.keys.decrypt_value(out) == want
    okeys = O.OracleKeys(SEED)
    oq = OP.encrypt_query(okeys, wl.query, wl.l_I, 7)
    mid = A.to_host(prog.intermediate())

    def one(i):
        r, p = OP.server_enc_record(okeys, wl.key_seed + 1, i, [int(v) for v in wl.records[i]], int(wl.payloads[i]),
                                    wl.l_I, wl.l_S)
        return OC.record_outputs(OC.TfheBackend(okeys), wl.mode, oq, r, p, wl.l_I, wl.d, wl.flags)

    for i, (v, masked) in zip(sample, POOL.map(one, sample)):
        assert np.array_equal(mid[prog.node_row(0, i), :631], v), ("v", i)
        for j in range(wl.l_S):
            assert np.array_equal(mid[prog.node_row(1, i, j), :631], masked[j]), ("mask", i, j)
    if keep_all:  # plus pure-function parity of per_level random gates of every level (SURVEY 4 layer 3)
        regions = {0: q, 1: db, 2: mid, 3: out}
        assert _gate_checks(prog, regions, okeys, per_level=per_level, seed=cfg) >= per_level * (prog.info.levels - 6)
    return wl, want


def _trivial_run(server, mode, d, l_I, l_S, flags, records, payloads, query):
    """P11 on explicit records: every input trivial (0, Ecd(bit)); returns the l_S output rows."""
    m = A.meta(mode, len(records), l_I, l_S, d, flags)
    per = A.record_cts(m)
    W = len(records[0])
    db = np.zeros((len(records) * per, 632), np.uint32)
    for i, (rec, pay) in enumerate(zip(records, payloads)):
        bits = [(int(rec[k]) >> j) & 1 for k in range(W) for j in range(l_I)] + [(int(pay) >> j) & 1 for j in range(l_S)]
        db[i * per:(i + 1) * per, 630] = np.where(np.array(bits) == 1, 0x20000000, 0xE0000000)
    q = np.zeros((len(query) * l_I, 632), np.uint32)
    for w, v in enumerate(query):
        for j in range(l_I):
            q[w * l_I + j, 630] = 0x20000000 if (int(v) >> j) & 1 else 0xE0000000
    out = torch.zeros((l_S, 632), dtype=torch.int32, device="cuda:0")
    server.eval(m, A.to_device(q), A.to_device(db), out)
    torch.cuda.synchronize()
    return A.to_host(out)


@pytest.mark.parametrize("case", ["idm32x64", "rect32x64", "rect32x64_prefix", "intv32_prefix_halfopen", "cov32",
                                  "intv2x1_single", "idm_or_serial"])
def test_all_trivial_extreme_widths(server, case):
    """P11 at the width limits of the ABI (l_I = 32, l_S = 64), a single record (no aggregation tree), the
    minimum comparator width l_I = 2, non-power-of-two M, and the paper-literal serial/OR variants: the
    output must be exactly (0, Ecd(bit)) of the plain predicate."""
    rng = np.random.default_rng(hash(case) & 0xFFFF)
    full = lambda l: int(rng.integers(0, 2 ** l, dtype=np.uint64))  # noqa: E731
    if case == "idm32x64":
        mode, d, l_I, l_S, flags = OC.MODE_IDM, 1, 32, 64, OC.CONFIG_FLAGS
        q = [full(32)]
        recs = [(full(32),), (q[0],), (full(32),)]
    elif case in ("rect32x64", "rect32x64_prefix"):
        mode, d, l_I, l_S, flags = OC.MODE_INTV, 2, 32, 64, OC.CONFIG_FLAGS | (OC.F_PREFIX_COMP if "prefix" in case else 0)
        q = [full(31), full(31)]
        recs = [(q[0] - 5, q[0] + 9, q[1] - 1, q[1]), (q[0], q[0], q[1] + 1, q[1] + 2), (0, 2 ** 32 - 1, 0, 2 ** 32 - 1),
                (q[0] + 1, q[0] + 3, 0, 7), (0, q[0], q[1], 2 ** 32 - 1)]
    elif case == "intv32_prefix_halfopen":
        mode, d, l_I, l_S, flags = OC.MODE_INTV, 1, 32, 33, OC.F_UNSIGNED | OC.F_SUM_TREE | OC.F_PREFIX_COMP
        q = [full(32)]
        recs = [(q[0], q[0] + 1), (q[0] - 3, q[0]), (0, 2 ** 32 - 1), (q[0] ^ 1, q[0] ^ 1), (0, q[0])]
        recs = [(lo % 2 ** 32, hi % 2 ** 32) for lo, hi in recs]
    elif case == "cov32":
        mode, d, l_I, l_S, flags = OC.MODE_COV, 2, 32, 40, OC.CONFIG_FLAGS
        q = [full(32), full(32)]
        recs = [(q[0], q[1]), (q[0], q[1] ^ 1), (q[0], q[1])]
    elif case == "intv2x1_single":
        mode, d, l_I, l_S, flags = OC.MODE_INTV, 1, 2, 1, OC.CONFIG_FLAGS
        q = [2]
        recs = [(1, 3)]
    else:
        mode, d, l_I, l_S, flags = OC.MODE_IDM, 1, 9, 7, OC.F_OR_REDUCE
        q = [300]
        recs = [(300,), (5,), (300,), (511,), (0,), (300,), (299,)]
    pays = [full(l_S) for _ in recs]
    out = _trivial_run(server, mode, d, l_I, l_S, flags, recs, pays, q)
    want = OC.plain_result(mode, q, [list(r) for r in recs], pays, d, flags, l_I)
    assert not out[:, :630].any()
    assert [int(x) for x in out[:, 630]] == [0x20000000 if (want >> j) & 1 else 0xE0000000 for j in range(l_S)]


def test_fft_rounding_margin_at_scale(server, route):
    """K2F's exactness argument measured on the product kernel: with the rounding monitor on
    (vlp_debug_fft_error), every limb result of a full config-2 evaluation (132,080 bootstraps x 630 steps x 4,096
    roundings = 3.4e11) and of a wave of extreme-digit inputs (accumulator words near +-2^31: digits of magnitude
    64) lies within 2^-10 of the integer it rounds to -- the margin is 1/2 -- and the monitored build gives the same
    bytes as the product build."""
    err = torch.zeros(1, dtype=torch.int64, device="cuda:0")
    wl = make_workload(2, key_seed=SEED)
    k = server.keys
    _, _, _, plain = _run_config(server, wl)
    A.check(A.lib().vlp_debug_fft_error(ctypes.c_void_p(err.data_ptr())))
    try:
        _, _, _, mon = _run_config(server, wl)
        assert np.array_equal(mon, plain)
        cts = k.encrypt_bits(np.random.default_rng(8).integers(0, 2, 1184, dtype=np.uint8), 41)
        cts[:, 631] = 0x80000000  # acc = +-mu everywhere after the test-vector rotation: D = +-2 mu
        route(2, 8)
        server.debug_blind_rotate(A.to_device(cts), 630)
        torch.cuda.synchronize()
    finally:
        A.check(A.lib().vlp_debug_fft_error(None))
    worst = float(np.array([int(err.item())], dtype=np.int64).view(np.float64)[0])
    print(f"K2F largest rounding distance: {worst:.3e}")
    assert 0.0 < worst < 2.0 ** -10


def test_server_eval_host_equals_device_call(server):
    """vlp_server_eval_host (the e2e call of bench.py at N = 1: host query in, host result out) gives the bytes of
    vlp_server_eval on device buffers, on config 1 and on a 512-record shard of config 2."""
    k = server.keys
    for cfg, first, count in ((1, 0, None), (2, 512, 512)):
        wl = make_workload(cfg, key_seed=SEED)
        count = wl.M if count is None else count
        m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
        q = k.encrypt_query(m, wl.query, 7)
        db = A.to_device(k.encrypt_db(m, wl.records[first:first + count], wl.payloads[first:first + count],
                                      pk_seed=9, first=first, count=count))
        dev_out = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
        server.eval(m, A.to_device(q), db, dev_out, first=first, count=count)
        host_out = np.zeros((wl.l_S, 632), np.uint32)
        server.eval_host(m, np.ascontiguousarray(q, dtype=np.uint32), db, host_out, first=first, count=count)
        assert np.array_equal(host_out, A.to_host(dev_out)), cfg


def test_config2_full_size_sampled(server):
    """Config 2 at full size (IntV 1D, 1024 records, 132,080 BR) in the production layout (rows recycled by
    liveness, as bench.py runs it): predicate + records 3 and 1023 byte-equal."""
    _full_size_sampled(server, 2, [3, 1023], keep_all=False)


def test_config3_full_size_sampled(server):
    """Config 3 at full size (rectangle containment, 4096 records, 1,060,832 BR; the bench headline): predicate +
    8 records (incl. 0, 4095 and every record containing the query) byte-equal, and 16 random gates of every level
    recomputed by the oracle from the GPU's own inputs."""
    wl = make_workload(3, key_seed=SEED)
    hits = [i for i in range(wl.M) if _contains(wl, i)]
    sample = sorted(set([0, 4095] + hits[:4] + random.Random(3).sample(range(wl.M), 6)))
    _full_size_sampled(server, 3, sample, per_level=16)


def test_config4_full_size_sampled(server):
    """Config 4 at full size (IdM, 65,536 records, 6,750,176 BR on one GPU): predicate + 8 records (the matching
    record if the seed put the query id in the DB, the last one, 6 random) byte-equal, and 16 random gates of every
    level recomputed by the oracle."""
    wl = make_workload(4, key_seed=SEED)
    hits = [i for i in range(wl.M) if int(wl.records[i][0]) == int(wl.query[0])]
    sample = sorted(set((hits[:1] or [1]) + [wl.M - 1] + random.Random(4).sample(range(wl.M), 6)))
    _full_size_sampled(server, 4, sample, per_level=16)


def test_paper_cov_4096_full_size_sampled(server):
    """the paper's CoV mode (alg:BB2: HomEQ trees on both coordinates + AND) on a
    4096-point database (config 10): predicate + 8 records (incl. the matching one, if any) byte-equal, and 16
    random gates of every level recomputed by the oracle from the GPU's own inputs."""
    wl = make_workload(10, key_seed=SEED)
    sample = sorted(set(wl.forced[:1] + [0, wl.M - 1] + random.Random(10).sample(range(wl.M), 6)))
    _full_size_sampled(server, 10, sample, per_level=16)


def _contains(wl, i):
    r = [int(v) for v in wl.records[i]]
    return all(r[2 * k] <= int(wl.query[k]) <= r[2 * k + 1] for k in range(wl.d))


def _full_parity_small(server, mode, d, l_I, l_S, flags, records, payloads, query, okeys_seed=SEED):
    """Full byte parity of a small instance (every record's v and masked payload, and R) vs the oracle."""
    m = A.meta(mode, len(records), l_I, l_S, d, flags)
    k = server.keys
    okeys = O.OracleKeys(okeys_seed)
    q = k.encrypt_query(m, query, 7)
    db = k.encrypt_db(m, np.array(records, np.uint64), np.array(payloads, np.uint64), pk_seed=99)
    prog = A.Program.velopir(server, m)
    out = torch.zeros((l_S, 632), dtype=torch.int32, device="cuda:0")
    prog.eval(A.to_device(q), A.to_device(db), out)
    torch.cuda.synchronize()
    out = A.to_host(out)
    oq = OP.encrypt_query(okeys, query, l_I, 7)
    recs, pays = [], []
    for i in range(len(records)):
        r, p = OP.server_enc_record(okeys, 99, i, list(records[i]), payloads[i], l_I, l_S)
        recs.append(r)
        pays.append(p)
    R, vs, masked = OC.velopir(OC.TfheBackend(okeys), mode, oq, recs, pays, l_I, d, l_S, flags)
    mid = A.to_host(prog.intermediate())
    for i in range(len(records)):
        if len(records) > 1 or not (flags & OC.F_SUM_TREE):
            assert np.array_equal(mid[prog.node_row(0, i), :631], vs[i]), ("v", i)
    for j in range(l_S):
        assert np.array_equal(out[j, :631], R[j]), ("R", j)
    want = OC.plain_result(mode, query, records, payloads, d, flags, l_I)
    assert k.decrypt_value(out) == want
    return want


def test_paper_cov_mode_full_parity(server):
    """Paper CoV (alg:BB2: HomEQ(x, loc_x) AND HomEQ(y, loc_y)), EQ tree, d = 2, l = 4, 3 records (not a
    power of two), one exact match."""
    recs = [(3, 9), (5, 12), (3, 12)]
    want = _full_parity_small(server, OC.MODE_COV, 2, 4, 3, OC.CONFIG_FLAGS, recs, [5, 2, 6], [5, 12])
    assert want == 2


def test_prefix_rectangle_half_open_full_parity(server):
    """R23 prefix comparators on the rectangle circuit with half-open upper bounds (CompL(x, hi) = [hi > x])
    and the serial HomSum: every record's v and the result byte-equal to the oracle."""
    recs = [(2, 9, 0, 15), (5, 6, 3, 4), (0, 15, 7, 8), (6, 7, 3, 5)]
    _full_parity_small(server, OC.MODE_INTV, 2, 4, 3, OC.F_UNSIGNED | OC.F_PREFIX_COMP, recs, [5, 2, 6, 1], [6, 3])


def test_paper_literal_intv_serial_full_parity(server):
    """Paper-literal IntV: signed comparators (final MUX on ct1[l-1]), half-open upper bound via
    HomCompL, serial HomEQ flag irrelevant, serial HomSum from trivial Enc(0)."""
    recs = [(-3 & 15, 2), (1, 7), (-8 & 15, -1 & 15)]
    flags = 0
    _full_parity_small(server, OC.MODE_INTV, 1, 4, 2, flags, recs, [1, 2, 3], [1])


def test_idm_serial_eq_or_reduce_full_parity(server):
    """IdM with the serial alg:HomEQ and the OR reduction flag (R19), 4 records."""
    flags = OC.F_SUM_TREE | OC.F_OR_REDUCE
    _full_parity_small(server, OC.MODE_IDM, 1, 5, 2, flags, [(7,), (19,), (7,), (30,)], [1, 2, 2, 3], [7])


def test_problem_statement_calls(server, okeys):
    """vlp_server_eval / vlp_server_combine / vlp_gate_batch / vlp_decrypt_result: config 1
    through server_eval equals the program path byte for byte; two shards of 2 records + combine(G=2)
    equal the single-shot result (R15); a MUX batch with separate b and c buffers equals the oracle."""
    wl = make_workload(1, key_seed=SEED)
    k = server.keys
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    q = A.to_device(k.encrypt_query(m, wl.query, 7))
    db_h = k.encrypt_db(m, wl.records, wl.payloads, pk_seed=wl.key_seed + 1)
    db = A.to_device(db_h)
    prog = A.Program.velopir(server, m)
    ref = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
    prog.eval(q, db, ref)
    out = torch.zeros_like(ref)
    server.eval(m, q, db, out)
    torch.cuda.synchronize()
    assert np.array_equal(A.to_host(out), A.to_host(ref))
    bits, value = k.decrypt_result(A.to_host(out), wl.l_S)
    want = OC.plain_result(wl.mode, wl.query, [list(map(int, r)) for r in wl.records], wl.payloads, wl.d, wl.flags)
    assert value == want and list(bits) == [(want >> j) & 1 for j in range(wl.l_S)]
    # two shards of M/2 records, then the top tree level
    per = A.record_cts(m)
    half = wl.M // 2
    roots = torch.zeros((2, wl.l_S, 632), dtype=torch.int32, device="cuda:0")
    for r in range(2):
        server.eval(m, q, db[r * half * per:(r + 1) * half * per], roots[r], first=r * half, count=half)
    comb = torch.zeros_like(ref)
    server.combine(m, 2, roots, comb)
    torch.cuda.synchronize()
    assert np.array_equal(A.to_host(comb), A.to_host(ref))
    # MUX with separate b / c device buffers
    rng = np.random.default_rng(11)
    bits3 = rng.integers(0, 2, (3, 9), dtype=np.uint8)
    a, b, c = (k.encrypt_bits(bits3[i], 800 + i, 0) for i in range(3))
    o = torch.zeros((9, 632), dtype=torch.int32, device="cuda:0")
    server.gate_batch(L.MUX, A.to_device(a), A.to_device(b), o, c_dev=A.to_device(c))
    torch.cuda.synchronize()
    got = A.to_host(o)
    want_ct = list(POOL.map(lambda i: okeys.mux(a[i, :631], b[i, :631], c[i, :631]), range(9)))
    for i in range(9):
        assert np.array_equal(got[i, :631], want_ct[i]), i
    assert np.array_equal(k.decrypt_bits(got), np.where(bits3[0] == 1, bits3[1], bits3[2]))


def test_linear_aggregation_sharded_decrypts(server):
    """R24 with sharding: every shard refreshes its own sum into the standard encoding and the roots combine
    through the XOR tree (vlp_server_combine), so 2- and 4-shard results decrypt to the same predicate as the
    single-shot result (decrypt-equal; R24 bytes depend on the shard count)."""
    wl = make_workload(6, key_seed=SEED)
    wl = make_workload(6, key_seed=SEED, M=8, flags=wl.flags | OC.F_LINEAR_SUM)
    k = server.keys
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    q = A.to_device(k.encrypt_query(m, wl.query, 7))
    db = A.to_device(k.encrypt_db(m, wl.records, wl.payloads, pk_seed=wl.key_seed + 1))
    want = expected_result(wl)
    one = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
    server.eval(m, q, db, one)
    torch.cuda.synchronize()
    assert k.decrypt_value(A.to_host(one)) == want
    per = A.record_cts(m)
    for G in (2, 4):
        sh = wl.M // G
        roots = torch.zeros((G, wl.l_S, 632), dtype=torch.int32, device="cuda:0")
        for r in range(G):
            server.eval(m, q, db[r * sh * per:(r + 1) * sh * per], roots[r], first=r * sh, count=sh)
        comb = torch.zeros_like(one)
        server.combine(m, G, roots, comb)
        torch.cuda.synchronize()
        assert k.decrypt_value(A.to_host(comb)) == want, G


def test_single_record_min_width_full_parity(server):
    """Degenerate instance on real encryptions: one record (no aggregation tree, the masked payload is the
    result), the minimum comparator width l_I = 2 and a 1-bit payload."""
    want = _full_parity_small(server, OC.MODE_INTV, 1, 2, 1, OC.CONFIG_FLAGS, [(1, 3)], [1], [2])
    assert want == 1


@pytest.mark.parametrize("cfg", [6, 7, 8, 9])
def test_dataset_shapes_predicate(server, cfg):
    """Synthetic stand-ins with the shapes of the paper's datasets (covid-kor / covid-usa IntV rectangles,
    gdacs CoV points, weather-usa IdM with a 128-bit payload): the decrypted answer equals the plain
    predicate; for the gdacs shape, record 0's validation bit and masked payload are byte-equal to the oracle."""
    sample = [0] if cfg == 8 else []
    wl = make_workload(cfg, key_seed=SEED)
    if sample:
        _full_size_sampled(server, cfg, sample, keep_all=False)
        return
    prog, q, db, out = _run_config(server, wl)
    want = OC.plain_result(wl.mode, wl.query, [list(map(int, r)) for r in wl.records], wl.payloads, wl.d, wl.flags)
    assert server.keys.decrypt_value(out) == want


@pytest.mark.parametrize("cfg,extra", [(8, 0), (6, OC.F_PREFIX_COMP | OC.F_LINEAR_SUM)])
def test_multi_query_batch_equals_single(server, cfg, extra):
    """Multi-query packing (vlp_server_eval_batch): 3 queries against the gdacs-shaped DB (and the covid-kor
    shape with the R23 + R24 options) in one schedule; each result is byte-equal to its own single-query
    vlp_server_eval and decrypts to its plain predicate."""
    wl = make_workload(cfg, key_seed=SEED)
    if extra:
        wl = make_workload(cfg, key_seed=SEED, flags=wl.flags | extra)
    k = server.keys
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    db = A.to_device(k.encrypt_db(m, wl.records, wl.payloads, pk_seed=wl.key_seed + 1))
    if wl.mode == OC.MODE_INTV:  # points inside record 0's box, record 5's box, and an arbitrary point
        qvals = [[int(wl.records[r][2 * a]) for a in range(wl.d)] for r in (0, 5)] + [[123, 456][:wl.d]]
    else:
        qvals = [[int(v) for v in wl.records[0]], [int(v) for v in wl.records[5]], [123, 456]]
    qs = [k.encrypt_query(m, qv, 40 + i) for i, qv in enumerate(qvals)]
    out = torch.zeros((3 * wl.l_S, 632), dtype=torch.int32, device="cuda:0")
    server.eval_batch(m, A.to_device(np.concatenate(qs)), db, out, 3)
    torch.cuda.synchronize()
    got = A.to_host(out)
    for i, qv in enumerate(qvals):
        one = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
        server.eval(m, A.to_device(qs[i]), db, one)
        torch.cuda.synchronize()
        assert np.array_equal(got[i * wl.l_S:(i + 1) * wl.l_S], A.to_host(one)), i
        want = OC.plain_result(wl.mode, qv, [list(map(int, r)) for r in wl.records], wl.payloads, wl.d, wl.flags)
        assert k.decrypt_value(got[i * wl.l_S:(i + 1) * wl.l_S]) == want, i


def test_noise_over_depth_at_scale(server):
    """P6 at scale on the GPU path: 20 levels of AND(x, Enc(1)) over 16,384 independent chains (327,680 gate
    bootstraps) never mis-decrypt, and the output phase error has the bootstrapped level predicted by the
    noise model (sigma ~ 3.5e-3; band [2e-3, 5e-3]) at every depth (no growth)."""
    k = server.keys
    s_bits = k.export()[0]
    s = s_bits.astype(np.int64)
    count = 16384
    x = A.to_device(k.encrypt_bits(np.ones(count, np.uint8), 3001, 0))
    sds = []
    for lvl in range(20):
        one = A.to_device(k.encrypt_bits(np.ones(count, np.uint8), 3002 + lvl, 0))
        out = torch.zeros((count, 632), dtype=torch.int32, device="cuda:0")
        server.gate_batch(L.AND, x, one, out)
        torch.cuda.synchronize()
        h = A.to_host(out).astype(np.int64)
        phase = (h[:, 630] - (h[:, :630] * s).sum(axis=1)) % 2 ** 32
        err = ((phase - 0x20000000 + 2 ** 31) % 2 ** 32 - 2 ** 31) / 2 ** 32
        assert np.all(np.abs(err) < 1 / 8), lvl  # every output still decrypts to 1
        sds.append(float(np.sqrt(np.mean(err ** 2))))
        x = out
    assert all(2e-3 < v < 5e-3 for v in sds), sds
    assert max(sds) / min(sds) < 1.1, sds  # bootstrapping refreshes: no growth with depth


def test_device_keygen_equals_host():
    """vlp_keygen_device (masks, ring products a*z and <a, s> on the device, noise on the host)
    gives the same s, z, bsk and ksk as vlp_keygen, byte for byte."""
    kh, kd = A.Keys(321), A.Keys(321, device=0)
    for x, y in zip(kh.export(), kd.export()):
        assert np.array_equal(x, y)


def _next_key(key):
    os.environ["VLP_TEST_HOOKS"] = "1"  # the hook is disabled without it
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32))
    A.check(A.lib().vlp_debug_next_secure_key(A._u32p(k)))


def test_device_secure_preprocessing_equals_host_secure(server):
    """The secure device calls draw their masks from ChaCha20 on the device: under one key (the test hook
    vlp_debug_next_secure_key) vlp_keygen_device_secure == vlp_keygen_secure and vlp_pubkeygen_device_secure ==
    vlp_pubkeygen_secure, byte for byte; the default Python calls (no seed) give fresh samples that decrypt to the
    records' bits."""
    key = (np.arange(8, dtype=np.uint32) * 0x9E3779B9 + 17).astype(np.uint32)
    _next_key(key)
    kh = A.Keys()
    _next_key(key)
    kd = A.Keys(device=0)
    for x, y in zip(kh.export(), kd.export()):
        assert np.array_equal(x, y)
    wl = make_workload(9, key_seed=SEED)
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    k = server.keys
    _next_key(key)
    host = k.encrypt_db(m, wl.records[:16], wl.payloads[:16], count=16)
    _next_key(key)
    pk = A.pubkeygen_device(k, m, None, 0, 16)
    db = A.server_encrypt_db_device(m, pk, wl.records[:16], wl.payloads[:16])
    assert np.array_equal(A.to_host(db), host)
    fresh = A.to_host(A.server_encrypt_db_device(m, A.pubkeygen_device(k, m, None, 0, 16), wl.records[:16],
                                                 wl.payloads[:16]))
    assert not np.array_equal(fresh, host)
    assert np.array_equal(k.decrypt_bits(fresh), k.decrypt_bits(host))


@pytest.mark.parametrize("cfg,count", [(1, None), (9, 16), (3, 512)])
def test_role_separated_device_preprocessing(server, cfg, count):
    """P:192 roles on the GPU: the client's device PubKeyGen (takes sk) then the server's device ServerEnc (takes
    only the pk samples) equal the host PubKeyGen + ServerEnc and the fused device call, byte for byte."""
    wl = make_workload(cfg, key_seed=SEED)
    count = wl.M if count is None else count
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    k = server.keys
    pk = A.pubkeygen_device(k, m, 4321, 0, count)
    db = A.server_encrypt_db_device(m, pk, wl.records[:count], wl.payloads[:count])
    host = k.encrypt_db(m, wl.records[:count], wl.payloads[:count], pk_seed=4321, count=count)
    assert np.array_equal(A.to_host(db), host)
    fused = A.encrypt_db_device(k, m, wl.records[:count], wl.payloads[:count], pk_seed=4321, count=count)
    assert np.array_equal(A.to_host(fused), host)


def test_server_load_records_single_use(server):
    """SURVEY 8(b) load records: the server's vlp_server_load_records of a received host pk equals the host
    PubKeyGen + ServerEnc byte for byte, and the pk is single-use (VLP_EPKUSED)."""
    wl = make_workload(9, key_seed=SEED)
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    k = server.keys
    pk = A.PublicKey(k, m, 0, 16, seed=777)
    db = A.server_load_records(pk, wl.records[:16], wl.payloads[:16])
    assert np.array_equal(A.to_host(db), k.encrypt_db(m, wl.records[:16], wl.payloads[:16], pk_seed=777, count=16))
    with pytest.raises(L.VlpError) as err:
        A.server_load_records(pk, wl.records[:16], wl.payloads[:16])
    assert err.value.code == L.VLP_EPKUSED


@pytest.mark.parametrize("cfg,count", [(1, None), (9, 16), (4, 4096)])
def test_device_encrypt_db_equals_host(server, cfg, count):
    """Device PubKeyGen + ServerEnc (vlp_encrypt_db_device) is byte-identical to the host vlp_pubkeygen +
    vlp_server_encrypt_db (which test_library_host pins to the oracle): config 1, 16 records of the 128-bit
    payload weather shape, and 4096 records of config 4 starting at record 1000."""
    wl = make_workload(cfg, key_seed=SEED)
    k = server.keys
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    first = 1000 if cfg == 4 else 0
    count = wl.M if count is None else count
    recs, pays = wl.records[first:first + count], wl.payloads[first:first + count]
    host = k.encrypt_db(m, recs, pays, pk_seed=77, first=first, count=count)
    dev = A.encrypt_db_device(k, m, recs, pays, pk_seed=77, first=first, count=count)
    torch.cuda.synchronize()
    assert np.array_equal(A.to_host(dev), host)


# ------------------------------------------------------------------ pure-function parity of every gate
# linear form (k0, ax, ay) -> (oracle gate, negate x, negate y); the sign-flipped ANDs are AND gates with
# NOT (free negation, O11) on an input: the R23 prefix comparator's leaves and the AND of two CompLE results
_FORMS = {(0xE0000000, 1, 1): (O.AND, 0, 0), (0x20000000, -1, -1): (O.NAND, 0, 0), (0x20000000, 1, 1): (O.OR, 0, 0),
          (0x40000000, 2, 2): (O.XOR, 0, 0), (0xC0000000, -2, -2): (O.XNOR, 0, 0),
          (0xE0000000, 1, -1): (O.AND, 0, 1), (0xE0000000, -1, 1): (O.AND, 1, 0), (0xE0000000, -1, -1): (O.AND, 1, 1)}


def _gate_checks(prog, regions, okeys, levels=None, per_level=None, seed=0):
    """For every key switch (= gate output) of the chosen levels: rebuild the gate from the schedule's jobs
    (linear form -> op; two half bootstraps -> MUX), recompute it with the oracle from the GPU's own input
    ciphertexts and compare with the GPU's output ciphertext.  Returns the number of gates checked."""
    rng = random.Random(seed)

    def ct(slot):
        return regions[slot >> 28][slot & 0x0FFFFFFF, :631]

    todo = []
    jobs = [prog.level_jobs(lvl) for lvl in range(prog.info.levels)]
    nrows = sum(len(b) for b, _ in jobs)
    by_row = np.zeros(nrows, jobs[0][0].dtype)  # N-LWE row -> its bootstrap job (rows are unique)
    for b, _ in jobs:
        by_row[b["row"]] = b
    for lvl in (range(prog.info.levels) if levels is None else levels):
        ks = jobs[lvl][1]
        idx = range(len(ks)) if per_level is None or len(ks) <= per_level else rng.sample(range(len(ks)), per_level)
        for i in idx:
            k = ks[i]
            if int(k["n1"]) == 0xFFFFFFFF:
                j = by_row[int(k["n0"])]
                form = (int(j["k0"]), int(j["ax"]), int(j["ay"]))
                if int(j["tv"]) == 0 and int(k["add"]) == 0 and form in _FORMS:
                    todo.append((int(k["out"]), "gate", _FORMS[form], int(j["x"]), int(j["y"])))
                else:  # R24 bootstraps: test vector 1/4 and / or a constant after the key switch
                    assert int(k["add"]) in (0, 0x40000000) and int(j["tv"]) in (0, 1), (form, k)
                    todo.append((int(k["out"]), "lin-form", form + (int(j["tv"]), int(k["add"])), int(j["x"]), int(j["y"])))
            else:
                j1, j2 = by_row[int(k["n0"])], by_row[int(k["n1"])]
                assert (int(j1["k0"]), int(j1["ax"]), int(j1["ay"])) == (0xE0000000, 1, 1)
                assert (int(j2["k0"]), int(j2["ax"]), int(j2["ay"])) == (0xE0000000, -1, 1)
                assert int(j1["x"]) == int(j2["x"])
                todo.append((int(k["out"]), "mux", int(j1["x"]), int(j1["y"]), int(j2["y"])))

    def one(t):
        if t[1] == "gate":
            op, nx, ny = t[2]
            x, y = ct(t[3]), ct(t[4])
            return okeys.gate(op, O.OracleKeys.not_(x) if nx else x, O.OracleKeys.not_(y) if ny else y)
        if t[1] == "lin-form":  # c = (0, k0) + ax x + ay y; bootstrap with test vector 1/8 or 1/4; + (0, add)
            k0, ax, ay, tv, add = t[2]
            c = (ax * ct(t[3]).astype(np.int64) + ay * ct(t[4]).astype(np.int64)) % 2 ** 32
            c[-1] = (c[-1] + k0) % 2 ** 32
            o = okeys.bootstrap_mu(c.astype(np.uint32), 0x40000000 if tv else 0x20000000)
            o[-1] = np.uint32((int(o[-1]) + add) % 2 ** 32)
            return o
        return okeys.mux(ct(t[2]), ct(t[3]), ct(t[4]))

    for t, want in zip(todo, POOL.map(one, todo)):
        assert np.array_equal(ct(t[0]), want), t
    return len(todo)


def _linear_checks(prog, regions):
    """R24: every linear job's output row equals the sum of its input rows mod 2^32.  Returns the count."""
    def ct(slot):
        return regions[slot >> 28][slot & 0x0FFFFFFF, :632].astype(np.uint64)

    n = 0
    for lvl in range(prog.info.levels):
        jobs, ins = prog.level_linear(lvl)
        for out, first, count, _ in jobs:
            want = sum(ct(int(ins[first + i])) for i in range(count)) % 2 ** 32
            assert np.array_equal(ct(int(out)), want), (lvl, out)
            n += 1
    return n


@pytest.mark.parametrize("variant", list(_VARIANT_FLAGS))
def test_config1_every_gate_pure_function(server, variant):
    """SURVEY 4 layer 3: every one of config 1's 188 gate outputs (every level) is byte-equal to the oracle's
    gate recomputed from the GPU's own inputs; with the R23 / R24 variants, every one of their gates and every
    linear sum."""
    wl = make_workload(1, key_seed=SEED, flags=OC.CONFIG_FLAGS | _VARIANT_FLAGS[variant] | L.F_KEEP_ALL)
    prog, q, db, out = _run_config(server, wl)
    okeys = O.OracleKeys(SEED)
    regions = {0: q, 1: db, 2: A.to_host(prog.intermediate()), 3: out}
    assert _gate_checks(prog, regions, okeys) == prog.info.gates
    nlin = _linear_checks(prog, regions)
    assert prog.info.levels == {"paper": 13, "prefix": 8, "linear": 12, "prefix+linear": 7}[variant]
    assert (nlin > 0) == ("linear" in variant)
    if variant == "paper":
        assert prog.info.gates == 188
    want = OC.plain_result(wl.mode, wl.query, [list(map(int, r)) for r in wl.records], wl.payloads, wl.d, wl.flags)
    assert server.keys.decrypt_value(out) == want


def test_config2_linear_aggregation(server):
    """R24 at config 2's full size (1024 records = 16 groups of 64): 115,984 BR in 21 levels instead of 132,080
    in 29; the result decrypts to the predicate; the refresh levels' gates (all of them), 8 masks and every
    linear sum are byte-equal to the oracle's recomputation from the GPU's own inputs."""
    wl = make_workload(2, key_seed=SEED, flags=OC.CONFIG_FLAGS | OC.F_LINEAR_SUM | L.F_KEEP_ALL)
    prog, q, db, out = _run_config(server, wl)
    assert (prog.info.br, prog.info.levels) == (115984, 21)
    assert server.keys.decrypt_value(out) == expected_result(wl)
    okeys = O.OracleKeys(SEED)
    regions = {0: q, 1: db, 2: A.to_host(prog.intermediate()), 3: out}
    assert _gate_checks(prog, regions, okeys, levels=[19, 20]) == 16 * 16 + 16
    assert _gate_checks(prog, regions, okeys, levels=[18], per_level=8, seed=3) == 8
    assert _linear_checks(prog, regions) == 16 * 16 + 16


def test_config2_sampled_gates_pure_function(server):
    """SURVEY 4 layer 3 at full size: 16 random gates of each of config 2's 29 levels (all of the narrow
    tree levels) are recomputed by the oracle from the GPU's own input ciphertexts and byte-equal."""
    wl = make_workload(2, key_seed=SEED, flags=OC.CONFIG_FLAGS | L.F_KEEP_ALL)
    prog, q, db, out = _run_config(server, wl)
    okeys = O.OracleKeys(SEED)
    regions = {0: q, 1: db, 2: A.to_host(prog.intermediate()), 3: out}
    assert _gate_checks(prog, regions, okeys, per_level=16, seed=3) >= 16 * 25


def test_nand_max_config5_size_sampled(server, okeys):
    """Config 5's largest batch (2^20 NAND gates on one GPU): every output decrypts to NAND of its inputs, and
    sampled outputs (incl. the first and last) are byte-equal to the oracle's gate."""
    count = 1 << 20
    a_bits, b_bits = nand_inputs(count, 91)
    k = server.keys
    a = k.encrypt_bits(a_bits, 4005, 0)
    b = k.encrypt_bits(b_bits, 4005, count)
    out = torch.zeros((count, 632), dtype=torch.int32, device="cuda:0")
    server.gate_batch(L.NAND, A.to_device(a), A.to_device(b), out)
    torch.cuda.synchronize()
    got = A.to_host(out)
    assert np.array_equal(k.decrypt_bits(got), 1 - (a_bits & b_bits))
    idx = [0, count - 1] + sorted(random.Random(9).sample(range(1, count - 1), 14))
    want = list(POOL.map(lambda i: okeys.gate(O.NAND, a[i, :631], b[i, :631]), idx))
    for i, w in zip(idx, want):
        assert np.array_equal(got[i, :631], w), i


def test_empty_inputs_are_no_ops(server):
    """Degenerate sizes: an empty gate batch and an empty blind-rotation batch launch nothing and succeed."""
    e = torch.zeros((0, 632), dtype=torch.int32, device="cuda:0")
    server.gate_batch(L.NAND, e, e, e)
    acc = server.debug_blind_rotate(e, 630)
    torch.cuda.synchronize()
    assert acc.shape[0] == 0


def test_gate_truth_tables_100_trials(server, okeys):
    """P5 at the SPEC's trial count: every gate type on every input combination, 100
    independent fresh encryptions each (800 for MUX) -- zero decryption errors -- plus byte parity of the
    first trial of each combination with the oracle."""
    k = server.keys
    f = {L.AND: lambda x, y: x & y, L.NAND: lambda x, y: 1 - (x & y), L.OR: lambda x, y: x | y,
         L.XOR: lambda x, y: x ^ y, L.XNOR: lambda x, y: 1 - (x ^ y)}
    for op in (L.AND, L.NAND, L.OR, L.XOR, L.XNOR, L.MUX):
        combos = [(x, y, z) for x in (0, 1) for y in (0, 1) for z in ((0, 1) if op == L.MUX else (0,))]
        bits = np.array([c for c in combos for _ in range(100)], np.uint8).T  # [3][n]
        n = bits.shape[1]
        a, b, c = (k.encrypt_bits(bits[i], 6000 + 10 * op + i, 0) for i in range(3))
        out = torch.zeros((n, 632), dtype=torch.int32, device="cuda:0")
        server.gate_batch(op, A.to_device(a), A.to_device(b), out, c_dev=A.to_device(c) if op == L.MUX else None)
        torch.cuda.synchronize()
        got = A.to_host(out)
        truth = np.where(bits[0] == 1, bits[1], bits[2]) if op == L.MUX else f[op](bits[0], bits[1])
        assert np.array_equal(k.decrypt_bits(got), truth), op
        firsts = list(range(0, n, 100))
        want = list(POOL.map(lambda i: okeys.mux(a[i, :631], b[i, :631], c[i, :631]) if op == L.MUX
                             else okeys.gate(op, a[i, :631], b[i, :631]), firsts))
        for i, w in zip(firsts, want):
            assert np.array_equal(got[i, :631], w), (op, i)


def test_mismatched_evaluation_key_is_detectable(server):
    """Failure detection: bootstrapping a key-A ciphertext with key B's evaluation key gives
    garbage -- about half of the decrypted NAND outputs are wrong -- while the matching key gives none."""
    other = A.Server(A.Keys(SEED + 1000), 0)
    k = server.keys
    count = 740
    a_bits, b_bits = nand_inputs(count, 17)
    a = A.to_device(k.encrypt_bits(a_bits, 7001, 0))
    b = A.to_device(k.encrypt_bits(b_bits, 7001, count))
    want = 1 - (a_bits & b_bits)
    for srv, lo, hi in ((server, 0.0, 0.0), (other, 0.3, 0.7)):
        out = torch.zeros((count, 632), dtype=torch.int32, device="cuda:0")
        srv.gate_batch(L.NAND, a, b, out)
        torch.cuda.synchronize()
        err = float(np.mean(k.decrypt_bits(A.to_host(out)) != want))
        assert lo <= err <= hi, err


@pytest.mark.gpu
def test_shared_scratch_between_programs(server):
    """One scratch buffer serving two programs in turn (AND, then XOR, then AND again), and a scratch filled
    with garbage between calls: every evaluation reloads its own job tables, so the outputs stay the truth
    tables (include/vlp.h vlp_program_eval)."""
    count = 37
    rng = np.random.default_rng(11)
    bits = rng.integers(0, 2, (2, count), dtype=np.uint8)
    k = server.keys
    a = A.to_device(k.encrypt_bits(bits[0], 901, 0))
    b = A.to_device(k.encrypt_bits(bits[1], 902, 0))
    p_and = A.Program.gates(server, L.AND, count)
    p_xor = A.Program.gates(server, L.XOR, count)
    shared = torch.empty(max(p_and.info.scratch_bytes, p_xor.info.scratch_bytes), dtype=torch.uint8, device="cuda:0")
    assert p_and.info.table_bytes >= count * 20 and p_xor.info.table_bytes >= count * 20
    p_and.scratch = shared
    p_xor.scratch = shared
    want = {L.AND: bits[0] & bits[1], L.XOR: bits[0] ^ bits[1]}
    for prog, op in [(p_and, L.AND), (p_xor, L.XOR), (p_and, L.AND), (p_xor, L.XOR)]:
        out = torch.zeros((count, 632), dtype=torch.int32, device="cuda:0")
        prog.eval(a, b, out)
        torch.cuda.synchronize()
        assert np.array_equal(k.decrypt_bits(A.to_host(out)), want[op]), op
        shared.random_(0, 256)  # whatever the buffer holds next time must not matter


@pytest.mark.gpu
def test_concurrent_evals_on_two_streams(server):
    """Two host threads run vlp_server_eval on the same compiled schedule on two CUDA streams at once (separate
    scratch buffers per stream, shared cached program and key): both results decrypt to the predicate and are
    byte-equal to a serial evaluation."""
    import threading
    wl = make_workload(1, key_seed=SEED)
    k = server.keys
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags)
    q = A.to_device(k.encrypt_query(m, wl.query, 7))
    db = A.to_device(k.encrypt_db(m, wl.records, wl.payloads, pk_seed=wl.key_seed + 1))
    ref = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
    server.eval(m, q, db, ref)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.zeros_like(ref) for _ in streams]
    errs = []

    def run(i):
        try:
            for _ in range(3):
                server.eval(m, q, db, outs[i], stream=streams[i])
            streams[i].synchronize()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for o in outs:
        assert np.array_equal(A.to_host(o), A.to_host(ref))


@pytest.mark.gpu
def test_linear_aggregation_noise_and_three_group_levels(server):
    """R24 noise budget and grouping, measured: an IdM database of 4,160 records (65 groups -> 2 -> 1: three
    refresh levels) with colliding 4-bit ids, so many masks are 1.  Every linear sum's phase is within the
    refresh margin 1/4 of its exact XOR (bit / 2), the error of the 64-term sums has the predicted spread
    (sigma ~ 0.028 = sqrt(64) x the gate output sigma), and the result decrypts to the predicate."""
    M, l_I, l_S = 4160, 4, 8
    rng = np.random.default_rng(29)
    recs = rng.integers(0, 16, (M, 1), dtype=np.uint64)
    pays = rng.integers(0, 256, M, dtype=np.uint64)
    qv = 5
    flags = OC.CONFIG_FLAGS | OC.F_LINEAR_SUM | L.F_KEEP_ALL
    k = server.keys
    m = A.meta(OC.MODE_IDM, M, l_I, l_S, 1, flags)
    q = k.encrypt_query(m, [qv], 7)
    db = k.encrypt_db(m, recs, pays, pk_seed=31)
    prog = A.Program.velopir(server, m)
    out = torch.zeros((l_S, 632), dtype=torch.int32, device="cuda:0")
    prog.eval(A.to_device(q), A.to_device(db), out)
    torch.cuda.synchronize()
    want = 0
    for r, p in zip(recs[:, 0], pays):
        if int(r) == qv:
            want ^= int(p)
    assert k.decrypt_value(A.to_host(out)) == want
    s = k.export()[0].astype(np.uint64)
    mid = A.to_host(prog.intermediate())

    def phase(row):  # b - <a, s> mod 2^32, centered
        ph = (int(row[630]) - int((row[:630].astype(np.uint64) * s).sum() % 2 ** 32)) % 2 ** 32
        return ph

    errs, levels_with_sums = [], 0
    for lvl in range(prog.info.levels):
        jobs, ins = prog.level_linear(lvl)
        if len(jobs) == 0:
            continue
        levels_with_sums += 1
        for out_slot, first, count, _ in jobs[:64]:
            bit = 0
            for i in range(count):  # inputs are {0, 1/2}-encoded: the bit is the phase rounded to 0 or 1/2
                bit ^= int(round(phase(mid[int(ins[first + i]) & 0x0FFFFFFF]) / 2 ** 31)) & 1
            e = (phase(mid[int(out_slot) & 0x0FFFFFFF]) - bit * 2 ** 31 + 2 ** 31) % 2 ** 32 - 2 ** 31
            errs.append(e / 2 ** 32)
    errs = np.array(errs)
    print(f"R24 linear sums: {len(errs)} checked, |error| max {np.abs(errs).max():.4f}, std {errs.std():.4f}")
    assert levels_with_sums == 3
    assert np.abs(errs).max() < 0.15, np.abs(errs).max()   # margin 1/4
    assert 0.01 < errs.std() < 0.045, errs.std()            # predicted ~0.028 for 64-term sums


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [6, 7, 8, 9])
def test_dataset_shapes_with_options_predicate(server, cfg):
    """The paper-dataset shapes with both options outside the paper (R23 prefix comparators where there are
    comparators, R24 linear aggregation; weather-usa shape: 128-bit payloads, 304 records = 5 groups):
    the decrypted answer equals the plain predicate, with fewer levels than the paper's circuit."""
    wl0 = make_workload(cfg, key_seed=SEED)
    wl = make_workload(cfg, key_seed=SEED, flags=wl0.flags | OC.F_LINEAR_SUM |
                       (OC.F_PREFIX_COMP if wl0.mode == OC.MODE_INTV else 0))
    prog, q, db, out = _run_config(server, wl)
    assert server.keys.decrypt_value(out) == expected_result(wl)
    m0 = A.meta(wl0.mode, wl0.M, wl0.l_I, wl0.l_S, wl0.d, wl0.flags)
    h = ctypes.c_void_p()
    L.check(L.lib().vlp_program_create(None, ctypes.byref(m0), 0, wl0.M, ctypes.byref(h)))
    info = L.VlpProgramInfo()
    L.check(L.lib().vlp_program_get_info(h, ctypes.byref(info)))
    L.lib().vlp_free_program(h)
    assert prog.info.levels < info.levels


def test_config2_engines_agree_on_every_gate(route):
    """Config 2 at full size (132,080 BR) evaluated twice with VLP_F_KEEP_ALL (every intermediate keeps its own
    scratch row): the default routing (K2F waves + tails) and the integer-NTT engine alone (vlp_debug_route(1, 5)).
    The two exact engines share no arithmetic, so every gate output row must be byte-equal
    between them (tools/engine_crosscheck.py runs the same check on configs 3, 4 and 10)."""
    wl = make_workload(2)
    m = A.meta(wl.mode, wl.M, wl.l_I, wl.l_S, wl.d, wl.flags | L.F_KEEP_ALL)
    keys = A.Keys(wl.key_seed)
    srv = A.Server(keys, 0)
    pk = A.pubkeygen_device(keys, m, wl.key_seed + 1, 0, wl.M)
    db = A.server_encrypt_db_device(m, pk, wl.records, wl.payloads)
    q = A.to_device(keys.encrypt_query(m, wl.query, 7))
    prog = A.Program.velopir(srv, m)
    rows, outs = [], []
    for eng, par in ((0, 0), (1, 5)):
        route(eng, par)
        out = torch.zeros((wl.l_S, 632), dtype=torch.int32, device="cuda:0")
        prog.scratch.zero_()
        prog.eval(q, db, out)
        torch.cuda.synchronize()
        assert keys.decrypt_value(A.to_host(out)) == expected_result(wl)
        rows.append(prog.intermediate().clone())
        outs.append(out)
    written = int(((rows[0] != 0).any(dim=1) | (rows[1] != 0).any(dim=1)).sum())
    assert written > prog.info.ks  # every gate output row (plus the constants) was written
    assert torch.equal(rows[0], rows[1]), int((rows[0] != rows[1]).any(dim=1).sum())
    assert torch.equal(outs[0], outs[1])
