"""oracle/circuits.py -- TEST INFRASTRUCTURE ONLY.

VeLoPIR's circuits written once, step by step in the order and notation of the paper's listings, against
a gate backend.  Backends:

* ``TfheBackend(keys)`` -- every gate is a bootstrapped TFHE gate of the C oracle (ciphertexts are
  uint32[631] numpy arrays).
* ``PlainBackend()``    -- the PlainOracle (O15): the same DAG over Python booleans, counting
  gates and depth, used to pin the circuit topology against brute force.

Readings: R11 (``unsigned``), R12 (``closed_upper``), R13 (rectangle = IntV d=2),
R14 (``eq_tree``), R15/R19 (``sum_tree``, ``or_reduce``), R16 (mask S_i with its own v_i), R20 (LSB first);
R23 (``F_PREFIX_COMP``, the log-depth comparator of SURVEY 8(f) NEXT 4 -- not in the paper); R24
(``F_LINEAR_SUM``, linear XOR aggregation in the {0, 1/2} encoding -- not in the paper).
"""
from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
import os

import numpy as np

from . import AND, NAND, OR, XOR, XNOR, OracleKeys, trivial

# Modes and flags (same values as the product's header, defined independently here).
MODE_INTV, MODE_COV, MODE_IDM = 0, 1, 2
F_CLOSED_UPPER, F_UNSIGNED, F_EQ_TREE, F_SUM_TREE, F_OR_REDUCE, F_PREFIX_COMP, F_LINEAR_SUM = 1, 2, 4, 8, 16, 32, 64
CONFIG_FLAGS = F_CLOSED_UPPER | F_UNSIGNED | F_EQ_TREE | F_SUM_TREE


class PlainBackend:
    """Booleans with a depth counter (depth in bootstrapped-gate levels; MUX halves hoisted like S9)."""

    def __init__(self):
        self.br = 0
        self.ks = 0

    @staticmethod
    def const(bit):
        return (bool(bit), 0)

    def _g(self, val, *deps):
        self.br += 1
        self.ks += 1
        return (val, max(d[1] for d in deps) + 1)

    def AND(self, x, y): return self._g(x[0] and y[0], x, y)
    def NAND(self, x, y): return self._g(not (x[0] and y[0]), x, y)
    def OR(self, x, y): return self._g(x[0] or y[0], x, y)
    def XOR(self, x, y): return self._g(x[0] != y[0], x, y)
    def XNOR(self, x, y): return self._g(x[0] == y[0], x, y)

    def MUX(self, c, a, b):
        # two BR halves (each depends on c and one data input), one KS when both are done (R10, S9)
        self.br += 2
        self.ks += 1
        h1 = max(c[1], a[1]) + 1
        h2 = max(c[1], b[1]) + 1
        return (a[0] if c[0] else b[0], max(h1, h2))

    @staticmethod
    def NOT(x): return (not x[0], x[1])

    # R24 (not in the paper): the {0, 1/2} encoding -- a bit value plus a depth, like every other node
    def AND_Q(self, x, y): return self._g(x[0] and y[0], x, y)

    @staticmethod
    def LIN(xs):  # sum of {0, 1/2}-encoded bits = their XOR; no bootstrap, no level
        v = False
        for x in xs:
            v = v != x[0]
        return (v, max(x[1] for x in xs))

    def REFRESH(self, x, final): return self._g(x[0], x)


class TfheBackend:
    """Bootstrapped TFHE gates of the C oracle; trivial constants per R21."""

    def __init__(self, keys: OracleKeys):
        self.k = keys

    @staticmethod
    def const(bit):
        return trivial(bit)

    def AND(self, x, y): return self.k.gate(AND, x, y)
    def NAND(self, x, y): return self.k.gate(NAND, x, y)
    def OR(self, x, y): return self.k.gate(OR, x, y)
    def XOR(self, x, y): return self.k.gate(XOR, x, y)
    def XNOR(self, x, y): return self.k.gate(XNOR, x, y)
    def MUX(self, c, a, b): return self.k.mux(c, a, b)
    def NOT(self, x): return OracleKeys.not_(x)

    # R24 (not in the paper): bits in the {0, 1/2} encoding (phase b/2), whose sums are XORs
    def AND_Q(self, x, y):
        """AND(x, y) into the {0, 1/2} encoding: Bootstrap_{testv 1/4}((0, -1/8) + x + y) + (0, 1/4)."""
        c = (x.astype(np.uint64) + y.astype(np.uint64)).astype(np.uint32)
        c[-1] = np.uint32((int(c[-1]) + 0xE0000000) & 0xFFFFFFFF)
        o = self.k.bootstrap_mu(c, 0x40000000)
        o[-1] = np.uint32((int(o[-1]) + 0x40000000) & 0xFFFFFFFF)
        return o

    @staticmethod
    def LIN(xs):
        """Sum mod 2^32 of {0, 1/2}-encoded ciphertexts (exact, no bootstrap)."""
        acc = np.zeros_like(xs[0], dtype=np.uint64)
        for x in xs:
            acc = (acc + x.astype(np.uint64)) & 0xFFFFFFFF
        return acc.astype(np.uint32)

    def REFRESH(self, x, final):
        """Bootstrap x - (0, 1/4): phase +-1/4 -> the standard +-1/8 encoding (final), or -- test vector 1/4,
        then + (0, 1/4) -- back into the {0, 1/2} encoding."""
        c = x.copy()
        c[-1] = np.uint32((int(c[-1]) + 0xC0000000) & 0xFFFFFFFF)
        if final:
            return self.k.bootstrap_mu(c, 0x20000000)
        o = self.k.bootstrap_mu(c, 0x40000000)
        o[-1] = np.uint32((int(o[-1]) + 0x40000000) & 0xFFFFFFFF)
        return o


# ------------------------------------------------------------------------------- comparators
def hom_comp_le(B, ct1, ct2, l, unsigned=True):
    """alg:HomCompLE: 1 iff z1 <= z2.  ``unsigned`` (R11): the final MUX selects ct2[l-1]
    (unsigned order) instead of the paper's ct1[l-1] (two's complement)."""
    t0 = B.XOR(ct1[l - 1], ct2[l - 1])
    t2 = B.const(1)                      # Enc^TLWE(0, 1/8), trivial (R21)
    for i in range(0, l - 1):
        t1 = B.XNOR(ct1[i], ct2[i])
        t2 = B.MUX(t1, t2, ct2[i])
    r = B.MUX(t0, ct2[l - 1] if unsigned else ct1[l - 1], t2)
    return r


def hom_comp_l(B, ct1, ct2, l, unsigned=True):
    """alg:HomCompL: as HomCompLE with t2 initialised to trivial Enc(0); 1 iff z1 < z2."""
    t0 = B.XOR(ct1[l - 1], ct2[l - 1])
    t2 = B.const(0)                      # Enc^TLWE(0, -1/8)
    for i in range(0, l - 1):
        t1 = B.XNOR(ct1[i], ct2[i])
        t2 = B.MUX(t1, t2, ct2[i])
    r = B.MUX(t0, ct2[l - 1] if unsigned else ct1[l - 1], t2)
    return r


def hom_comp_gt_prefix(B, ct1, ct2, l):
    """Log-depth comparator, flag F_PREFIX_COMP -- NOT in the paper (DESIGN.md reading
    R23): 1 iff z1 > z2 (unsigned).  Per bit i (LSB first): G_i = AND(ct1[i], NOT ct2[i]) (greater at bit i),
    E_i = XNOR(ct1[i], ct2[i]) (equal at bit i).  Adjacent ranges are merged level by level, range 2k+1 as
    the high part H and range 2k as the low part L (a last unpaired range is carried up unchanged):
    G = MUX(H.E, L.G, H.G) -- equal on the high part: the low part decides, else the high part does --
    and E = AND(H.E, L.E).  Every E is computed here (the product builds only the ones a G uses; unused gates
    do not change any output)."""
    G = [B.AND(ct1[i], B.NOT(ct2[i])) for i in range(l)]
    E = [B.XNOR(ct1[i], ct2[i]) for i in range(l)]
    while len(G) > 1:
        nG, nE = [], []
        for k in range(0, len(G), 2):
            if k + 1 < len(G):
                nG.append(B.MUX(E[k + 1], G[k], G[k + 1]))
                nE.append(B.AND(E[k + 1], E[k]))
            else:
                nG.append(G[k])
                nE.append(E[k])
        G, E = nG, nE
    return G[0]


def hom_comp_le_prefix(B, ct1, ct2, l, unsigned=True):
    """[z1 <= z2] = NOT [z1 > z2] (free negation)."""
    assert unsigned, "the prefix comparator is unsigned only"
    return B.NOT(hom_comp_gt_prefix(B, ct1, ct2, l))


def hom_comp_l_prefix(B, ct1, ct2, l, unsigned=True):
    """[z1 < z2] = [z2 > z1]."""
    assert unsigned, "the prefix comparator is unsigned only"
    return hom_comp_gt_prefix(B, ct2, ct1, l)


# ------------------------------------------------------------------------------- equality
def hom_eq_serial(B, ct1, ct2, l):
    """alg:HomEQ: r = trivial Enc(1); r <- AND(r, XNOR(ct1[i], ct2[i])) for every bit."""
    r = B.const(1)
    for i in range(0, l):
        t = B.XNOR(ct1[i], ct2[i])
        r = B.AND(r, t)
    return r


def hom_eq_tree(B, ct1, ct2, l):
    """alg:HomEquiOPT: XNORs, then the pairwise AND reduction (i, i+k), k doubling."""
    t1 = [B.XNOR(ct1[i], ct2[i]) for i in range(l)]
    k = 1
    while k < l:
        for i in range(0, l, 2 * k):
            if i + k < l:
                t1[i] = B.AND(t1[i], t1[i + k])
        k *= 2
    return t1[0]


# ------------------------------------------------------------------------------- validation modules
def intv(B, q, rec, l, d, flags):
    """alg:InterValid.  q = [Enc(x)] or [Enc(x), Enc(y)]; rec = [Enc(x_left), Enc(x_right)]
    (+ [Enc(y_left), Enc(y_right)] for d = 2).  CLOSED_UPPER (R12): the right bound uses
    HomCompLE(x, x_right) (lo <= x <= hi) instead of the paper's HomCompL (x < x_right)."""
    uns = bool(flags & F_UNSIGNED)
    le, lt = (hom_comp_le_prefix, hom_comp_l_prefix) if flags & F_PREFIX_COMP else (hom_comp_le, hom_comp_l)
    right = le if flags & F_CLOSED_UPPER else lt
    v_xl = le(B, rec[0], q[0], l, uns)
    v_xr = right(B, q[0], rec[1], l, uns)
    if d == 1:
        return B.AND(v_xl, v_xr)
    v_yl = le(B, rec[2], q[1], l, uns)
    v_yr = right(B, q[1], rec[3], l, uns)
    v_x = B.AND(v_xl, v_xr)
    v_y = B.AND(v_yl, v_yr)
    return B.AND(v_x, v_y)


def cov(B, q, rec, l, flags):
    """alg:BB2: HomEQ(x, loc_x) AND HomEQ(y, loc_y)."""
    eq = hom_eq_tree if flags & F_EQ_TREE else hom_eq_serial
    v_x = eq(B, q[0], rec[0], l)
    v_y = eq(B, q[1], rec[1], l)
    return B.AND(v_x, v_y)


def idm(B, q, rec, l, flags):
    """IdM: a single HomEQ on the identifier, no final AND."""
    eq = hom_eq_tree if flags & F_EQ_TREE else hom_eq_serial
    return eq(B, q[0], rec[0], l)


def validate(B, mode, q, rec, l, d, flags):
    if mode == MODE_INTV:
        return intv(B, q, rec, l, d, flags)
    if mode == MODE_COV:
        return cov(B, q, rec, l, flags)
    return idm(B, q, rec, l, flags)


# ------------------------------------------------------------------------------- mask and aggregation
def hom_bitwise_and(B, v, S):
    """alg:HomBitwiseAND: S[j] <- AND(v, S[j])."""
    return [B.AND(v, s) for s in S]


def hom_sum_serial(B, Ss, l_S, or_reduce=False):
    """alg:HomSum: S <- Enc(0)^{l_S} (trivial), S[j] <- XOR(S[j], S_i[j]) over all i."""
    red = B.OR if or_reduce else B.XOR
    S = [B.const(0) for _ in range(l_S)]
    for Si in Ss:
        for j in range(l_S):
            S[j] = red(S[j], Si[j])
    return S


def hom_sum_tree(B, Ss, l_S, or_reduce=False, pool=None):
    """Outermost HomSum: S_i[j] <- XOR(S_i[j], S_{i+k}[j]) pairing (i, i+k), k doubling
    (R15; same pairing rule as P:742-748).  Returns S_0."""
    red = B.OR if or_reduce else B.XOR
    Ss = [list(s) for s in Ss]
    M = len(Ss)
    k = 1
    while k < M:
        pairs = [(i, j) for i in range(0, M, 2 * k) if i + k < M for j in range(l_S)]
        if pool is not None:
            outs = list(pool.map(lambda ij: red(Ss[ij[0]][ij[1]], Ss[ij[0] + k][ij[1]]), pairs))
        else:
            outs = [red(Ss[i][j], Ss[i + k][j]) for (i, j) in pairs]
        for (i, j), o in zip(pairs, outs):
            Ss[i][j] = o
        k *= 2
    return Ss[0]


LIN_GROUP = 64


def hom_sum_linear(B, Ss, l_S):
    """R24 (NOT in the paper): XOR aggregation by sums.  Ss are masked payload bits in the
    {0, 1/2} encoding.  While more than LIN_GROUP rows remain, each group of LIN_GROUP consecutive rows is
    summed and refreshed back into the {0, 1/2} encoding; the last sum is refreshed into the standard encoding."""
    Ss = [list(s) for s in Ss]
    while len(Ss) > LIN_GROUP:
        Ss = [[B.REFRESH(B.LIN([Ss[i][j] for i in range(g0, min(len(Ss), g0 + LIN_GROUP))]), False)
               for j in range(l_S)] for g0 in range(0, len(Ss), LIN_GROUP)]
    return [B.REFRESH(B.LIN([S[j] for S in Ss]), True) for j in range(l_S)]


def record_outputs(B, mode, q, rec, S, l, d, flags):
    """One iteration of alg:VeLoPIR's record loop: v, then S_i <- HomBitwiseAND(v, S_i)
    (R24: into the {0, 1/2} encoding)."""
    v = validate(B, mode, q, rec, l, d, flags)
    if flags & F_LINEAR_SUM:
        return v, [B.AND_Q(v, s) for s in S]
    return v, hom_bitwise_and(B, v, S)


def velopir(B, mode, q, records, payloads, l, d, l_S, flags, threads=None):
    """alg:VeLoPIR with the outermost parallelism of P:781-802 (records in parallel).
    q: list of query words (each a list of l bit-ciphertexts); records[i]: list of record words;
    payloads[i]: list of l_S ciphertexts.  Returns (R, v list, masked payload list)."""
    M = len(records)
    threads = threads or (os.cpu_count() or 1)
    pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None
    try:
        fn = lambda i: record_outputs(B, mode, q, records[i], payloads[i], l, d, flags)
        outs = list(pool.map(fn, range(M))) if pool else [fn(i) for i in range(M)]
        vs = [o[0] for o in outs]
        masked = [o[1] for o in outs]
        orr = bool(flags & F_OR_REDUCE)
        if flags & F_LINEAR_SUM:
            assert not orr, "linear aggregation computes XOR only"
            R = hom_sum_linear(B, masked, l_S)
        elif flags & F_SUM_TREE:
            R = hom_sum_tree(B, masked, l_S, orr, pool)
        else:
            R = hom_sum_serial(B, masked, l_S, orr)
    finally:
        if pool:
            pool.shutdown()
    return R, vs, masked


# ------------------------------------------------------------------------------- plain predicate (8(c))
def plain_match(mode, qvals, rec_words, d, flags, l=None):
    """The plaintext predicate of thm:bb1 / thm:bb2 / IdM (R11-R13).  Values are l-bit words; without
    F_UNSIGNED (and with l given) they are compared as two's complement, as the paper's comparators do."""
    if mode == MODE_INTV and l is not None and not flags & F_UNSIGNED:
        sg = lambda v: int(v) - (1 << l) if (int(v) >> (l - 1)) & 1 else int(v)  # noqa: E731
        qvals = [sg(v) for v in qvals]
        rec_words = [sg(v) for v in rec_words]
    if mode == MODE_INTV:
        ok = True
        for a in range(d):
            lo, hi, x = rec_words[2 * a], rec_words[2 * a + 1], qvals[a]
            ok = ok and (lo <= x) and ((x <= hi) if flags & F_CLOSED_UPPER else (x < hi))
        return ok
    if mode == MODE_COV:
        return all(qvals[a] == rec_words[a] for a in range(d))
    return qvals[0] == rec_words[0]


def plain_result(mode, qvals, records, payloads, d, flags, l=None):
    """R = XOR (OR with F_OR_REDUCE) of the payloads of all matching records; 0 if none (R19)."""
    r = 0
    for rec, pay in zip(records, payloads):
        if plain_match(mode, qvals, rec, d, flags, l):
            r = (r | int(pay)) if flags & F_OR_REDUCE else (r ^ int(pay))
    return r
