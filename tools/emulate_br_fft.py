"""Developer tool (not product code): lane-level emulation of the FP64 negacyclic-FFT external product of
kernels_fft.cu ("K2F").  One warp = one bootstrap, 32 lanes x 16 complex points.

Checks the index maps (fold/twist, four-step 16 x 32 FFT with a smem transpose and one lane-pair
exchange, the point held by lane L / register rho, the key layout) against an exact integer negacyclic
product, and measures the rounding margin of the 2-limb (and 1-limb) key split.

    python tools/emulate_br_fft.py [trials]
"""
import sys

import numpy as np

N, M = 1024, 512
PSI = np.exp(1j * np.pi * np.arange(2048) / 1024)  # psi^e, psi = exp(i pi / 1024)
W16 = np.exp(2j * np.pi * np.arange(16) / 16)
W32 = np.exp(2j * np.pi * np.arange(32) / 32)


def mrev(rho):  # register rho of a radix-4 x 4 DIF 16-point DFT holds output m = mrev(rho)
    return (rho >> 2) | ((rho & 3) << 2)


MREV = np.array([mrev(r) for r in range(16)])


def bfly4(a, b, c, d, sgn):  # X0..X3 of the 4-point DFT with omega_4 = exp(sgn * 2 pi i / 4)
    s02, d02, s13, d13 = a + c, a - c, b + d, b - d
    return s02 + s13, d02 + sgn * 1j * d13, s02 - s13, d02 - sgn * 1j * d13


def dft16_fwd(v):  # v: [..., 16] natural a -> out[..., rho] = X[mrev(rho)]
    v = v.copy()
    t = np.empty_like(v)
    for a0 in range(4):  # stage 1 over a1 (stride 4), twiddle w16^(a0 k0)
        outs = bfly4(v[..., a0], v[..., a0 + 4], v[..., a0 + 8], v[..., a0 + 12], +1)
        for k0 in range(4):
            t[..., a0 + 4 * k0] = outs[k0] * W16[(a0 * k0) % 16]
    o = np.empty_like(v)
    for k0 in range(4):  # stage 2 over a0 -> X[k0 + 4 k1] in register k1 + 4 k0
        outs = bfly4(t[..., 4 * k0], t[..., 4 * k0 + 1], t[..., 4 * k0 + 2], t[..., 4 * k0 + 3], +1)
        for k1 in range(4):
            o[..., k1 + 4 * k0] = outs[k1]
    return o


def dft16_inv(o):  # exact mirror: in[..., rho] = X[mrev(rho)] -> 16 * x[a] natural
    t = np.empty_like(o)
    for k0 in range(4):
        # inverse 4-point DFT over k1 -> a0 (input register k1 + 4 k0)
        outs = bfly4(o[..., 4 * k0], o[..., 4 * k0 + 1], o[..., 4 * k0 + 2], o[..., 4 * k0 + 3], -1)
        for a0 in range(4):
            t[..., 4 * k0 + a0] = outs[a0] * np.conj(W16[(a0 * k0) % 16])
    v = np.empty_like(o)
    for a0 in range(4):
        outs = bfly4(t[..., a0], t[..., a0 + 4], t[..., a0 + 8], t[..., a0 + 12], -1)
        for a1 in range(4):
            v[..., a0 + 4 * a1] = outs[a1]
    return v


# per-lane twiddles tw[b][rho] = psi^(b (1 + 4 k1)), k1 = mrev(rho)
LANE = np.arange(32)
TW = PSI[(LANE[:, None] * (1 + 4 * MREV[None, :])) % 2048]  # [32][16]
TWIST = PSI[32 * np.arange(16)]  # psi^(32 a), uniform


def fwd(x):
    """x: [1024] real (integers) -> out[L][rho] = A_k, k = L + 32 mrev(rho)."""
    # lane b, register a: (x[32a+b] + i x[32a+b+512]) psi^(32a)
    u = np.empty((32, 16), complex)
    for b in range(32):
        for a in range(16):
            u[b, a] = (x[32 * a + b] + 1j * x[32 * a + b + 512]) * TWIST[a]
    y = dft16_fwd(u) * TW  # lane b, register rho <-> k1 = mrev(rho)
    T = np.empty((16, 32), complex)  # smem transpose T[k1][b]
    for b in range(32):
        for rho in range(16):
            T[MREV[rho], b] = y[b, rho]
    # lane L = (e, k1): reads Y_i, Y_{16+i} for i in [8e, 8e+8), computes s, d; exchange with L ^ 16
    V = np.empty((32, 16), complex)
    s = np.empty((32, 8), complex)
    d = np.empty((32, 8), complex)
    for L in range(32):
        e, k1 = L >> 4, L & 15
        for r in range(8):
            i = 8 * e + r
            s[L, r] = T[k1, i] + T[k1, 16 + i]
            d[L, r] = (T[k1, i] - T[k1, 16 + i]) * W32[r] * (1j if e else 1)
    for L in range(32):
        e = L >> 4
        P = L ^ 16
        if e == 0:  # keeps s (i < 8), receives s (i >= 8) from the partner
            V[L, :8], V[L, 8:] = s[L], s[P]
        else:  # receives d (i < 8), keeps d (i >= 8)
            V[L, :8], V[L, 8:] = d[P], d[L]
    return dft16_fwd(V)


def inv(C):
    """C[L][rho] at point k = L + 32 mrev(rho) -> 512 * (c_j + i c_{j+512}) psi^(-j) ... returns real [1024]."""
    V = dft16_inv(C)  # 16 * V_e[i]
    s = np.empty((32, 8), complex)
    d = np.empty((32, 8), complex)
    for L in range(32):
        e, P = L >> 4, L ^ 16
        if e == 0:
            s[L], d[L] = V[L, :8], V[P, :8]
        else:
            s[L], d[L] = V[P, 8:], V[L, 8:]
    T = np.empty((16, 32), complex)
    for L in range(32):
        e, k1 = L >> 4, L & 15
        for r in range(8):
            i = 8 * e + r
            dd = d[L, r] * np.conj(W32[r]) * (-1j if e else 1)
            T[k1, i] = s[L, r] + dd
            T[k1, 16 + i] = s[L, r] - dd
    y = np.empty((32, 16), complex)
    for b in range(32):
        for rho in range(16):
            y[b, rho] = T[MREV[rho], b] * np.conj(TW[b, rho])
    u = dft16_inv(y)  # lane b, register a (natural)
    out = np.empty(1024)
    res = np.empty(1024)
    for b in range(32):
        for a in range(16):
            z = u[b, a] * np.conj(TWIST[a])
            out[32 * a + b], out[32 * a + b + 512] = z.real, z.imag
    return out


def key_fft(p):
    """Direct DFT of one key polynomial (exact-ish), scaled 1/512, in the lane layout [L][rho]."""
    j = np.arange(512)
    z = (p[:512] + 1j * p[512:]) * PSI[j]
    k = np.arange(512)
    A = (np.exp(2j * np.pi * np.outer(k, j) / 512) @ z) / 512
    out = np.empty((32, 16), complex)
    for L in range(32):
        for rho in range(16):
            out[L, rho] = A[L + 32 * MREV[rho]]
    return out


def negacyclic(a, b):  # exact integer product mod X^N + 1 (python ints)
    res = [0] * N
    for i in range(N):
        if a[i] == 0:
            continue
        for j in range(N):
            k = i + j
            if k < N:
                res[k] += a[i] * b[j]
            else:
                res[k - N] -= a[i] * b[j]
    return res


def limbs(b, nl):
    s = b.astype(np.int64)
    s = np.where(s >= 2 ** 31, s - 2 ** 32, s)
    if nl == 1:
        return [s]
    lo = ((s + 2 ** 15) & 0xFFFF) - 2 ** 15
    hi = (s - lo) >> 16
    return [lo, hi]


def main():
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    rng = np.random.default_rng(5)
    # index check: single product vs exact
    x = rng.integers(-64, 64, N)
    p = rng.integers(-2 ** 15, 2 ** 15, N)
    got = inv(fwd(x) * key_fft(p))
    want = np.convolve(x, p)
    want = want[:N] - np.concatenate([want[N:], [0]])
    err = np.max(np.abs(got - want))
    print("single product max |err| =", err)
    assert err < 1e-3, "index maps wrong"
    for nl in (2, 1):
        worst = 0.0
        for t in range(trials):
            mode = t % 3
            if mode == 0:
                digits = [rng.integers(-64, 64, N) for _ in range(6)]
            elif mode == 1:  # extreme digits
                digits = [rng.choice([-64, 63], N) for _ in range(6)]
            else:  # structured: test-vector-like rotation step functions
                digits = [np.where(np.arange(N) < rng.integers(0, N), 32, 0) * rng.choice([-1, 1]) for _ in range(6)]
            keys = [rng.integers(0, 2 ** 32, N, dtype=np.uint64) for _ in range(6)]
            Xs = [fwd(d.astype(float)) for d in digits]
            for li in range(nl):
                acc = np.zeros((32, 16), complex)
                want = np.zeros(N)
                for r in range(6):
                    kl = limbs(keys[r], nl)[li]
                    acc += Xs[r] * key_fft(kl.astype(float))
                    c = np.convolve(digits[r].astype(float), kl.astype(float))
                    want += c[:N] - np.concatenate([c[N:], [0]])
                got = inv(acc)
                worst = max(worst, float(np.max(np.abs(got - want))))
        print(f"{nl} limb(s): worst |err| over {trials} trials = {worst:.3g}")


if __name__ == "__main__" and "--v3" not in sys.argv:
    main()


# ---------------------------------------------------------------------------- v3: select-free lane pairs
# Lane b = 16 h + bb.  Lanes h = 1 negate odd inputs a, so their first 16-point DFT comes out shifted by 8:
# register rho holds k1 = mrev(rho) ^ 8h.  Registers A (mrev(rho) < 8) are a lane's own k1 set; the partner's
# matching values sit in register rho | 2.  The lane pair (bb, bb + 16) forms s = Y_bb + Y_bb+16 and
# d = (Y_bb - Y_bb+16) w32^bb for the 8 k1 of each lane; T[g][k1][bb] (g = 0: s, 1: d); lane L = (g, k1) reads
# 16 values and runs the second 16-point DFT -> point L + 32 mrev(rho), as before.
A_REGS = [r for r in range(16) if not (r & 2)]


def k1_of(b, rho):
    return MREV[rho] ^ (8 * (b >> 4))


TW3 = np.array([[PSI[(b * (1 + 4 * k1_of(b, r))) % 2048] for r in range(16)] for b in range(32)])
TAU = np.array([(-1 if b >> 4 else 1) * W32[b & 15] for b in range(32)])
SIG = np.array([[(-1) ** a if b >> 4 else 1 for a in range(16)] for b in range(32)])


def fwd3(x):
    u = np.empty((32, 16), complex)
    for b in range(32):
        for a in range(16):
            u[b, a] = SIG[b, a] * (x[32 * a + b] + 1j * x[32 * a + b + 512]) * TWIST[a]
    y = dft16_fwd(u) * TW3
    T = np.zeros((2, 16, 16), complex)
    for b in range(32):
        P = b ^ 16
        for ra in A_REGS:
            recv = y[P, ra | 2]
            s = y[b, ra] + recv
            d = (y[b, ra] - recv) * TAU[b]
            k1 = k1_of(b, ra)
            T[0, k1, b & 15], T[1, k1, b & 15] = s, d
    V = np.empty((32, 16), complex)
    for L in range(32):
        V[L] = T[L >> 4, L & 15, :]
    return dft16_fwd(V)


def inv3(C):
    V = dft16_inv(C)
    T = np.zeros((2, 16, 16), complex)
    for L in range(32):
        T[L >> 4, L & 15, :] = V[L]
    y = np.empty((32, 16), complex)
    part = np.empty((32, 16), complex)
    for b in range(32):
        for ra in A_REGS:
            k1 = k1_of(b, ra)
            s, d = T[0, k1, b & 15], T[1, k1, b & 15]
            dd = d * np.conj(TAU[b])
            y[b, ra] = s + dd
            part[b, ra] = s - dd
    for b in range(32):
        for ra in A_REGS:
            y[b, ra | 2] = part[b ^ 16, ra]
    u = dft16_inv(y * np.conj(TW3))
    out = np.empty(1024)
    for b in range(32):
        for a in range(16):
            z = u[b, a] * np.conj(TWIST[a]) * SIG[b, a]
            out[32 * a + b], out[32 * a + b + 512] = z.real, z.imag
    return out


def check_v3():
    rng = np.random.default_rng(9)
    x = rng.integers(-64, 64, N)
    p = rng.integers(-2 ** 15, 2 ** 15, N)
    assert np.max(np.abs(fwd3(x.astype(float)) - fwd(x.astype(float)))) < 1e-6, "v3 forward layout"
    got = inv3(fwd3(x.astype(float)) * key_fft(p.astype(float)))
    want = np.convolve(x, p)
    want = want[:N] - np.concatenate([want[N:], [0]])
    err = np.max(np.abs(got - want))
    print("v3 single product max |err| =", err)
    assert err < 1e-3


if __name__ == "__main__" and "--v3" in sys.argv:
    check_v3()
