"""Developer tool: a numpy emulation of the GPU external-product arithmetic (layouts A/B/C, lazy
Harvey butterflies with Shoup twiddles, Montgomery MAC, 3-limb key split) used to validate index math and
bounds before writing CUDA.  Not product code, not the oracle.  Run: python tools/emulate_br_ntt.py"""
import numpy as np

P = 0x3FFF7801
N = 1024
M32 = (1 << 32) - 1


def find_psi():
    for g in range(2, 1000):
        x = pow(g, (P - 1) // 2048, P)
        if pow(x, 1024, P) == P - 1:
            return x


def brv(x, bits=10):
    return int(f"{x:0{bits}b}"[::-1], 2)


PSI = find_psi()
PSI_INV = pow(PSI, P - 2, P)
W = [pow(PSI, brv(k), P) for k in range(N)]
WI = [pow(PSI_INV, brv(k), P) for k in range(N)]
WS = [(w << 32) // P for w in W]
WIS = [(w << 32) // P for w in WI]
NINV = pow(N, P - 2, P)
R = (1 << 32) % P
PINV_NEG = (-pow(P, -1, 1 << 32)) % (1 << 32)


def shoup(y, w, ws):
    q = (y * ws) >> 32
    return (y * w - q * P) & M32  # in [0, 2P)


def jA(t, r): return t + 64 * r
def jB(t, r): return ((t >> 2) << 6) | (r << 2) | (t & 3)
def jC(t, r): return (t << 4) | r


def fwd(vals):
    """vals: dict (t, r)->value in layout A; returns layout-C dict."""
    a = np.zeros(N, dtype=object)
    for t in range(64):
        for r in range(16):
            a[jA(t, r)] = vals[t][r]
    lay = jA
    for s in range(10):
        if s == 4:
            lay = jB
        if s == 8:
            lay = jC
        tt = 512 >> s
        for t in range(64):
            for r in range(16):
                j = lay(t, r)
                if j & tt:
                    continue
                k = (1 << s) + (j >> (10 - s))
                x, y = a[j], a[j + tt]
                assert x < 4 * P and y < 4 * P
                x = x - 2 * P if x >= 2 * P else x
                T = shoup(y, W[k], WS[k])
                a[j], a[j + tt] = x + T, x - T + 2 * P
    return a


def inv(a):
    a = a.copy()
    for s in range(9, -1, -1):
        lay = jC if s >= 8 else (jB if s >= 4 else jA)
        tt = 512 >> s
        for t in range(64):
            for r in range(16):
                j = lay(t, r)
                if j & tt:
                    continue
                k = (1 << s) + (j >> (10 - s))
                x, y = a[j], a[j + tt]
                assert x < 2 * P and y < 2 * P, (s, x, y)
                X = x + y
                X = X - 2 * P if X >= 2 * P else X
                T = x - y + 2 * P
                a[j], a[j + tt] = X, shoup(T, WI[k], WIS[k])
    return a


def redc(T):
    m = ((T & M32) * PINV_NEG) & M32
    return (T + m * P) >> 32


def main():
    rng = np.random.default_rng(1)
    digits = rng.integers(-64, 64, (6, N))
    key = rng.integers(0, 2 ** 32, (6, 2, N), dtype=np.uint64)
    # limbs b = b0 + 2^11 b1 + 2^22 b2
    def limbs(b):
        b = int(b)
        b0 = ((b + 1024) & 2047) - 1024
        r1 = (b - b0) >> 11
        b1 = ((r1 + 1024) & 2047) - 1024
        r2 = (r1 - b1) >> 11
        b2 = ((r2 + 512) & 1023) - 512
        assert (b0 + (b1 << 11) + (b2 << 22) - b) % 2 ** 32 == 0
        return b0, b1, b2
    # key NTT: plain (non-lazy) forward on limb polys, Montgomery * N^-1
    def plain_fwd(poly):
        a = [int(x) % P for x in poly]
        for s in range(10):
            tt = 512 >> s
            for i in range(1 << s):
                w = W[(1 << s) + i]
                for j in range(2 * i * tt, 2 * i * tt + tt):
                    u, v = a[j], a[j + tt] * w % P
                    a[j], a[j + tt] = (u + v) % P, (u - v) % P
        return a
    khat = np.zeros((6, 2, 3, N), dtype=object)
    for r in range(6):
        for u in range(2):
            L = [limbs(b) for b in key[r, u]]
            for l in range(3):
                f = plain_fwd([x[l] for x in L])
                khat[r, u, l] = [(x * NINV % P) * R % P for x in f]
    # digits -> forward lazy (inputs ((v>>s)&127) + P - 64 in [P-64, P+64))
    dhat = []
    for r in range(6):
        vals = [[int(digits[r][jA(t, q)]) + P for q in range(16)] for t in range(64)]
        dhat.append(fwd(vals))
    out = {}
    for u in range(2):
        res = np.zeros(N, dtype=object)
        for l in range(3):
            acc = np.zeros(N, dtype=object)
            for j in range(N):
                Tsum = 0
                for r in range(6):
                    x = dhat[r][j]
                    x = x - 2 * P if x >= 2 * P else x  # [0, 2P)
                    Tsum += x * khat[r, u, l][j]
                assert Tsum < 2 ** 64
                y = redc(Tsum)
                assert y < 4 * P
                acc[j] = y - 2 * P if y >= 2 * P else y
            c = inv(acc)
            for j in range(N):
                v = c[j] % P
                v = v - P if v > P // 2 else v
                res[j] = (res[j] + (v << (11 * l))) % 2 ** 32
        out[u] = res
    # reference: schoolbook of sum_r digits_r * key[r][u] mod 2^32
    for u in range(2):
        want = np.zeros(N, dtype=object)
        for r in range(6):
            a = [int(x) for x in digits[r]]
            b = [int(x) for x in key[r, u]]
            conv = np.convolve(np.array(a, dtype=object), np.array(b, dtype=object))
            for k in range(N):
                want[k] += conv[k] - (conv[k + N] if k + N < len(conv) else 0)
        want = [int(w) % 2 ** 32 for w in want]
        assert [int(x) for x in out[u]] == want, u
    print("emulation OK: psi=%d" % PSI)


if __name__ == "__main__":
    main()
