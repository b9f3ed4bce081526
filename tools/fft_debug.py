"""Developer tool: one CMux step of K2F against an exact numpy external product, with the error split by
digit row and limb (which part of the glue is wrong)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12761_b200 import _lib as L  # noqa: E402
from paper_2506_12761_b200 import api as A  # noqa: E402

N = 1024


def nega(a, b):
    c = np.convolve(a.astype(np.int64), b.astype(np.int64))
    return c[:N] - np.concatenate([c[N:], [0]])


def mono(p, e):  # X^e * p mod X^N + 1 (u32), e in [0, 2N)
    out = np.zeros(N, np.uint64)
    for j in range(N):
        k = j + e
        s = 1
        while k >= N:
            k -= N
            s = -s
        out[k] = (int(p[j]) * s) % (1 << 32)
    return out.astype(np.uint32)


def main():
    keys = A.Keys(123)
    srv = A.Server(keys, 0)
    s, z, bsk, ksk = keys.export()
    rng = np.random.default_rng(1)
    ct = rng.integers(0, 2 ** 32, (1, 632), dtype=np.uint64).astype(np.uint32)
    ct[:, 631] = 0
    ms = lambda v: ((int(v) + (1 << 20)) >> 21) & 2047
    abar0, bbar = ms(ct[0, 0]), ms(ct[0, 630])
    testv = np.full(N, 0x20000000, np.uint32)
    acc = [np.zeros(N, np.uint32), mono(testv, (2 * N - bbar) % (2 * N))]
    D = [(mono(acc[u], abar0).astype(np.int64) - acc[u].astype(np.int64)) % (1 << 32) for u in range(2)]
    digits = []
    for u in range(2):
        w = (D[u] + 0x81020400) % (1 << 32)
        for j in range(3):
            digits.append((((w >> (25 - 7 * j)) & 127) - 64).astype(np.int64))
    parts = {}
    for r in range(6):
        for o in range(2):
            sv = bsk[0, r, o].astype(np.int64)
            sv = np.where(sv >= 2 ** 31, sv - 2 ** 32, sv)
            lo = ((sv + 32768) & 65535) - 32768
            hi = (sv - lo) >> 16
            parts[(r, o, 0)] = nega(digits[r], lo)
            parts[(r, o, 1)] = nega(digits[r], hi)
    want = []
    for o in range(2):
        tot = sum(parts[(r, o, 0)] + (parts[(r, o, 1)] << 16) for r in range(6))
        want.append((acc[o].astype(np.int64) + tot) % (1 << 32))
    for eng, par in ((1, 5), (2, 1)):
        L.lib().vlp_debug_route(eng, par)
        got = A.to_host(srv.debug_blind_rotate(A.to_device(ct), 1))[0].astype(np.int64)
        for o in range(2):
            diff = (got[o * N:(o + 1) * N] - want[o]) % (1 << 32)
            diff = np.where(diff >= 2 ** 31, diff - 2 ** 32, diff)
            print(f"engine {eng} comp {o}: {np.count_nonzero(diff)} differ, max |diff| {np.max(np.abs(diff))}", flush=True)
            if np.count_nonzero(diff):
                # try explaining diff by single parts
                for key, p in parts.items():
                    for sc in (1, 1 << 16):
                        for sg in (1, -1):
                            if np.array_equal((sg * sc * p - diff) % (1 << 32), np.zeros(N)):
                                print("   diff ==", sg, sc, key)
                print("   diff[:8]", diff[:8], "diff mod 2^16", diff[:8] % 65536)
    L.lib().vlp_debug_route(0, 0)
    np.savez("gpurun_out/fft_debug.npz", got=got, want0=want[0], want1=want[1],
             **{f"p{r}{o}{l}": parts[(r, o, l)] for r in range(6) for o in range(2) for l in range(2)})


if __name__ == "__main__":
    main()
