"""Developer tool: index/swizzle/bounds check of the v2 blind-rotate layout (8 coefficients per thread,
128 threads per bootstrap, stage 9 via a lane-pair register exchange).  Not product code."""
import numpy as np
import sys
sys.path.insert(0, "tools")
from emulate_br_ntt import P, W, WS, WI, WIS, shoup

def jA(t, r): return t | (r << 7)
def jB(t, r): return ((t >> 4) << 7) | (r << 4) | (t & 15)
def jC(t, r): return ((t >> 1) << 4) | (r << 1) | (t & 1)

def h(j):
    b = lambda k: (j >> k) & 1
    return (b(5) << 1) ^ (b(6) << 2) ^ (b(7) << 3) ^ (b(7) << 4)
def phys(j): return j ^ h(j)

# swizzle: bijection + conflict-free per warp for all layouts
assert sorted(phys(j) for j in range(1024)) == list(range(1024))
for lay in (jA, jB, jC):
    assert sorted(lay(t, r) for t in range(128) for r in range(8)) == list(range(1024))
    for w in range(4):
        for r in range(8):
            banks = [phys(lay(32 * w + l, r)) % 32 for l in range(32)]
            assert len(set(banks)) == 32, (lay.__name__, w, r)
# base^c decomposition used by the kernel
def bA(t): return t ^ (((t >> 5) & 1) << 1) ^ (((t >> 6) & 1) << 2)
def cA(r): return (r << 7) ^ ((r & 1) * 24)
def bB(t): return ((((t >> 4) << 7) | (t & 15)) ^ (((t >> 4) & 1) * 24))
def cB(r): return (r << 4) ^ (((r >> 1) & 1) << 1) ^ (((r >> 2) & 1) << 2)
def bC(t): return ((((t >> 1) << 4) | (t & 1)) ^ (((t >> 2) & 1) << 1) ^ (((t >> 3) & 1) << 2) ^ (((t >> 4) & 1) * 24))
def cC(r): return r << 1
for t in range(128):
    for r in range(8):
        assert bA(t) ^ cA(r) == phys(jA(t, r))
        assert bB(t) ^ cB(r) == phys(jB(t, r))
        assert bC(t) ^ cC(r) == phys(jC(t, r))

def posF(t, s):
    i = s & 3
    r = 4 + i if t & 1 else i
    tt = (t & ~1) if s < 4 else (t | 1)
    return jC(tt, r)
def inv_pos(pos):
    b0 = pos & 1; r = (pos >> 1) & 7
    t = ((pos >> 4) << 1) | (1 if r >= 4 else 0)
    s = (4 if b0 else 0) + (r & 3)
    return t, s
assert sorted(posF(t, s) for t in range(128) for s in range(8)) == list(range(1024))
for t in range(128):
    for s in range(8):
        assert inv_pos(posF(t, s)) == (t, s)

def twk(stage, t, q):
    th = t >> 4; tc = t >> 1
    return {3: 8 + th, 4: 16 + 2 * th + q, 5: 32 + 4 * th + q, 6: 64 + tc, 7: 128 + 2 * tc + q,
            8: 256 + 4 * tc + q, 9: 512 + 8 * tc + ((4 + q) if t & 1 else q)}[stage]

def fwd(vals):  # vals[t][r] layout A, each in [0, 4P)
    reg = [list(v) for v in vals]
    a = {}
    def stage(lay, s, rb, qf):
        tt = 512 >> s
        for t in range(128):
            for r in range(8):
                if r & rb: continue
                j = lay(t, r); assert lay(t, r | rb) == j + tt
                k = (1 << s) + (j >> (10 - s))
                if s >= 3: assert k == twk(s, t, qf(r)), (s, t, r)
                x, y = reg[t][r], reg[t][r | rb]
                assert x < 4 * P and y < 4 * P
                x = x - 2 * P if x >= 2 * P else x
                T = shoup(y, W[k], WS[k])
                reg[t][r], reg[t][r | rb] = x + T, x - T + 2 * P
    def exch(src, dst):
        buf = [0] * 1024
        for t in range(128):
            for r in range(8): buf[phys(src(t, r))] = reg[t][r]
        for t in range(128):
            for r in range(8): reg[t][r] = buf[phys(dst(t, r))]
    for s in range(3): stage(jA, s, 4 >> s, None)
    exch(jA, jB)
    stage(jB, 3, 4, lambda r: 0); stage(jB, 4, 2, lambda r: r >> 2); stage(jB, 5, 1, lambda r: r >> 1)
    exch(jB, jC)
    stage(jC, 6, 4, lambda r: 0); stage(jC, 7, 2, lambda r: r >> 2); stage(jC, 8, 1, lambda r: r >> 1)
    # stage 9: lane-pair exchange then in-register butterflies on (reg[i], reg[4+i])
    new = [list(v) for v in reg]
    for t in range(128):
        lo = (t & 1) == 0; p = t ^ 1
        for i in range(4):
            send_p = reg[p][4 + i] if (p & 1) == 0 else reg[p][i]
            recv = send_p
            new[t][i] = reg[t][i] if lo else recv
            new[t][4 + i] = recv if lo else reg[t][4 + i]
    reg = new
    for t in range(128):
        for i in range(4):
            k = twk(9, t, i)
            x, y = reg[t][i], reg[t][4 + i]
            assert k == 512 + (posF(t, i) >> 1) and posF(t, 4 + i) == posF(t, i) + 1
            x = x - 2 * P if x >= 2 * P else x
            T = shoup(y, W[k], WS[k])
            reg[t][i], reg[t][4 + i] = x + T, x - T + 2 * P
    out = [0] * 1024
    for t in range(128):
        for s in range(8): out[posF(t, s)] = reg[t][s]
    return out

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

rng = np.random.default_rng(3)
poly = rng.integers(-64, 64, 1024)
vals = [[int(poly[jA(t, r)]) + P for r in range(8)] for t in range(128)]
got = fwd(vals)
want = plain_fwd(poly)
assert [g % P for g in got] == want
print("v2 layout emulation OK")
