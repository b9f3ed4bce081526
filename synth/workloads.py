"""Seeded synthetic workloads.

Configs (BASELINE.json):
  1 IntV 1D tiny   l_I=8,  M=4,      l_S=8   x ~ U[0,2^8); (lo,hi) sorted pair of U[0,2^8) draws
  2 IntV 1D        l_I=16, M=1024,   l_S=16  widths round(2^u), u ~ U[4,12]; K in {0,1,2..4} forced hits
  3 rectangle      l_I=16, M=4096,   l_S=32  d=2, sides round(2^u), u ~ U[6,12] per axis; K forced hits
  4 IdM            l_I=20, M=65536,  l_S=32  distinct U[0,2^20) ids; query id present or absent by seed
  5 NAND sweep     2^10 / 2^14 / 2^17 / 2^20 pairs of U{0,1} bits
Synthetic stand-ins with the SHAPES of the paper's four datasets.  No
dataset record is reproduced: regions are disjoint random boxes in a 16 x 16 grid of the 2^16 x 2^16
plane, points / ids are distinct uniform draws, payloads uniform; the query hits one record or none by seed.
  6 covid-kor shape  IntV d=2 (rectangles)  M=9,   l_I=16, l_S=9
  7 covid-usa shape  IntV d=2 (rectangles)  M=58,  l_I=16, l_S=22
  8 gdacs shape      CoV  d=2 (points)      M=9,   l_I=16, l_S=16
  9 weather-usa shape IdM                   M=304, l_I=16, l_S=128
 10 paper CoV (alg:BB2) at scale: M=4096 distinct 16-bit (lat, lon) points, l_I=16, l_S=32; the
    query is one of the points (probability 3/4) or none ("paper CoV on a 4096-point shape")
Seeds: keys 1000 + cfg, data 2000 + cfg (overridable).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MODE_INTV, MODE_COV, MODE_IDM = 0, 1, 2
F_CLOSED_UPPER, F_UNSIGNED, F_EQ_TREE, F_SUM_TREE, F_OR_REDUCE = 1, 2, 4, 8, 16
CONFIG_FLAGS = F_CLOSED_UPPER | F_UNSIGNED | F_EQ_TREE | F_SUM_TREE


@dataclass
class Workload:
    cfg: int
    mode: int
    M: int
    l_I: int
    l_S: int
    d: int
    flags: int
    query: list            # query words (x) / (x, y) / (id)
    records: np.ndarray    # (M, W) uint64 record words
    payloads: np.ndarray   # (M,) uint64
    key_seed: int
    data_seed: int
    forced: list = field(default_factory=list)  # indices of records forced to match

    @property
    def name(self):
        return CONFIGS[self.cfg]["name"]


CONFIGS = {
    1: dict(name="intv1d_tiny", mode=MODE_INTV, M=4, l_I=8, l_S=8, d=1),
    2: dict(name="intv1d_1024", mode=MODE_INTV, M=1024, l_I=16, l_S=16, d=1),
    3: dict(name="rect2d_4096", mode=MODE_INTV, M=4096, l_I=16, l_S=32, d=2),
    4: dict(name="idm_65536", mode=MODE_IDM, M=65536, l_I=20, l_S=32, d=1),
    6: dict(name="kor_shape_intv2d_9", mode=MODE_INTV, M=9, l_I=16, l_S=9, d=2),
    7: dict(name="usa_shape_intv2d_58", mode=MODE_INTV, M=58, l_I=16, l_S=22, d=2),
    8: dict(name="gdacs_shape_cov_9", mode=MODE_COV, M=9, l_I=16, l_S=16, d=2),
    9: dict(name="weather_shape_idm_304", mode=MODE_IDM, M=304, l_I=16, l_S=128, d=1),
    10: dict(name="cov_points_4096", mode=MODE_COV, M=4096, l_I=16, l_S=32, d=2),
}


def _interval_containing(rng, x, w, top):
    lo_min = max(0, x - w + 1)
    lo_max = min(x, top - w)
    lo = int(rng.integers(lo_min, lo_max + 1))
    return lo, lo + w - 1


def _interval_random(rng, w, top):
    lo = int(rng.integers(0, top - w + 1))
    return lo, lo + w - 1


def _hit_count(rng):
    k = int(rng.integers(0, 3))
    return k if k < 2 else int(rng.integers(2, 5))


def make_workload(cfg: int, data_seed: int | None = None, key_seed: int | None = None,
                  M: int | None = None, flags: int = CONFIG_FLAGS, hits: int | None = None) -> Workload:
    """Draw the plaintext inputs of config ``cfg`` (1-4).  ``M`` overrides the record count (tests),
    ``hits`` the number of records forced to match."""
    c = CONFIGS[cfg]
    data_seed = 2000 + cfg if data_seed is None else data_seed
    key_seed = 1000 + cfg if key_seed is None else key_seed
    M = c["M"] if M is None else M
    rng = np.random.default_rng(data_seed)
    l_I, l_S, d, mode = c["l_I"], c["l_S"], c["d"], c["mode"]
    top = 1 << l_I
    if l_S <= 64:
        payloads = rng.integers(0, 1 << l_S, size=M, dtype=np.uint64) if l_S < 64 else \
            rng.integers(0, 2 ** 64, size=M, dtype=np.uint64)
    else:  # l_S up to 128: Python ints (two 64-bit draws)
        lo = rng.integers(0, 2 ** 64, size=M, dtype=np.uint64)
        hi = rng.integers(0, 1 << (l_S - 64), size=M, dtype=np.uint64)
        payloads = np.array([int(a) | (int(b) << 64) for a, b in zip(lo, hi)], dtype=object)
    forced = []
    if cfg == 1:
        x = int(rng.integers(0, top))
        recs = np.zeros((M, 2), np.uint64)
        for i in range(M):
            a, b = sorted(int(v) for v in rng.integers(0, top, size=2))
            recs[i] = (a, b)
        query = [x]
    elif cfg in (2, 3):
        lo_u, hi_u = (4, 12) if cfg == 2 else (6, 12)
        query = [int(rng.integers(0, top)) for _ in range(d)]
        K = _hit_count(rng) if hits is None else hits
        forced = sorted(int(i) for i in rng.choice(M, size=min(K, M), replace=False))
        recs = np.zeros((M, 2 * d), np.uint64)
        for i in range(M):
            while True:
                row = []
                inside = True
                for a in range(d):
                    w = int(round(2.0 ** rng.uniform(lo_u, hi_u)))
                    if i in forced:
                        lo, hi = _interval_containing(rng, query[a], w, top)
                    else:
                        lo, hi = _interval_random(rng, w, top)
                    inside = inside and lo <= query[a] <= hi
                    row += [lo, hi]
                if i in forced or not inside:
                    break
            recs[i] = row
    elif cfg == 4:
        ids = rng.choice(top, size=M, replace=False).astype(np.uint64)
        recs = ids.reshape(M, 1)
        present = bool(rng.integers(0, 2)) if hits is None else hits > 0
        if present:
            k = int(rng.integers(0, M))
            query = [int(ids[k])]
            forced = [k]
        else:
            idset = set(int(v) for v in ids)
            while True:
                q = int(rng.integers(0, top))
                if q not in idset:
                    break
            query = [q]
    elif cfg in (6, 7):  # disjoint boxes: distinct cells of a 16 x 16 grid, a random sub-box in each
        cells = rng.choice(256, size=M, replace=False)
        recs = np.zeros((M, 4), np.uint64)
        for i, c in enumerate(cells):
            row = []
            for a, cell in enumerate((int(c) % 16, int(c) // 16)):
                side = int(rng.integers(256, 4097))
                lo = cell * 4096 + int(rng.integers(0, 4096 - side + 1))
                row += [lo, lo + side - 1]
            recs[i] = [row[0], row[1], row[2], row[3]]
        if bool(rng.integers(0, 4)) if hits is None else hits > 0:  # hit with probability 3/4
            k = int(rng.integers(0, M))
            forced = [k]
            query = [int(rng.integers(recs[k][0], recs[k][1] + 1)), int(rng.integers(recs[k][2], recs[k][3] + 1))]
        else:
            while True:
                query = [int(rng.integers(0, top)), int(rng.integers(0, top))]
                if not any(r[0] <= query[0] <= r[1] and r[2] <= query[1] <= r[3] for r in recs.tolist()):
                    break
    elif cfg in (8, 9, 10):  # distinct points (CoV, d = 2) or distinct ids (IdM)
        W = 1 if cfg == 9 else 2
        flat = rng.choice(top ** W, size=M, replace=False)
        recs = np.array([[(int(v) >> (16 * a)) & (top - 1) for a in range(W)] for v in flat], np.uint64)
        if bool(rng.integers(0, 4)) if hits is None else hits > 0:
            k = int(rng.integers(0, M))
            forced = [k]
            query = [int(v) for v in recs[k]]
        else:
            seen = set(tuple(int(v) for v in r) for r in recs)
            while True:
                query = [int(rng.integers(0, top)) for _ in range(W)]
                if tuple(query) not in seen:
                    break
    else:
        raise ValueError(f"config {cfg} is not a circuit config")
    return Workload(cfg, mode, M, l_I, l_S, d, flags, query, recs, payloads, key_seed, data_seed, forced)


def nand_inputs(count: int, data_seed: int = 2005):
    """Config 5: ``count`` pairs of U{0,1} plaintext bits (a, b)."""
    rng = np.random.default_rng(data_seed)
    a = rng.integers(0, 2, size=count, dtype=np.uint8)
    b = rng.integers(0, 2, size=count, dtype=np.uint8)
    return a, b


def extra_queries(wl: Workload, count: int, seed: int = 7):
    """``count`` further plaintext queries for multi-query packing runs: uniform points for IntV, a random
    record's point / id (probability 1/2) or a uniform one for CoV / IdM."""
    rng = np.random.default_rng(seed)
    out = []
    top = 1 << wl.l_I
    W = len(wl.query)
    for _ in range(count):
        if wl.mode != MODE_INTV and rng.integers(0, 2):
            out.append([int(v) for v in wl.records[int(rng.integers(0, wl.M))]])
        else:
            out.append([int(rng.integers(0, top)) for _ in range(W)])
    return out


def expected_result(wl: Workload, query=None) -> int:
    """The plaintext answer the query must decrypt to (thm:VeLoPIR; R12/R13/R19): XOR (OR with
    F_OR_REDUCE) of the payloads of the records whose plaintext bounds match the query; 0 if none.
    Ground truth of the drawn inputs (used by bench.py's sanity check), not the homomorphic method."""
    q = wl.query if query is None else query
    r = 0
    for rec, pay in zip(wl.records.tolist(), wl.payloads.tolist()):
        if wl.mode == MODE_INTV:
            ok = all(rec[2 * a] <= q[a] and (q[a] <= rec[2 * a + 1] if wl.flags & F_CLOSED_UPPER
                                             else q[a] < rec[2 * a + 1]) for a in range(wl.d))
        elif wl.mode == MODE_COV:
            ok = all(q[a] == rec[a] for a in range(wl.d))
        else:
            ok = q[0] == rec[0]
        if ok:
            r = (r | int(pay)) if wl.flags & F_OR_REDUCE else (r ^ int(pay))
    return r
