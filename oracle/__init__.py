"""oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow CPU implementation of the TFHE gate bootstrapping and VeLoPIR circuits (arXiv 2506.12761).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg
may import this package.  It shares no code with ``paper_2506_12761_b200`` (the CUDA product path) and
never imports it.

* ``tfhe_oracle.c``  -- torus32 arithmetic, PRNG/Gaussian, KeyGen, TLWE Enc/Dec, exact negacyclic
  products, external product, BlindRotate, SampleExtract, KeySwitch, gates.
* ``circuits.py``    -- alg:HomCompLE / HomCompL / HomEQ / HomEqOPT / IntV / CoV / IdM / HomBitwiseAND /
  HomSum / VeLoPIR, written once against a gate backend: ``TfheBackend`` (ciphertexts through the C
  oracle) or ``PlainBackend`` (booleans: the PlainOracle, O15) -- plus the plain predicate.
* ``protocol.py``    -- PubKeyGen / ServerEnc / query encryption / decryption.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "tfhe_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

n = 630
N = 1024
MU = 0x20000000  # 1/8
SIGMA_LWE = 2.0 ** -15  # R2
SIGMA_BK = 2.0 ** -25
SIGMA_KS = 2.0 ** -15

AND, NAND, OR, XOR, XNOR = 0, 1, 2, 3, 4
KIND_FRESH, KIND_QUERY, KIND_PK = 0, 1, 2

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no -ffast-math, no FMA contraction: R3 determinism)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
             "-o", LIB + ".tmp", SRC, "-lm"])
        os.replace(LIB + ".tmp", LIB)
    return LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(LIB)
            u32p = ctypes.POINTER(ctypes.c_uint32)
            i32p = ctypes.POINTER(ctypes.c_int32)
            i64p = ctypes.POINTER(ctypes.c_int64)
            vp = ctypes.c_void_p
            sig = {
                "oracle_prng": (ctypes.c_uint64, [ctypes.c_uint64] * 4),
                "oracle_gaussian": (ctypes.c_int32, [ctypes.c_uint64] * 4 + [ctypes.c_double]),
                "oracle_ecd": (ctypes.c_uint32, [ctypes.c_int]),
                "oracle_negacyclic_schoolbook": (None, [u32p, u32p, u32p, ctypes.c_int]),
                "oracle_negacyclic_dot": (None, [ctypes.c_int, i64p, i64p, u32p]),
                "oracle_negacyclic_mul": (None, [u32p, u32p, u32p]),
                "oracle_gadget_digits": (None, [ctypes.c_uint32, i32p]),
                "oracle_ks_digits": (None, [ctypes.c_uint32, i32p]),
                "oracle_modswitch": (ctypes.c_int, [ctypes.c_uint32]),
                "oracle_keygen": (vp, [ctypes.c_uint64, ctypes.c_double, ctypes.c_double]),
                "oracle_free_keys": (None, [vp]),
                "oracle_export_keys": (None, [vp, u32p, u32p, u32p, u32p]),
                "oracle_encrypt": (None, [vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                          ctypes.c_double, u32p]),
                "oracle_phase": (ctypes.c_uint32, [vp, u32p]),
                "oracle_decrypt": (ctypes.c_int, [vp, u32p]),
                "oracle_trlwe_phase": (None, [vp, u32p, u32p]),
                "oracle_external_product": (None, [vp, ctypes.c_int, u32p, u32p]),
                "oracle_blind_rotate": (None, [vp, u32p, ctypes.c_int, u32p]),
                "oracle_sample_extract": (None, [u32p, u32p]),
                "oracle_keyswitch": (None, [vp, u32p, u32p]),
                "oracle_bootstrap_nlwe": (None, [vp, u32p, u32p]),
                "oracle_bootstrap": (None, [vp, u32p, u32p]),
                "oracle_bootstrap_mu": (None, [vp, u32p, ctypes.c_uint32, u32p]),
                "oracle_gate": (None, [vp, ctypes.c_int, u32p, u32p, u32p]),
                "oracle_mux": (None, [vp, u32p, u32p, u32p, u32p]),
            }
            for name, (res, args) in sig.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def _p(a: np.ndarray, t=ctypes.c_uint32):
    return a.ctypes.data_as(ctypes.POINTER(t))


def u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


# ---------------------------------------------------------------- exact primitives (pins use these)
def prng(seed, domain, obj, word) -> int:
    return int(lib().oracle_prng(seed, domain, obj, word))


def gaussian(seed, domain, obj, t, sigma) -> int:
    return int(lib().oracle_gaussian(seed, domain, obj, t, sigma))


def negacyclic_schoolbook(a, b) -> np.ndarray:
    a, b = u32(a), u32(b)
    c = np.zeros_like(a)
    lib().oracle_negacyclic_schoolbook(_p(a), _p(b), _p(c), len(a))
    return c


def negacyclic_dot(a_list, b_list) -> np.ndarray:
    """sum_t a_t * b_t in Z[X]/(X^1024+1) mod 2^32 for signed integer polynomials (exact NTT path)."""
    a = np.ascontiguousarray(np.asarray(a_list, dtype=np.int64).reshape(-1, N))
    b = np.ascontiguousarray(np.asarray(b_list, dtype=np.int64).reshape(-1, N))
    out = np.zeros(N, dtype=np.uint32)
    lib().oracle_negacyclic_dot(a.shape[0], _p(a, ctypes.c_int64), _p(b, ctypes.c_int64), _p(out))
    return out


def gadget_digits(x: int):
    d = (ctypes.c_int32 * 3)()
    lib().oracle_gadget_digits(x, d)
    return list(d)


def ks_digits(x: int):
    d = (ctypes.c_int32 * 8)()
    lib().oracle_ks_digits(x, d)
    return list(d)


def modswitch(x: int) -> int:
    return int(lib().oracle_modswitch(x))


def trivial(bit: int) -> np.ndarray:
    """Noiseless (0, Ecd(bit)) (R21)."""
    ct = np.zeros(n + 1, dtype=np.uint32)
    ct[n] = MU if bit else (0x100000000 - MU)
    return ct


def trivial_mu(mu: int) -> np.ndarray:
    ct = np.zeros(n + 1, dtype=np.uint32)
    ct[n] = mu & 0xFFFFFFFF
    return ct


def sample_extract(acc) -> np.ndarray:
    acc = u32(acc)
    out = np.zeros(N + 1, dtype=np.uint32)
    lib().oracle_sample_extract(_p(acc), _p(out))
    return out


class OracleKeys:
    """Secret key s, ring key z, bootstrapping key and key-switching key for one seed."""

    def __init__(self, seed: int, sigma_bk: float = SIGMA_BK, sigma_ks: float = SIGMA_KS):
        self.seed = seed
        self._h = lib().oracle_keygen(seed, sigma_bk, sigma_ks)
        self.gates = 0  # BR count (MUX counts 2)

    def __del__(self):
        try:
            if self._h:
                lib().oracle_free_keys(self._h)
                self._h = None
        except Exception:
            pass

    # -- keys --
    def export(self):
        s = np.zeros(n, np.uint32)
        z = np.zeros(N, np.uint32)
        bsk = np.zeros(n * 6 * 2 * N, np.uint32)
        ksk = np.zeros(N * 8 * 3 * (n + 1), np.uint32)
        lib().oracle_export_keys(self._h, _p(s), _p(z), _p(bsk), _p(ksk))
        return s, z, bsk.reshape(n, 6, 2, N), ksk.reshape(N, 8, 3, n + 1)

    # -- TLWE --
    def encrypt(self, bit: int, seed: int, obj: int, kind: int = KIND_FRESH, sigma: float = SIGMA_LWE):
        ct = np.zeros(n + 1, np.uint32)
        lib().oracle_encrypt(self._h, int(bit), seed, kind, obj, sigma, _p(ct))
        return ct

    def phase(self, ct) -> int:
        return int(lib().oracle_phase(self._h, _p(u32(ct))))

    def decrypt(self, ct) -> int:
        return int(lib().oracle_decrypt(self._h, _p(u32(ct))))

    def trlwe_phase(self, trlwe) -> np.ndarray:
        out = np.zeros(N, np.uint32)
        lib().oracle_trlwe_phase(self._h, _p(u32(trlwe)), _p(out))
        return out

    # -- bootstrapping pieces --
    def external_product(self, i: int, D) -> np.ndarray:
        out = np.zeros(2 * N, np.uint32)
        lib().oracle_external_product(self._h, i, _p(u32(D)), _p(out))
        return out

    def blind_rotate(self, c, steps: int = n) -> np.ndarray:
        acc = np.zeros(2 * N, np.uint32)
        lib().oracle_blind_rotate(self._h, _p(u32(c)), steps, _p(acc))
        return acc

    def keyswitch(self, nlwe) -> np.ndarray:
        out = np.zeros(n + 1, np.uint32)
        lib().oracle_keyswitch(self._h, _p(u32(nlwe)), _p(out))
        return out

    def bootstrap_nlwe(self, c) -> np.ndarray:
        out = np.zeros(N + 1, np.uint32)
        lib().oracle_bootstrap_nlwe(self._h, _p(u32(c)), _p(out))
        return out

    def bootstrap(self, c) -> np.ndarray:
        out = np.zeros(n + 1, np.uint32)
        lib().oracle_bootstrap(self._h, _p(u32(c)), _p(out))
        return out

    def bootstrap_mu(self, c, mu: int) -> np.ndarray:
        """R24 (not in the paper): bootstrap with test vector mu in every coefficient (R8 uses 1/8)."""
        out = np.zeros(n + 1, np.uint32)
        lib().oracle_bootstrap_mu(self._h, _p(u32(c)), mu, _p(out))
        return out

    # -- gates (R10) --
    def gate(self, op: int, x, y) -> np.ndarray:
        out = np.zeros(n + 1, np.uint32)
        lib().oracle_gate(self._h, op, _p(u32(x)), _p(u32(y)), _p(out))
        self.gates += 1
        return out

    def mux(self, c, a, b) -> np.ndarray:
        out = np.zeros(n + 1, np.uint32)
        lib().oracle_mux(self._h, _p(u32(c)), _p(u32(a)), _p(u32(b)), _p(out))
        self.gates += 2
        return out

    @staticmethod
    def not_(x) -> np.ndarray:
        return (np.uint32(0) - u32(x)).astype(np.uint32)
