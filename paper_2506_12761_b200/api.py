"""Thin Python layer over the C ABI (include/vlp.h).  Argument marshalling only.

PyTorch provides device memory (uint8 / int32 tensors) and streams; every computation of the hot path runs in
libvlp.so's CUDA kernels.  Host ciphertext arrays are numpy uint32 [count, 632]; device ciphertext
tensors are torch.int32 [count, 632] (same bytes).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L
from ._lib import CT_STRIDE, NLWE_STRIDE, VlpMeta, VlpParams, VlpProgramInfo, check, lib


def _u32p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def meta(mode, M, l_I, l_S, d, flags=L.CONFIG_FLAGS) -> VlpMeta:
    return VlpMeta(mode, M, l_I, l_S, d, flags)


def _stream_handle(stream, device=None) -> int:
    """The raw cudaStream_t of `stream`; None -> the current torch stream of `device` (the server's GPU, not the
    caller's current device)."""
    if stream is None:
        import torch
        return torch.cuda.current_stream(device).cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


class Keys:
    """vlp_keygen: secret key + evaluation key, host side."""

    def __init__(self, seed: int | None = None, device: int | None = None):
        """KeyGen.  seed=None (the default): fresh keys from OS randomness (vlp_keygen_secure; with device= the
        device KeyGen, vlp_keygen_device_secure).  An integer seed: the reproducible test / benchmark keys of
        vlp_keygen (only as secret as the seed), on the host, or with device= the byte-identical device KeyGen
        (vlp_keygen_device)."""
        self.seed = seed
        sk, evk = ctypes.c_void_p(), ctypes.c_void_p()
        if device is None:
            if seed is None:
                check(lib().vlp_keygen_secure(None, ctypes.byref(sk), ctypes.byref(evk)))
            else:
                check(lib().vlp_keygen(seed, None, ctypes.byref(sk), ctypes.byref(evk)))
        else:
            import torch
            sc = torch.empty(lib().vlp_keygen_device_scratch_bytes(), dtype=torch.uint8, device=f"cuda:{device}")
            st = _stream_handle(None, device)
            if seed is None:
                check(lib().vlp_keygen_device_secure(None, ctypes.c_void_p(sc.data_ptr()), sc.numel(), st,
                                                     ctypes.byref(sk), ctypes.byref(evk)))
            else:
                check(lib().vlp_keygen_device(seed, None, ctypes.c_void_p(sc.data_ptr()), sc.numel(), st,
                                              ctypes.byref(sk), ctypes.byref(evk)))
        self.sk, self.evk = sk, evk

    def __del__(self):
        try:
            lib().vlp_free_sk(self.sk)
            lib().vlp_free_evk(self.evk)
        except Exception:
            pass

    def export(self):
        s = np.zeros(L.n, np.uint32)
        z = np.zeros(L.N, np.uint32)
        bsk = np.zeros(L.n * 6 * 2 * L.N, np.uint32)
        ksk = np.zeros(L.N * 8 * 3 * (L.n + 1), np.uint32)
        check(lib().vlp_sk_export(self.sk, _u32p(s), _u32p(z)))
        check(lib().vlp_evk_export(self.evk, _u32p(bsk), _u32p(ksk)))
        return s, z, bsk.reshape(L.n, 6, 2, L.N), ksk.reshape(L.N, 8, 3, L.n + 1)

    def encrypt_bits(self, bits, seed: int | None = None, obj0: int = 0) -> np.ndarray:
        """Fresh encryptions; seed=None: OS randomness (vlp_encrypt_bits_secure), else the seeded test mode."""
        bits = np.ascontiguousarray(np.asarray(bits, dtype=np.uint8))
        out = np.zeros((len(bits), CT_STRIDE), np.uint32)
        bp = bits.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
        if seed is None:
            check(lib().vlp_encrypt_bits_secure(self.sk, bp, len(bits), _u32p(out)))
        else:
            check(lib().vlp_encrypt_bits(self.sk, bp, len(bits), seed, obj0, _u32p(out)))
        return out

    def encrypt_query(self, m: VlpMeta, values, seed: int | None = None) -> np.ndarray:
        """encrypt_query; seed=None: OS randomness (vlp_encrypt_query_secure), else the seeded test mode."""
        vals = np.ascontiguousarray(np.asarray(values, dtype=np.uint64))
        words = 1 if m.mode == L.MODE_IDM else m.d
        out = np.zeros((words * m.l_I, CT_STRIDE), np.uint32)
        if seed is None:
            check(lib().vlp_encrypt_query_secure(self.sk, ctypes.byref(m), _u64p(vals), _u32p(out)))
        else:
            check(lib().vlp_encrypt_query(self.sk, ctypes.byref(m), _u64p(vals), seed, _u32p(out)))
        return out

    def decrypt_bits(self, ct: np.ndarray) -> np.ndarray:
        ct = np.ascontiguousarray(ct, dtype=np.uint32).reshape(-1, CT_STRIDE)
        out = np.zeros(ct.shape[0], np.uint8)
        check(lib().vlp_decrypt_bits(self.sk, _u32p(ct), ct.shape[0], out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
        return out

    def decrypt_result(self, ct: np.ndarray, l_S: int | None = None):
        """decrypt_result: (bits LSB first, value) of the l_S result ciphertexts."""
        ct = np.ascontiguousarray(ct, dtype=np.uint32)
        l_S = ct.shape[0] if l_S is None else l_S
        bits = np.zeros(l_S, np.uint8)
        v = ctypes.c_uint64()
        check(lib().vlp_decrypt_result(self.sk, _u32p(ct), l_S, bits.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                                       ctypes.byref(v) if l_S <= 64 else None))
        return bits, v.value

    def decrypt_value(self, ct: np.ndarray) -> int:  # any l_S (Python int)
        return int(sum(int(b) << j for j, b in enumerate(self.decrypt_bits(ct))))

    def encrypt_db(self, m: VlpMeta, words, payloads, pk_seed: int | None = None, first: int = 0,
                   count: int | None = None):
        """Client PubKeyGen (alg:PubKeyGen) + server ServerEnc (alg:ServerEnc) for records [first, first+count);
        pk_seed=None: the pk from OS randomness (vlp_pubkeygen_secure), else the seeded test mode."""
        words = np.ascontiguousarray(np.asarray(words, dtype=np.uint64))
        count = len(payloads) if count is None else count
        pw = (m.l_S + 63) // 64  # payload words per record (l_S up to 128)
        if pw == 1:
            payloads = np.ascontiguousarray(np.asarray(payloads, dtype=np.uint64))
        else:
            payloads = np.array([[(int(v) >> (64 * w)) & (2 ** 64 - 1) for w in range(pw)] for v in payloads],
                                dtype=np.uint64)
        pk = ctypes.c_void_p()
        if pk_seed is None:
            check(lib().vlp_pubkeygen_secure(self.sk, ctypes.byref(m), first, count, ctypes.byref(pk)))
        else:
            check(lib().vlp_pubkeygen(self.sk, ctypes.byref(m), pk_seed, first, count, ctypes.byref(pk)))
        try:
            per = record_cts(m)
            out = np.zeros((count * per, CT_STRIDE), np.uint32)
            check(lib().vlp_server_encrypt_db(pk, _u64p(words), _u64p(payloads), _u32p(out)))
        finally:
            lib().vlp_free_pk(pk)
        return out


class PublicKey:
    """alg:PubKeyGen's single-use samples (vlp_pk), held on the host until the server consumes them."""

    def __init__(self, keys: "Keys", m: VlpMeta, first: int, count: int, seed: int | None = None):
        self.m, self.first, self.count = m, first, count
        h = ctypes.c_void_p()
        if seed is None:
            check(lib().vlp_pubkeygen_secure(keys.sk, ctypes.byref(m), first, count, ctypes.byref(h)))
        else:
            check(lib().vlp_pubkeygen(keys.sk, ctypes.byref(m), seed, first, count, ctypes.byref(h)))
        self.h = h

    def __del__(self):
        try:
            lib().vlp_free_pk(self.h)
        except Exception:
            pass


def server_load_records(pk: PublicKey, words, payloads, device: int = 0, stream=None):
    """Server side (vlp_server_load_records): ServerEnc of a received pk straight into a torch int32
    [count * per, 632] tensor on `device`; consumes the pk (a second call raises VLP_EPKUSED)."""
    import torch
    words = np.ascontiguousarray(np.asarray(words, dtype=np.uint64))
    pays = _payload_words(pk.m, payloads)
    per = record_cts(pk.m)
    out = torch.empty((pk.count * per, CT_STRIDE), dtype=torch.int32, device=f"cuda:{device}")
    sb = ctypes.c_size_t()
    check(lib().vlp_server_encrypt_db_device_scratch_bytes(ctypes.byref(pk.m), pk.count, ctypes.byref(sb)))
    sc = torch.empty(max(256, sb.value), dtype=torch.uint8, device=f"cuda:{device}")
    check(lib().vlp_server_load_records(pk.h, _u64p(words), _u64p(pays), ctypes.c_void_p(out.data_ptr()),
                                        ctypes.c_void_p(sc.data_ptr()), sc.numel(), _stream_handle(stream, device)))
    return out


def _payload_words(m: VlpMeta, payloads):
    pw = (m.l_S + 63) // 64  # payload words per record (l_S up to 128)
    if pw == 1:
        return np.ascontiguousarray(np.asarray(payloads, dtype=np.uint64))
    return np.array([[(int(v) >> (64 * w)) & (2 ** 64 - 1) for w in range(pw)] for v in payloads], dtype=np.uint64)


def pubkeygen_device(keys: "Keys", m: VlpMeta, pk_seed: int | None, first: int, count: int, device: int = 0,
                     stream=None):
    """Client side, device PubKeyGen (alg:PubKeyGen P:194-219): the records' single-use TLWE(0) samples as a torch
    int32 [count * per, 632] tensor, byte-identical to vlp_pubkeygen's samples.  pk_seed=None: OS randomness
    (vlp_pubkeygen_device_secure)."""
    import torch
    per = record_cts(m)
    pk = torch.empty((count * per, CT_STRIDE), dtype=torch.int32, device=f"cuda:{device}")
    sb = ctypes.c_size_t()
    check(lib().vlp_pubkeygen_device_scratch_bytes(ctypes.byref(m), count, ctypes.byref(sb)))
    sc = torch.empty(max(256, sb.value), dtype=torch.uint8, device=f"cuda:{device}")
    if pk_seed is None:
        check(lib().vlp_pubkeygen_device_secure(keys.sk, ctypes.byref(m), first, count, ctypes.c_void_p(pk.data_ptr()),
                                                ctypes.c_void_p(sc.data_ptr()), sc.numel(), _stream_handle(stream, device)))
    else:
        check(lib().vlp_pubkeygen_device(keys.sk, ctypes.byref(m), pk_seed, first, count, ctypes.c_void_p(pk.data_ptr()),
                                         ctypes.c_void_p(sc.data_ptr()), sc.numel(), _stream_handle(stream, device)))
    return pk


def server_encrypt_db_device(m: VlpMeta, pk_dev, words, payloads, out=None, stream=None):
    """Server side, device ServerEnc (alg:ServerEnc P:223-247): pk + (0, Ecd(bit)) for every DB row, in place in
    pk_dev unless out is given.  Takes no secret key."""
    import torch
    words = np.ascontiguousarray(np.asarray(words, dtype=np.uint64))
    pays = _payload_words(m, payloads)
    count = len(payloads)
    dev = pk_dev.device.index
    out = pk_dev if out is None else out
    sb = ctypes.c_size_t()
    check(lib().vlp_server_encrypt_db_device_scratch_bytes(ctypes.byref(m), count, ctypes.byref(sb)))
    sc = torch.empty(max(256, sb.value), dtype=torch.uint8, device=pk_dev.device)
    check(lib().vlp_server_encrypt_db_device(ctypes.byref(m), count, ctypes.c_void_p(pk_dev.data_ptr()), _u64p(words),
                                             _u64p(pays), ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(sc.data_ptr()),
                                             sc.numel(), _stream_handle(stream, dev)))
    return out


def encrypt_db_device(keys: "Keys", m: VlpMeta, words, payloads, pk_seed: int, first: int = 0,
                      count: int | None = None, device: int = 0, stream=None):
    """Device PubKeyGen + ServerEnc: the encrypted DB as a torch int32 [count * per, 632] tensor on `device`,
    byte-identical to Keys.encrypt_db."""
    import torch
    words = np.ascontiguousarray(np.asarray(words, dtype=np.uint64))
    count = len(payloads) if count is None else count
    pw = (m.l_S + 63) // 64
    if pw == 1:
        pays = np.ascontiguousarray(np.asarray(payloads, dtype=np.uint64))
    else:
        pays = np.array([[(int(v) >> (64 * w)) & (2 ** 64 - 1) for w in range(pw)] for v in payloads], dtype=np.uint64)
    per = record_cts(m)
    out = torch.empty((count * per, CT_STRIDE), dtype=torch.int32, device=f"cuda:{device}")
    sb = ctypes.c_size_t()
    check(lib().vlp_encrypt_db_device_scratch_bytes(ctypes.byref(m), count, ctypes.byref(sb)))
    sc = torch.empty(max(256, sb.value), dtype=torch.uint8, device=f"cuda:{device}")
    check(lib().vlp_encrypt_db_device(keys.sk, ctypes.byref(m), pk_seed, first, count, _u64p(words), _u64p(pays),
                                      ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(sc.data_ptr()), sc.numel(),
                                      _stream_handle(stream, device)))
    return out


def record_cts(m: VlpMeta) -> int:
    v = ctypes.c_size_t()
    check(lib().vlp_db_record_cts(ctypes.byref(m), ctypes.byref(v)))
    return v.value


class Server:
    """vlp_server_create: the evaluation key resident on one GPU (bsk converted to the NTT domain)."""

    def __init__(self, keys: Keys, device: int = 0, stream=None):
        import torch
        self.device = device
        self.keys = keys
        nbytes = lib().vlp_server_evk_bytes()
        self.evk_dev = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            check(lib().vlp_server_create(device, keys.evk, ctypes.c_void_p(self.evk_dev.data_ptr()), nbytes,
                                          _stream_handle(stream, device), ctypes.byref(h)))
        self.h = h

    def __del__(self):
        try:
            lib().vlp_free_server(self.h)
        except Exception:
            pass

    # ---- the problem-statement calls (vlp_server_eval / vlp_server_combine / vlp_gate_batch): schedules are
    # compiled and cached inside the library; the scratch buffers are torch tensors owned here
    def _scratch(self, key, nbytes, stream_handle):
        """One scratch tensor per (call shape, stream): evaluations on one stream are ordered (each reloads its
        job tables first), evaluations on different streams may run concurrently and get separate buffers."""
        import torch
        cache = self.__dict__.setdefault("_scratch_cache", {})
        key = key + (stream_handle,)
        t = cache.get(key)
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(256, nbytes), dtype=torch.uint8, device=f"cuda:{self.device}")
            cache[key] = t
        return t

    def eval(self, m: VlpMeta, query_dev, db_dev, out_dev, first: int = 0, count: int | None = None, stream=None):
        """server_eval: the shard [first, first+count)'s l_S aggregate ciphertexts into out_dev."""
        count = m.M - first if count is None else count
        key = ("eval", bytes(m), first, count)
        if key not in self.__dict__.setdefault("_ws", {}):
            sb = ctypes.c_size_t()
            check(lib().vlp_server_workspace_bytes(ctypes.byref(m), count, None, None, ctypes.byref(sb)))
            self._ws[key] = sb.value
        sh = _stream_handle(stream, self.device)
        sc = self._scratch(key, self._ws[key], sh)
        check(lib().vlp_server_eval(self.h, ctypes.byref(m), first, count, ctypes.c_void_p(query_dev.data_ptr()),
                                    ctypes.c_void_p(db_dev.data_ptr()), ctypes.c_void_p(out_dev.data_ptr()),
                                    ctypes.c_void_p(sc.data_ptr()), sc.numel(), sh))

    def eval_host(self, m: VlpMeta, query_host: np.ndarray, db_dev, out_host: np.ndarray, first: int = 0,
                  count: int | None = None, stream=None):
        """server_eval with host buffers (vlp_server_eval_host): query_host [query cts, 632] u32 in, the l_S result
        ciphertexts into out_host [l_S, 632] u32 (both C-contiguous; pinned memory makes the copies asynchronous).
        Returns once the result is on the host."""
        count = m.M - first if count is None else count
        key = ("eval_host", bytes(m), first, count)
        if key not in self.__dict__.setdefault("_ws", {}):
            sb = ctypes.c_size_t()
            check(lib().vlp_server_eval_host_workspace_bytes(ctypes.byref(m), count, ctypes.byref(sb)))
            self._ws[key] = sb.value
        sh = _stream_handle(stream, self.device)
        sc = self._scratch(key, self._ws[key], sh)
        check(lib().vlp_server_eval_host(self.h, ctypes.byref(m), first, count, _u32p(query_host),
                                         ctypes.c_void_p(db_dev.data_ptr()), _u32p(out_host),
                                         ctypes.c_void_p(sc.data_ptr()), sc.numel(), sh))

    def eval_batch(self, m: VlpMeta, queries_dev, db_dev, out_dev, nq: int, first: int = 0,
                   count: int | None = None, stream=None):
        """Multi-query packing: nq queries (queries_dev [nq * query cts, 632]) -> out_dev [nq * l_S, 632]."""
        count = m.M - first if count is None else count
        key = ("batch", bytes(m), first, count, nq)
        if key not in self.__dict__.setdefault("_ws", {}):
            sb = ctypes.c_size_t()
            check(lib().vlp_server_batch_workspace_bytes(ctypes.byref(m), count, nq, ctypes.byref(sb)))
            self._ws[key] = sb.value
        sh = _stream_handle(stream, self.device)
        sc = self._scratch(key, self._ws[key], sh)
        check(lib().vlp_server_eval_batch(self.h, ctypes.byref(m), nq, first, count,
                                          ctypes.c_void_p(queries_dev.data_ptr()), ctypes.c_void_p(db_dev.data_ptr()),
                                          ctypes.c_void_p(out_dev.data_ptr()), ctypes.c_void_p(sc.data_ptr()),
                                          sc.numel(), sh))

    def combine(self, m: VlpMeta, G: int, partials_dev, out_dev, stream=None):
        key = ("combine", bytes(m), G)
        if key not in self.__dict__.setdefault("_ws", {}):
            sb = ctypes.c_size_t()
            check(lib().vlp_server_combine_workspace_bytes(ctypes.byref(m), G, ctypes.byref(sb)))
            self._ws[key] = sb.value
        sh = _stream_handle(stream, self.device)
        sc = self._scratch(key, self._ws[key], sh)
        check(lib().vlp_server_combine(self.h, ctypes.byref(m), G, ctypes.c_void_p(partials_dev.data_ptr()),
                                       ctypes.c_void_p(out_dev.data_ptr()), ctypes.c_void_p(sc.data_ptr()),
                                       sc.numel(), sh))

    def gate_batch(self, op: int, a_dev, b_dev, out_dev, c_dev=None, stream=None):
        """A batch of independent gates (config 5): out = op(a, b), or MUX(a, b, c) = a ? b : c."""
        count = a_dev.shape[0]
        key = ("gates", op, count)
        if key not in self.__dict__.setdefault("_ws", {}):
            sb = ctypes.c_size_t()
            check(lib().vlp_gate_batch_workspace_bytes(op, count, ctypes.byref(sb)))
            self._ws[key] = sb.value
        sh = _stream_handle(stream, self.device)
        sc = self._scratch(key, self._ws[key], sh)
        p = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        check(lib().vlp_gate_batch(self.h, op, p(a_dev), p(b_dev), p(c_dev), p(out_dev), count,
                                   ctypes.c_void_p(sc.data_ptr()), sc.numel(), sh))

    def debug_blind_rotate(self, in_dev, steps: int, stream=None):
        import torch
        count = in_dev.shape[0]
        acc = torch.zeros((count, 2 * L.N), dtype=torch.int32, device=in_dev.device)
        scratch = torch.empty(max(256, lib().vlp_debug_scratch_bytes(count)), dtype=torch.uint8, device=in_dev.device)
        check(lib().vlp_debug_blind_rotate(self.h, ctypes.c_void_p(in_dev.data_ptr()), count, steps,
                                           ctypes.c_void_p(acc.data_ptr()), ctypes.c_void_p(scratch.data_ptr()),
                                           _stream_handle(stream, self.device)))
        return acc

    def debug_keyswitch(self, nlwe_dev, stream=None):
        import torch
        count = nlwe_dev.shape[0]
        out = torch.zeros((count, CT_STRIDE), dtype=torch.int32, device=nlwe_dev.device)
        scratch = torch.empty(max(256, lib().vlp_debug_scratch_bytes(count)), dtype=torch.uint8, device=nlwe_dev.device)
        check(lib().vlp_debug_keyswitch(self.h, ctypes.c_void_p(nlwe_dev.data_ptr()), count,
                                        ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(scratch.data_ptr()),
                                        _stream_handle(stream, self.device)))
        return out


class Program:
    """A compiled level schedule (vlp_program_create*), with its torch-owned scratch."""

    def __init__(self, server: Server, handle: ctypes.c_void_p):
        import torch
        self.server = server
        self.h = handle
        info = VlpProgramInfo()
        check(lib().vlp_program_get_info(self.h, ctypes.byref(info)))
        self.info = info
        self.scratch = torch.empty(max(256, info.scratch_bytes), dtype=torch.uint8, device=f"cuda:{server.device}")

    @classmethod
    def velopir(cls, server: Server, m: VlpMeta, first: int = 0, count: int | None = None):
        count = m.M - first if count is None else count
        h = ctypes.c_void_p()
        check(lib().vlp_program_create(server.h, ctypes.byref(m), first, count, ctypes.byref(h)))
        return cls(server, h)

    @classmethod
    def queries(cls, server: Server, m: VlpMeta, nq: int, first: int = 0, count: int | None = None):
        count = m.M - first if count is None else count
        h = ctypes.c_void_p()
        check(lib().vlp_program_create_queries(server.h, ctypes.byref(m), first, count, nq, ctypes.byref(h)))
        return cls(server, h)

    @classmethod
    def gates(cls, server: Server, op: int, count: int):
        h = ctypes.c_void_p()
        check(lib().vlp_program_create_gates(server.h, op, count, ctypes.byref(h)))
        return cls(server, h)

    @classmethod
    def combine(cls, server: Server, m: VlpMeta, G: int):
        h = ctypes.c_void_p()
        check(lib().vlp_program_create_combine(server.h, ctypes.byref(m), G, ctypes.byref(h)))
        return cls(server, h)

    def __del__(self):
        try:
            lib().vlp_free_program(self.h)
        except Exception:
            pass

    def eval(self, in0, in1, out, stream=None):
        p = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        check(lib().vlp_program_eval(self.h, ctypes.c_void_p(self.scratch.data_ptr()), self.scratch.numel(),
                                     p(in0), p(in1), p(out), _stream_handle(stream, self.server.device)))

    def profile(self, enable: bool = True):
        check(lib().vlp_program_profile(self.h, 1 if enable else 0))

    def profile_read(self, reset: bool = True):
        """(br_ms, ks_ms, br_launches, ks_launches) accumulated since the last reset."""
        br, ks = ctypes.c_double(), ctypes.c_double()
        nb, nk = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib().vlp_program_profile_read(self.h, ctypes.byref(br), ctypes.byref(ks), ctypes.byref(nb),
                                             ctypes.byref(nk), 1 if reset else 0))
        return br.value, ks.value, nb.value, nk.value

    def node_row(self, kind: int, record: int, bit: int = 0) -> int:
        r = ctypes.c_uint64()
        check(lib().vlp_program_node_row(self.h, kind, record, bit, ctypes.byref(r)))
        return r.value

    def level_jobs(self, level: int):
        """(br jobs, ks jobs) of one level of the compiled schedule as numpy structured arrays with the fields
        of vlp_br_job (x, y, k0, ax, ay, tv, row) and vlp_ks_job (n0, n1, add, out)."""
        nb, nk = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib().vlp_program_level_jobs(self.h, level, None, ctypes.byref(nb), None, ctypes.byref(nk)))
        br_t = np.dtype([("x", "<u4"), ("y", "<u4"), ("k0", "<u4"), ("ax", "i1"), ("ay", "i1"), ("tv", "<u2"),
                         ("row", "<u4")])
        ks_t = np.dtype([("n0", "<u4"), ("n1", "<u4"), ("add", "<u4"), ("out", "<u4")])
        br = np.zeros(max(1, nb.value), br_t)
        ks = np.zeros(max(1, nk.value), ks_t)
        check(lib().vlp_program_level_jobs(self.h, level, br.ctypes.data_as(ctypes.POINTER(L.VlpBrJob)),
                                           ctypes.byref(nb), ks.ctypes.data_as(ctypes.POINTER(L.VlpKsJob)),
                                           ctypes.byref(nk)))
        return br[:nb.value], ks[:nk.value]

    def level_linear(self, level: int):
        """R24 linear jobs of one level: (jobs uint32 [n, 4] = (out slot, first, count, 0), input slots)."""
        nj, ni = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib().vlp_program_level_linear(self.h, level, None, ctypes.byref(nj), None, ctypes.byref(ni)))
        jobs = np.zeros((max(1, nj.value), 4), np.uint32)
        ins = np.zeros(max(1, ni.value), np.uint32)
        check(lib().vlp_program_level_linear(self.h, level, jobs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                             ctypes.byref(nj), ins.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                                             ctypes.byref(ni)))
        return jobs[:nj.value], ins[:ni.value]

    def intermediate(self):
        """The intermediate-row region of the scratch as an int32 [rows, 632] view (parity dumps)."""
        off = ctypes.c_uint64()
        check(lib().vlp_program_intermediate_offset(self.h, ctypes.byref(off)))
        rows = (self.scratch.numel() - off.value) // (CT_STRIDE * 4)
        return self.scratch[off.value: off.value + rows * CT_STRIDE * 4].view(dtype=__import__("torch").int32).view(rows, CT_STRIDE)


def to_device(ct: np.ndarray, device: int = 0):
    import torch
    return torch.from_numpy(np.ascontiguousarray(ct, dtype=np.uint32).view(np.int32)).to(f"cuda:{device}")


def to_host(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)
