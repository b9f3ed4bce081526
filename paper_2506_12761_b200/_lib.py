"""ctypes binding of libvlp.so (include/vlp.h).  Argument marshalling only: every step of the hot path runs
in the library's CUDA kernels.  Importing fails loudly if the in-tree library is missing (no fallback)."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VLP_LIB", os.path.join(HERE, "libvlp.so"))  # VLP_LIB: dev builds (tools/)

CT_STRIDE = 632
NLWE_STRIDE = 1028
n = 630
N = 1024

VLP_OK, VLP_EINVAL, VLP_EMODE, VLP_EWIDTH, VLP_ERANGE, VLP_EPKUSED, VLP_ECUDA, VLP_ENOMEM, VLP_ENODEV = (
    0, -1, -2, -3, -4, -5, -6, -7, -8)
MODE_INTV, MODE_COV, MODE_IDM = 0, 1, 2
F_CLOSED_UPPER, F_UNSIGNED, F_EQ_TREE, F_SUM_TREE, F_OR_REDUCE, F_PREFIX_COMP, F_LINEAR_SUM, F_KEEP_ALL = 1, 2, 4, 8, 16, 32, 64, 128
CONFIG_FLAGS = F_CLOSED_UPPER | F_UNSIGNED | F_EQ_TREE | F_SUM_TREE
AND, NAND, OR, XOR, XNOR, MUX = 0, 1, 2, 3, 4, 5


class VlpParams(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint32), ("N", ctypes.c_uint32), ("k", ctypes.c_uint32),
                ("bg_bits", ctypes.c_uint32), ("ell", ctypes.c_uint32), ("ks_base_bits", ctypes.c_uint32),
                ("ks_t", ctypes.c_uint32), ("sigma_lwe", ctypes.c_double), ("sigma_bk", ctypes.c_double),
                ("sigma_ks", ctypes.c_double)]


class VlpMeta(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_uint32), ("M", ctypes.c_uint32), ("l_I", ctypes.c_uint32),
                ("l_S", ctypes.c_uint32), ("d", ctypes.c_uint32), ("flags", ctypes.c_uint32)]


class VlpProgramInfo(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_uint32), ("br", ctypes.c_uint64), ("ks", ctypes.c_uint64),
                ("gates", ctypes.c_uint64), ("in0_cts", ctypes.c_uint64), ("in1_cts", ctypes.c_uint64),
                ("out_cts", ctypes.c_uint64), ("scratch_bytes", ctypes.c_uint64),
                ("max_level_br", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint32),
                ("table_bytes", ctypes.c_uint64)]


class VlpBrJob(ctypes.Structure):
    _fields_ = [("x", ctypes.c_uint32), ("y", ctypes.c_uint32), ("k0", ctypes.c_uint32), ("ax", ctypes.c_int8),
                ("ay", ctypes.c_int8), ("tv", ctypes.c_uint16), ("row", ctypes.c_uint32)]


class VlpKsJob(ctypes.Structure):
    _fields_ = [("n0", ctypes.c_uint32), ("n1", ctypes.c_uint32), ("add", ctypes.c_uint32), ("out", ctypes.c_uint32)]


# every symbol include/vlp.h declares: name -> (restype, argtypes)
_vp, _u32p, _u64p, _u8p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64), \
    ctypes.POINTER(ctypes.c_uint8)
_pp = ctypes.POINTER(ctypes.c_void_p)
_i, _u64, _sz = ctypes.c_int, ctypes.c_uint64, ctypes.c_size_t
SIGNATURES = {
    "vlp_last_error": (ctypes.c_char_p, []),
    "vlp_params_tfhe128": (_i, [ctypes.POINTER(VlpParams)]),
    "vlp_keygen": (_i, [_u64, ctypes.POINTER(VlpParams), _pp, _pp]),
    "vlp_keygen_secure": (_i, [ctypes.POINTER(VlpParams), _pp, _pp]),
    "vlp_encrypt_query_secure": (_i, [_vp, ctypes.POINTER(VlpMeta), _u64p, _u32p]),
    "vlp_encrypt_bits_secure": (_i, [_vp, ctypes.POINTER(ctypes.c_uint8), _sz, _u32p]),
    "vlp_pubkeygen_secure": (_i, [_vp, ctypes.POINTER(VlpMeta), _sz, _sz, _pp]),
    "vlp_debug_chacha20_block": (_i, [_u32p, ctypes.c_uint32, _u32p, _u32p]),
    "vlp_debug_next_secure_key": (_i, [_u32p]),
    "vlp_sk_export": (_i, [_vp, _u32p, _u32p]),
    "vlp_evk_export": (_i, [_vp, _u32p, _u32p]),
    "vlp_encrypt_bits": (_i, [_vp, _u8p, _sz, _u64, _u64, _u32p]),
    "vlp_encrypt_query": (_i, [_vp, ctypes.POINTER(VlpMeta), _u64p, _u64, _u32p]),
    "vlp_decrypt_bits": (_i, [_vp, _u32p, _sz, _u8p]),
    "vlp_pubkeygen": (_i, [_vp, ctypes.POINTER(VlpMeta), _u64, _sz, _sz, _pp]),
    "vlp_db_record_cts": (_i, [ctypes.POINTER(VlpMeta), ctypes.POINTER(ctypes.c_size_t)]),
    "vlp_server_encrypt_db": (_i, [_vp, _u64p, _u64p, _u32p]),
    "vlp_encrypt_db_device_scratch_bytes": (_i, [ctypes.POINTER(VlpMeta), _sz, ctypes.POINTER(ctypes.c_size_t)]),
    "vlp_encrypt_db_device": (_i, [_vp, ctypes.POINTER(VlpMeta), _u64, _sz, _sz, _u64p, _u64p, _vp, _vp, _sz, _u64]),
    "vlp_keygen_device_scratch_bytes": (_sz, []),
    "vlp_keygen_device": (_i, [_u64, ctypes.POINTER(VlpParams), _vp, _sz, _u64, _pp, _pp]),
    "vlp_keygen_device_secure": (_i, [ctypes.POINTER(VlpParams), _vp, _sz, _u64, _pp, _pp]),
    "vlp_pubkeygen_device_scratch_bytes": (_i, [ctypes.POINTER(VlpMeta), _sz, ctypes.POINTER(ctypes.c_size_t)]),
    "vlp_pubkeygen_device": (_i, [_vp, ctypes.POINTER(VlpMeta), _u64, _sz, _sz, _vp, _vp, _sz, _u64]),
    "vlp_pubkeygen_device_secure": (_i, [_vp, ctypes.POINTER(VlpMeta), _sz, _sz, _vp, _vp, _sz, _u64]),
    "vlp_server_encrypt_db_device_scratch_bytes": (_i, [ctypes.POINTER(VlpMeta), _sz, ctypes.POINTER(ctypes.c_size_t)]),
    "vlp_server_load_records": (_i, [_vp, _u64p, _u64p, _vp, _vp, _sz, _u64]),
    "vlp_server_encrypt_db_device": (_i, [ctypes.POINTER(VlpMeta), _sz, _vp, _u64p, _u64p, _vp, _vp, _sz, _u64]),
    "vlp_server_evk_bytes": (_sz, []),
    "vlp_server_create": (_i, [_i, _vp, _vp, _sz, _u64, _pp]),
    "vlp_program_create": (_i, [_vp, ctypes.POINTER(VlpMeta), _sz, _sz, _pp]),
    "vlp_program_create_queries": (_i, [_vp, ctypes.POINTER(VlpMeta), _sz, _sz, ctypes.c_uint32, _pp]),
    "vlp_program_create_gates": (_i, [_vp, _i, _sz, _pp]),
    "vlp_program_create_combine": (_i, [_vp, ctypes.POINTER(VlpMeta), ctypes.c_uint32, _pp]),
    "vlp_program_get_info": (_i, [_vp, ctypes.POINTER(VlpProgramInfo)]),
    "vlp_program_node_row": (_i, [_vp, _i, _sz, ctypes.c_uint32, _u64p]),
    "vlp_program_intermediate_offset": (_i, [_vp, _u64p]),
    "vlp_program_level_linear": (_i, [_vp, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32), _u64p,
                                     ctypes.POINTER(ctypes.c_uint32), _u64p]),
    "vlp_program_level_jobs": (_i, [_vp, ctypes.c_uint32, ctypes.POINTER(VlpBrJob), _u64p, ctypes.POINTER(VlpKsJob),
                                    _u64p]),
    "vlp_program_eval": (_i, [_vp, _vp, _sz, _vp, _vp, _vp, _u64]),
    "vlp_program_profile": (_i, [_vp, _i]),
    "vlp_program_profile_read": (_i, [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                      _u64p, _u64p, _i]),
    "vlp_debug_scratch_bytes": (_sz, [_sz]),
    "vlp_debug_blind_rotate": (_i, [_vp, _vp, _sz, _i, _vp, _vp, _u64]),
    "vlp_debug_keyswitch": (_i, [_vp, _vp, _sz, _vp, _vp, _u64]),
    "vlp_debug_route": (_i, [_i, _i]),
    "vlp_debug_fft_error": (_i, [_vp]),
    "vlp_server_workspace_bytes": (_i, [ctypes.POINTER(VlpMeta), _sz, ctypes.POINTER(ctypes.c_size_t),
                                        ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]),
    "vlp_server_eval": (_i, [_vp, ctypes.POINTER(VlpMeta), _sz, _sz, _vp, _vp, _vp, _vp, _sz, _u64]),
    "vlp_server_eval_host_workspace_bytes": (_i, [ctypes.POINTER(VlpMeta), _sz, ctypes.POINTER(ctypes.c_size_t)]),
    "vlp_server_eval_host": (_i, [_vp, ctypes.POINTER(VlpMeta), _sz, _sz, _u32p, _vp, _u32p, _vp, _sz, _u64]),
    "vlp_server_batch_workspace_bytes": (_i, [ctypes.POINTER(VlpMeta), _sz, ctypes.c_uint32,
                                              ctypes.POINTER(ctypes.c_size_t)]),
    "vlp_server_eval_batch": (_i, [_vp, ctypes.POINTER(VlpMeta), ctypes.c_uint32, _sz, _sz, _vp, _vp, _vp, _vp, _sz,
                                   _u64]),
    "vlp_server_combine_workspace_bytes": (_i, [ctypes.POINTER(VlpMeta), ctypes.c_uint32,
                                                ctypes.POINTER(ctypes.c_size_t)]),
    "vlp_server_combine": (_i, [_vp, ctypes.POINTER(VlpMeta), ctypes.c_uint32, _vp, _vp, _vp, _sz, _u64]),
    "vlp_gate_batch_workspace_bytes": (_i, [_i, _sz, ctypes.POINTER(ctypes.c_size_t)]),
    "vlp_gate_batch": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _sz, _vp, _sz, _u64]),
    "vlp_decrypt_result": (_i, [_vp, _u32p, ctypes.c_uint32, _u8p, _u64p]),
    "vlp_free_sk": (None, [_vp]),
    "vlp_free_evk": (None, [_vp]),
    "vlp_free_pk": (None, [_vp]),
    "vlp_free_server": (None, [_vp]),
    "vlp_free_program": (None, [_vp]),
}

_lib = None


class VlpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"vlp error {code}: {msg}")
        self.code = code


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2506_12761_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    if rc != VLP_OK:
        raise VlpError(rc, (lib().vlp_last_error() or b"").decode())
    return rc
