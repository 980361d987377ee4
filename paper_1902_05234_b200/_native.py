"""ctypes loader for libaes_b200.so (the C ABI of include/aes_b200.h).

Argument marshalling only: every step of the AES path runs in the library's
CUDA kernels.  There is no fallback -- if the shared library is missing,
importing the package raises ImportError.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libaes_b200.so")

AES_OK, AES_EKEYBITS, AES_ENR, AES_ENULL, AES_EALIGN, AES_EOVERLAP, AES_ERANGE, \
    AES_ENOTDEVICE, AES_ECUDA, AES_EVARIANT, AES_ECAPTURE = range(11)

AES_VAR_DEFAULT, AES_VAR_SMEM_REPL, AES_VAR_SMEM_PLAIN, AES_VAR_CONST, AES_VAR_SMEM_REPL_TMA, AES_VAR_SMEM_ROT, \
    AES_VAR_GLOBAL, AES_VAR_HYBRID, AES_VAR_BITSLICE = range(9)
AES_LAUNCH_TRUSTED_PTRS, AES_LAUNCH_NO_PDL = 1, 2

# every symbol include/aes_b200.h declares
EXPORTS = ("aes_expand_key", "aes_ecb_encrypt", "aes_ecb_decrypt", "aes_ecb_launch",
           "aes_ctr_xcrypt", "aes_cbc_decrypt", "aes_ecb_trace", "aes_ecb_batch", "aes_pipeline_create", "aes_pipeline_run", "aes_pipeline_destroy",
           "aes_mb_lds_gather", "aes_status_string", "aes_last_cuda_error", "aes_abi_version")


class aes_round_keys(ctypes.Structure):
    _fields_ = [("ek", ctypes.c_uint32 * 60), ("dk", ctypes.c_uint32 * 60),
                ("nr", ctypes.c_int32), ("keybits", ctypes.c_int32)]


class aes_segment(ctypes.Structure):
    _fields_ = [("in_offset", ctypes.c_uint64), ("out_offset", ctypes.c_uint64), ("nblocks", ctypes.c_uint64),
                ("key_index", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class aes_launch_config(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("states_per_thread", ctypes.c_int32),
                ("grid", ctypes.c_int32), ("flags", ctypes.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    p, u64, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
    RKP = ctypes.POINTER(aes_round_keys)
    L.aes_expand_key.restype = i32
    L.aes_expand_key.argtypes = [ctypes.c_char_p, i32, RKP]
    for f in (L.aes_ecb_encrypt, L.aes_ecb_decrypt):
        f.restype = i32
        f.argtypes = [RKP, i32, p, p, u64, p]
    L.aes_ecb_launch.restype = i32
    L.aes_ecb_launch.argtypes = [RKP, i32, i32, p, p, u64, p, ctypes.POINTER(aes_launch_config)]
    L.aes_ctr_xcrypt.restype = i32
    L.aes_ctr_xcrypt.argtypes = [RKP, i32, ctypes.c_char_p, u64, p, p, u64, p]
    L.aes_cbc_decrypt.restype = i32
    L.aes_cbc_decrypt.argtypes = [RKP, i32, ctypes.c_char_p, p, p, u64, p]
    L.aes_ecb_trace.restype = i32
    L.aes_ecb_trace.argtypes = [RKP, i32, i32, i32, p, p, u64, p]
    L.aes_ecb_batch.restype = i32
    L.aes_ecb_batch.argtypes = [RKP, i32, i32, ctypes.POINTER(aes_segment), ctypes.c_uint32, p, p, p]
    L.aes_pipeline_create.restype = i32
    L.aes_pipeline_create.argtypes = [u64, i32, ctypes.POINTER(p)]
    L.aes_pipeline_run.restype = i32
    L.aes_pipeline_run.argtypes = [p, RKP, i32, i32, p, p, u64]
    L.aes_pipeline_destroy.restype = i32
    L.aes_pipeline_destroy.argtypes = [p]
    L.aes_mb_lds_gather.restype = i32
    L.aes_mb_lds_gather.argtypes = [p, i32, i32, p]
    L.aes_status_string.restype = ctypes.c_char_p
    L.aes_status_string.argtypes = [i32]
    L.aes_last_cuda_error.restype = i32
    L.aes_last_cuda_error.argtypes = []
    L.aes_abi_version.restype = i32
    L.aes_abi_version.argtypes = []
    return L


lib = _load()


def status_string(code: int) -> str:
    return lib.aes_status_string(code).decode()
