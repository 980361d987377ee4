"""CPU parity oracle for the B200 AES-ECB path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` (including ``tests/golden/make_samples.py``, which writes the
golden samples the bench/tool parity gates read), ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` and ``--impl reference`` legs may import this package.  The product package
``paper_1902_05234_b200`` never imports it, and this package imports nothing
from the product.

The arithmetic lives in ``aes_oracle.c`` (plain byte-oriented C: SubBytes /
ShiftRows / MixColumns / AddRoundKey written from PAPER.md Defs 1-7 and
Algorithm 1 as corrected by DESIGN.md reading R1; no T-tables).  This module
only compiles it with gcc (if needed) and marshals arguments with ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "aes_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def _digest() -> str:
    import hashlib
    with open(_SRC, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, -O2, pthreads); content-hash staleness."""
    stamp = _LIB + ".stamp"
    stale = not os.path.exists(_LIB) or not os.path.exists(stamp) or open(stamp).read().strip() != _digest()
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-fno-semantic-interposition", "-shared", "-pthread",
                               "-o", tmp, _SRC], stdout=subprocess.DEVNULL)
        os.replace(tmp, _LIB)
        with open(stamp, "w") as f:
            f.write(_digest())
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            u8, i32, u64, p = ctypes.c_uint8, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p
            L.oracle_gf_add.restype = u8; L.oracle_gf_add.argtypes = [u8, u8]
            L.oracle_gf_mul.restype = u8; L.oracle_gf_mul.argtypes = [u8, u8]
            L.oracle_xtime.restype = u8; L.oracle_xtime.argtypes = [u8]
            L.oracle_gf_inv.restype = u8; L.oracle_gf_inv.argtypes = [u8]
            L.oracle_sbox.restype = u8; L.oracle_sbox.argtypes = [u8]
            L.oracle_inv_sbox.restype = u8; L.oracle_inv_sbox.argtypes = [u8]
            L.oracle_nr.restype = i32; L.oracle_nr.argtypes = [i32]
            L.oracle_key_expansion.restype = i32; L.oracle_key_expansion.argtypes = [p, i32, p]
            L.oracle_aes_ecb.restype = i32
            L.oracle_aes_ecb.argtypes = [p, i32, i32, p, p, u64, i32]
            L.oracle_cipher_trace.restype = i32; L.oracle_cipher_trace.argtypes = [p, i32, p, p]
            L.oracle_inv_cipher_trace.restype = i32; L.oracle_inv_cipher_trace.argtypes = [p, i32, p, p]
            L.oracle_sbox_table.restype = None; L.oracle_sbox_table.argtypes = [p]
            L.oracle_inv_sbox_table.restype = None; L.oracle_inv_sbox_table.argtypes = [p]
            L.oracle_transform.restype = i32; L.oracle_transform.argtypes = [i32, p]
            _lib = L
    return _lib


def _buf(b: bytes):
    return ctypes.create_string_buffer(bytes(b), len(b))


# --- GF(2^8), PAPER.md Defs 1-3 -------------------------------------------
def gf_add(a: int, b: int) -> int: return lib().oracle_gf_add(a, b)
def gf_mul(a: int, b: int) -> int: return lib().oracle_gf_mul(a, b)
def xtime(a: int) -> int: return lib().oracle_xtime(a)
def gf_inv(a: int) -> int: return lib().oracle_gf_inv(a)
def sbox(a: int) -> int: return lib().oracle_sbox(a)
def inv_sbox(a: int) -> int: return lib().oracle_inv_sbox(a)


def sbox_table() -> bytes:
    out = ctypes.create_string_buffer(256)
    lib().oracle_sbox_table(out)
    return out.raw


def inv_sbox_table() -> bytes:
    out = ctypes.create_string_buffer(256)
    lib().oracle_inv_sbox_table(out)
    return out.raw


TRANSFORMS = {"sub_bytes": 0, "shift_rows": 1, "mix_columns": 2,
              "inv_sub_bytes": 3, "inv_shift_rows": 4, "inv_mix_columns": 5}


def transform(op: str, block: bytes) -> bytes:
    assert len(block) == 16
    b = _buf(block)
    if lib().oracle_transform(TRANSFORMS[op], b) != 0:
        raise ValueError(op)
    return b.raw


# --- key schedule / cipher -------------------------------------------------
def nr(keybits: int) -> int: return lib().oracle_nr(keybits)


def key_expansion(key: bytes) -> bytes:
    """Expanded key bytes, 16*(Nr+1); word i = bytes [4i, 4i+4)."""
    keybits = 8 * len(key)
    n = nr(keybits)
    if n == 0:
        raise ValueError("key must be 16, 24 or 32 bytes")
    out = ctypes.create_string_buffer(16 * (n + 1))
    lib().oracle_key_expansion(_buf(key), keybits, out)
    return out.raw


def cipher_trace(key: bytes, block: bytes) -> list[bytes]:
    """State after AddRoundKey(r) for r = 0..Nr (FIPS-197 App B layout)."""
    n = nr(8 * len(key))
    tr = ctypes.create_string_buffer(16 * (n + 1))
    lib().oracle_cipher_trace(_buf(key), 8 * len(key), _buf(block), tr)
    return [tr.raw[16 * r:16 * r + 16] for r in range(n + 1)]


def inv_cipher_trace(key: bytes, block: bytes) -> list[bytes]:
    """InvCipher states: [after ARK(Nr), after iteration Nr-1, ..., after iteration 1, output]."""
    n = nr(8 * len(key))
    tr = ctypes.create_string_buffer(16 * (n + 1))
    lib().oracle_inv_cipher_trace(_buf(key), 8 * len(key), _buf(block), tr)
    return [tr.raw[16 * r:16 * r + 16] for r in range(n + 1)]


def ecb(key: bytes, data, decrypt: bool = False, nthreads: int = 1, out=None) -> np.ndarray:
    """ECB over a whole-block buffer (Eq 1).  ``data``: bytes or a
    contiguous uint8 numpy array; returns a new uint8 array (or fills ``out``)."""
    arr = np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray)) else data
    if arr.dtype != np.uint8 or not arr.flags["C_CONTIGUOUS"]:
        raise TypeError("need a contiguous uint8 array")
    if arr.size % 16:
        raise ValueError("length must be a multiple of 16")
    if out is None:
        out = np.empty_like(arr)
    rc = lib().oracle_aes_ecb(_buf(key), 8 * len(key), int(bool(decrypt)),
                              arr.ctypes.data, out.ctypes.data, arr.size // 16, int(nthreads))
    if rc != 0:
        raise ValueError("bad key size")
    return out


def encrypt(key: bytes, data, nthreads: int = 1) -> np.ndarray:
    return ecb(key, data, False, nthreads)


def decrypt(key: bytes, data, nthreads: int = 1) -> np.ndarray:
    return ecb(key, data, True, nthreads)


# --- CTR / CBC (NEXT-1 / NEXT-4) -------------------------------------------
def _lib_modes():
    L = lib()
    if not getattr(L, "_modes", False):
        p, i32, u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64
        L.oracle_aes_ctr.restype = i32
        L.oracle_aes_ctr.argtypes = [p, i32, p, u64, p, p, u64, i32]
        L.oracle_aes_cbc.restype = i32
        L.oracle_aes_cbc.argtypes = [p, i32, p, i32, p, p, u64]
        L._modes = True
    return L


def _arr(data):
    arr = np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray)) else data
    if arr.dtype != np.uint8 or not arr.flags["C_CONTIGUOUS"] or arr.size % 16:
        raise ValueError("need a contiguous uint8 buffer of whole blocks")
    return arr


def ctr(key: bytes, iv: bytes, data, block_offset: int = 0, nthreads: int = 1) -> np.ndarray:
    """CTR (Eq 5, reading R24): block j uses counter iv + block_offset + j (BE, mod 2^128)."""
    arr = _arr(data)
    out = np.empty_like(arr)
    assert len(iv) == 16
    rc = _lib_modes().oracle_aes_ctr(_buf(key), 8 * len(key), _buf(iv), block_offset & (2**64 - 1),
                                     arr.ctypes.data, out.ctypes.data, arr.size // 16, nthreads)
    if rc:
        raise ValueError("bad key size")
    return out


def cbc(key: bytes, iv: bytes, data, decrypt: bool) -> np.ndarray:
    """CBC (Eq 2, reading R25), sequential."""
    arr = _arr(data)
    out = np.empty_like(arr)
    assert len(iv) == 16
    rc = _lib_modes().oracle_aes_cbc(_buf(key), 8 * len(key), _buf(iv), int(bool(decrypt)),
                                     arr.ctypes.data, out.ctypes.data, arr.size // 16)
    if rc:
        raise ValueError("bad key size")
    return out
