"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic: only the splitmix64 counter-based
stream of DESIGN.md "Input recipe".  Host twin in numpy
here; device twin in ``fill.cu`` (``libsynth.so``).  Block i of a buffer is
words 2i and 2i+1 (little-endian), so any block of any shard can be
regenerated on the host for sampled parity without copying the device buffer.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

DATA_SEED = 190205234
KIND = {"random": 0, "zeros": 1, "repeat": 2, "ascii": 3}

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libsynth.so")
_lib = None


def words(seed: int, first: int, count: int) -> np.ndarray:
    """splitmix64 words m = first .. first+count-1 of stream ``seed``."""
    return words_at(seed, np.arange(first, first + count, dtype=np.uint64))


def blocks(first_block: int, nblocks: int, seed: int = DATA_SEED, kind: str = "random") -> np.ndarray:
    """Bytes of blocks [first_block, first_block+nblocks) as a flat uint8 array."""
    k = KIND[kind]
    if k == 1:
        return np.zeros(16 * nblocks, np.uint8)
    if k == 2:
        w = np.tile(words(seed, 0, 2), nblocks)
    else:
        w = words(seed, 2 * first_block, 2 * nblocks)
    b = w.astype("<u8").view(np.uint8).copy()
    if k == 3:
        b = (0x20 + b % 95).astype(np.uint8)
    return b


def blocks_at(idx: np.ndarray, seed: int = DATA_SEED) -> np.ndarray:
    """Random-kind blocks at arbitrary global indices, shape (len(idx), 16)."""
    idx = np.asarray(idx, dtype=np.uint64)
    w0 = words_at(seed, 2 * idx)
    w1 = words_at(seed, 2 * idx + np.uint64(1))
    return np.stack([w0, w1], 1).astype("<u8").view(np.uint8).reshape(-1, 16)


def words_at(seed: int, m: np.ndarray) -> np.ndarray:
    m = np.asarray(m, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (m + np.uint64(1)) * _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def key(keybits: int) -> bytes:
    """Synthetic key: first keybits/8 bytes of stream 5234 + keybits."""
    return words(5234 + keybits, 0, 4).astype("<u8").view(np.uint8)[: keybits // 8].tobytes()


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(_LIB)
        L.synth_fill.restype = ctypes.c_int
        L.synth_fill.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
        _lib = L
    return _lib


def fill_device(t, first_block: int = 0, seed: int = DATA_SEED, kind: str = "random", stream=None):
    """Fill a CUDA uint8 tensor (16-byte aligned, numel % 16 == 0) on its device."""
    import torch
    assert t.is_cuda and t.dtype == torch.uint8 and t.is_contiguous() and t.numel() % 16 == 0
    s = stream if stream is not None else torch.cuda.current_stream(t.device)
    with torch.cuda.device(t.device):
        rc = lib().synth_fill(ctypes.c_void_p(t.data_ptr()), first_block, t.numel() // 16, seed,
                              KIND[kind], ctypes.c_void_p(s.cuda_stream))
    if rc:
        raise RuntimeError(f"synth_fill failed ({rc})")
    return t
