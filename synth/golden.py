"""Reader for tests/golden/samples.txt (expected outputs at sampled global
block indices, written by tests/golden/make_samples.py from oracle/ only).

Lets bench.py and tools/ gate their timings on parity without executing the
oracle.  Holds no AES arithmetic: it parses text and compares bytes.
"""
from __future__ import annotations

import os

import numpy as np

_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "samples.txt")
_cache: dict = {}


def samples(op: str, keybits: int) -> tuple[np.ndarray, np.ndarray]:
    """(global indices uint64 [m], expected blocks uint8 [m,16]) for op in
    {ecb_enc, ecb_dec, ctr, cbc_dec}."""
    if not _cache:
        acc: dict = {}
        with open(_PATH) as f:
            for ln in f:
                if ln.startswith("#") or not ln.strip():
                    continue
                o, kb, i, h = ln.split()
                acc.setdefault((o, int(kb)), []).append((int(i), bytes.fromhex(h)))
        for k, v in acc.items():
            v.sort()
            _cache[k] = (np.array([a for a, _ in v], np.uint64),
                         np.frombuffer(b"".join(b for _, b in v), np.uint8).reshape(-1, 16))
    return _cache[(op, keybits)]


def check(op: str, keybits: int, first_block: int, nblocks: int, gather) -> int:
    """Compare the sampled blocks that fall in [first_block, first_block+nblocks).
    ``gather(local_idx: np.ndarray[int64]) -> np.ndarray[m,16] uint8`` reads the
    device result.  Returns the number of blocks checked; raises AssertionError
    on any mismatch."""
    idx, want = samples(op, keybits)
    sel = (idx >= np.uint64(first_block)) & (idx < np.uint64(first_block + nblocks))
    if not sel.any():
        return 0
    local = (idx[sel] - np.uint64(first_block)).astype(np.int64)
    got = gather(local)
    bad = np.nonzero((got != want[sel]).any(axis=1))[0]
    if len(bad):
        raise AssertionError(f"parity: {op} AES-{keybits} mismatch at global block {int(idx[sel][bad[0]])}"
                             f" ({len(bad)} of {int(sel.sum())} samples)")
    return int(sel.sum())
