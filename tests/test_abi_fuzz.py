"""Fuzz the C ABI's argument validation (CPU, no device needed): arbitrary
nr / keybits / pointer / size / config combinations never crash and always
return a defined aes_status; a call rejected for a decided-before-launch
reason returns that reason."""
import ctypes

import pytest

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st

from paper_1902_05234_b200 import _native
import paper_1902_05234_b200 as aes

PTRS = st.sampled_from([0, 16, 0x10000, 0x10008, 0x10010, 2**47 - 16, 2**63 - 16])
CODES = set(range(11))


@settings(max_examples=400, deadline=None, derandomize=True)
@given(nr=st.integers(-2, 20), inp=PTRS, out=PTRS, n=st.sampled_from([0, 1, 2, 31, 2**20, 2**40, 2**59, 2**60, 2**64 - 1]),
       dec=st.integers(0, 1), variant=st.integers(-1, 8), spt=st.integers(-1, 5), grid=st.integers(-2, 3),
       flags=st.integers(-1, 5))
def test_launch_validation_total(nr, inp, out, n, dec, variant, spt, grid, flags):
    rk = aes.expand_key(bytes(16))
    cfg = _native.aes_launch_config(variant, spt, grid, flags)
    code = _native.lib.aes_ecb_launch(ctypes.byref(rk.c), nr, dec, inp, out, n, None, ctypes.byref(cfg))
    assert code in CODES
    if nr != 10:
        assert code == _native.AES_ENR
    elif code == _native.AES_OK:
        assert n == 0          # nothing can launch on a CPU-only box


@settings(max_examples=200, deadline=None, derandomize=True)
@given(keybits=st.integers(-1, 300), key=st.binary(min_size=0, max_size=40))
def test_expand_key_total(keybits, key):
    rk = _native.aes_round_keys()
    buf = key + bytes(40 - len(key))
    code = _native.lib.aes_expand_key(buf, keybits, ctypes.byref(rk))
    if keybits in (128, 192, 256):
        assert code == _native.AES_OK and rk.nr == keybits // 32 + 6
    else:
        assert code == _native.AES_EKEYBITS


@settings(max_examples=200, deadline=None, derandomize=True)
@given(nsegs=st.integers(0, 5), nkeys=st.integers(-1, 130), kidx=st.integers(0, 200),
       off=st.sampled_from([0, 8, 16, 2**40]), n=st.sampled_from([0, 1, 2**59, 2**61]))
def test_batch_validation_total(nsegs, nkeys, kidx, off, n):
    k = aes.expand_key(bytes(16)).c
    cnt = max(1, min(nkeys, 130))
    keys = (_native.aes_round_keys * cnt)(*([k] * cnt))
    segs = (_native.aes_segment * max(1, nsegs))(*[_native.aes_segment(off, off, n, kidx, 0)] * max(1, nsegs))
    code = _native.lib.aes_ecb_batch(keys, nkeys, 0, segs, nsegs, 0x10000, 0x10000, None)
    assert code in CODES
    if nkeys < 1 or nkeys > 128:
        assert code == _native.AES_ERANGE
