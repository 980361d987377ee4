"""Host-side tests of the C ABI (no GPU needed, no compute calls).

* the library loads and exports every symbol include/aes_b200.h declares;
* aes_expand_key (steps A1/A2, host C++) against FIPS-197 App A and the
  pinned oracle's key expansion / InvMixColumns (parity of the host logic);
* every validation error code that is decided before any CUDA call;
* the Python layer's argument checks.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from conftest import ROOT, golden


def test_library_exports_every_declared_symbol():
    from paper_1902_05234_b200 import _native
    hdr = open(os.path.join(ROOT, "include", "aes_b200.h")).read()
    declared = set(re.findall(r"\b(aes_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(_native.EXPORTS), declared ^ set(_native.EXPORTS)
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert _native.lib.aes_abi_version() == 3


def test_library_is_sm100a_and_has_no_oracle_symbols():
    from paper_1902_05234_b200 import _native
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    syms = subprocess.run(["nm", "-D", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle_" not in syms


def _le_words(b: bytes):
    return [int.from_bytes(b[4 * i:4 * i + 4], "little") for i in range(len(b) // 4)]


def test_expand_key_matches_fips197_appendix_a():
    import paper_1902_05234_b200 as aes
    for key, idx, word in (ln.split() for ln in open(golden("fips197_appA.txt")) if ln.strip() and not ln.startswith("#")):
        rk = aes.expand_key(bytes.fromhex(key))
        # FIPS prints word i as its 4 bytes in order; the ABI stores LE memory-order words (R21)
        assert rk.ek[int(idx)] == int.from_bytes(bytes.fromhex(word), "little"), (key, idx)
    rk = aes.expand_key(bytes(range(16)))
    assert rk.ek[0] == 0x03020100 and rk.nr == 10 and rk.keybits == 128


@pytest.mark.parametrize("keybits", [128, 192, 256])
def test_expand_key_matches_oracle_and_equivalent_inverse(keybits):
    import paper_1902_05234_b200 as aes
    rng = np.random.default_rng(keybits)
    for _ in range(50):
        key = rng.integers(0, 256, keybits // 8, dtype=np.uint8).tobytes()
        rk = aes.expand_key(key)
        nr = rk.nr
        assert nr == keybits // 32 + 6
        w = oracle.key_expansion(key)
        assert rk.ek == _le_words(w)
        dk = rk.dk
        assert dk[0:4] == rk.ek[4 * nr:4 * nr + 4]
        assert dk[4 * nr:4 * nr + 4] == rk.ek[0:4]
        for r in range(1, nr):
            rkey = w[16 * (nr - r):16 * (nr - r) + 16]
            assert dk[4 * r:4 * r + 4] == _le_words(oracle.transform("inv_mix_columns", rkey)), r


def test_equivalent_inverse_round1_value():
    # InvMixColumns(a0fafe17 88542cb1 23a33939 2a6c7605) for key 2b7e..3c
    import paper_1902_05234_b200 as aes
    rk = aes.expand_key(bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c"))
    want = bytes.fromhex("2b3708a7f262d405bc3ebdbf4b617d62")
    assert rk.dk[4 * 9:4 * 10] == _le_words(want)   # dk[Nr-1] = InvMix(ek[1])


def test_expand_key_errors():
    from paper_1902_05234_b200 import _native
    import paper_1902_05234_b200 as aes
    rk = _native.aes_round_keys()
    assert _native.lib.aes_expand_key(bytes(16), 100, ctypes.byref(rk)) == _native.AES_EKEYBITS
    assert _native.lib.aes_expand_key(None, 128, ctypes.byref(rk)) == _native.AES_ENULL
    assert _native.lib.aes_expand_key(bytes(16), 128, None) == _native.AES_ENULL
    with pytest.raises(ValueError):
        aes.expand_key(bytes(15))


def _call(rk, nr, inp, out, n, decrypt=0, cfg=None):
    from paper_1902_05234_b200 import _native
    L = _native.lib
    rkp = ctypes.byref(rk.c) if rk is not None else None
    if cfg is None:
        f = L.aes_ecb_decrypt if decrypt else L.aes_ecb_encrypt
        return f(rkp, nr, inp, out, n, None)
    return L.aes_ecb_launch(rkp, nr, decrypt, inp, out, n, None, ctypes.byref(cfg))


def test_validation_errors_before_any_cuda_call():
    from paper_1902_05234_b200 import _native
    import paper_1902_05234_b200 as aes
    rk = aes.expand_key(bytes(16))
    A = 0x10000
    assert _call(None, 10, A, A, 1) == _native.AES_ENULL
    assert _call(rk, 12, A, A, 1) == _native.AES_ENR          # nr != rk->nr
    assert _call(rk, 11, A, A, 1) == _native.AES_ENR
    assert _call(rk, 10, A, A, 0) == _native.AES_OK           # no-op, no launch
    assert _call(rk, 10, None, A, 0) == _native.AES_OK
    assert _call(rk, 10, None, A, 4) == _native.AES_ENULL
    assert _call(rk, 10, A, None, 4, decrypt=1) == _native.AES_ENULL
    assert _call(rk, 10, A + 8, A + 4096, 4) == _native.AES_EALIGN
    assert _call(rk, 10, A, A + 16, 4) == _native.AES_EOVERLAP
    assert _call(rk, 10, A + 16, A, 4) == _native.AES_EOVERLAP
    assert _call(rk, 10, A, A, 1 << 62) == _native.AES_ERANGE
    cfg = _native.aes_launch_config(9, 0, 0, 0)                 # unknown variant
    assert _call(rk, 10, A, A, 4, cfg=cfg) == _native.AES_EVARIANT
    for v in (_native.AES_VAR_HYBRID, _native.AES_VAR_BITSLICE):   # one state per thread only
        cfg = _native.aes_launch_config(v, 2, 0, 0)
        assert _call(rk, 10, A, A, 4, cfg=cfg) == _native.AES_EVARIANT
    cfg = _native.aes_launch_config(_native.AES_VAR_SMEM_REPL, 3, 0, 0)
    assert _call(rk, 10, A, A, 4, cfg=cfg) == _native.AES_EVARIANT
    cfg = _native.aes_launch_config(_native.AES_VAR_SMEM_REPL_TMA, 2, 0, 0)
    assert _call(rk, 10, A, A, 4, cfg=cfg) == _native.AES_EVARIANT
    cfg = _native.aes_launch_config(_native.AES_VAR_SMEM_REPL, 1, -1, 0)
    assert _call(rk, 10, A, A, 4, cfg=cfg) == _native.AES_ERANGE
    for bad_flags in (4, 8, -1):                               # unknown aes_launch_config.flags bits
        cfg = _native.aes_launch_config(_native.AES_VAR_SMEM_REPL, 1, 0, bad_flags)
        assert _call(rk, 10, A, A, 4, cfg=cfg) == _native.AES_ERANGE
    cfg = _native.aes_launch_config(_native.AES_VAR_GLOBAL, 2, 0, 0)
    assert _call(rk, 10, A, A, 4, cfg=cfg) == _native.AES_EVARIANT
    # a tampered schedule (keybits inconsistent with nr) is rejected
    bad = aes.expand_key(bytes(16))
    bad.c.keybits = 256
    assert _call(bad, 10, A, A, 1) == _native.AES_ENR


def test_pipeline_argument_errors():
    from paper_1902_05234_b200 import _native
    h = ctypes.c_void_p()
    assert _native.lib.aes_pipeline_create(15, 2, ctypes.byref(h)) == _native.AES_ERANGE
    assert _native.lib.aes_pipeline_create(1 << 20, 0, ctypes.byref(h)) == _native.AES_ERANGE
    assert _native.lib.aes_pipeline_create(1 << 20, 9, ctypes.byref(h)) == _native.AES_ERANGE
    assert _native.lib.aes_pipeline_create(1 << 20, 2, None) == _native.AES_ENULL
    assert _native.lib.aes_pipeline_run(None, None, 10, 0, None, None, 1) == _native.AES_ENULL
    assert _native.lib.aes_pipeline_destroy(None) == _native.AES_ENULL
    assert _native.lib.aes_mb_lds_gather(None, 1, 1, None) == _native.AES_ENULL


def test_status_strings():
    from paper_1902_05234_b200 import _native
    for code in range(10):
        s = _native.status_string(code)
        assert s.startswith("AES_")
    assert "unknown" in _native.status_string(99)


def test_python_layer_rejects_cpu_tensors():
    import torch
    import paper_1902_05234_b200 as aes
    rk = aes.expand_key(bytes(16))
    with pytest.raises(TypeError):
        aes.ecb_encrypt(rk, torch.zeros(32, dtype=torch.uint8))
    with pytest.raises(TypeError):
        aes.ecb_encrypt(rk, np.zeros(32, np.uint8))


def test_ctr_cbc_validation_errors():
    from paper_1902_05234_b200 import _native
    import paper_1902_05234_b200 as aes
    rk = aes.expand_key(bytes(32))
    L = _native.lib
    A = 0x10000
    iv = bytes(16)
    assert L.aes_ctr_xcrypt(ctypes.byref(rk.c), 14, None, 0, A, A, 4, None) == _native.AES_ENULL
    assert L.aes_ctr_xcrypt(ctypes.byref(rk.c), 10, iv, 0, A, A, 4, None) == _native.AES_ENR
    assert L.aes_ctr_xcrypt(ctypes.byref(rk.c), 14, iv, 0, A, A, 0, None) == _native.AES_OK
    assert L.aes_ctr_xcrypt(ctypes.byref(rk.c), 14, iv, 0, A, A + 32, 4, None) == _native.AES_EOVERLAP
    assert L.aes_cbc_decrypt(ctypes.byref(rk.c), 14, None, A, A + 4096, 4, None) == _native.AES_ENULL
    assert L.aes_cbc_decrypt(ctypes.byref(rk.c), 14, iv, A, A, 4, None) == _native.AES_EOVERLAP
    assert L.aes_cbc_decrypt(ctypes.byref(rk.c), 14, iv, A + 4, A + 4096, 4, None) == _native.AES_EALIGN


def test_trace_validation():
    from paper_1902_05234_b200 import _native
    import paper_1902_05234_b200 as aes
    rk = aes.expand_key(bytes(16))
    L = _native.lib
    assert L.aes_ecb_trace(ctypes.byref(rk.c), 10, 0, 11, 0x10000, 0x10000, 1, None) == _native.AES_ERANGE
    assert L.aes_ecb_trace(ctypes.byref(rk.c), 10, 0, -1, 0x10000, 0x10000, 1, None) == _native.AES_ERANGE
    assert L.aes_ecb_trace(ctypes.byref(rk.c), 10, 0, 3, 0x10000, 0x10000, 0, None) == _native.AES_OK


def test_batch_validation():
    from paper_1902_05234_b200 import _native
    import paper_1902_05234_b200 as aes
    L = _native.lib
    k128 = aes.expand_key(bytes(16)).c
    k256 = aes.expand_key(bytes(32)).c
    keys = (_native.aes_round_keys * 2)(k128, k128)
    seg = (_native.aes_segment * 2)(_native.aes_segment(0, 0, 4, 0, 0), _native.aes_segment(64, 64, 4, 1, 0))
    A = 0x10000
    assert L.aes_ecb_batch(None, 1, 0, seg, 2, A, A, None) == _native.AES_ENULL
    assert L.aes_ecb_batch(keys, 0, 0, seg, 2, A, A, None) == _native.AES_ERANGE
    many = (_native.aes_round_keys * 129)(*([k128] * 129))
    assert L.aes_ecb_batch(many, 129, 0, seg, 2, A, A, None) == _native.AES_ERANGE
    assert L.aes_ecb_batch(keys, 2, 0, seg, 0, None, None, None) == _native.AES_OK
    assert L.aes_ecb_batch(keys, 2, 0, None, 2, A, A, None) == _native.AES_ENULL
    mixed = (_native.aes_round_keys * 2)(k128, k256)
    assert L.aes_ecb_batch(mixed, 2, 0, seg, 2, A, A, None) == _native.AES_ENR
    bad_key = (_native.aes_segment * 1)(_native.aes_segment(0, 0, 4, 2, 0))
    assert L.aes_ecb_batch(keys, 2, 0, bad_key, 1, A, A, None) == _native.AES_ERANGE
    mis = (_native.aes_segment * 1)(_native.aes_segment(8, 8, 4, 0, 0))
    assert L.aes_ecb_batch(keys, 2, 0, mis, 1, A, A, None) == _native.AES_EALIGN
    ovl = (_native.aes_segment * 1)(_native.aes_segment(0, 16, 4, 0, 0))
    assert L.aes_ecb_batch(keys, 2, 0, ovl, 1, A, A, None) == _native.AES_EOVERLAP
    assert L.aes_ecb_batch(keys, 2, 0, seg, 2, A + 8, A, None) == _native.AES_EALIGN


def test_python_binding_mirrors_abi_names():
    import paper_1902_05234_b200 as aes
    for name in ("aes_expand_key", "aes_ecb_encrypt", "aes_ecb_decrypt", "aes_ctr_xcrypt", "aes_cbc_decrypt",
                 "aes_ecb_batch", "aes_ecb_trace", "aes_mb_lds_gather"):
        assert callable(getattr(aes, name)), name
    assert aes.aes_expand_key(bytes(16)).ek[:4] == [0, 0, 0, 0]


def test_batch_overlap_rules_host_side():
    """ecb_batch's O(m log m) overlap check: outputs pairwise
    disjoint; an output may overlap only its own input, exactly (in place)."""
    from paper_1902_05234_b200 import _check_batch_overlap as check
    check([0, 256], [0, 256], [256, 256])                       # both in place
    check([0, 0], [256, 512], [256, 256])                       # shared input
    check([0, 4096], [8192, 12288], [256, 256])                 # disjoint
    for ip, op in (([0, 256], [512, 512]), ([0, 256], [256, 512]), ([0], [16]), ([0, 1024], [1024, 0])):
        with pytest.raises(ValueError):
            check(ip, op, [256] * len(ip))
