"""B200 (sm_100a) AES-128/192/256 ECB -- thin Python binding over libaes_b200.so.

The hot path of arXiv 1902.05234 (T-box rounds, one state per thread, ECB):
    rk = expand_key(key)                      # aes_expand_key (host, C++)
    ct = ecb_encrypt(rk, x)                   # aes_ecb_encrypt (CUDA kernel)
    pt = ecb_decrypt(rk, ct)                  # aes_ecb_decrypt (CUDA kernel)
``x`` is a contiguous torch.uint8 CUDA tensor whose length is a multiple of 16
(padding is the caller's job, R17).  Work is enqueued on
``torch.cuda.current_stream()``.  This module only marshals arguments; every
step of the path runs in the library's kernels.  There is no CPU fallback:
CPU tensors raise TypeError.
"""
from __future__ import annotations

import ctypes

from . import _native
from ._native import (AES_LAUNCH_NO_PDL, AES_LAUNCH_TRUSTED_PTRS, AES_VAR_BITSLICE, AES_VAR_CONST, AES_VAR_DEFAULT,
                      AES_VAR_GLOBAL, AES_VAR_HYBRID, AES_VAR_SMEM_PLAIN, AES_VAR_SMEM_REPL, AES_VAR_SMEM_REPL_TMA, AES_VAR_SMEM_ROT, aes_launch_config,
                      aes_round_keys, status_string)

__all__ = ["RoundKeys", "expand_key", "ecb_encrypt", "ecb_decrypt", "ecb", "ecb_batch", "ecb_batch_offsets", "KeySet", "ctr_xcrypt", "cbc_decrypt",
           "ecb_trace", "Pipeline",
           "lds_gather", "AesError", "AES_VAR_DEFAULT", "AES_VAR_SMEM_REPL", "AES_VAR_SMEM_PLAIN",
           "AES_VAR_CONST", "AES_VAR_SMEM_REPL_TMA", "AES_VAR_SMEM_ROT", "AES_VAR_GLOBAL", "AES_VAR_HYBRID", "AES_VAR_BITSLICE",
           "AES_LAUNCH_TRUSTED_PTRS",
           "AES_LAUNCH_NO_PDL", "abi_version", "prepare_ecb", "EcbCall"]


class AesError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        msg = status_string(code)
        if code == _native.AES_ECUDA:
            msg += f" (cudaError {_native.lib.aes_last_cuda_error()})"
        super().__init__(f"{what}: {msg}" if what else msg)


def _check(code: int, what: str):
    if code != _native.AES_OK:
        raise AesError(code, what)


class RoundKeys:
    """Expanded key (aes_round_keys): ek, dk (equivalent inverse), nr, keybits."""

    __slots__ = ("c", "c_ref")

    def __init__(self, c: aes_round_keys):
        self.c = c
        self.c_ref = ctypes.byref(c)   # built once: byref() per call costs ~0.3 us

    @property
    def nr(self) -> int:
        return self.c.nr

    @property
    def keybits(self) -> int:
        return self.c.keybits

    @property
    def ek(self) -> list[int]:
        return list(self.c.ek[: 4 * (self.nr + 1)])

    @property
    def dk(self) -> list[int]:
        return list(self.c.dk[: 4 * (self.nr + 1)])


def abi_version() -> int:
    return _native.lib.aes_abi_version()


def expand_key(key: bytes) -> RoundKeys:
    """aes_expand_key: 16/24/32-byte key -> round keys (ValueError otherwise)."""
    key = bytes(key)
    if len(key) not in (16, 24, 32):
        raise ValueError("AES key must be 16, 24 or 32 bytes")
    rk = aes_round_keys()
    _check(_native.lib.aes_expand_key(key, 8 * len(key), ctypes.byref(rk)), "aes_expand_key")
    return RoundKeys(rk)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


_NULL = _Null()


def _raw_stream(dev_index: int) -> int:
    """cudaStream_t of torch's current stream on ``dev_index`` (cheap path)."""
    import torch
    try:
        return torch._C._cuda_getCurrentRawStream(dev_index)
    except AttributeError:   # pragma: no cover - older torch
        return torch.cuda.current_stream(dev_index).cuda_stream


def _on_device(dev):
    """torch.cuda.device(dev) only when dev is not already current (cheap path)."""
    import torch
    return _NULL if dev.index == torch.cuda.current_device() else torch.cuda.device(dev)


def _check_tensor(x, name):
    import torch
    if type(x) is torch.Tensor and x.dtype is torch.uint8 and x.is_cuda and x.is_contiguous() \
            and not x.numel() & 15:
        return                                  # the common case: one combined test
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if not x.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if x.dtype != torch.uint8:
        raise TypeError(f"{name} must be torch.uint8")
    if not x.is_contiguous():
        raise TypeError(f"{name} must be contiguous")
    if x.numel() % 16:
        raise ValueError(f"{name}.numel() must be a multiple of 16 (whole AES blocks)")


def ecb(rk: RoundKeys, x, decrypt: bool, out=None, variant: int = AES_VAR_DEFAULT,
        states_per_thread: int = 0, grid: int = 0, stream=None, flags: int = 0):
    """ECB over a device buffer; ``out`` may be ``x`` (in place) or None (new tensor).
    ``variant``: AES_VAR_* (default: the hybrid T-table + bitsliced kernel from
    2^23 blocks, the replicated T-table kernel below); ``flags``: AES_LAUNCH_*
    bits (aes_launch_config.flags).  Every variant returns identical bytes."""
    import torch
    _check_tensor(x, "x")
    if out is None:
        out = torch.empty_like(x)
    elif out is not x:
        _check_tensor(out, "out")
        if out.numel() != x.numel():
            raise ValueError("out must have the same size as x")
    n = x.numel() >> 4
    with _on_device(x.device):
        sp = stream.cuda_stream if stream is not None else _raw_stream(x.device.index)
        if variant == AES_VAR_DEFAULT and not states_per_thread and not grid and not flags:
            fn = _native.lib.aes_ecb_decrypt if decrypt else _native.lib.aes_ecb_encrypt
            code = fn(rk.c_ref, rk.nr, x.data_ptr(), out.data_ptr(), n, sp)
        else:
            cfg = aes_launch_config(variant, states_per_thread, grid, flags)
            code = _native.lib.aes_ecb_launch(rk.c_ref, rk.nr, int(bool(decrypt)),
                                              x.data_ptr(), out.data_ptr(), n, sp, ctypes.byref(cfg))
    if code:
        _check(code, "aes_ecb_decrypt" if decrypt else "aes_ecb_encrypt")
    return out


class EcbCall:
    """A prepared ECB call over fixed device buffers -- the per-call fast path.

    Everything that does not change between calls is decided once here: the
    tensors are validated (contiguous uint8 CUDA memory of one device, sizes,
    in == out or disjoint), the ctypes arguments are packed, and the launch
    carries AES_LAUNCH_TRUSTED_PTRS so the library skips its per-call
    cudaPointerGetAttributes queries (torch already guarantees device memory).
    Each ``call()`` (or ``__call__``) then costs one raw-stream query plus the
    C ABI call: aes_ecb_launch on torch's current stream (or ``stream``).
    The tensors must stay alive (and in place) while the object is used."""

    __slots__ = ("_fn", "_args", "_dev", "x", "out")

    def __init__(self, rk: RoundKeys, x, out=None, decrypt: bool = False, variant: int = AES_VAR_DEFAULT,
                 states_per_thread: int = 0, grid: int = 0, flags: int = 0):
        import torch
        _check_tensor(x, "x")
        if out is None:
            out = torch.empty_like(x)
        _check_tensor(out, "out")
        if out.numel() != x.numel() or out.device != x.device:
            raise ValueError("out must have the size and device of x")
        self.x, self.out = x, out
        self._dev = x.device.index
        cfg = aes_launch_config(variant, states_per_thread, grid, flags | AES_LAUNCH_TRUSTED_PTRS)
        self._fn = _native.lib.aes_ecb_launch
        # the keys are copied into the object: later changes to rk do not leak in
        kc = aes_round_keys.from_buffer_copy(rk.c)
        self._args = [ctypes.byref(kc), rk.nr, int(bool(decrypt)), ctypes.c_void_p(x.data_ptr()),
                      ctypes.c_void_p(out.data_ptr()), x.numel() >> 4, None, ctypes.byref(cfg), kc, cfg]
        # what the library would check per call, checked once: alignment,
        # overlap (in == out allowed), then variant/flags/keys via a zero-block call
        pi, po, nb = x.data_ptr(), out.data_ptr(), x.numel()
        if (pi | po) & 15:
            raise AesError(_native.AES_EALIGN, "aes_ecb_launch")
        if pi != po and pi < po + nb and po < pi + nb:
            raise AesError(_native.AES_EOVERLAP, "aes_ecb_launch")
        code = self._fn(*self._args[:5], 0, None, self._args[7])
        if code:
            _check(code, "aes_ecb_launch")

    def __call__(self, stream=None):
        import torch
        a = self._args
        dev = self._dev
        if torch.cuda.current_device() != dev:
            with torch.cuda.device(dev):
                return self.__call__(stream)
        code = self._fn(a[0], a[1], a[2], a[3], a[4], a[5],
                        stream.cuda_stream if stream is not None else _raw_stream(dev), a[7])
        if code:
            _check(code, "aes_ecb_launch")
        return self.out

    call = __call__


def prepare_ecb(rk: RoundKeys, x, out=None, decrypt: bool = False, **kw) -> EcbCall:
    """EcbCall(rk, x, out, decrypt): the per-call fast path over fixed buffers."""
    return EcbCall(rk, x, out, decrypt, **kw)


def ecb_encrypt(rk: RoundKeys, x, out=None, **kw):
    return ecb(rk, x, False, out, **kw)


def ecb_decrypt(rk: RoundKeys, x, out=None, **kw):
    return ecb(rk, x, True, out, **kw)


def _prep_out(x, out):
    import torch
    _check_tensor(x, "x")
    if out is None:
        return torch.empty_like(x)
    _check_tensor(out, "out")
    if out.numel() != x.numel():
        raise ValueError("out must have the same size as x")
    return out


def ctr_xcrypt(rk: RoundKeys, iv: bytes, x, out=None, block_offset: int = 0, stream=None):
    """CTR (Eq 5, reading R24): out_j = x_j ^ E(iv + block_offset + j); iv = 16-byte BE counter."""
    import torch
    iv = bytes(iv)
    if len(iv) != 16:
        raise ValueError("iv must be 16 bytes")
    out = _prep_out(x, out)
    with _on_device(x.device):
        sp = stream.cuda_stream if stream is not None else _raw_stream(x.device.index)
        code = _native.lib.aes_ctr_xcrypt(rk.c_ref, rk.nr, iv, block_offset & (2**64 - 1),
                                          x.data_ptr(), out.data_ptr(), x.numel() // 16, sp)
    _check(code, "aes_ctr_xcrypt")
    return out


def cbc_decrypt(rk: RoundKeys, iv: bytes, x, out=None, stream=None):
    """CBC decryption (Eq 2, reading R25): out_i = D(x_i) ^ x_{i-1}, x_{-1} = iv.  Not in place."""
    import torch
    iv = bytes(iv)
    if len(iv) != 16:
        raise ValueError("iv must be 16 bytes")
    out = _prep_out(x, out)
    with _on_device(x.device):
        sp = stream.cuda_stream if stream is not None else _raw_stream(x.device.index)
        code = _native.lib.aes_cbc_decrypt(rk.c_ref, rk.nr, iv, x.data_ptr(), out.data_ptr(),
                                           x.numel() // 16, sp)
    _check(code, "aes_cbc_decrypt")
    return out


class KeySet:
    """A fixed list of RoundKeys packed once as the C array aes_ecb_batch takes."""

    __slots__ = ("arr", "n")

    def __init__(self, rks):
        self.n = len(rks)
        self.arr = (aes_round_keys * self.n)(*[r.c for r in rks])


_SEG_DTYPE = None


def ecb_batch_offsets(rks, in_base: int, out_base: int, in_offsets, out_offsets, nblocks, key_index,
                      decrypt: bool = False, device=None, stream=None):
    """aes_ecb_batch over raw device addresses: message i = nblocks[i] blocks at
    in_base + in_offsets[i] -> out_base + out_offsets[i] with rks[key_index[i]].
    ``rks``: a KeySet (cheapest) or a list of RoundKeys.  Array arguments are
    vectors of equal length (numpy or lists); no per-message Python work beyond
    packing them."""
    import numpy as np
    import torch
    global _SEG_DTYPE
    if _SEG_DTYPE is None:
        _SEG_DTYPE = np.dtype([("in", "<u8"), ("out", "<u8"), ("n", "<u8"), ("k", "<u4"), ("r", "<u4")])
    m = len(nblocks)
    segs = np.empty(m, dtype=_SEG_DTYPE)
    segs["in"], segs["out"], segs["n"], segs["k"], segs["r"] = in_offsets, out_offsets, nblocks, key_index, 0
    ks = rks if isinstance(rks, KeySet) else KeySet(rks)
    keys = ks.arr
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    with _on_device(dev):
        sp = stream.cuda_stream if stream is not None else _raw_stream(dev.index)
        code = _native.lib.aes_ecb_batch(keys, ks.n, int(bool(decrypt)),
                                         segs.ctypes.data_as(ctypes.POINTER(_native.aes_segment)), m,
                                         in_base, out_base, sp)
    _check(code, "aes_ecb_batch")


def _check_batch_overlap(ip, op, nbytes):
    """Outputs must be pairwise disjoint, and an output may overlap an input
    only when it IS that message's own input (in place).  O(m log m)."""
    import numpy as np
    i0, o0, ln = (np.asarray(v, dtype=np.uint64) for v in (ip, op, nbytes))
    order = np.argsort(o0, kind="stable")
    so, se = o0[order], o0[order] + ln[order]
    if len(so) > 1 and np.any(so[1:] < se[:-1]):
        raise ValueError("aes_ecb_batch: output buffers of two messages overlap")
    # for every input, the output with the largest start below the input's end
    k = np.searchsorted(so, i0 + ln, side="left").astype(np.int64) - 1
    hit = k >= 0
    kk = np.where(hit, k, 0)
    hit &= se[kk] > i0                                          # that output overlaps the input
    own = order[kk] == np.arange(len(i0))                       # ... and is the message's own output
    exact = so[kk] == i0
    if np.any(hit & ~(own & exact)):
        raise ValueError("aes_ecb_batch: an output overlaps another message's input (or its own, partially)")


def ecb_batch(rks, xs, outs=None, key_index=None, decrypt: bool = False, stream=None):
    """aes_ecb_batch: ECB of many messages (each its own key) in ONE launch.

    rks: list of RoundKeys (same key size); xs: list of contiguous CUDA uint8
    tensors on one device (numel % 16 == 0, 16-byte aligned); key_index[i]
    picks rks for xs[i] (default: i).  Returns the list of outputs (``outs``
    if given; an output may be its own input, but must not overlap any other
    message's input or output: ValueError)."""
    import torch
    n = len(xs)
    if key_index is None:
        key_index = list(range(n))
    if len(key_index) != n or not rks:
        raise ValueError("need one key index per message and at least one key")
    if outs is None:
        outs = [torch.empty_like(x) for x in xs]
    if len(outs) != n:
        raise ValueError("one output per message")
    dev0 = xs[0].device if n else None
    for x, o in zip(xs, outs):
        _check_tensor(x, "x")
        _check_tensor(o, "out")
        if o.numel() != x.numel():
            raise ValueError("out must match x")
        if x.device != dev0 or o.device != dev0:
            raise ValueError("all messages and outputs must be on one CUDA device")
    live = [i for i in range(n) if xs[i].numel()]
    if not live:
        return outs
    ip = [xs[i].data_ptr() for i in live]
    op = [outs[i].data_ptr() for i in live]
    _check_batch_overlap(ip, op, [xs[i].numel() for i in live])
    ib, ob = min(ip), min(op)
    ecb_batch_offsets(rks, ib, ob, [p - ib for p in ip], [p - ob for p in op], [xs[i].numel() // 16 for i in live],
                      [key_index[i] for i in live], decrypt, xs[live[0]].device, stream)
    return outs


def ecb_trace(rk: RoundKeys, x, rounds: int, decrypt: bool = False, out=None):
    """aes_ecb_trace: state after ARK(0) + `rounds` rounds (round-by-round parity pin)."""
    out = _prep_out(x, out)
    with _on_device(x.device):
        code = _native.lib.aes_ecb_trace(rk.c_ref, rk.nr, int(bool(decrypt)), int(rounds), x.data_ptr(),
                                         out.data_ptr(), x.numel() // 16, _raw_stream(x.device.index))
    _check(code, "aes_ecb_trace")
    return out


class Pipeline:
    """Host-resident end-to-end path: aes_pipeline_create/run/destroy.

    ``run`` takes host buffers (numpy arrays or CPU uint8 tensors, ideally
    pinned), copies chunks to the device, ciphers them there and copies them
    back, overlapping the three stages across ``depth`` streams.  Synchronous.
    """

    def __init__(self, chunk_bytes: int = 64 << 20, depth: int = 3, device=None):
        import torch
        self.h = ctypes.c_void_p()
        dev = torch.cuda.current_device() if device is None else device
        with torch.cuda.device(dev):
            _check(_native.lib.aes_pipeline_create(chunk_bytes, depth, ctypes.byref(self.h)),
                   "aes_pipeline_create")

    @staticmethod
    def _ptr_len(a):
        import numpy as np
        import torch
        if isinstance(a, torch.Tensor):
            if a.is_cuda or a.dtype != torch.uint8 or not a.is_contiguous():
                raise TypeError("host buffers must be contiguous CPU uint8 tensors")
            return a.data_ptr(), a.numel()
        if isinstance(a, np.ndarray):
            if a.dtype != np.uint8 or not a.flags["C_CONTIGUOUS"]:
                raise TypeError("host buffers must be contiguous uint8 arrays")
            return a.ctypes.data, a.size
        raise TypeError("host buffer must be a numpy array or CPU tensor")

    def run(self, rk: RoundKeys, src, dst, decrypt: bool = False):
        ps, ns = self._ptr_len(src)
        pd, nd = self._ptr_len(dst)
        if ns != nd or ns % 16:
            raise ValueError("src/dst must have equal sizes, a multiple of 16")
        _check(_native.lib.aes_pipeline_run(self.h, rk.c_ref, rk.nr, int(bool(decrypt)),
                                            ctypes.c_void_p(ps), ctypes.c_void_p(pd), ns // 16),
               "aes_pipeline_run")
        return dst

    def close(self):
        if self.h:
            _native.lib.aes_pipeline_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def lds_gather(sink, grid: int, iters: int, stream=None):
    """Launch the shared-memory gather microbenchmark (aes_mb_lds_gather)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(sink.device)
    with torch.cuda.device(sink.device):
        _check(_native.lib.aes_mb_lds_gather(ctypes.c_void_p(sink.data_ptr()), grid, iters,
                                             ctypes.c_void_p(s.cuda_stream)), "aes_mb_lds_gather")
    return 16 * iters * grid * 1024  # lookups issued


# The C ABI's own names (include/aes_b200.h), for callers who mirror the C API.
aes_expand_key = expand_key
aes_ecb_encrypt = ecb_encrypt
aes_ecb_decrypt = ecb_decrypt
aes_ctr_xcrypt = ctr_xcrypt
aes_cbc_decrypt = cbc_decrypt
aes_ecb_batch = ecb_batch
aes_ecb_trace = ecb_trace
aes_mb_lds_gather = lds_gather
__all__ += ["aes_expand_key", "aes_ecb_encrypt", "aes_ecb_decrypt", "aes_ctr_xcrypt", "aes_cbc_decrypt",
            "aes_ecb_batch", "aes_ecb_trace", "aes_mb_lds_gather"]
