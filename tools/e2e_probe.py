#!/usr/bin/env python
"""The host-buffer path (NEXT-3) against its own roofline, the PCIe link:
  * copy ceiling: 1 GiB H2D and 1 GiB D2H at the same time on two streams
    (pinned), and each direction alone;
  * aes_pipeline_run (encrypt, 1 GiB, pinned in/out) over chunk sizes and depths.
Parity of every pipeline configuration is checked against the device path."""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1902_05234_b200 as aes
import synth

G = 1 << 30
x = torch.empty(G, dtype=torch.uint8, device="cuda")
synth.fill_device(x)
dev_out = torch.empty_like(x)
hx = x.cpu().pin_memory()
ho = torch.empty_like(hx).pin_memory()
rk = aes.expand_key(synth.key(128))
ref = aes.ecb_encrypt(rk, x).cpu()


def t_copy(both):
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        dev_out.copy_(hx, non_blocking=True)
    if both:
        with torch.cuda.stream(s2):
            ho.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for _ in range(2):
    t_copy(True)
h2d = min(t_copy(False) for _ in range(3))
both = min(t_copy(True) for _ in range(3))
print(json.dumps({"what": "copy_ceiling", "h2d_GBps": G / h2d / 1e9, "bidir_GBps_each": G / both / 1e9}))
# zero copy at full size: one kernel reads and writes the pinned (UVA-mapped)
# host buffers over the link directly (AES_LAUNCH_TRUSTED_PTRS: the ABI's
# device-pointer check would refuse host memory), T-table and hybrid kernels
from paper_1902_05234_b200 import _native  # noqa: E402
for v, name in ((aes.AES_VAR_SMEM_REPL, "t_table"), (aes.AES_VAR_HYBRID, "hybrid")):
    cfg = _native.aes_launch_config(v, 0, 0, aes.AES_LAUNCH_TRUSTED_PTRS)
    sp = torch.cuda.current_stream().cuda_stream
    def zc():
        code = _native.lib.aes_ecb_launch(rk.c_ref, rk.nr, 0, hx.data_ptr(), ho.data_ptr(), G // 16, sp,
                                          ctypes.byref(cfg))
        assert code == 0, code
    ho.zero_()
    zc()
    torch.cuda.synchronize()
    ok = torch.equal(ho, ref)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        zc()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(json.dumps({"what": "zero_copy", "kernel": name, "ok": ok, "t_s": min(ts), "GBps": G / min(ts) / 1e9,
                      "Gbps": 8 * G / min(ts) / 1e9}), flush=True)
for chunk_mb in (8, 32, 64, 128, 256):
    for depth in (2, 3, 4, 6, 8):
        p = aes.Pipeline(chunk_bytes=chunk_mb << 20, depth=depth)
        p.run(rk, hx, ho)
        ok = torch.equal(ho, ref)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            p.run(rk, hx, ho)
            ts.append(time.perf_counter() - t0)
        p.close()
        print(json.dumps({"what": "pipeline", "chunk_MiB": chunk_mb, "depth": depth, "ok": ok,
                          "t_s": min(ts), "GBps": G / min(ts) / 1e9, "Gbps": 8 * G / min(ts) / 1e9}))
