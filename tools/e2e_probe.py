#!/usr/bin/env python
"""The host-buffer path (NEXT-3) against its own roofline, the PCIe link:
  * copy ceiling: 1 GiB H2D and 1 GiB D2H at the same time on two streams
    (pinned), and each direction alone;
  * aes_pipeline_run (encrypt, 1 GiB, pinned in/out) over chunk sizes and depths.
Parity of every pipeline configuration is checked against the device path."""
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
