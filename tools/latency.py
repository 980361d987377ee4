#!/usr/bin/env python
"""Host launch-path cost of one small call (the t0 of the config-4 fit):
direct ctypes call into aes_ecb_encrypt vs the Python wrapper, 1 block and
64 Ki blocks, 2000 calls each, plus the device time of a 1-block kernel from
events around a CUDA graph of 100 launches (host cost excluded)."""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1902_05234_b200 as aes
from paper_1902_05234_b200 import _native

rk = aes.expand_key(bytes(16))
for nb in (1, 65536):
    x = torch.zeros(16 * nb, dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    s = torch.cuda.current_stream()
    L = _native.lib
    args = (ctypes.byref(rk.c), 10, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), nb,
            ctypes.c_void_p(s.cuda_stream))
    for _ in range(100):
        L.aes_ecb_encrypt(*args)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2000):
        L.aes_ecb_encrypt(*args)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    for _ in range(2000):
        aes.ecb_encrypt(rk, x, out=y)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    g = torch.cuda.CUDAGraph()
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        with torch.cuda.graph(g, stream=gs):
            for _ in range(100):
                aes.ecb_encrypt(rk, x, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"nblocks": nb, "ctypes_call_us": (t1 - t0) / 2000 * 1e6,
                      "ctypes_drain_us": (t2 - t0) / 2000 * 1e6,
                      "python_wrapper_call_us": (t3 - t2) / 2000 * 1e6,
                      "python_wrapper_drain_us": (t4 - t2) / 2000 * 1e6,
                      "graph_device_us_per_launch": e0.elapsed_time(e1) * 1e3 / 100}))
