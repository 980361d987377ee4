#!/usr/bin/env python
"""Small-message regime (BASELINE config 4): host-call
latency and device time reported SEPARATELY (SURVEY.md 8(d) "back-to-back
throughput and single-call latency are reported separately").

Per size (AES-128 encrypt, one buffer, L2-warm):
  host_*_us          host cost of one call, measured as the mean over 2000
                     calls issued back to back (the GPU queue absorbs them;
                     the kernels are shorter than the calls): raw ctypes into
                     aes_ecb_encrypt, the Python wrapper aes.ecb_encrypt, and
                     the prepared fast path aes.prepare_ecb(...)() (trusted
                     pointers, packed arguments)
  single_device_us   one launch between two CUDA events, all three queued
                     behind a ~20 us GPU spin so the host enqueue cost is
                     outside the interval (launch latency + table fill +
                     work of ONE isolated launch; median of 50)
  graph_b2b_us       per-launch device time of 100 back-to-back launches
                     captured in a CUDA graph and replayed, timed with events
                     (no host cost) -- with PDL (default) and with
                     AES_LAUNCH_NO_PDL
Then the device-side fit t = t0 + n/R_inf over the graph-timed points.
Parity: every size's output is compared with the golden (oracle-written)
samples before timing.  JSON lines on stdout.
"""
import ctypes
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1902_05234_b200 as aes
import synth
from paper_1902_05234_b200 import _native
from synth import golden

SIZES = [1, 1024, 4096, 16384, 65536, 262144, 1048576]   # blocks: 16 B .. 16 MiB


def host_calls(fn, reps=2000):
    for _ in range(100):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / reps * 1e6


def graph_b2b(fn, s, reps=100):
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    g.replay()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        s.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


def single_device(fn, s, reps=50):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        time.sleep(2e-4)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            torch.cuda._sleep(40000)      # ~20 us spin: e0, fn and e1 are all queued before e0 fires
            e0.record(s)
            fn()
            e1.record(s)
        s.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def main():
    key = synth.key(128)
    rk = aes.expand_key(key)
    s = torch.cuda.Stream()
    pts = []
    for nb in SIZES:
        x = torch.empty(16 * nb, dtype=torch.uint8, device="cuda")
        synth.fill_device(x)
        y = torch.empty_like(x)
        aes.ecb_encrypt(rk, x, out=y)
        torch.cuda.synchronize()
        gather = lambda loc: y.view(-1, 16)[torch.from_numpy(loc).cuda()].cpu().numpy()
        checked = golden.check("ecb_enc", 128, 0, nb, gather)
        L = _native.lib
        cs = torch.cuda.current_stream()
        args = (rk.c_ref, 10, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), nb,
                ctypes.c_void_p(cs.cuda_stream))
        prep = aes.prepare_ecb(rk, x, y)
        row = {"what": "latency", "nblocks": nb, "bytes": 16 * nb, "parity_samples": checked,
               "host_ctypes_us": host_calls(lambda: L.aes_ecb_encrypt(*args)),
               "host_wrapper_us": host_calls(lambda: aes.ecb_encrypt(rk, x, out=y)),
               "host_prepared_us": host_calls(prep)}
        f = (lambda: aes.ecb_encrypt(rk, x, out=y))
        fnp = (lambda: aes.ecb_encrypt(rk, x, out=y, flags=aes.AES_LAUNCH_NO_PDL))
        row["single_device_us"] = single_device(f, s)
        row["graph_b2b_us"] = graph_b2b(f, s)
        row["graph_b2b_no_pdl_us"] = graph_b2b(fnp, s)
        row["graph_b2b_GBps"] = 16 * nb / (row["graph_b2b_us"] * 1e-6) / 1e9
        assert torch.equal(y, aes.ecb_encrypt(rk, x))
        pts.append((nb, row["graph_b2b_us"], row["graph_b2b_no_pdl_us"]))
        print(json.dumps(row), flush=True)
    n = np.array([p[0] for p in pts], float)
    for col, name in ((1, "pdl"), (2, "no_pdl")):
        t = np.array([p[col] for p in pts], float) * 1e-6
        A = np.stack([np.ones_like(n), n], 1)
        (t0, inv), *_ = np.linalg.lstsq(A, t, rcond=None)
        print(json.dumps({"what": "device_fit", "launch": name, "t0_us": t0 * 1e6,
                          "R_inf_GBps": 16 / inv / 1e9 if inv > 0 else None,
                          "points": "graph_b2b per-launch device time, sizes " + ",".join(str(int(v)) for v in n),
                          "gpu": torch.cuda.get_device_name(0)}), flush=True)


if __name__ == "__main__":
    main()
