#!/usr/bin/env python
"""Run tools/mb/corun.cu: 32-warp T-table kernel + a co-resident bitsliced
kernel on a second stream, static split f swept (AES-128 encrypt, 1 GiB).
Reports GB/s per (bitsliced CTA size, f) and whether the output matches the
library's default kernel.  JSON lines."""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
SO = os.path.join(HERE, "libcorun.so")
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(os.path.join(HERE, "corun.cu")):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                           "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                           "-I", os.path.join(ROOT, "paper_1902_05234_b200", "csrc"),
                           "-o", SO, os.path.join(HERE, "corun.cu")])
import paper_1902_05234_b200 as aes  # noqa: E402
import synth  # noqa: E402

L = ctypes.CDLL(SO)
L.corun_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int,
                        ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int)]
nsm = torch.cuda.get_device_properties(0).multi_processor_count
n = 1 << 26
x = torch.empty(16 * n, dtype=torch.uint8, device="cuda")
synth.fill_device(x)
rk = aes.expand_key(synth.key(128))
ref = aes.ecb_encrypt(rk, x)
y = torch.empty_like(x)
ek = (ctypes.c_uint32 * 60)(*rk.c.ek)
ms = (ctypes.c_float * 32)()
regs = (ctypes.c_int * 3)()
k = L.corun_run(x.data_ptr(), y.data_ptr(), n, ctypes.cast(ek, ctypes.c_void_p), nsm, ms, regs)
torch.cuda.synchronize()
fs = [0.0, 0.06, 0.08, 0.10, 0.12, 0.14, 0.16]
print(json.dumps({"regs": {"t_kernel": regs[0], "b_kernel_192": regs[1], "b_kernel_128": regs[2]}}))
for i in range(k):
    bt = 192 if i < len(fs) else 128
    f = fs[i % len(fs)]
    print(json.dumps({"b_cta_threads": bt, "f_bitsliced": f, "ms": ms[i], "GBps": 16 * n / (ms[i] * 1e-3) / 1e9}))
print(json.dumps({"last_output_matches_default": bool(torch.equal(y, ref))}))
