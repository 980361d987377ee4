#!/usr/bin/env python
"""Run tools/mb/hyb.cu: AES-128 encrypt of 1 GiB by the hybrid kernel under
several knob settings; reports time and how many blocks the bitsliced warps
took.  JSON lines."""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
SO = os.path.join(HERE, "libhyb.so")
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(os.path.join(HERE, "hyb.cu")):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                           "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                           "-I", os.path.join(ROOT, "paper_1902_05234_b200", "csrc"),
                           "-o", SO, os.path.join(HERE, "hyb.cu")])
import paper_1902_05234_b200 as aes  # noqa: E402
import synth  # noqa: E402

L = ctypes.CDLL(SO)
L.hyb_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int,
                      ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_void_p]
nsm = torch.cuda.get_device_properties(0).multi_processor_count
n = 1 << 26
x = torch.empty(16 * n, dtype=torch.uint8, device="cuda")
synth.fill_device(x)
rk = aes.expand_key(synth.key(128))
ref = aes.ecb_encrypt(rk, x)
y = torch.empty_like(x)
ek = (ctypes.c_uint32 * 60)(*rk.c.ek)
scratch = torch.zeros(1, dtype=torch.int64, device="cuda")
ms = (ctypes.c_float * 16)()
bb = (ctypes.c_ulonglong * 16)()
k = L.hyb_run(x.data_ptr(), y.data_ptr(), n, ctypes.cast(ek, ctypes.c_void_p), nsm, ms, bb, scratch.data_ptr())
torch.cuda.synchronize()
names = ["T28 alone", "T28+B4 hybrid", "T24 alone (48 regs)", "T24+B8 (48/112 regs)", "T24+B8 (56/88 regs)",
         "T20+B12 (48/88 regs)"]
for i in range(k):
    print(json.dumps({"cfg": names[i], "ms": ms[i], "GBps": 16 * n / (ms[i] * 1e-3) / 1e9,
                      "b_blocks_frac": bb[i] / n}))
print(json.dumps({"last_output_matches_default": bool(torch.equal(y, ref))}))
