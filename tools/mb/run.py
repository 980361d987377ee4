#!/usr/bin/env python
"""Run tools/mb/lds_width.cu: lookups/clk/SM and bytes/clk/SM for 32/64/128-bit
lane-replicated shared-memory gathers, constant-memory gathers and L1-resident
global gathers.  One JSON line per kind."""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmb.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                       "-o", SO, os.path.join(HERE, "lds_width.cu")])
L = ctypes.CDLL(SO)
L.mb_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                     ctypes.POINTER(ctypes.c_float)]
nsm = torch.cuda.get_device_properties(0).multi_processor_count
sink = torch.empty(nsm * 1024, dtype=torch.int32, device="cuda")
tab = torch.randint(0, 2**31, (256 * 32,), dtype=torch.int32, device="cuda")
clk = float(sys.argv[1]) if len(sys.argv) > 1 else 1.965e9
for kind, name, lookups_per_it, bytes_per in ((1, "smem LDS.32", 16, 4), (2, "smem LDS.64", 16, 8),
                                             (4, "smem LDS.128", 16, 16), (10, "__constant__ LDC", 8, 4),
                                             (11, "L1-resident LDG.32", 16, 4)):
    iters = 2048 if kind < 10 else 64
    ms = ctypes.c_float()
    rc = L.mb_run(kind, sink.data_ptr(), tab.data_ptr(), nsm, iters, ctypes.byref(ms))
    n = nsm * 1024 * iters * lookups_per_it
    rate = n / (ms.value * 1e-3)
    print(json.dumps({"kind": name, "rc": rc, "ms": ms.value, "lookups_per_s": rate,
                      "lookups_per_clk_per_sm": rate / nsm / clk, "bytes_per_clk_per_sm": rate * bytes_per / nsm / clk}))
