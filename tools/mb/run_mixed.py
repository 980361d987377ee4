#!/usr/bin/env python
"""Run tools/mb/mixed.cu: time of 16 LDS chains + E extra chains through LDS /
L1-resident LDG / texture.  Extra chains that add ~no time would be a lookup
path independent of the shared-memory data path."""
import ctypes
import json
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmixed.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                       "-o", SO, os.path.join(HERE, "mixed.cu")])
L = ctypes.CDLL(SO)
L.mixed_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
nsm = torch.cuda.get_device_properties(0).multi_processor_count
sink = torch.empty(nsm * 1024, dtype=torch.int32, device="cuda")
tab = torch.randint(0, 2**31, (256 * 32,), dtype=torch.int32, device="cuda")
out = (ctypes.c_float * 7)()
rc = L.mixed_run(tab.data_ptr(), sink.data_ptr(), nsm, 1024, out)
names = ["16 LDS", "16 LDS + 2 LDS", "16 LDS + 4 LDS", "16 LDS + 2 LDG(L1)", "16 LDS + 4 LDG(L1)",
         "16 LDS + 2 TEX", "16 LDS + 4 TEX"]
for nm, ms in zip(names, out):
    print(json.dumps({"kernel": nm, "ms": ms, "rel_to_16_lds": ms / out[0] if out[0] > 0 else None, "rc": rc}))
