#!/usr/bin/env python
"""Run tools/mb/alu.cu: LOP3 / PRMT / IMAD lane-ops per clock per SM."""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libalu.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                       "-o", SO, os.path.join(HERE, "alu.cu")])
L = ctypes.CDLL(SO)
L.alu_run.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
nsm = torch.cuda.get_device_properties(0).multi_processor_count
clk = float(sys.argv[1]) if len(sys.argv) > 1 else 1.965e9
sink = torch.empty(nsm * 1024, dtype=torch.int32, device="cuda")
out = (ctypes.c_float * 6)()
iters = 4096
rc = L.alu_run(sink.data_ptr(), nsm, iters, out)
for name, ms in zip(("LOP3", "PRMT", "IMAD", "IMAD.HI", "SHF.L.W", "IMAD.WIDE+IMAD (2 instr)"), out):
    ops = nsm * 1024 * iters * 16
    print(json.dumps({"op": name, "rc": rc, "ms": ms, "lane_ops_per_clk_per_sm": ops / (ms * 1e-3) / nsm / clk}))
