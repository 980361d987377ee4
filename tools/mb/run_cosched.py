#!/usr/bin/env python
"""Run tools/mb/cosched.cu: AES-128 ECB T-table warps + side warps doing LOP3 /
IMAD chains in the same CTA.  Reports the T path's time relative to the
all-T baseline and the side warps' retired lane-ops per clock per SM, i.e.
how much ALU / FMA work a hybrid (T-table + bitsliced) kernel could add for
free.  One JSON line per configuration."""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
SO = os.path.join(HERE, "libcosched.so")
if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(os.path.join(HERE, "cosched.cu")):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                           "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                           "-I", os.path.join(ROOT, "paper_1902_05234_b200", "csrc"),
                           "-o", SO, os.path.join(HERE, "cosched.cu")])
L = ctypes.CDLL(SO)
L.cosched_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int,
                          ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_void_p]
nsm = torch.cuda.get_device_properties(0).multi_processor_count
clk = float(sys.argv[1]) if len(sys.argv) > 1 else 1.965e9
n = 1 << 26                                       # 1 GiB of blocks
x = torch.randint(0, 256, (n * 16,), dtype=torch.uint8, device="cuda")
y = torch.empty_like(x)
rkw = (ctypes.c_uint32 * 60)(*[(0x9E3779B9 * (i + 1)) & 0xFFFFFFFF for i in range(60)])
scratch = torch.zeros(1, dtype=torch.int64, device="cuda")
ms = (ctypes.c_float * 16)()
side = (ctypes.c_ulonglong * 16)()
k = L.cosched_run(x.data_ptr(), y.data_ptr(), n, ctypes.cast(rkw, ctypes.c_void_p), nsm, ms, side,
                  scratch.data_ptr())
cfgs = [(32, "lop3", 8, "prmt"), (28, "lop3", 8, "prmt"), (24, "lop3", 8, "prmt"), (24, "imad", 8, "prmt"),
        (32, "lop3", 8, "fma03"), (28, "lop3", 8, "fma03"), (24, "lop3", 8, "fma03"), (20, "lop3", 8, "fma03"),
        (28, "imad", 8, "fma03"), (24, "imad", 8, "fma03")]
for i in range(k):
    wt, kind, e, addr = cfgs[i]
    t = ms[i] * 1e-3
    print(json.dumps({"t_warps": wt, "side_warps": 32 - wt, "side_kind": kind, "side_chains": e, "t_addressing": addr, "ms": ms[i],
                      "t_rel_to_baseline": ms[i] / ms[0], "aes_blocks_per_clk_per_sm": n / t / nsm / clk,
                      "side_lane_ops_per_clk_per_sm": side[i] / t / nsm / clk,
                      "side_bitslice_equiv_blocks_per_clk_per_sm_at_550_ops": side[i] / 550 / t / nsm / clk,
                      "total_equiv_rel": (n / t + side[i] / 550 / t) / (n / (ms[0] * 1e-3))}))
