#!/usr/bin/env python
"""Hybrid (T-table + bitsliced warps) probe: parity of AES_VAR_HYBRID /
AES_VAR_BITSLICE against the default kernel (itself oracle-checked in tests/),
then CUDA-event timings of 1 GiB
encrypt / decrypt per variant and key size.  JSONL on stdout."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import paper_1902_05234_b200 as aes
import synth

NAMES = {aes.AES_VAR_SMEM_REPL: "smem_repl", aes.AES_VAR_HYBRID: "hybrid", aes.AES_VAR_BITSLICE: "bitslice"}


def timeit(fn, s, reps=10):
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    s.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            fn()
            e1.record(s)
        s.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[0], ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, nargs="*", default=[1024])
    ap.add_argument("--keybits", type=int, nargs="*", default=[128, 192, 256])
    ap.add_argument("--variants", type=int, nargs="*", default=[1, 7, 8])
    a = ap.parse_args()
    s = torch.cuda.Stream()
    for mib in a.mib:
        run_size(a, s, mib << 16)


def run_size(a, s, n):
    for kb in a.keybits:
        rk = aes.expand_key(synth.key(kb))
        x = torch.empty(16 * n, dtype=torch.uint8, device="cuda")
        synth.fill_device(x)
        ref_c = aes.ecb_encrypt(rk, x)
        ref_p = aes.ecb_decrypt(rk, x)
        for v in a.variants:
            out = torch.empty_like(x)
            for dec, ref in ((False, ref_c), (True, ref_p)):
                aes.ecb(rk, x, dec, out=out, variant=v)
                torch.cuda.synchronize()
                ok = torch.equal(out, ref)
                if not ok:
                    bad = (out.view(-1, 16) != ref.view(-1, 16)).any(1).nonzero()
                    print(json.dumps({"variant": NAMES[v], "keybits": kb, "dec": dec, "parity": False,
                                      "first_bad_block": int(bad[0]), "n_bad": int(bad.numel())}), flush=True)
                    continue
                tmin, tmed = timeit(lambda: aes.ecb(rk, x, dec, out=out, variant=v), s)
                print(json.dumps({"variant": NAMES[v], "keybits": kb, "dir": "dec" if dec else "enc", "parity": True,
                                  "n": n, "ms_min": tmin, "ms_med": tmed, "Gbps": 8 * 16 * n / (tmin * 1e-3) / 1e9,
                                  "GBps": 16 * n / (tmin * 1e-3) / 1e9}), flush=True)
        del x, ref_c, ref_p
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
