#!/usr/bin/env python
"""NEXT-2 table-placement ablation under ncu ("ncu
conflict and pipe counters for each").

Launches each T-table placement ONCE (AES-128 encrypt of a 256 MiB random
buffer, 1024-thread CTAs x 148), after a parity check of every variant
against the default kernel (itself oracle-checked in tests/) and the golden
(oracle-written) samples.  Meant to run under

  ncu --set full --clock-control none -k regex:'ecb|hybrid|bs_kernel' -o prof_variants \
      python tools/ncu_variants.py

so the capture holds the reference launch (default kernel) and then exactly
one launch per variant, in the order of VARIANTS.  Without ncu it prints the event-timed duration of each launch.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1902_05234_b200 as aes
import synth
from synth import golden

VARIANTS = [(aes.AES_VAR_SMEM_REPL, "smem_repl (default)"), (aes.AES_VAR_SMEM_REPL_TMA, "smem_repl + TMA staging"),
            (aes.AES_VAR_SMEM_ROT, "one table + rotations"), (aes.AES_VAR_SMEM_PLAIN, "smem_plain (Li et al.)"),
            (aes.AES_VAR_GLOBAL, "global __ldg (L1)"), (aes.AES_VAR_CONST, "const (the paper's choice)"),
            (aes.AES_VAR_HYBRID, "hybrid: T-table + bitsliced warps"), (aes.AES_VAR_BITSLICE, "bitsliced only")]
if os.environ.get("AES_NCU_ONLY"):        # e.g. AES_NCU_ONLY=7,8: just these variants
    _keep = {int(v) for v in os.environ["AES_NCU_ONLY"].split(",")}
    VARIANTS = [(v, nm) for v, nm in VARIANTS if v in _keep]


def main():
    nbytes = int(os.environ.get("AES_NCU_BYTES", 256 << 20))
    x = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    synth.fill_device(x)
    rk = aes.expand_key(synth.key(128))
    ref = aes.ecb_encrypt(rk, x)
    torch.cuda.synchronize()
    gather = lambda loc: ref.view(-1, 16)[torch.from_numpy(loc).cuda()].cpu().numpy()
    assert golden.check("ecb_enc", 128, 0, nbytes // 16, gather) > 0
    # capture order: the reference launch above (default kernel), then one launch
    # per variant; each variant's output must equal the reference byte for byte
    outs = {}
    for v, name in VARIANTS:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        out = torch.empty_like(x)
        e0.record()
        aes.ecb_encrypt(rk, x, out=out, variant=v)
        e1.record()
        torch.cuda.synchronize()
        outs[name] = out
        print(json.dumps({"what": "ncu_variant_launch", "variant": name, "bytes": nbytes,
                          "ms": e0.elapsed_time(e1), "identical_to_default": bool(torch.equal(out, ref))}), flush=True)
    assert all(torch.equal(o, ref) for o in outs.values())


if __name__ == "__main__":
    main()
