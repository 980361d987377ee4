#!/usr/bin/env python
"""NEXT-1 / NEXT-4 on the hybrid kernel under ncu: one CTR launch and one CBC
decryption launch (AES-128, 1 GiB, the default kernel at this size), each
parity-checked against the golden (oracle-written) samples first.  Meant to run
under

  ncu --set full --clock-control none -k regex:hybrid -o prof_modes python tools/ncu_modes.py

Without ncu it prints the event-timed duration of each launch."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_1902_05234_b200 as aes
import synth
from synth import golden


def main():
    nbytes = int(os.environ.get("AES_NCU_BYTES", 1 << 30))
    n = nbytes // 16
    x = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    synth.fill_device(x)
    rk = aes.expand_key(synth.key(128))
    out = torch.empty_like(x)
    gather = lambda loc: out.view(-1, 16)[torch.from_numpy(loc).cuda()].cpu().numpy()
    iv = bytes(range(16))                 # the IV of the golden samples (tests/golden/make_samples.py)
    for mode in ("ctr", "cbc_dec"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if mode == "ctr":
            aes.ctr_xcrypt(rk, iv, x, out=out)
        else:
            aes.cbc_decrypt(rk, iv, x, out=out)
        e1.record()
        torch.cuda.synchronize()
        checked = golden.check(mode, 128, 0, n, gather)
        print(json.dumps({"what": "ncu_mode_launch", "mode": mode, "bytes": nbytes, "ms": e0.elapsed_time(e1),
                          "golden_samples_checked": checked}), flush=True)
        assert checked > 0


if __name__ == "__main__":
    main()
