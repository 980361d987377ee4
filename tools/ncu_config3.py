#!/usr/bin/env python
"""BASELINE config 3 under ncu: AES-256 ECB decrypt of 4 GiB (the default,
hybrid kernel at this size), after the GPU encrypt that makes its input;
parity: D(E(x)) == x and the golden samples of E.  Run as
  ncu --set full --clock-control none -k regex:hybrid -s 1 -c 1 -o prof python tools/ncu_config3.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1902_05234_b200 as aes, synth
from synth import golden
n = (4 << 30) // 16
x = torch.empty(16 * n, dtype=torch.uint8, device="cuda")
synth.fill_device(x)
rk = aes.expand_key(synth.key(256))
ct = aes.ecb_encrypt(rk, x)          # outside the captured launch (-s 1 skips it)
out = torch.empty_like(x)
aes.ecb_decrypt(rk, ct, out=out)
torch.cuda.synchronize()
assert torch.equal(out, x)
gather = lambda loc: ct.view(-1, 16)[torch.from_numpy(loc).cuda()].cpu().numpy()
print(json.dumps({"config3_golden_checked": golden.check("ecb_enc", 256, 0, n, gather)}))
