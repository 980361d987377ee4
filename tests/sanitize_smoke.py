#!/usr/bin/env python
"""Small enc/dec runs of every kernel variant for compute-sanitizer
(memcheck / racecheck / initcheck / synccheck): ragged tails, in-place,
tiny grids, and the hybrid kernel with its bitsliced warps active in every
mode.  Exit code 0 iff every output matches the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # repo root
sys.path.insert(0, ROOT)
import numpy as np
import torch

import oracle
import paper_1902_05234_b200 as aes
import synth

ok = True
for kb in (128, 256):
    key = synth.key(kb)
    rk = aes.expand_key(key)
    for n in (1, 33, 2 * 1024 + 5):
        x = torch.empty(16 * n, dtype=torch.uint8, device="cuda")
        synth.fill_device(x)
        host = synth.blocks(0, n)
        variants = [(1, 1), (1, 2), (1, 4), (2, 1), (3, 1), (4, 1), (5, 1), (6, 1), (7, 1), (8, 1)]
        if os.environ.get("AES_SANITIZE_VARIANTS"):
            variants = [tuple(int(x) for x in p.split(":")) for p in os.environ["AES_SANITIZE_VARIANTS"].split(",")]
        for v, spt in variants:
            for dec in (False, True):
                out = aes.ecb(rk, x, dec, variant=v, states_per_thread=spt, grid=2)
                ok &= np.array_equal(out.cpu().numpy(), oracle.ecb(key, host, dec, 4))
        y = x.clone()
        aes.ecb_encrypt(rk, y, out=y)
        aes.ecb_decrypt(rk, y, out=y)
        ok &= bool(torch.equal(x, y))
# CTR (counter-mode-cached kernel: warp-private group tables) and CBC decryption
for kb in (128, 256):
    key = synth.key(kb)
    rk = aes.expand_key(key)
    for n in (1, 300, 3 * 1024 + 17):
        x = torch.empty(16 * n, dtype=torch.uint8, device="cuda")
        synth.fill_device(x)
        host = synth.blocks(0, n)
        for iv in (bytes([0xFF] * 15 + [0xC8]), bytes(range(16))):
            ok &= np.array_equal(aes.ctr_xcrypt(rk, iv, x, block_offset=77).cpu().numpy(),
                                 oracle.ctr(key, iv, host, block_offset=77, nthreads=4))
        ok &= np.array_equal(aes.cbc_decrypt(rk, bytes(16), x).cpu().numpy(), oracle.cbc(key, bytes(16), host, True))
# hybrid kernel with ONE CTA and > 384 units, so its bitsliced warps claim
# units next to the T-table warps (shared-memory unit queue, setmaxnreg): ECB
# both directions, and CTR / CBC decryption through the crossover knob
os.environ["AES_B200_HYBRID_MIN_BLOCKS"] = "0"
n = 16 * 1024 + 77
for kb in (128, 256):
    key = synth.key(kb)
    rk = aes.expand_key(key)
    x = torch.empty(16 * n, dtype=torch.uint8, device="cuda")
    synth.fill_device(x)
    host = synth.blocks(0, n)
    for dec in (False, True):
        out = aes.ecb(rk, x, dec, variant=aes.AES_VAR_HYBRID, grid=1)
        ok &= np.array_equal(out.cpu().numpy(), oracle.ecb(key, host, dec, 4))
    ok &= np.array_equal(aes.ctr_xcrypt(rk, bytes(range(16)), x, block_offset=5).cpu().numpy(),
                         oracle.ctr(key, bytes(range(16)), host, block_offset=5, nthreads=4))
    ok &= np.array_equal(aes.cbc_decrypt(rk, bytes(16), x).cpu().numpy(), oracle.cbc(key, bytes(16), host, True))
os.environ.pop("AES_B200_HYBRID_MIN_BLOCKS")
torch.cuda.synchronize()
print("sanitize_smoke", "ok" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
