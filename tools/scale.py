#!/usr/bin/env python
"""BASELINE config 5: AES-128 ECB encrypt of a 64 GiB buffer (2^32 blocks)
sharded across N GPUs -- strong scaling (total work fixed).

    python tools/scale.py                                   # N = 1 (64 GiB on one GPU, in place)
    python tools/scale.py --gpus N                          # spawns N ranks itself
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/scale.py --gpus N

Rank r owns blocks [r*n/N, (r+1)*n/N) of the global splitmix64 stream
(dist.shard_range), fills them on its own GPU, checks sampled blocks against
the oracle (including the shard edges and block 2^32-1), and then encrypts its
shard in place K times.  Time = max over ranks of the CUDA-event time of the K
launches between two barriers.  No data-path collective.  One JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1902_05234_b200 as aes
import synth
from paper_1902_05234_b200 import dist as pdist
from synth import golden


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return float(json.load(open(p))["hbm_gbs"]) if os.path.exists(p) else 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--global-bytes", type=int, default=64 << 30)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", 1)))
    ap.add_argument("--keybits", type=int, default=128, choices=[128, 192, 256])
    ap.add_argument("--dir", default="enc", choices=["enc", "dec"], help="the timed in-place operation")
    ap.add_argument("--variant", default="default", choices=["default", "smem_repl", "hybrid", "bitslice"])
    a = ap.parse_args()
    kw = {} if a.variant == "default" else {"variant": {"smem_repl": aes.AES_VAR_SMEM_REPL,
                                                        "hybrid": aes.AES_VAR_HYBRID,
                                                        "bitslice": aes.AES_VAR_BITSLICE}[a.variant]}
    rc = pdist.respawn_under_torchrun(a.gpus, [os.path.abspath(__file__), *sys.argv[1:]])
    if rc is not None:
        return rc
    pdist.require_world(a.gpus)
    rank, world, local = pdist.init(os.environ.get("AES_BENCH_BACKEND") or None)
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    n = a.global_bytes // 16
    b0, b1 = pdist.shard_range(n, rank, world)
    m = b1 - b0
    key = synth.key(a.keybits)
    rk = aes.expand_key(key)
    x = torch.empty(16 * m, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s):
        synth.fill_device(x, first_block=b0)
        aes.ecb(rk, x, False, out=x, **kw)
    s.synchronize()
    # sampled parity: oracle-written golden samples (incl. shard edges and block
    # 2^32-1) for E(x); after an in-place decrypt the same samples must be the input
    gather = lambda loc: x.view(-1, 16)[torch.from_numpy(loc).to(dev)].cpu().numpy()
    try:
        checked = golden.check("ecb_enc", a.keybits, b0, m, gather)
        ok = checked >= 3
    except AssertionError as e:
        print(f"[rank {rank}] {e}", file=sys.stderr)
        ok = False
    idx, _ = golden.samples("ecb_enc", a.keybits)
    g = idx[(idx >= np.uint64(b0)) & (idx < np.uint64(b1))]
    with torch.cuda.stream(s):
        aes.ecb(rk, x, True, out=x, **kw)
    s.synchronize()
    ok &= bool(np.array_equal(gather((g - np.uint64(b0)).astype(np.int64)), synth.blocks_at(g)))
    if pdist.sum_over_ranks(0.0 if ok else 1.0, dev):
        if rank == 0:
            print(json.dumps({"error": "parity failed"}))
        return 1
    with torch.cuda.stream(s):
        for _ in range(a.warmup):
            aes.ecb(rk, x, a.dir == "dec", out=x, **kw)
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pdist.barrier(dev)
    torch.cuda.synchronize(dev)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(a.steps):
            aes.ecb(rk, x, a.dir == "dec", out=x, **kw)
        e1.record(s)
    s.synchronize()
    pdist.barrier(dev)
    ms_local = e0.elapsed_time(e1)
    ms = pdist.max_over_ranks(ms_local, dev)
    ms_min = pdist.min_over_ranks(ms_local, dev)
    devices = pdist.gather_objects(f"{torch.cuda.get_device_name(dev)}#{dev.index}")
    total = pdist.sum_over_ranks(16.0 * m * a.steps, dev)
    if rank == 0:
        gbps = 8 * total / (ms * 1e-3) / 1e9
        what = "encrypt" if a.dir == "enc" else "decrypt"
        print(json.dumps({"metric": f"AES-{a.keybits} ECB {what} Gbps, {a.global_bytes / 2**30:g} GiB sharded"
                                    + (" (BASELINE config 5)" if (a.keybits, a.dir, a.global_bytes) == (128, "enc", 64 << 30)
                                       else ""),
                          "variant": a.variant,
                          "value": gbps, "unit": "Gbps", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
                          "ms_per_step": ms / a.steps, "scaling": "strong", "global_bytes": a.global_bytes,
                          "bytes_per_gpu": 16 * m, "GBps": gbps / 8,
                          "hbm_frac": 32 * total / 16 / (ms * 1e-3) / 1e9 / hbm_peak() / world,
                          "parity": "golden (oracle-written) samples incl. shard edges and block 2^32-1; in-place round trip on the samples",
                          "ranks": {"world": world, "backend": pdist.backend_name(), "ms_min": ms_min,
                                    "ms_max": ms, "devices": devices},
                          "gpu": torch.cuda.get_device_name(dev)}), flush=True)
    pdist.barrier(dev)
    pdist.finalize()
    return 0


if __name__ == "__main__":
    sys.exit(main())
