#!/usr/bin/env python
"""Measurement sweeps beyond bench.py's headline line.

  --what sizes     config 4: sizes 16 KiB .. 16 GiB x {128,192,256} x {enc,dec};
                   fit t = t0 + n/R_inf per (keybits, dir) like the paper's Tables 4-5
  --what variants  NEXT-2 ablation: table placement (replicated smem / plain smem /
                   constant, the paper's choice) x states-per-thread, 1 GiB AES-128,
                   plus data-structure variants (random / zeros / repeat / ascii)
  --what config3   config 3: AES-256 decrypt, 4 GiB
  --what ladder    the paper's file-size ladder (Tables 4-5), device-resident and e2e

Every timed point is preceded by a parity check of that configuration: sampled
blocks against tests/golden/samples.txt (expected values written by the oracle,
tests/golden/make_samples.py) for the random stream, and against the default
kernel (itself oracle-checked in tests/) for the other data kinds.  Buffers smaller than 2x L2 are measured with an
L2 flush (a 512 MiB write) before every rep; larger ones are not.  JSONL on stdout.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_1902_05234_b200 as aes
import synth
from synth import golden

NR = {128: 10, 192: 12, 256: 14}
HYBRID_MIN_BLOCKS = 1 << 23   # aes_ecb.cu: the default kernel is the hybrid one from here up


def kernel_of(n, variant=0):
    if variant == 7 or (variant == 0 and n >= HYBRID_MIN_BLOCKS):
        return "hybrid"
    return {8: "bitslice"}.get(variant, "t_table")


def lds_fields(lookups_per_block, n, t, ldsp, kernel):
    """Lookup-rate fraction of the measured LDS-gather ceiling.  For the hybrid
    kernel 'lookups' are dense-equivalent (every block counted with the T-table
    lookups although the bitsliced warps cipher some blocks without any), so the
    fraction can exceed 1."""
    f = lookups_per_block * n / t / ldsp
    if kernel == "t_table":
        return {"lds_frac": f}
    return {"lds_equiv_frac": f, "lds_note": "dense-equivalent lookups (bitsliced warps do part of the blocks "
                                              "without lookups): > 1 means beyond the T-table-only ceiling"}


def peaks():
    d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    return float(d["hbm_gbs"])


def lds_peak(s):
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    sink = torch.empty(nsm * 1024, dtype=torch.int32, device="cuda")
    best = 0.0
    with torch.cuda.stream(s):
        aes.lds_gather(sink, nsm, 64)
    for _ in range(3):                    # best of 3 x ~4 ms (short runs under-read the ceiling)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            n = aes.lds_gather(sink, nsm, 16384)
            e1.record(s)
        s.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) * 1e-3))
    return best


def _gather(t):
    return lambda loc: t.view(-1, 16)[torch.from_numpy(loc).cuda()].cpu().numpy()


def parity(keybits, out, op):
    """Sampled blocks of `out` (result of `op` on the random stream from block 0)
    against the oracle-written golden samples."""
    n = out.numel() // 16
    if golden.check(op, keybits, 0, n, _gather(out)) < 1:
        raise SystemExit(f"no golden samples for n={n}")


def time_op(fn, s, reps, flush=None):
    ts = []
    for _ in range(reps):
        if flush is not None:
            with torch.cuda.stream(s):
                flush.zero_()          # on the timed stream, so it completes before e0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            fn()
            e1.record(s)
        s.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return min(ts), statistics.median(ts)


def time_graph_b2b(fn, s, reps):
    """Per-launch DEVICE time of `reps` back-to-back launches captured in a CUDA
    graph and replayed between two events (no host enqueue cost inside)."""
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    g.replay()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        s.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3 / reps)
    del g
    return best


def time_eager_b2b(fn, s, reps):
    """Mean time per launch of `reps` eager launches issued back to back (the
    host enqueue cost bounds it when a launch is shorter than its call)."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        fn()
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


def time_device_single(fn, s, reps, flush=None):
    """One launch between two events, queued behind a GPU spin so the host
    enqueue cost is outside the interval (isolated-launch device time)."""
    ts = []
    for _ in range(reps):
        with torch.cuda.stream(s):
            if flush is not None:
                flush.zero_()
            torch.cuda._sleep(40000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
        s.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return min(ts), statistics.median(ts)


def time_host_call(fn, reps=200):
    """Host cost of one call (Python wrapper -> C ABI -> cudaLaunchKernelExC),
    mean over back-to-back calls."""
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / reps


def record(**kw):
    print(json.dumps(kw), flush=True)


def sizes(a, s, hbm, ldsp):
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    sz = [16 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20, 1 << 30, 4 << 30]
    if a.big:
        sz.append(16 << 30)
    fits = {}
    for nbytes in sz:
        x = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        synth.fill_device(x)
        out = torch.empty_like(x)
        n = nbytes // 16
        for kb in (128, 192, 256):
            key = synth.key(kb)
            rk = aes.expand_key(key)
            for dec in (False, True):
                f = (lambda: aes.ecb(rk, x, dec, out=out))
                f()
                torch.cuda.synchronize()
                parity(kb, out, "ecb_dec" if dec else "ecb_enc")
                reps = 20 if nbytes < (4 << 30) else 5
                warm = nbytes >= 2 * l2
                for _ in range(3):
                    f()
                torch.cuda.synchronize()   # warm-ups ran on the default stream; s is non-blocking
                tmin, tmed = time_op(f, s, reps, None if warm else flush)
                dmin, dmed = time_device_single(f, s, reps, None if warm else flush)
                tb2b = time_graph_b2b(f, s, 20) if nbytes < (256 << 20) else dmin
                thost = time_host_call(f, 200 if nbytes < (16 << 20) else 5)
                g = 8 * nbytes / dmin / 1e9
                fits.setdefault((kb, dec), []).append((n, dmin, tb2b))
                record(what="size", bytes=nbytes, keybits=kb, dir="dec" if dec else "enc",
                       t_call_min_s=tmin, t_call_med_s=tmed, t_device_min_s=dmin, t_device_med_s=dmed,
                       t_graph_b2b_s=tb2b, t_host_call_s=thost, Gbps=g, GBps=g / 8,
                       Gbps_graph_b2b=8 * nbytes / tb2b / 1e9,
                       hbm_frac=32 * n / dmin / 1e9 / hbm, kernel=kernel_of(n),
                       **lds_fields(16 * NR[kb], n, dmin, ldsp, kernel_of(n)),
                       l2="flushed" if not warm else "input>2xL2",
                       note="t_call: events around one call incl. host enqueue; t_device: one launch queued "
                            "behind a GPU spin (device time of an isolated launch, L2 flushed if small); "
                            "t_graph_b2b: per-launch device time of 20 back-to-back launches in a CUDA graph "
                            "(PDL overlap, L2 warm if small; = t_device for >= 256 MiB); t_host_call: host "
                            "cost of one Python-wrapper call")
        del x, out
        torch.cuda.empty_cache()
    for (kb, dec), pts in fits.items():
        nn = np.array([p[0] for p in pts], float)
        A = np.stack([np.ones_like(nn), nn], 1)
        for col, which in ((1, "device_single"), (2, "graph_b2b")):
            tt = np.array([p[col] for p in pts], float)
            (t0, inv), *_ = np.linalg.lstsq(A, tt, rcond=None)
            record(what="fit", keybits=kb, dir="dec" if dec else "enc", timing=which, t0_us=t0 * 1e6,
                   R_inf_GBps=16 / inv / 1e9 if inv > 0 else None)


def variants(a, s, hbm, ldsp):
    nbytes = 1 << 30
    x = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    out = torch.empty_like(x)
    n = nbytes // 16
    key = synth.key(128)
    rk = aes.expand_key(key)
    names = {1: "smem_repl", 2: "smem_plain", 3: "const (paper)", 4: "smem_repl + TMA staging", 5: "one table + rotations",
             6: "global __ldg (L1)", 7: "hybrid (T-table + bitsliced warps)", 8: "bitsliced only"}
    for kind in ("random", "zeros", "repeat", "ascii"):
        synth.fill_device(x, kind=kind)
        for v, spt in ((1, 1), (1, 2), (1, 4), (4, 1), (5, 1), (2, 1), (6, 1), (3, 1), (7, 1), (8, 1)):
            if kind != "random" and (v == 1 and spt != 1 or v in (4, 5, 8)):
                continue
            for dec in (False, True):
                f = (lambda: aes.ecb(rk, x, dec, out=out, variant=v, states_per_thread=spt))
                f()
                torch.cuda.synchronize()
                if kind == "random":
                    parity(128, out, "ecb_dec" if dec else "ecb_enc")
                else:
                    assert torch.equal(out, aes.ecb(rk, x, dec)), ("variant mismatch", v, spt, kind)
                reps = 10 if v not in (3, 6) else 3
                tmin, tmed = time_op(f, s, reps)
                g = 8 * nbytes / tmin / 1e9
                record(what="variant", variant=names[v], spt=spt, data=kind, dir="dec" if dec else "enc",
                       keybits=128, bytes=nbytes, t_min_s=tmin, t_med_s=tmed, Gbps=g,
                       hbm_frac=32 * n / tmin / 1e9 / hbm, **lds_fields(160, n, tmin, ldsp, kernel_of(n, v)))


def config3(a, s, hbm, ldsp):
    nbytes = 4 << 30
    x = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    synth.fill_device(x)
    key = synth.key(256)
    rk = aes.expand_key(key)
    ct = aes.ecb_encrypt(rk, x)               # made outside the timed region
    out = torch.empty_like(x)
    f = (lambda: aes.ecb_decrypt(rk, ct, out=out))
    f()
    torch.cuda.synchronize()
    assert torch.equal(out, x)
    parity(256, ct, "ecb_enc")
    for _ in range(3):
        f()
    torch.cuda.synchronize()   # warm-ups ran on the default stream; s is non-blocking
    tmin, tmed = time_op(f, s, 10)
    n = nbytes // 16
    g = 8 * nbytes / tmin / 1e9
    record(what="config3", keybits=256, dir="dec", bytes=nbytes, t_min_s=tmin, t_med_s=tmed, Gbps=g,
           hbm_frac=32 * n / tmin / 1e9 / hbm, kernel=kernel_of(n), **lds_fields(224, n, tmin, ldsp, kernel_of(n)))


def ladder(a, s, hbm, ldsp):
    files = [1202, 4652, 9302, 18602, 37202, 74402, 148802, 297602, 595202, 1190402]
    key = synth.key(128)
    rk = aes.expand_key(key)
    pipe = aes.Pipeline(chunk_bytes=1 << 20, depth=2)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for fb in files:
        nb = (fb + 15) // 16
        x = torch.empty(16 * nb, dtype=torch.uint8, device="cuda")
        synth.fill_device(x)
        out = torch.empty_like(x)
        hx = x.cpu().pin_memory()
        ho = torch.empty_like(hx).pin_memory()
        for dec in (False, True):
            f = (lambda: aes.ecb(rk, x, dec, out=out))
            f()
            torch.cuda.synchronize()
            parity(128, out, "ecb_dec" if dec else "ecb_enc")
            tmin, tmed = time_op(f, s, 20, flush)
            import time
            pipe.run(rk, hx, ho, decrypt=dec)
            te = []
            for _ in range(20):
                t0 = time.perf_counter()
                pipe.run(rk, hx, ho, decrypt=dec)
                te.append(time.perf_counter() - t0)
            assert np.array_equal(ho.numpy(), out.cpu().numpy())
            record(what="ladder", file_bytes=fb, blocks=nb, dir="dec" if dec else "enc",
                   kernel_t_min_s=tmin, kernel_Bps=fb / tmin, e2e_t_min_s=min(te), e2e_Bps=fb / min(te),
                   paper_gpu_Bps=None)


def modes(a, s, hbm, ldsp):
    """NEXT-1 CTR and NEXT-4 CBC decryption at 1 GiB, all key sizes."""
    nbytes = 1 << 30
    x = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    synth.fill_device(x)
    out = torch.empty_like(x)
    n = nbytes // 16
    iv = bytes(range(16))
    for kb in (128, 192, 256):
        key = synth.key(kb)
        rk = aes.expand_key(key)
        for mode in ("ctr", "cbc_dec"):
            if mode == "ctr":
                f = (lambda: aes.ctr_xcrypt(rk, iv, x, out=out))
            else:
                f = (lambda: aes.cbc_decrypt(rk, iv, x, out=out))
            # default kernel (hybrid at 1 GiB), then the T-table-only kernel of the mode
            for kern, knob in (("hybrid", None), ("t_table", str(1 << 62))):
                if knob:
                    os.environ["AES_B200_HYBRID_MIN_BLOCKS"] = knob
                try:
                    f()
                    torch.cuda.synchronize()
                    parity(kb, out, "ctr" if mode == "ctr" else "cbc_dec")
                    for _ in range(3):
                        f()
                    torch.cuda.synchronize()   # warm-ups ran on the default stream; s is non-blocking
                    tmin, tmed = time_op(f, s, 10)
                finally:
                    os.environ.pop("AES_B200_HYBRID_MIN_BLOCKS", None)
                g = 8 * nbytes / tmin / 1e9
                # the method's own work: CTR with counter-mode caching does 16(Nr-2)+5 lookups per
                # block plus 27 per warp per 16 trips for its group tables (27/512 per block);
                # CBC decryption moves 32 DRAM bytes per block (the neighbour block re-read
                # hits L1/L2) while requesting 48
                looks = 16 * (NR[kb] - 2) + 5 + 27 / 512 if mode == "ctr" else 16 * NR[kb]
                record(what="mode", mode=mode, kernel=kern, keybits=kb, bytes=nbytes, t_min_s=tmin, t_med_s=tmed,
                       Gbps=g, hbm_frac=32 * n / tmin / 1e9 / hbm,
                       requested_bytes_per_block=48 if mode == "cbc_dec" else 32,
                       lookups_per_block=looks, **lds_fields(looks, n, tmin, ldsp, kern),
                       note="hbm_frac counts 32 DRAM bytes per block (16 read + 16 written); lookups count "
                            "the T-table work of this mode")


def batch(a, s, hbm, ldsp):
    """The paper's file ladder as a serving workload: M files of one size,
    each with its own key, encrypted by ONE aes_ecb_batch launch vs M calls."""
    import time
    files = [1202, 4652, 9302, 18602, 37202, 74402, 148802, 297602, 595202, 1190402]
    rng = np.random.default_rng(7)
    rks = [aes.expand_key(rng.integers(0, 256, 16, dtype=np.uint8).tobytes()) for _ in range(64)]
    for fb in files:
        nb = (fb + 15) // 16
        M = max(64, min(4096, (1 << 28) // (16 * nb)))
        base = torch.empty(16 * nb * M, dtype=torch.uint8, device="cuda")
        synth.fill_device(base)
        out = torch.empty_like(base)
        xs = [base[16 * nb * i:16 * nb * (i + 1)] for i in range(M)]
        os_ = [out[16 * nb * i:16 * nb * (i + 1)] for i in range(M)]
        kidx = [i % 64 for i in range(M)]
        offs = np.arange(M, dtype=np.uint64) * np.uint64(16 * nb)
        nbs = np.full(M, nb, dtype=np.uint64)
        kid = np.array(kidx, dtype=np.uint32)
        kset = aes.KeySet(rks)
        fbatch = (lambda: aes.ecb_batch_offsets(kset, base.data_ptr(), out.data_ptr(), offs, offs, nbs, kid))
        fbatch()
        torch.cuda.synchronize()
        # parity: message i under key i % 64 -- check message 0 and 1 against the
        # per-call path (itself golden/oracle-checked)
        for i in (0, 1, M - 1):
            assert torch.equal(os_[i], aes.ecb_encrypt(rks[kidx[i]], xs[i]))
        for _ in range(3):
            fbatch()
        torch.cuda.synchronize()
        tb, _ = time_op(fbatch, s, 10)
        tbd = time_eager_b2b(fbatch, s, 10)     # back to back, eager (aes_ecb_batch is not graph-capturable)
        # M separate calls, back to back (host launch path included, as a user would see it)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            for i in range(M):
                aes.ecb_encrypt(rks[kidx[i]], xs[i], out=os_[i])
        s.synchronize()
        tc = time.perf_counter() - t0
        payload = 16 * nb * M
        record(what="batch", file_bytes=fb, blocks_per_file=nb, files=M, batch_t_s=tb, batch_GBps=payload / tb / 1e9,
               batch_b2b_t_s=tbd, batch_b2b_GBps=payload / tbd / 1e9,
               per_call_t_s=tc, per_call_GBps=payload / tc / 1e9, speedup=tc / tb,
               lds_frac=160 * nb * M / tb / ldsp)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="variants", choices=["sizes", "variants", "config3", "ladder", "modes", "batch", "all"])
    ap.add_argument("--big", action="store_true", help="include 16 GiB in the size sweep")
    a = ap.parse_args()
    s = torch.cuda.Stream()
    hbm = peaks()
    ldsp = lds_peak(s)
    record(what="peaks", hbm_gbs=hbm, lds_lookups_per_s=ldsp, gpu=torch.cuda.get_device_name(0))
    todo = ["variants", "config3", "modes", "sizes", "ladder", "batch"] if a.what == "all" else [a.what]
    from bench import ClockSampler
    clk = ClockSampler(torch.cuda.current_device())
    clk.start()
    clk.mark_start()
    for w in todo:
        globals()[w](a, s, hbm, ldsp)
    clk.mark_end()
    record(what="clocks", **clk.stop())


if __name__ == "__main__":
    main()
