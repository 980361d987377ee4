"""Command line: encrypt / decrypt files on the B200, the way the paper's
program is used (sec 5: files of 1,202 .. 1,190,402 bytes, Tables 4-5).

    python -m paper_1902_05234_b200 enc --key 2b7e1516...3c --in plain.bin --out cipher.bin
    python -m paper_1902_05234_b200 dec --key 2b7e1516...3c --in cipher.bin --out plain.bin
    python -m paper_1902_05234_b200 ladder            # the paper's file-size ladder, timed

ECB files are PKCS#7-padded on encryption and unpadded on decryption (the
library itself only takes whole blocks, R17; --no-pad requires a
whole-block file).  --mode ctr (with --iv) needs no padding.  Files go through
the pipelined host path (aes_pipeline_run): H2D, kernel and D2H of 64 MiB
chunks overlapped on 3 streams.  Timing is printed like the paper's tables
(bytes, seconds, bytes per second).
"""
from __future__ import annotations

import argparse
import sys
import time

import numpy as np


def _pad(data: bytes) -> bytes:
    k = 16 - len(data) % 16
    return data + bytes([k]) * k


def _unpad(data: bytes) -> bytes:
    if not data or len(data) % 16:
        raise SystemExit("ciphertext is not a whole number of blocks")
    k = data[-1]
    if not 1 <= k <= 16 or data[-k:] != bytes([k]) * k:
        raise SystemExit("bad PKCS#7 padding (wrong key?)")
    return data[:-k]


def _run_file(a) -> int:
    import torch

    import paper_1902_05234_b200 as aes
    key = bytes.fromhex(a.key)
    rk = aes.expand_key(key)
    data = open(a.inp, "rb").read()
    decrypt = a.cmd == "dec"
    t0 = time.perf_counter()
    if a.mode == "ecb":
        if not decrypt and not a.no_pad:
            data = _pad(data)
        if len(data) % 16:
            raise SystemExit("input is not a whole number of 16-byte blocks (use padding or --mode ctr)")
        buf = torch.from_numpy(np.frombuffer(data, np.uint8).copy())
        if len(data) >= (1 << 20):
            buf = buf.pin_memory()
        out = torch.empty_like(buf)
        p = aes.Pipeline(chunk_bytes=64 << 20, depth=3)
        p.run(rk, buf, out, decrypt=decrypt)
        p.close()
        res = out.numpy().tobytes()
        if decrypt and not a.no_pad:
            res = _unpad(res)
    else:   # CTR: keystream on the device, any length
        iv = bytes.fromhex(a.iv)
        n = (len(data) + 15) // 16
        x = torch.zeros(16 * n, dtype=torch.uint8)
        x[:len(data)] = torch.from_numpy(np.frombuffer(data, np.uint8).copy())
        y = aes.ctr_xcrypt(rk, iv, x.cuda())
        res = y.cpu().numpy().tobytes()[:len(data)]
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    open(a.out, "wb").write(res)
    size = len(open(a.inp, "rb").read())
    print(f"{a.cmd} {a.mode} AES-{8 * len(key)}: {size} bytes in {dt:.6f} s = {size / dt:,.2f} bytes/s "
          f"(incl. host<->device copies)")
    return 0


def _ladder(a) -> int:
    """The paper's Tables 4-5 file sizes with random
    content: per-file end-to-end time through aes_pipeline_run and the
    device-only time, printed in the paper's columns (GPU side only)."""
    import torch

    import paper_1902_05234_b200 as aes
    sizes = [1202, 4652, 9302, 18602, 37202, 74402, 148802, 297602, 595202, 1190402]
    rng = np.random.default_rng(1)
    rk = aes.expand_key(rng.integers(0, 256, 16, dtype=np.uint8).tobytes())
    p = aes.Pipeline(chunk_bytes=1 << 20, depth=2)
    print(f"{'file size (bytes)':>18} {'dir':>4} {'e2e time (s)':>13} {'e2e bytes/s':>18} {'device time (s)':>16} {'device bytes/s':>18}")
    print("(e2e: host buffers through aes_pipeline_run, best of reps; device: per-launch time of a CUDA graph of reps "
          "back-to-back launches, no host cost)")
    for size in sizes:
        data = _pad(rng.integers(0, 256, size, dtype=np.uint8).tobytes())
        h = torch.from_numpy(np.frombuffer(data, np.uint8).copy()).pin_memory()
        o = torch.empty_like(h).pin_memory()
        d = h.cuda()
        for decrypt in (False, True):
            for _ in range(3):
                p.run(rk, h, o, decrypt=decrypt)
            te = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                p.run(rk, h, o, decrypt=decrypt)
                te.append(time.perf_counter() - t0)
            # device time per launch: a CUDA graph of `reps` launches into a
            # preallocated output, replayed between two events (no host cost)
            out = torch.empty_like(d)
            gs = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            torch.cuda.synchronize()
            with torch.cuda.stream(gs):
                with torch.cuda.graph(g, stream=gs):
                    for _ in range(a.reps):
                        aes.ecb(rk, d, decrypt, out=out)
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(gs):
                e0.record(gs)
                g.replay()
                e1.record(gs)
            torch.cuda.synchronize()
            td = e0.elapsed_time(e1) * 1e-3 / a.reps
            print(f"{size:>18} {'dec' if decrypt else 'enc':>4} {min(te):>13.6f} {size / min(te):>18,.2f} "
                  f"{td:>16.6f} {size / td:>18,.2f}")
    p.close()
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1902_05234_b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("enc", "dec"):
        s = sub.add_parser(name)
        s.add_argument("--key", required=True, help="hex, 16/24/32 bytes")
        s.add_argument("--in", dest="inp", required=True)
        s.add_argument("--out", required=True)
        s.add_argument("--mode", choices=["ecb", "ctr"], default="ecb")
        s.add_argument("--iv", default="00" * 16, help="CTR initial counter block (hex, 16 bytes)")
        s.add_argument("--no-pad", action="store_true", help="ECB without PKCS#7 (whole-block input)")
    s = sub.add_parser("ladder")
    s.add_argument("--reps", type=int, default=20)
    a = ap.parse_args(argv)
    return _ladder(a) if a.cmd == "ladder" else _run_file(a)


if __name__ == "__main__":
    sys.exit(main())
