"""tests/golden/samples.txt (used by bench.py / tools/ parity gates) is what
the oracle computes today: re-derive a subset of every op and key size."""
import numpy as np

import oracle
import synth
from synth import golden

IV = bytes(range(16))


def test_samples_file_matches_the_oracle():
    for kb in (128, 192, 256):
        key = synth.key(kb)
        for op in ("ecb_enc", "ecb_dec", "ctr", "cbc_dec"):
            idx, want = golden.samples(op, kb)
            assert len(idx) > 500
            pick = np.r_[0:8, len(idx) - 8:len(idx), np.arange(8, len(idx) - 8, 97)]
            for j in pick:
                i = int(idx[j])
                x = synth.blocks(i, 1)
                if op == "ecb_enc":
                    w = oracle.encrypt(key, x)
                elif op == "ecb_dec":
                    w = oracle.decrypt(key, x)
                elif op == "ctr":
                    w = oracle.ctr(key, IV, x, block_offset=i)
                else:
                    prev = IV if i == 0 else synth.blocks(i - 1, 1).tobytes()
                    w = oracle.cbc(key, prev, x, True)
                assert np.array_equal(w, want[j]), (op, kb, i)


def test_check_helper_detects_mismatch():
    idx, want = golden.samples("ecb_enc", 128)
    first, n = 0, 1 << 20
    table = {int(i): w for i, w in zip(idx, want)}
    n_ok = golden.check("ecb_enc", 128, first, n, lambda loc: np.stack([table[int(l)] for l in loc]))
    assert n_ok > 50
    try:
        golden.check("ecb_enc", 128, first, n, lambda loc: np.zeros((len(loc), 16), np.uint8))
    except AssertionError:
        pass
    else:
        raise AssertionError("mismatch not detected")
