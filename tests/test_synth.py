"""The seeded input generator (synth/): host numpy twin pinned to the
published splitmix64 stream; the device twin is compared in test_gpu_parity."""
import numpy as np

import synth


def test_splitmix64_reference_values():
    # splitmix64 from state 0: first outputs (Vigna's reference generator)
    w = synth.words(0, 0, 2)
    assert int(w[0]) == 0xE220A8397B1DCDAF
    assert int(w[1]) == 0x6E789E6AA1B965F4


def test_blocks_are_counter_based_and_sliceable():
    a = synth.blocks(0, 100)
    b = synth.blocks(37, 20)
    assert np.array_equal(a[16 * 37:16 * 57], b)
    idx = np.array([0, 5, 99, 2**32 - 1, 2**32, 2**33 + 7], dtype=np.uint64)
    at = synth.blocks_at(idx)
    assert np.array_equal(at[2], a[16 * 99:16 * 100])
    assert np.array_equal(at[4], synth.blocks(2**32, 1))
    assert synth.blocks(0, 3, kind="zeros").sum() == 0
    r = synth.blocks(0, 4, kind="repeat").reshape(4, 16)
    assert (r == r[0]).all()
    t = synth.blocks(0, 64, kind="ascii")
    assert t.min() >= 0x20 and t.max() <= 0x7E


def test_keys():
    for kb in (128, 192, 256):
        k = synth.key(kb)
        assert len(k) == kb // 8
    assert synth.key(128) != synth.key(256)[:16]
