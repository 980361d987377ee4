"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact, zero tolerance (integer work with a unique result, R23).
Inputs are the seeded splitmix64 stream (synth/), the same bytes on both
sides; expected values come only from oracle/.  Sizes span one warp, several
CTAs and ragged tails; full BASELINE sizes are checked on sampled blocks the
oracle computes one by one, plus an on-device round trip.
"""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle
import synth
from conftest import golden

VARIANTS = [(1, 1), (1, 2), (1, 4), (2, 1), (3, 1), (4, 1), (5, 1), (6, 1), (7, 1), (8, 1)]   # (variant, states_per_thread)
# one warp .. several CTAs, ragged tails, 1 MiB, and whole grid-stride trips + a per-CTA tail split
SIZES = [1, 2, 31, 32, 33, 1023, 1024, 1025, 4096 + 17, 148 * 1024 + 7, 65536, 2 * 148 * 1024 + 30011]


@pytest.fixture(scope="module")
def aes():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1902_05234_b200 as m
    assert torch.cuda.is_available(), "GPU test on a box without CUDA"
    return m


def _dev_rand(n, first=0, kind="random"):
    x = torch.empty(16 * n, dtype=torch.uint8, device="cuda")
    synth.fill_device(x, first_block=first, kind=kind)
    return x


def test_device_generator_matches_host_twin(aes):
    for first, n in ((0, 1000), (12345, 777)):
        x = _dev_rand(n, first)
        assert np.array_equal(x.cpu().numpy(), synth.blocks(first, n))
    for kind in ("zeros", "repeat", "ascii"):
        x = _dev_rand(300, 0, kind)
        assert np.array_equal(x.cpu().numpy(), synth.blocks(0, 300, kind=kind))


def test_fips197_and_sp800_38a_vectors_all_variants(aes):
    rows = [ln.split() for ln in open(golden("fips197_appC.txt")) if ln.strip() and not ln.startswith("#")]
    sp = [ln.split() for ln in open(golden("sp800_38a_ecb.txt")) if ln.strip() and not ln.startswith("#")]
    pt4 = bytes.fromhex("".join(sp[0][1:]))
    for i in range(1, 7, 2):
        rows.append([sp[i][1], pt4.hex(), "".join(sp[i + 1][1:])])
    for key, pt, ct in rows:
        rk = aes.expand_key(bytes.fromhex(key))
        x = torch.frombuffer(bytearray(bytes.fromhex(pt)), dtype=torch.uint8).cuda()
        c = torch.frombuffer(bytearray(bytes.fromhex(ct)), dtype=torch.uint8).cuda()
        for v, spt in VARIANTS:
            got = aes.ecb_encrypt(rk, x, variant=v, states_per_thread=spt)
            assert got.cpu().numpy().tobytes().hex() == ct, (key, v, spt)
            back = aes.ecb_decrypt(rk, c, variant=v, states_per_thread=spt)
            assert back.cpu().numpy().tobytes().hex() == pt, (key, v, spt)


@pytest.mark.parametrize("keybits", [128, 192, 256])
def test_random_buffers_against_oracle(aes, keybits):
    key = synth.key(keybits)
    rk = aes.expand_key(key)
    for n in SIZES:
        x = _dev_rand(n, first=n)
        host = synth.blocks(n, n)
        want_ct = oracle.encrypt(key, host, nthreads=8)
        want_pt = oracle.decrypt(key, host, nthreads=8)   # decrypt of arbitrary input
        for v, spt in VARIANTS:
            ct = aes.ecb_encrypt(rk, x, variant=v, states_per_thread=spt).cpu().numpy()
            assert np.array_equal(ct, want_ct), (keybits, n, v, spt, int(np.argmax(ct != want_ct)) // 16)
            pt = aes.ecb_decrypt(rk, x, variant=v, states_per_thread=spt).cpu().numpy()
            assert np.array_equal(pt, want_pt), (keybits, n, v, spt)


def test_small_grids_many_trips_and_in_place(aes):
    key = synth.key(128)
    rk = aes.expand_key(key)
    n = 3 * 1024 * 4 + 5
    x = _dev_rand(n)
    want = oracle.encrypt(key, synth.blocks(0, n), nthreads=8)
    for grid in (1, 2, 3, 7):
        for spt in (1, 2, 4):
            ct = aes.ecb_encrypt(rk, x, grid=grid, variant=1, states_per_thread=spt)
            assert np.array_equal(ct.cpu().numpy(), want), (grid, spt)
    y = x.clone()
    aes.ecb_encrypt(rk, y, out=y)
    assert np.array_equal(y.cpu().numpy(), want)
    aes.ecb_decrypt(rk, y, out=y)
    assert torch.equal(y, x)


@pytest.mark.parametrize("keybits", [128, 192, 256])
def test_hybrid_both_paths_against_oracle(aes, keybits):
    """AES_VAR_HYBRID with few CTAs: each CTA then needs > kTailUnits units, so
    its bitsliced warps take part (they stop claiming kTailUnits units before
    the end) next to the T-table warps; ragged tail, in place, both directions."""
    key = synth.key(keybits)
    rk = aes.expand_key(key)
    for n, grid in ((65536 + 1234, 1), (3 * 32 * 1024 + 77, 3), (148 * 32 * 400 + 5, 148)):
        x = _dev_rand(n, first=7 * n)
        src = synth.blocks(7 * n, n)
        want_ct = oracle.encrypt(key, src, nthreads=16)
        want_pt = oracle.decrypt(key, src, nthreads=16)
        ct = aes.ecb_encrypt(rk, x, grid=grid, variant=aes.AES_VAR_HYBRID)
        assert np.array_equal(ct.cpu().numpy(), want_ct), (keybits, n, grid)
        pt = aes.ecb_decrypt(rk, x, grid=grid, variant=aes.AES_VAR_HYBRID)
        assert np.array_equal(pt.cpu().numpy(), want_pt), (keybits, n, grid)
        y = x.clone()
        aes.ecb_encrypt(rk, y, out=y, grid=grid, variant=aes.AES_VAR_HYBRID)
        assert np.array_equal(y.cpu().numpy(), want_ct), ("in place", keybits, n, grid)
    for grid in (1, 2, 5):   # the bitsliced-only kernel: partial 8-unit groups at every grid size
        n = 8 * 256 * grid + 129
        x = _dev_rand(n)
        want = oracle.encrypt(key, synth.blocks(0, n), nthreads=16)
        ct = aes.ecb_encrypt(rk, x, grid=grid, variant=aes.AES_VAR_BITSLICE)
        assert np.array_equal(ct.cpu().numpy(), want), ("bitslice", keybits, n, grid)


def _cbc_decrypt_oracle(key, iv, ct, parts=16):
    """oracle.cbc decryption in independent chunks (chunk k's IV is the last
    ciphertext block of chunk k-1), run on host threads (ctypes drops the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    n = ct.size // 16
    cuts = [n * k // parts for k in range(parts + 1)]
    cb = ct.reshape(-1, 16)

    def one(k):
        a, b = cuts[k], cuts[k + 1]
        v = iv if a == 0 else cb[a - 1].tobytes()
        return oracle.cbc(key, v, cb[a:b].reshape(-1).copy(), decrypt=True)
    with ThreadPoolExecutor(parts) as ex:
        return np.concatenate(list(ex.map(one, range(parts))))


@pytest.mark.parametrize("keybits", [128, 256])
def test_hybrid_ctr_and_cbc_against_oracle(aes, keybits, monkeypatch):
    """The NEXT modes on the hybrid kernel (T-table warps with counter-mode
    caching / CBC chaining + bitsliced warps).  The crossover knob puts the
    hybrid under a 3M-block input (~640 units per CTA, so the bitsliced warps
    take part), checked on every block against the oracle."""
    monkeypatch.setenv("AES_B200_HYBRID_MIN_BLOCKS", "0")
    key = synth.key(keybits)
    rk = aes.expand_key(key)
    n = 3 * 2**20 + 12345
    x = _dev_rand(n, first=11)
    host = synth.blocks(11, n)
    iv = bytes(8) + bytes([0xFF] * 7) + bytes([0xF0])          # low counter half wraps inside the buffer
    for off in (0, 2**64 - 2**20):
        got = aes.ctr_xcrypt(rk, iv, x, block_offset=off).cpu().numpy()
        want = oracle.ctr(key, iv, host, block_offset=off, nthreads=16)
        assert np.array_equal(got, want), ("ctr", keybits, off, int(np.argmax(got != want)) // 16)
    civ = bytes(range(16))
    got = aes.cbc_decrypt(rk, civ, x).cpu().numpy()
    want = _cbc_decrypt_oracle(key, civ, host)
    assert np.array_equal(got, want), ("cbc", keybits, int(np.argmax(got != want)) // 16)


def test_data_structure_variants(aes):
    key = synth.key(128)
    rk = aes.expand_key(key)
    for kind in ("zeros", "repeat", "ascii"):
        x = _dev_rand(5000, kind=kind)
        want = oracle.encrypt(key, synth.blocks(0, 5000, kind=kind), nthreads=8)
        assert np.array_equal(aes.ecb_encrypt(rk, x).cpu().numpy(), want), kind


def test_empty_buffer_and_errors_on_device(aes):
    from paper_1902_05234_b200 import _native
    rk = aes.expand_key(bytes(16))
    e = torch.empty(0, dtype=torch.uint8, device="cuda")
    assert aes.ecb_encrypt(rk, e).numel() == 0
    host = np.zeros(64, np.uint8)
    code = _native.lib.aes_ecb_encrypt(ctypes.byref(rk.c), 10, ctypes.c_void_p(host.ctypes.data),
                                       ctypes.c_void_p(host.ctypes.data), 4, None)
    assert code == _native.AES_ENOTDEVICE
    pinned = torch.zeros(64, dtype=torch.uint8).pin_memory()
    code = _native.lib.aes_ecb_encrypt(ctypes.byref(rk.c), 10, ctypes.c_void_p(pinned.data_ptr()),
                                       ctypes.c_void_p(pinned.data_ptr()), 4, None)
    assert code == _native.AES_ENOTDEVICE
    x = torch.zeros(64 + 8, dtype=torch.uint8, device="cuda")
    with pytest.raises(aes.AesError):
        aes.ecb_encrypt(rk, x[8:], out=torch.empty(64, dtype=torch.uint8, device="cuda"))


def test_concurrent_streams_different_keys(aes):
    n = 200000
    x = _dev_rand(n)
    host = synth.blocks(0, n)
    outs = []
    streams = [torch.cuda.Stream() for _ in range(3)]
    keys = [synth.key(128), synth.key(192), synth.key(256)]
    torch.cuda.synchronize()
    for s, k in zip(streams, keys):
        with torch.cuda.stream(s):
            outs.append(aes.ecb_encrypt(aes.expand_key(k), x))
    torch.cuda.synchronize()
    for o, k in zip(outs, keys):
        sel = np.r_[0:64, n - 64:n]
        want = oracle.encrypt(k, host.reshape(-1, 16)[sel].copy().reshape(-1))
        assert np.array_equal(o.cpu().numpy().reshape(-1, 16)[sel].reshape(-1), want)


def test_host_pipeline_end_to_end(aes):
    key = synth.key(256)
    rk = aes.expand_key(key)
    n = 70001
    host = synth.blocks(0, n)
    src = torch.from_numpy(host.copy()).pin_memory()
    dst = torch.empty_like(src).pin_memory()
    p = aes.Pipeline(chunk_bytes=16 * 4099, depth=3)
    p.run(rk, src, dst)
    want = oracle.encrypt(key, host, nthreads=8)
    assert np.array_equal(dst.numpy(), want)
    p.run(rk, dst, dst, decrypt=True)   # in place
    assert np.array_equal(dst.numpy(), host)
    p.close()


def _sample_idx(n, k=4096, seed=0):
    rng = np.random.default_rng(seed)
    edges = [0, 1, 2, n // 2 - 1, n // 2, n - 2, n - 1]
    return np.unique(np.r_[edges, rng.integers(0, n, k)]).astype(np.int64)


def test_config2_aes128_1gib_sampled_parity_and_round_trip(aes):
    """BASELINE config 2 at full size: 1 GiB, AES-128, enc and dec, the
    bench launch configuration (default variant, persistent grid)."""
    n = (1 << 30) // 16
    key = synth.key(128)
    rk = aes.expand_key(key)
    x = _dev_rand(n)
    ct = aes.ecb_encrypt(rk, x)
    back = aes.ecb_decrypt(rk, ct)
    assert torch.equal(back, x)
    idx = _sample_idx(n)
    want = oracle.encrypt(key, synth.blocks_at(idx.astype(np.uint64)).reshape(-1), nthreads=8)
    got = ct.view(-1, 16)[torch.from_numpy(idx).cuda()].cpu().numpy().reshape(-1)
    assert np.array_equal(got, want)


def test_config3_aes256_4gib_decrypt_sampled(aes):
    """BASELINE config 3: AES-256 decrypt of a 4 GiB buffer (byte offsets
    >= 2^32).  The ciphertext is the ORACLE's encryption at the sampled
    blocks; the GPU decrypt must give back the generator's plaintext."""
    free, _ = torch.cuda.mem_get_info()
    if free < 10 * (1 << 30):
        pytest.skip("needs ~10 GiB free")
    n = (4 << 30) // 16
    key = synth.key(256)
    rk = aes.expand_key(key)
    x = _dev_rand(n)
    ct = aes.ecb_encrypt(rk, x)
    idx = _sample_idx(n, seed=1)
    idx = np.unique(np.r_[idx, (1 << 28) - 1, (1 << 28) - 2, ((1 << 32) // 16) - 1, (1 << 32) // 16])
    idx = idx[idx < n]
    sample_pt = synth.blocks_at(idx.astype(np.uint64)).reshape(-1)
    sample_ct = oracle.encrypt(key, sample_pt, nthreads=8)
    tidx = torch.from_numpy(idx).cuda()
    assert np.array_equal(ct.view(-1, 16)[tidx].cpu().numpy().reshape(-1), sample_ct)
    # overwrite the sampled blocks with the oracle's ciphertext, then GPU-decrypt all 4 GiB
    ct.view(-1, 16)[tidx] = torch.from_numpy(sample_ct.reshape(-1, 16)).cuda()
    pt = aes.ecb_decrypt(rk, ct, out=ct)
    assert torch.equal(pt, x)
    del x, ct


def test_config3_aes256_4gib_decrypt_full_parity(aes):
    """BASELINE config 3, FULL parity (Table 5,
    PAPER.md:525-553): the GPU decrypts the whole 4 GiB AES-256 buffer (the
    splitmix64 stream read as ciphertext; byte offsets >= 2^32) in the bench's
    launch configuration, and every one of its 2^28 blocks is compared with
    the oracle's InvCipher of the host twin of the same stream, chunk by chunk
    on all host cores.  Then the GPU round trip E(D(x)) == x."""
    import os
    import time
    free, _ = torch.cuda.mem_get_info()
    if free < 10 * (1 << 30):
        pytest.skip("needs ~10 GiB free")
    n = (4 << 30) // 16
    key = synth.key(256)
    rk = aes.expand_key(key)
    x = _dev_rand(n)
    pt = aes.ecb_decrypt(rk, x)
    torch.cuda.synchronize()
    cores = len(os.sched_getaffinity(0))
    chunk = 1 << 22                                    # 64 MiB of host memory per side
    t0 = time.perf_counter()
    for first in range(0, n, chunk):
        nb = min(chunk, n - first)
        want = oracle.decrypt(key, synth.blocks(first, nb), nthreads=cores)
        got = pt[16 * first:16 * (first + nb)].cpu().numpy()
        if not np.array_equal(got, want):
            bad = np.nonzero((got.reshape(-1, 16) != want.reshape(-1, 16)).any(axis=1))[0]
            pytest.fail(f"AES-256 decrypt mismatch: first bad block {first + int(bad[0])} "
                        f"({len(bad)} bad blocks in chunk at {first})")
    print(f"config 3 full parity: {n} blocks on {cores} cores in {time.perf_counter() - t0:.1f} s")
    back = aes.ecb_encrypt(rk, pt, out=pt)
    assert torch.equal(back, x)
    del x, pt


def test_lds_gather_microbenchmark_runs(aes):
    sink = torch.zeros(148 * 1024, dtype=torch.int32, device="cuda")
    aes.lds_gather(sink, 148, 4)
    torch.cuda.synchronize()
    assert int(sink.abs().sum().item()) != 0


# ---------------------------------------------------------------------------
# NEXT-1 CTR and NEXT-4 CBC decryption
# ---------------------------------------------------------------------------
def _modes_golden():
    rows = [ln.split() for ln in open(golden("sp800_38a_ctr_cbc.txt")) if ln.strip() and not ln.startswith("#")]
    sp = [ln.split() for ln in open(golden("sp800_38a_ecb.txt")) if ln.strip() and not ln.startswith("#")]
    pt = bytes.fromhex("".join(sp[0][1:]))
    sets = [(bytes.fromhex(rows[i][1]), bytes.fromhex("".join(rows[i + 1][1:])),
             bytes.fromhex("".join(rows[i + 2][1:]))) for i in range(2, len(rows), 3)]
    return bytes.fromhex(rows[0][1]), bytes.fromhex(rows[1][1]), pt, sets


def test_ctr_cbc_sp800_38a_vectors(aes):
    ctr_iv, cbc_iv, pt, sets = _modes_golden()
    tp = torch.frombuffer(bytearray(pt), dtype=torch.uint8).cuda()
    for key, ctr_ct, cbc_ct in sets:
        rk = aes.expand_key(key)
        assert aes.ctr_xcrypt(rk, ctr_iv, tp).cpu().numpy().tobytes() == ctr_ct
        tc = torch.frombuffer(bytearray(cbc_ct), dtype=torch.uint8).cuda()
        assert aes.cbc_decrypt(rk, cbc_iv, tc).cpu().numpy().tobytes() == pt


@pytest.mark.parametrize("keybits", [128, 192, 256])
def test_ctr_random_against_oracle_wrap_and_offsets(aes, keybits):
    key = synth.key(keybits)
    rk = aes.expand_key(key)
    rng = np.random.default_rng(keybits)
    ivs = [bytes([0xFF] * 16), bytes(8) + bytes([0xFF] * 8), rng.integers(0, 256, 16, dtype=np.uint8).tobytes()]
    for n in (1, 33, 1025, 148 * 1024 + 7):
        x = _dev_rand(n, first=7 * n)
        host = synth.blocks(7 * n, n)
        for iv in ivs:
            for off in (0, 12345, 2**64 - 3):
                got = aes.ctr_xcrypt(rk, iv, x, block_offset=off).cpu().numpy()
                assert np.array_equal(got, oracle.ctr(key, iv, host, block_offset=off, nthreads=8)), (n, iv.hex(), off)
    # in place round trip
    x = _dev_rand(5000)
    y = x.clone()
    aes.ctr_xcrypt(rk, ivs[2], y, out=y)
    aes.ctr_xcrypt(rk, ivs[2], y, out=y)
    assert torch.equal(x, y)


@pytest.mark.parametrize("keybits", [128, 256])
def test_cbc_decrypt_against_oracle_and_sharding(aes, keybits):
    key = synth.key(keybits)
    rk = aes.expand_key(key)
    iv = bytes(range(16))
    for n in (1, 2, 33, 1025, 148 * 1024 + 7):
        pt = synth.blocks(0, n)
        ct = oracle.cbc(key, iv, pt, decrypt=False)            # sequential oracle encryption
        tc = torch.from_numpy(ct.copy()).cuda()
        got = aes.cbc_decrypt(rk, iv, tc).cpu().numpy()
        assert np.array_equal(got, pt), n
        if n > 2:                                             # two shards, second uses C_{m-1} as its IV
            m = n // 2
            a = aes.cbc_decrypt(rk, iv, tc[:16 * m]).cpu().numpy()
            b = aes.cbc_decrypt(rk, ct[16 * (m - 1):16 * m].tobytes(), tc[16 * m:]).cpu().numpy()
            assert np.array_equal(np.r_[a, b], pt)
    with pytest.raises(aes.AesError):
        aes.cbc_decrypt(rk, iv, tc, out=tc)


def test_config5_64gib_in_place_block_indices_past_2_32(aes):
    """BASELINE config 5's buffer on one GPU: 64 GiB = 2^32 blocks (block
    indices and byte offsets beyond 32 bits), AES-128 encrypt in place,
    sampled oracle parity around block 2^32-1 and at both ends, then decrypt
    in place and check the same samples against the generator."""
    free, _ = torch.cuda.mem_get_info()
    nbytes = 64 << 30
    if free < nbytes + (4 << 30):
        pytest.skip("needs ~68 GiB free")
    n = nbytes // 16
    key = synth.key(128)
    rk = aes.expand_key(key)
    x = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    synth.fill_device(x)
    aes.ecb_encrypt(rk, x, out=x)
    idx = _sample_idx(n, k=2048, seed=5)
    idx = np.unique(np.r_[idx, n - 1, n - 2, (1 << 32) - 1, (1 << 28), (1 << 28) - 1])
    idx = idx[idx < n]
    plain = synth.blocks_at(idx.astype(np.uint64)).reshape(-1)
    tidx = torch.from_numpy(idx).cuda()
    got = x.view(-1, 16)[tidx].cpu().numpy().reshape(-1)
    assert np.array_equal(got, oracle.encrypt(key, plain, nthreads=8))
    aes.ecb_decrypt(rk, x, out=x)
    assert np.array_equal(x.view(-1, 16)[tidx].cpu().numpy().reshape(-1), plain)
    del x
    torch.cuda.empty_cache()


def test_host_threads_call_concurrently(aes):
    """The ABI is re-entrant: 8 host threads, each with its own key and stream."""
    import threading
    n = 4099
    host = synth.blocks(0, n)
    x = _dev_rand(n)
    results, errors = {}, []

    def work(t):
        try:
            kb = (128, 192, 256)[t % 3]
            key = bytes((t * 31 + i) & 0xFF for i in range(kb // 8))
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(20):
                    rk = aes.expand_key(key)
                    ct = aes.ecb_encrypt(rk, x)
                    back = aes.ecb_decrypt(rk, ct)
            s.synchronize()
            results[t] = (key, ct.cpu().numpy(), bool(torch.equal(back, x)))
        except Exception as e:   # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=work, args=(t,)) for t in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors
    for t, (key, ct, ok) in results.items():
        assert ok
        assert np.array_equal(ct, oracle.encrypt(key, host, nthreads=4)), t


@pytest.mark.parametrize("keybits", [128, 192, 256])
def test_round_by_round_trace_against_oracle(aes, keybits):
    """SURVEY.md 8(c) per-round pin: after ARK(0) and r Eq-26 rounds the GPU
    state equals the oracle's state after AddRoundKey(r) (encryption), and
    the equivalent-inverse state after r rounds equals the straightforward
    InvCipher's state after r iterations (decryption), for every r."""
    key = synth.key(keybits)
    rk = aes.expand_key(key)
    n = 333
    host = synth.blocks(11, n)
    x = _dev_rand(n, first=11)
    E = [oracle.cipher_trace(key, host[16 * i:16 * i + 16].tobytes()) for i in range(n)]
    C = np.frombuffer(b"".join(e[-1] for e in E), np.uint8)
    D = [oracle.inv_cipher_trace(key, C[16 * i:16 * i + 16].tobytes()) for i in range(n)]
    tc = torch.from_numpy(C.copy()).cuda()
    for r in range(rk.nr + 1):
        ge = aes.ecb_trace(rk, x, r).cpu().numpy().tobytes()
        assert ge == b"".join(e[r] for e in E), ("enc", keybits, r)
        gd = aes.ecb_trace(rk, tc, r, decrypt=True).cpu().numpy().tobytes()
        assert gd == b"".join(d[r] for d in D), ("dec", keybits, r)


def test_round_trace_fips197_appendix_b(aes):
    d = {ln.split()[0]: ln.split()[1] for ln in open(golden("fips197_appB.txt")) if ln.strip() and not ln.startswith("#")}
    rk = aes.expand_key(bytes.fromhex(d["key"]))
    x = torch.frombuffer(bytearray(bytes.fromhex(d["pt"])), dtype=torch.uint8).cuda()
    for r in range(10):
        assert aes.ecb_trace(rk, x, r).cpu().numpy().tobytes().hex() == d[f"r{r}"], r
    assert aes.ecb_trace(rk, x, 10).cpu().numpy().tobytes().hex() == d["ct"]


@pytest.mark.parametrize("keybits", [128, 192, 256])
@pytest.mark.parametrize("decrypt", [False, True])
def test_batch_many_messages_many_keys_against_oracle(aes, keybits, decrypt):
    """aes_ecb_batch: messages of the paper's file sizes (PAPER.md:509-518,
    ceil(size/16) blocks) plus empty / 1-block / ragged ones, each with its
    own key, some in place; every output byte checked against the oracle."""
    rng = np.random.default_rng(keybits + int(decrypt))
    ladder = [76, 291, 582, 1163, 2326, 4651, 9301, 18601, 37201, 74401]
    sizes = ladder + [0, 1, 2, 31, 32, 33] + [int(v) for v in rng.integers(1, 3000, 40)]
    rng.shuffle(sizes)
    nkeys = 7
    keys = [rng.integers(0, 256, keybits // 8, dtype=np.uint8).tobytes() for _ in range(nkeys)]
    rks = [aes.expand_key(k) for k in keys]
    kidx = [int(v) for v in rng.integers(0, nkeys, len(sizes))]
    xs, hosts = [], []
    first = 0
    for n in sizes:
        h = synth.blocks(first, n)
        first += n
        hosts.append(h)
        xs.append(torch.from_numpy(h.copy()).cuda())
    outs = [x if i % 5 == 0 else None for i, x in enumerate(xs)]      # every 5th in place
    outs = [o if o is not None else torch.empty_like(x) for o, x in zip(outs, xs)]
    got = aes.ecb_batch(rks, xs, outs, key_index=kidx, decrypt=decrypt)
    torch.cuda.synchronize()
    for i, (g, h) in enumerate(zip(got, hosts)):
        want = oracle.ecb(keys[kidx[i]], h, decrypt, nthreads=4)
        assert np.array_equal(g.cpu().numpy(), want), (i, sizes[i])


def test_batch_rejects_overlapping_messages(aes):
    rk = [aes.expand_key(synth.key(128))]
    buf = _dev_rand(64)
    a, b, c = buf[:256], buf[256:512], buf[512:768]
    outs = aes.ecb_batch(rk * 2, [a, b], outs=[a, b], key_index=[0, 0])      # each in place: fine
    assert outs[0].data_ptr() == a.data_ptr()
    with pytest.raises(ValueError):
        aes.ecb_batch(rk * 2, [a, b], outs=[c, c], key_index=[0, 0])          # two outputs on one buffer
    with pytest.raises(ValueError):
        aes.ecb_batch(rk * 2, [a, b], outs=[b, c], key_index=[0, 0])          # output = another input
    with pytest.raises(ValueError):
        aes.ecb_batch(rk, [a], outs=[buf[16:272]], key_index=[0])             # partial self-overlap
    aes.ecb_batch(rk * 2, [a, a], outs=[b, c], key_index=[0, 0])              # shared input: fine


def test_batch_thousand_small_files_one_launch(aes):
    key = synth.key(128)
    rk = aes.expand_key(key)
    n = 76   # 1,202-byte file of Table 4, padded to whole blocks
    base = _dev_rand(1000 * n)
    xs = [base[16 * n * i:16 * n * (i + 1)] for i in range(1000)]
    outs = aes.ecb_batch([rk], xs, key_index=[0] * 1000)
    got = torch.cat(outs).cpu().numpy()
    assert np.array_equal(got, oracle.encrypt(key, synth.blocks(0, 1000 * n), nthreads=8))


def test_pipeline_pageable_numpy_and_errors(aes):
    """aes_pipeline_run with pageable numpy buffers (no overlap, still correct),
    chunk sizes that do not divide the message, and its argument errors."""
    key = synth.key(192)
    rk = aes.expand_key(key)
    n = 12345
    host = synth.blocks(3, n)
    dst = np.empty_like(host)
    p = aes.Pipeline(chunk_bytes=16 * 1000, depth=2)
    p.run(rk, host, dst)
    assert np.array_equal(dst, oracle.encrypt(key, host, nthreads=8))
    back = np.empty_like(host)
    p.run(rk, dst, back, decrypt=True)
    assert np.array_equal(back, host)
    with pytest.raises(aes.AesError):
        p.run(rk, host[:-16 * 5], host[16:-16 * 4])       # partial overlap
    with pytest.raises(ValueError):
        p.run(rk, host, dst[:-16])
    p.close()


def test_cuda_graph_capture_and_replay(aes):
    """The launches are stream-ordered and capture-safe: a CUDA graph of
    encrypt -> decrypt -> CTR, replayed twice on fresh inputs, matches the oracle."""
    key = synth.key(128)
    rk = aes.expand_key(key)
    iv = bytes(range(16))
    n = 5000
    x = _dev_rand(n)
    ct, pt, ks = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            aes.ecb_encrypt(rk, x, out=ct)
            aes.ecb_decrypt(rk, ct, out=pt)
            aes.ctr_xcrypt(rk, iv, x, out=ks)
    for first in (77, 4242):
        synth.fill_device(x, first_block=first)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        host = synth.blocks(first, n)
        assert np.array_equal(ct.cpu().numpy(), oracle.encrypt(key, host, nthreads=8))
        assert torch.equal(pt, x)
        assert np.array_equal(ks.cpu().numpy(), oracle.ctr(key, iv, host, nthreads=8))


def test_hybrid_threads_streams_and_graph(aes):
    """The hybrid kernel (bitsliced round keys built per call on the host,
    per-CTA unit queue) from 6 host threads on their own streams with
    different keys, and captured into a CUDA graph (CTR / CBC through the
    crossover knob at capture time) and replayed on fresh inputs."""
    import os
    import threading
    n = 16 * 1024 + 77                      # one CTA: both warp kinds take units
    host = synth.blocks(0, n)
    x = _dev_rand(n)
    results, errors = {}, []

    def work(t):
        try:
            kb = (128, 192, 256)[t % 3]
            key = bytes((t * 17 + i) & 0xFF for i in range(kb // 8))
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(10):
                    rk = aes.expand_key(key)
                    ct = aes.ecb_encrypt(rk, x, variant=aes.AES_VAR_HYBRID, grid=1)
                    back = aes.ecb_decrypt(rk, ct, variant=aes.AES_VAR_HYBRID, grid=1)
            s.synchronize()
            results[t] = (key, ct.cpu().numpy(), bool(torch.equal(back, x)))
        except Exception as e:   # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=work, args=(t,)) for t in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors
    for t, (key, ct, ok) in results.items():
        assert ok
        assert np.array_equal(ct, oracle.encrypt(key, host, nthreads=4)), t

    key = synth.key(192)
    rk = aes.expand_key(key)
    iv = bytes(range(16))
    m = 3 * 2**20 + 5                       # default grid, > kTailUnits units per CTA
    y = _dev_rand(m)
    ct, pt, ks, cb = (torch.empty_like(y) for _ in range(4))
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    os.environ["AES_B200_HYBRID_MIN_BLOCKS"] = "0"
    try:
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                aes.ecb_encrypt(rk, y, out=ct)
                aes.ecb_decrypt(rk, ct, out=pt)
                aes.ctr_xcrypt(rk, iv, y, out=ks)
                aes.cbc_decrypt(rk, iv, y, out=cb)
    finally:
        os.environ.pop("AES_B200_HYBRID_MIN_BLOCKS", None)
    for first in (5, 999):
        synth.fill_device(y, first_block=first)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        hy = synth.blocks(first, m)
        sel = np.r_[0:4096, m - 4096:m]
        assert np.array_equal(ct.cpu().numpy().reshape(-1, 16)[sel],
                              oracle.encrypt(key, hy.reshape(-1, 16)[sel].copy().reshape(-1), nthreads=8).reshape(-1, 16))
        assert torch.equal(pt, y)
        assert np.array_equal(ks.cpu().numpy(), oracle.ctr(key, iv, hy, nthreads=16))
        assert np.array_equal(cb.cpu().numpy(), _cbc_decrypt_oracle(key, iv, hy))


def test_cli_file_round_trip(aes, tmp_path):
    """python -m paper_1902_05234_b200 enc/dec on a non-block-multiple file
    (PKCS#7): ciphertext equals OpenSSL-free oracle ECB of the padded file,
    and decryption restores the file; CTR on a ragged file too."""
    import subprocess
    import sys
    from conftest import ROOT
    rng = np.random.default_rng(5)
    data = rng.integers(0, 256, 1190402, dtype=np.uint8).tobytes()   # the paper's largest file
    key = rng.integers(0, 256, 32, dtype=np.uint8).tobytes()
    src, enc, dec = tmp_path / "p.bin", tmp_path / "c.bin", tmp_path / "d.bin"
    src.write_bytes(data)
    for cmd, a, b in (("enc", src, enc), ("dec", enc, dec)):
        r = subprocess.run([sys.executable, "-m", "paper_1902_05234_b200", cmd, "--key", key.hex(), "--in", str(a),
                            "--out", str(b)], cwd=ROOT, capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]
    k = 16 - len(data) % 16
    padded = np.frombuffer(data + bytes([k]) * k, np.uint8).copy()
    assert enc.read_bytes() == oracle.encrypt(key, padded, nthreads=8).tobytes()
    assert dec.read_bytes() == data
    iv = bytes(range(16))
    r = subprocess.run([sys.executable, "-m", "paper_1902_05234_b200", "enc", "--mode", "ctr", "--iv", iv.hex(),
                        "--key", key.hex(), "--in", str(src), "--out", str(enc)], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    n = (len(data) + 15) // 16
    padded0 = np.zeros(16 * n, np.uint8)
    padded0[:len(data)] = np.frombuffer(data, np.uint8)
    assert enc.read_bytes() == oracle.ctr(key, iv, padded0, nthreads=8).tobytes()[:len(data)]


def test_pipeline_zero_copy_and_staged_paths(aes):
    """Pinned messages <= 8 MiB run on mapped host memory (zero copy), larger
    ones through the chunked staging; both equal the oracle."""
    key = synth.key(128)
    rk = aes.expand_key(key)
    p = aes.Pipeline(chunk_bytes=1 << 20, depth=3)
    for n in ((8 << 20) // 16, (8 << 20) // 16 + 1, (9 << 20) // 16 + 7):
        host = synth.blocks(0, n)
        src = torch.from_numpy(host.copy()).pin_memory()
        dst = torch.empty_like(src).pin_memory()
        p.run(rk, src, dst)
        idx = np.r_[0:64, n // 2:n // 2 + 64, n - 64:n]
        want = oracle.encrypt(key, host.reshape(-1, 16)[idx].copy().reshape(-1), nthreads=8)
        assert np.array_equal(dst.numpy().reshape(-1, 16)[idx].reshape(-1), want), n
        p.run(rk, dst, dst, decrypt=True)
        assert np.array_equal(dst.numpy(), host), n
    p.close()


@pytest.mark.parametrize("keybits", [128, 256])
def test_ctr_large_many_table_refreshes(aes, keybits):
    """The cached CTR kernel refreshes its per-warp group tables every 16
    trips: 80 MiB (> 32 trips per warp) with a block_offset that puts byte 15
    mid-group, checked on sampled blocks against the oracle (incl. warp and
    group boundaries) and by an on-device round trip."""
    key = synth.key(keybits)
    rk = aes.expand_key(key)
    n = (80 << 20) // 16 + 13
    x = _dev_rand(n, first=3)
    iv = bytes([0xFF] * 8) + bytes([0x12, 0x34, 0x56, 0x78, 0xFF, 0xFF, 0xFF, 0xF0])
    off = 2**64 - 1000
    y = aes.ctr_xcrypt(rk, iv, x, block_offset=off)
    rng = np.random.default_rng(keybits)
    T = 148 * 1024
    idx = np.unique(np.r_[0:40, 16 * T - 40:16 * T + 40, 32 * T - 3:32 * T + 3, n - 40:n, rng.integers(0, n, 2048)])
    idx = idx[idx < n].astype(np.int64)
    got = y.view(-1, 16)[torch.from_numpy(idx).cuda()].cpu().numpy()
    plain = synth.blocks_at((idx + 3).astype(np.uint64))
    for j, i in enumerate(idx):
        want = oracle.ctr(key, iv, plain[j].copy(), block_offset=(off + int(i)) % 2**64)
        # block_offset is 64-bit in the ABI: off + i wraps into the high counter half only via the counter add
        if off + int(i) >= 2**64:
            hi = int.from_bytes(iv, "big") + off + int(i)
            want = oracle.ctr(key, (hi % 2**128).to_bytes(16, "big"), plain[j].copy())
        assert np.array_equal(got[j], want), int(i)
    back = aes.ctr_xcrypt(rk, iv, y, block_offset=off)
    assert torch.equal(back, x)


def test_config2_full_parity_every_byte(aes):
    """BASELINE config 2 with FULL parity: all 67,108,864 blocks of the 1 GiB
    AES-128 encryption compared with the oracle (threaded over all host cores),
    in the bench's launch configuration."""
    import os
    n = (1 << 30) // 16
    key = synth.key(128)
    rk = aes.expand_key(key)
    x = _dev_rand(n)
    ct = aes.ecb_encrypt(rk, x).cpu().numpy()
    want = oracle.encrypt(key, synth.blocks(0, n), nthreads=len(os.sched_getaffinity(0)))
    bad = np.nonzero((ct.reshape(-1, 16) != want.reshape(-1, 16)).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} blocks differ, first {int(bad[0])}"


def test_ctr_plain_kernel_matches_cached(aes, tmp_path):
    """AES_B200_CTR_KERNEL=plain (uncached A/B reference) gives the same bytes."""
    import subprocess
    import sys
    from conftest import ROOT
    code = (
        "import sys; sys.path.insert(0, '.');"
        "import torch, numpy as np, synth, paper_1902_05234_b200 as aes;"
        "x = torch.empty(16 * 300007, dtype=torch.uint8, device='cuda'); synth.fill_device(x);"
        "rk = aes.expand_key(synth.key(192));"
        "np.save(sys.argv[1], aes.ctr_xcrypt(rk, bytes(range(16)), x, block_offset=251).cpu().numpy())")
    outs = []
    for env_val in ("plain", "cached"):
        f = str(tmp_path / f"{env_val}.npy")
        env = dict(__import__("os").environ, AES_B200_CTR_KERNEL=env_val)
        r = subprocess.run([sys.executable, "-c", code, f], cwd=ROOT, env=env, capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


def test_pipeline_unaligned_host_buffers(aes):
    """Host buffers need no alignment: a pinned buffer at an 8-byte offset takes
    the staged path (the zero-copy path is only used for 16-byte-aligned ones)."""
    key = synth.key(128)
    rk = aes.expand_key(key)
    n = 1000
    host = synth.blocks(0, n)
    big = torch.empty(16 * n + 16, dtype=torch.uint8).pin_memory()
    src = big[8:8 + 16 * n]
    src.copy_(torch.from_numpy(host))
    dst = torch.empty(16 * n + 16, dtype=torch.uint8).pin_memory()[8:8 + 16 * n]
    p = aes.Pipeline(chunk_bytes=1 << 20, depth=2)
    p.run(rk, src, dst)
    assert np.array_equal(dst.numpy(), oracle.encrypt(key, host, nthreads=4))
    p.close()


def test_launch_flags_trusted_pointers_and_no_pdl(aes):
    """aes_launch_config.flags: TRUSTED_PTRS (no per-call pointer queries) and
    NO_PDL give the same bytes as the default (checked pointers + PDL)."""
    from paper_1902_05234_b200 import _native
    key = synth.key(192)
    rk = aes.expand_key(key)
    n = 70001
    x = _dev_rand(n, first=3)
    want = oracle.encrypt(key, synth.blocks(3, n), nthreads=8)
    for fl in (0, aes.AES_LAUNCH_TRUSTED_PTRS, aes.AES_LAUNCH_NO_PDL, aes.AES_LAUNCH_TRUSTED_PTRS | aes.AES_LAUNCH_NO_PDL):
        ct = aes.ecb_encrypt(rk, x, flags=fl)
        assert np.array_equal(ct.cpu().numpy(), want), fl
        assert torch.equal(aes.ecb_decrypt(rk, ct, flags=fl), x), fl
    cfg = _native.aes_launch_config(0, 0, 0, 4)
    code = _native.lib.aes_ecb_launch(rk.c_ref, 12, 0, x.data_ptr(), x.data_ptr(), n, None, ctypes.byref(cfg))
    assert code == _native.AES_ERANGE


def test_back_to_back_pdl_chain_in_place(aes):
    """A chain of dependent in-place launches (each kernel reads what the
    previous one wrote) with PDL overlap: 2k+1 alternating encrypt/decrypt
    launches == one encrypt, for sizes from one warp to several trips, eagerly
    and inside a CUDA graph."""
    key = synth.key(128)
    rk = aes.expand_key(key)
    s = torch.cuda.Stream()
    for n in (32, 4099, 65536, 148 * 1024 * 3 + 77):
        x = _dev_rand(n, first=n)
        want = oracle.encrypt(key, synth.blocks(n, n), nthreads=8)
        y = x.clone()
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            for k in range(41):
                aes.ecb(rk, y, decrypt=bool(k & 1), out=y)
        s.synchronize()
        assert np.array_equal(y.cpu().numpy(), want), n
        y.copy_(x)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for k in range(21):
                    aes.ecb(rk, y, decrypt=bool(k & 1), out=y)
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), want), ("graph", n)


def test_prepared_call_fast_path(aes):
    """EcbCall: validated once, then each call is one C-ABI launch with trusted
    pointers on the current stream; same bytes as the checked path."""
    key = synth.key(256)
    rk = aes.expand_key(key)
    n = 65536 + 3
    x = _dev_rand(n, first=11)
    out = torch.empty_like(x)
    enc = aes.prepare_ecb(rk, x, out)
    dec = aes.prepare_ecb(rk, out, out, decrypt=True)     # in place
    assert enc() is out
    assert np.array_equal(out.cpu().numpy(), oracle.encrypt(key, synth.blocks(11, n), nthreads=8))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    dec(stream=s)
    s.synchronize()
    assert torch.equal(out, x)
    with pytest.raises(aes.AesError):                     # partial overlap
        aes.prepare_ecb(rk, x[16:], x[:-16])
    z = torch.zeros(64 + 8, dtype=torch.uint8, device="cuda")
    with pytest.raises(aes.AesError):                     # misaligned view
        aes.prepare_ecb(rk, z[8:], torch.empty(64, dtype=torch.uint8, device="cuda"))
    with pytest.raises(TypeError):
        aes.prepare_ecb(rk, x.cpu())


def test_small_message_work_split_every_cta_busy(aes):
    """Messages below one grid-stride trip are split into per-CTA chunks:
    parity at sizes around the chunk rounding (multiples of 32 per CTA) and
    with explicit grids, for every key size and direction."""
    for kb in (128, 256):
        key = synth.key(kb)
        rk = aes.expand_key(key)
        for n in (33, 148 * 32 - 1, 148 * 32 + 1, 74401, 148 * 1024 - 1):
            x = _dev_rand(n, first=7 * n)
            host = synth.blocks(7 * n, n)
            want = oracle.encrypt(key, host, nthreads=8)
            wantd = oracle.decrypt(key, host, nthreads=8)
            for grid in (0, 5, 148):
                assert np.array_equal(aes.ecb_encrypt(rk, x, grid=grid, variant=1).cpu().numpy(), want), (kb, n, grid)
                assert np.array_equal(aes.ecb_decrypt(rk, x, grid=grid, variant=1).cpu().numpy(), wantd), (kb, n, grid)
            cbc = aes.cbc_decrypt(rk, bytes(16), x)
            assert np.array_equal(cbc.cpu().numpy(), oracle.cbc(key, bytes(16), host, decrypt=True)), (kb, n)
