"""Pins for the CPU oracle (oracle/aes_oracle.c) against things other than itself.

Every check here compares the oracle with a value the paper or a standard
prints (tests/golden/*, each with its citation), a closed form written a
DIFFERENT way than the oracle writes it, an invariant, or an independent
library (OpenSSL through ``cryptography``).  A dropped term, a wrong index,
a transposed operand or the w[i-4] key-schedule trap (R3) each fail
at least one of them.  CPU only (no gpu marker).
"""
import os
import random

import numpy as np
import pytest

import oracle
from conftest import golden


def _lines(name):
    with open(golden(name)) as f:
        for ln in f:
            ln = ln.split(";")[0].strip()
            if ln and not ln.startswith("#"):
                yield ln.split()


# --------------------------------------------------------------------------
# GF(2^8): PAPER.md Defs 1-3
# --------------------------------------------------------------------------
def test_paper_gf_worked_examples():
    seen = set()
    for op, a, b, r in _lines("paper_gf_examples.txt"):
        a, r = int(a, 16), int(r, 16)
        if op == "add":
            assert oracle.gf_add(a, int(b, 16)) == r
        elif op == "mul":
            assert oracle.gf_mul(a, int(b, 16)) == r
            assert oracle.gf_mul(int(b, 16), a) == r
        elif op == "xtime":
            assert oracle.xtime(a) == r
        seen.add(op)
    assert seen == {"add", "mul", "xtime"}


def _clmul_mod(a, b):
    """Independent multiply: full carry-less product (up to x^14), then long
    division by m(x) = 0x11B (Eq 8) from the top bit down."""
    p = 0
    for i in range(8):
        if (b >> i) & 1:
            p ^= a << i
    for deg in range(14, 7, -1):
        if (p >> deg) & 1:
            p ^= 0x11B << (deg - 8)
    return p


def test_gf_mul_exhaustive_against_long_division():
    lib = oracle.lib()
    for a in range(256):
        for b in range(256):
            assert lib.oracle_gf_mul(a, b) == _clmul_mod(a, b), (a, b)


def test_xtime_is_mul_by_x_and_carry_case():
    for a in range(256):
        assert oracle.xtime(a) == _clmul_mod(a, 2)
    assert oracle.xtime(0x80) == 0x1B          # x^8 mod m(x)
    assert oracle.xtime(0x00) == 0x00


def test_gf_add_is_xor_and_field_axioms():
    rng = random.Random(7)
    for _ in range(2000):
        a, b, c = rng.randrange(256), rng.randrange(256), rng.randrange(256)
        assert oracle.gf_add(a, b) == a ^ b
        m = oracle.gf_mul
        assert m(a, m(b, c)) == m(m(a, b), c)
        assert m(a, b ^ c) == m(a, b) ^ m(a, c)
        assert m(a, 1) == a


def test_every_nonzero_element_has_inverse():
    for a in range(1, 256):
        inv = oracle.gf_inv(a)
        assert _clmul_mod(a, inv) == 1
    assert oracle.gf_inv(0) == 0


# --------------------------------------------------------------------------
# S-box: Definition 4 + FIPS-197 5.1.1 (R5)
# --------------------------------------------------------------------------
def _rotl8(b, n):
    return ((b << n) | (b >> (8 - n))) & 0xFF


def _sbox_closed_form(a):
    """S(a) = inv(a) xor rotl1 xor rotl2 xor rotl3 xor rotl4 xor 0x63 -- the
    circulant-matrix form of the affine map, with inv = a^254 by square-and-
    multiply over the independent multiply above."""
    inv, base, e = 1, a, 254
    while e:
        if e & 1:
            inv = _clmul_mod(inv, base)
        base = _clmul_mod(base, base)
        e >>= 1
    if a == 0:
        inv = 0
    return inv ^ _rotl8(inv, 1) ^ _rotl8(inv, 2) ^ _rotl8(inv, 3) ^ _rotl8(inv, 4) ^ 0x63


def test_sbox_closed_form_and_known_values():
    S = oracle.sbox_table()
    SI = oracle.inv_sbox_table()
    for a in range(256):
        assert S[a] == _sbox_closed_form(a), a
        assert oracle.sbox(a) == S[a]
    assert S[0x00] == 0x63 and S[0x53] == 0xED and S[0xFF] == 0x16
    assert SI[0x00] == 0x52
    assert sorted(S) == list(range(256))                               # bijection
    for a in range(256):
        assert SI[S[a]] == a
        assert oracle.inv_sbox(S[a]) == a


# --------------------------------------------------------------------------
# ShiftRows / MixColumns: Eqs 19-20
# --------------------------------------------------------------------------
def _state_rows(block):
    return [[block[r + 4 * c] for c in range(4)] for r in range(4)]


def test_shift_rows_rotates_row_i_left_by_i():
    blk = bytes(range(16))
    out = _state_rows(oracle.transform("shift_rows", blk))
    rows = _state_rows(blk)
    for i in range(4):
        assert out[i] == rows[i][i:] + rows[i][:i]
    # 4 applications = identity; inverse undoes it
    x = blk
    for _ in range(4):
        x = oracle.transform("shift_rows", x)
    assert x == blk
    assert oracle.transform("inv_shift_rows", oracle.transform("shift_rows", blk)) == blk


def test_mix_columns_known_column_and_inverse():
    col = bytes([0xDB, 0x13, 0x53, 0x45])          # SPEC.md:187, FIPS-197 / textbook example
    blk = col * 4
    out = oracle.transform("mix_columns", blk)
    assert out[:4] == bytes([0x8E, 0x4D, 0xA1, 0xBC])
    ones = bytes([1] * 16)
    assert oracle.transform("mix_columns", ones) == ones
    rng = np.random.default_rng(3)
    for _ in range(200):
        b = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        assert oracle.transform("inv_mix_columns", oracle.transform("mix_columns", b)) == b
        assert oracle.transform("inv_sub_bytes", oracle.transform("sub_bytes", b)) == b


def test_mix_columns_matches_matrix_A_by_hand():
    """Eq 20 with A, products via the independent multiply."""
    A = [[2, 3, 1, 1], [1, 2, 3, 1], [1, 1, 2, 3], [3, 1, 1, 2]]
    rng = np.random.default_rng(11)
    for _ in range(100):
        b = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        out = oracle.transform("mix_columns", b)
        for c in range(4):
            col = b[4 * c:4 * c + 4]
            for r in range(4):
                acc = 0
                for k in range(4):
                    acc ^= _clmul_mod(A[r][k], col[k])
                assert out[4 * c + r] == acc


# --------------------------------------------------------------------------
# Key schedule: FIPS-197 App A (R2, R3, R4)
# --------------------------------------------------------------------------
def test_key_expansion_fips197_appendix_a():
    n = 0
    for key, idx, word in _lines("fips197_appA.txt"):
        w = oracle.key_expansion(bytes.fromhex(key))
        i = int(idx)
        assert w[4 * i:4 * i + 4].hex() == word, (key, i)
        n += 1
    assert n >= 15
    for kb, nr in ((128, 10), (192, 12), (256, 14)):
        assert oracle.nr(kb) == nr
        assert len(oracle.key_expansion(bytes(kb // 8))) == 16 * (nr + 1)
    assert oracle.nr(100) == 0


# --------------------------------------------------------------------------
# Cipher: FIPS-197 App B per-round states, App C, SP 800-38A F.1
# --------------------------------------------------------------------------
def test_cipher_round_by_round_fips197_appendix_b():
    d = {k: v for k, v in _lines("fips197_appB.txt")}
    tr = oracle.cipher_trace(bytes.fromhex(d["key"]), bytes.fromhex(d["pt"]))
    assert len(tr) == 11
    for r in range(10):
        assert tr[r].hex() == d[f"r{r}"], r
    assert tr[10].hex() == d["ct"]


def test_fips197_appendix_c_both_directions():
    rows = list(_lines("fips197_appC.txt"))
    assert len(rows) == 3
    for key, pt, ct in rows:
        k = bytes.fromhex(key)
        assert oracle.encrypt(k, bytes.fromhex(pt)).tobytes().hex() == ct
        assert oracle.decrypt(k, bytes.fromhex(ct)).tobytes().hex() == pt


def test_sp800_38a_f1_ecb_vectors():
    it = list(_lines("sp800_38a_ecb.txt"))
    pt = bytes.fromhex("".join(it[0][1:]))
    pairs = [(bytes.fromhex(it[i][1]), bytes.fromhex("".join(it[i + 1][1:]))) for i in range(1, 7, 2)]
    assert len(pairs) == 3
    for key, ct in pairs:
        for nt in (1, 3):
            assert oracle.encrypt(key, pt, nthreads=nt).tobytes() == ct
            assert oracle.decrypt(key, ct, nthreads=nt).tobytes() == pt


# --------------------------------------------------------------------------
# Library special case: OpenSSL AES-*-ECB without padding (a third implementation)
# --------------------------------------------------------------------------
def _openssl_ecb(key, data, decrypt):
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes
    c = Cipher(algorithms.AES(key), modes.ECB())
    op = c.decryptor() if decrypt else c.encryptor()
    return op.update(data) + op.finalize()


@pytest.mark.parametrize("keybits", [128, 192, 256])
def test_matches_openssl_on_random_buffers(keybits):
    pytest.importorskip("cryptography")
    rng = np.random.default_rng(keybits)
    for nblocks in (1, 2, 31, 33, 1000):
        key = rng.integers(0, 256, keybits // 8, dtype=np.uint8).tobytes()
        pt = rng.integers(0, 256, 16 * nblocks, dtype=np.uint8)
        ct = oracle.encrypt(key, pt, nthreads=4)
        assert ct.tobytes() == _openssl_ecb(key, pt.tobytes(), False)
        back = oracle.decrypt(key, ct, nthreads=2)
        assert back.tobytes() == _openssl_ecb(key, ct.tobytes(), True) == pt.tobytes()


# --------------------------------------------------------------------------
# ECB structure (Eq 1, Table 1) and properties
# --------------------------------------------------------------------------
def test_ecb_block_independence_and_threads_invariance():
    rng = np.random.default_rng(5)
    key = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
    pt = rng.integers(0, 256, 16 * 257, dtype=np.uint8)
    pt[16 * 10:16 * 11] = pt[16 * 3:16 * 4]          # repeated block
    ct = oracle.encrypt(key, pt)
    assert ct[16 * 10:16 * 11].tobytes() == ct[16 * 3:16 * 4].tobytes()
    perm = rng.permutation(257)
    ptp = pt.reshape(-1, 16)[perm].copy().reshape(-1)
    assert np.array_equal(oracle.encrypt(key, ptp).reshape(-1, 16), ct.reshape(-1, 16)[perm])
    for nt in (2, 7, 64):
        assert np.array_equal(oracle.encrypt(key, pt, nthreads=nt), ct)
    # in place
    buf = pt.copy()
    oracle.ecb(key, buf, False, 3, out=buf)
    assert np.array_equal(buf, ct)


def test_round_trip_and_avalanche():
    rng = np.random.default_rng(9)
    for kb in (128, 192, 256):
        key = rng.integers(0, 256, kb // 8, dtype=np.uint8).tobytes()
        pt = rng.integers(0, 256, 16 * 4096, dtype=np.uint8)
        assert np.array_equal(oracle.decrypt(key, oracle.encrypt(key, pt, 4), 4), pt)
    key = bytes(16)
    flips = []
    for _ in range(200):
        b = bytearray(rng.integers(0, 256, 16, dtype=np.uint8).tobytes())
        c0 = oracle.encrypt(key, bytes(b)).tobytes()
        bit = int(rng.integers(0, 128))
        b[bit // 8] ^= 1 << (bit % 8)
        c1 = oracle.encrypt(key, bytes(b)).tobytes()
        flips.append(bin(int.from_bytes(c0, "big") ^ int.from_bytes(c1, "big")).count("1"))
    assert 40 <= np.mean(flips) <= 88


def test_empty_and_bad_inputs():
    assert oracle.encrypt(bytes(16), b"").size == 0
    with pytest.raises(ValueError):
        oracle.encrypt(bytes(15), bytes(16))
    with pytest.raises(ValueError):
        oracle.encrypt(bytes(16), bytes(17))


# --------------------------------------------------------------------------
# CTR (Eq 5, reading R24) and CBC (Eq 2, reading R25): SP 800-38A F.5 / F.2
# --------------------------------------------------------------------------
def _modes_golden():
    rows = list(_lines("sp800_38a_ctr_cbc.txt"))
    ctr_iv = bytes.fromhex(rows[0][1])
    cbc_iv = bytes.fromhex(rows[1][1])
    sets = []
    for i in range(2, len(rows), 3):
        sets.append((bytes.fromhex(rows[i][1]), bytes.fromhex("".join(rows[i + 1][1:])),
                     bytes.fromhex("".join(rows[i + 2][1:]))))
    pt = bytes.fromhex("".join(list(_lines("sp800_38a_ecb.txt"))[0][1:]))
    return ctr_iv, cbc_iv, pt, sets


def test_ctr_and_cbc_sp800_38a_vectors():
    ctr_iv, cbc_iv, pt, sets = _modes_golden()
    assert len(sets) == 3
    for key, ctr_ct, cbc_ct in sets:
        assert oracle.ctr(key, ctr_iv, pt).tobytes() == ctr_ct
        assert oracle.ctr(key, ctr_iv, ctr_ct).tobytes() == pt          # CTR is an involution
        assert oracle.cbc(key, cbc_iv, pt, False).tobytes() == cbc_ct
        assert oracle.cbc(key, cbc_iv, cbc_ct, True).tobytes() == pt


def test_ctr_counter_wrap_offset_and_openssl():
    pytest.importorskip("cryptography")
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes
    rng = np.random.default_rng(21)
    for kb in (128, 256):
        key = rng.integers(0, 256, kb // 8, dtype=np.uint8).tobytes()
        for iv in (bytes([0xFF] * 16), bytes([0xFF] * 8) + bytes([0xFF] * 7) + b"\xfd",
                   bytes(8) + bytes([0xFF] * 8), rng.integers(0, 256, 16, dtype=np.uint8).tobytes()):
            data = rng.integers(0, 256, 16 * 37, dtype=np.uint8)
            e = Cipher(algorithms.AES(key), modes.CTR(iv)).encryptor()
            want = e.update(data.tobytes()) + e.finalize()
            assert oracle.ctr(key, iv, data, nthreads=3).tobytes() == want
            # block_offset k == the tail of a longer stream
            assert oracle.ctr(key, iv, data[16 * 5:], block_offset=5).tobytes() == want[16 * 5:]
        data = rng.integers(0, 256, 16 * 23, dtype=np.uint8)
        iv = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        e = Cipher(algorithms.AES(key), modes.CBC(iv)).encryptor()
        ct = e.update(data.tobytes()) + e.finalize()
        assert oracle.cbc(key, iv, data, False).tobytes() == ct
        assert oracle.cbc(key, iv, np.frombuffer(ct, np.uint8), True).tobytes() == data.tobytes()


def test_inv_cipher_trace_mirrors_the_forward_trace():
    """InvCipher's state after its iteration for round r equals
    ShiftRows(SubBytes(E_{r-1})), E = the (App B-pinned) forward trace; the
    last entry is the plaintext.  Checked for every key size."""
    rng = np.random.default_rng(17)
    for kb in (128, 192, 256):
        for _ in range(20):
            key = rng.integers(0, 256, kb // 8, dtype=np.uint8).tobytes()
            p = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
            E = oracle.cipher_trace(key, p)
            nr = len(E) - 1
            D = oracle.inv_cipher_trace(key, E[nr])
            assert D[nr] == p
            for i in range(nr):
                assert D[i] == oracle.transform("shift_rows", oracle.transform("sub_bytes", E[nr - 1 - i])), (kb, i)
