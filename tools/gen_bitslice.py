#!/usr/bin/env python
"""Generate paper_1902_05234_b200/csrc/aes_bs_sbox.inc: bitsliced AES S-box and
inverse S-box circuits for the hybrid kernel's bitsliced warps.

Product-side code generator (it never touches oracle/): the S-box is rebuilt
here from its definition (GF(2^8) inverse, then the FIPS-197 5.1.1 affine map;
PAPER.md:280 only says "a 256-byte look-up table").

* Forward S-box: the Boyar-Peralta depth-16 circuit (top linear layer,
  shared GF(2^4)-tower inversion core, bottom linear layer; 128 gates,
  34 AND).  Checked here on all 256 inputs.
* Inverse S-box: the same inversion core; the top layer is composed with the
  inverse affine map U = A^-1 (Y ^ 0x63) and the bottom layer with A^-1
  (S = A inv(U) ^ 0x63  =>  inv(U) = A^-1 (S ^ 0x63)), both linear layers
  re-synthesised with a greedy common-pair (Paar) XOR heuristic.  Checked here
  on all 256 inputs.

Bit convention of the emitted code: x[b] holds bit b (b = 0 is the LSB) of a
byte in every bit lane of the 32-bit words; BP's U0 is the MSB, i.e. x[7].
Run: python tools/gen_bitslice.py  (rewrites the .inc, prints gate counts).
"""
import os
import sys

BP = """
T1 = U0 + U3
T2 = U0 + U5
T3 = U0 + U6
T4 = U3 + U5
T5 = U4 + U6
T6 = T1 + T5
T7 = U1 + U2
T8 = U7 + T6
T9 = U7 + T7
T10 = T6 + T7
T11 = U1 + U5
T12 = U2 + U5
T13 = T3 + T4
T14 = T6 + T11
T15 = T5 + T11
T16 = T5 + T12
T17 = T9 + T16
T18 = U3 + U7
T19 = T7 + T18
T20 = T1 + T19
T21 = U6 + U7
T22 = T7 + T21
T23 = T2 + T22
T24 = T2 + T10
T25 = T20 + T17
T26 = T3 + T16
T27 = T1 + T12
M1 = T13 x T6
M2 = T23 x T8
M3 = T14 + M1
M4 = T19 x U7
M5 = M4 + M1
M6 = T3 x T16
M7 = T22 x T9
M8 = T26 + M6
M9 = T20 x T17
M10 = M9 + M6
M11 = T1 x T15
M12 = T4 x T27
M13 = M12 + M11
M14 = T2 x T10
M15 = M14 + M11
M16 = M3 + M2
M17 = M5 + T24
M18 = M8 + M7
M19 = M10 + M15
M20 = M16 + M13
M21 = M17 + M15
M22 = M18 + M13
M23 = M19 + T25
M24 = M22 + M23
M25 = M22 x M20
M26 = M21 + M25
M27 = M20 + M21
M28 = M23 + M25
M29 = M28 x M27
M30 = M26 x M24
M31 = M20 x M23
M32 = M27 x M31
M33 = M27 + M25
M34 = M21 x M22
M35 = M24 x M34
M36 = M24 + M25
M37 = M21 + M29
M38 = M32 + M33
M39 = M23 + M30
M40 = M35 + M36
M41 = M38 + M40
M42 = M37 + M39
M43 = M37 + M38
M44 = M39 + M40
M45 = M42 + M41
M46 = M44 x T6
M47 = M40 x T8
M48 = M39 x U7
M49 = M43 x T16
M50 = M38 x T9
M51 = M37 x T17
M52 = M42 x T15
M53 = M45 x T27
M54 = M41 x T10
M55 = M44 x T13
M56 = M40 x T23
M57 = M39 x T19
M58 = M43 x T3
M59 = M38 x T22
M60 = M37 x T20
M61 = M42 x T1
M62 = M45 x T4
M63 = M41 x T2
L0 = M61 + M62
L1 = M50 + M56
L2 = M46 + M48
L3 = M47 + M55
L4 = M54 + M58
L5 = M49 + M61
L6 = M62 + L5
L7 = M46 + L3
L8 = M51 + M59
L9 = M52 + M53
L10 = M53 + L4
L11 = M60 + L2
L12 = M48 + M51
L13 = M50 + L0
L14 = M52 + M61
L15 = M55 + L1
L16 = M56 + L0
L17 = M57 + L1
L18 = M58 + L8
L19 = M63 + L4
L20 = L0 + L1
L21 = L1 + L7
L22 = L3 + L12
L23 = L18 + L2
L24 = L15 + L9
L25 = L6 + L10
L26 = L7 + L9
L27 = L8 + L10
L28 = L11 + L14
L29 = L11 + L17
S0 = L6 + L24
S1 = L16 # L26
S2 = L19 # L28
S3 = L6 + L21
S4 = L20 + L22
S5 = L25 + L29
S6 = L13 # L27
S7 = L6 # L23
"""


def netlist():
    g = []
    for line in BP.strip().splitlines():
        d, e = [x.strip() for x in line.split("=")]
        a, op, b = e.split()
        g.append((d, a, op, b))
    return g


def gf_mul(a, b):
    r = 0
    while b:
        if b & 1:
            r ^= a
        a <<= 1
        if a & 0x100:
            a ^= 0x11B
        b >>= 1
    return r


def sbox_table():
    inv = [0] * 256
    for a in range(1, 256):
        inv[a] = next(b for b in range(1, 256) if gf_mul(a, b) == 1)
    S = []
    for a in range(256):
        b, s = inv[a], 0x63
        for i in range(8):
            s ^= (((b >> i) ^ (b >> ((i + 4) % 8)) ^ (b >> ((i + 5) % 8)) ^ (b >> ((i + 6) % 8)) ^
                   (b >> ((i + 7) % 8))) & 1) << i
        S.append(s)
    return S, inv


def run(g, env):
    v = dict(env)
    for d, a, op, b in g:
        A, B = v[a], v[b]
        v[d] = A ^ B if op == "+" else (A & B if op == "x" else 1 ^ A ^ B)
    return v


# ---- linear algebra over GF(2): a linear form is an int bitmask over inputs ----
def forms(g, inputs, upto):
    """Linear forms (bitmask over `inputs`) of every XOR-only signal of g before `upto`."""
    f = {name: 1 << i for i, name in enumerate(inputs)}
    for d, a, op, b in g:
        if d == upto:
            break
        if op == "+" and a in f and b in f:
            f[d] = f[a] ^ f[b]
    return f


def paar(rows, nin, prefix):
    """Greedy common-pair XOR synthesis.  rows: list of int masks over nin inputs.
    Returns (gates, outsig) with gates = [(name, a, b)], outsig[i] = signal of row i."""
    sig = [f"in{i}" for i in range(nin)]
    rows = [set(i for i in range(nin) if r >> i & 1) for r in rows]
    gates = []
    while True:
        best, cnt = None, 1
        cands = {}
        for r in rows:
            s = sorted(r)
            for i in range(len(s)):
                for j in range(i + 1, len(s)):
                    cands[(s[i], s[j])] = cands.get((s[i], s[j]), 0) + 1
        for k, c in cands.items():
            if c > cnt:
                best, cnt = k, c
        if best is None:
            break
        name = f"{prefix}{len(gates)}"
        gates.append((name, sig[best[0]], sig[best[1]]))
        sig.append(name)
        idx = len(sig) - 1
        for r in rows:
            if best[0] in r and best[1] in r:
                r.discard(best[0])
                r.discard(best[1])
                r.add(idx)
    outs = []
    for r in rows:       # remaining rows: chain the leftovers
        s = sorted(r)
        if not s:
            outs.append(None)
            continue
        cur = sig[s[0]]
        for k in s[1:]:
            name = f"{prefix}{len(gates)}"
            gates.append((name, cur, sig[k]))
            cur = name
        outs.append(cur)
    return gates, outs


def inverse_circuit(g):
    """Inverse S-box netlist over inputs Y0..Y7 (Y0 = MSB) -> outputs S0..S7 = inv(A^-1(Y ^ 63))."""
    U = [f"U{i}" for i in range(8)]
    core_start = next(d for d, a, op, b in g if op == "x")              # M1
    top = forms(g, U, core_start)
    core = [x for x in g if x[0].startswith("M")]
    core_names = {x[0] for x in core}
    core_in = sorted({s for _, a, _, b in core for s in (a, b) if s not in core_names},
                     key=lambda s: (s[0], int(s[1:])))
    # U_i (MSB-first) as affine forms of Y: u = A^-1 (y ^ 0x63) (bit 0 of a byte = LSB = U7)
    S_tab, _ = sbox_table()
    inv_s = [0] * 256
    for a in range(256):
        inv_s[S_tab[a]] = a
    # A^-1 y ^ c  as columns: x(y) = inv_affine(y) with inv_affine(y) = A^-1 (y ^ 63) affine
    def inv_aff(y):
        # A^-1 (y ^ 0x63): invert the affine map numerically from S = A inv ^ 63
        return AINV[y]
    aff = [0] * 256
    for b in range(256):
        s = 0x63
        for i in range(8):
            s ^= (((b >> i) ^ (b >> ((i + 4) % 8)) ^ (b >> ((i + 5) % 8)) ^ (b >> ((i + 6) % 8)) ^
                   (b >> ((i + 7) % 8))) & 1) << i
        aff[b] = s
    AINV = [0] * 256
    for b in range(256):
        AINV[aff[b]] = b
    c0 = inv_aff(0)
    # U_i form over Y_k (MSB-first both): bit (7-i) of AINV(y) ^ c0 is linear in y
    u_form, u_const = [], []
    for i in range(8):
        m = 0
        for k in range(8):
            y = 1 << (7 - k)
            if ((inv_aff(y) ^ c0) >> (7 - i)) & 1:
                m |= 1 << k
        u_form.append(m)
        u_const.append((c0 >> (7 - i)) & 1)
    # core inputs as affine forms of Y
    rows, consts = [], []
    for s in core_in:
        f = top[s]
        m, c = 0, 0
        for i in range(8):
            if f >> i & 1:
                m ^= u_form[i]
                c ^= u_const[i]
        rows.append(m)
        consts.append(c)
    tg, tout = paar(rows, 8, "t")
    # bottom: S_j (before the XNOR constants, which are 0x63) as forms over M46..M63
    Mout = [f"M{i}" for i in range(46, 64)]
    Lf = {m: 1 << i for i, m in enumerate(Mout)}
    for d, a, op, b in g:
        if d[0] in "LS":
            Lf[d] = Lf[a] ^ Lf[b]
    s_form = [Lf[f"S{j}"] for j in range(8)]          # S (MSB-first) ^ 63 = A inv  (S_j linear part)
    # inv = A^-1 (S ^ 63): out_i = XOR over j of AINVLIN[i][j] * Slin_j
    out_rows = []
    for i in range(8):
        m = 0
        for j in range(8):
            s = 1 << (7 - j)
            if ((AINV[s ^ 0x63] ^ AINV[0x63]) >> (7 - i)) & 1:   # linear part of A^-1 . e_j
                m ^= s_form[j]
        out_rows.append(m)
    bg, bout = paar(out_rows, 18, "b")
    return core_in, consts, tg, tout, core, bg, bout


def check_inverse(core_in, consts, tg, tout, core, bg, bout):
    S_tab, _ = sbox_table()
    inv_s = [0] * 256
    for a in range(256):
        inv_s[S_tab[a]] = a
    for y in range(256):
        v = {f"in{k}": (y >> (7 - k)) & 1 for k in range(8)}
        for name, a, b in tg:
            v[name] = v[a] ^ v[b]
        env = {s: v[tout[i]] ^ consts[i] for i, s in enumerate(core_in)}
        env = run(core, env)
        w = {f"in{k}": env[f"M{46 + k}"] for k in range(18)}
        for name, a, b in bg:
            w[name] = w[a] ^ w[b]
        out = sum(w[bout[i]] << (7 - i) for i in range(8))
        assert out == inv_s[y], (y, out, inv_s[y])


def emit_core(core, ind):
    lines = []
    for d, a, op, b in core:
        lines.append(f"{ind}const uint32_t {d} = {a} {'^' if op == '+' else '&'} {b};")
    return lines


def emit():
    g = netlist()
    S_tab, _ = sbox_table()
    for x in range(256):
        v = run(g, {f"U{i}": (x >> (7 - i)) & 1 for i in range(8)})
        assert sum(v[f"S{i}"] << (7 - i) for i in range(8)) == S_tab[x]
    core_in, consts, tg, tout, core, bg, bout = inverse_circuit(g)
    check_inverse(core_in, consts, tg, tout, core, bg, bout)
    ind = "    "
    L = ["// aes_bs_sbox.inc -- GENERATED by tools/gen_bitslice.py; do not edit.",
         "// Bitsliced S-box / inverse S-box over 32 independent bytes per word:",
         "// x[b] = bit b (b = 0: LSB) of the byte in every bit lane.  Forward: the",
         "// Boyar-Peralta depth-16 circuit; inverse: the same GF(2^4)-tower inversion",
         "// core with the inverse affine map folded into re-synthesised linear layers.",
         "// Both checked on all 256 inputs by the generator and by static_asserts in",
         "// aes_bitslice.cuh.",
         "template <class W>",
         "__host__ __device__ __forceinline__ constexpr void bs_sbox(W (&x)[8]) {"]
    for i in range(8):
        L.append(f"{ind}const W U{i} = x[{7 - i}];")
    for d, a, op, b in g:
        if op == "#":
            L.append(f"{ind}x[{7 - int(d[1:])}] = ~({a} ^ {b});")
        elif d.startswith("S"):
            L.append(f"{ind}x[{7 - int(d[1:])}] = {a} ^ {b};")
        else:
            L.append(f"{ind}const W {d} = {a} {'^' if op == '+' else '&'} {b};")
    L.append("}")
    L.append("")
    L.append("template <class W>")
    L.append("__host__ __device__ __forceinline__ constexpr void bs_inv_sbox(W (&x)[8]) {")
    for k in range(8):
        L.append(f"{ind}const W in{k} = x[{7 - k}];")
    for name, a, b in tg:
        L.append(f"{ind}const W {name} = {a} ^ {b};")
    for i, s in enumerate(core_in):
        L.append(f"{ind}const W {s} = {'~' if consts[i] else ''}{tout[i]};")
    for d, a, op, b in core:
        L.append(f"{ind}const W {d} = {a} {'^' if op == '+' else '&'} {b};")
    for k in range(18):
        L.append(f"{ind}const W bin{k} = M{46 + k};")
    for name, a, b in bg:
        a = a.replace("in", "bin") if a.startswith("in") else a
        b = b.replace("in", "bin") if b.startswith("in") else b
        L.append(f"{ind}const W {name} = {a} ^ {b};")
    for i in range(8):
        o = bout[i].replace("in", "bin") if bout[i].startswith("in") else bout[i]
        L.append(f"{ind}x[{7 - i}] = {o};")
    L.append("}")
    fwd = len(g)
    inv = len(tg) + sum(consts) + len(core) + len(bg)
    return "\n".join(L) + "\n", fwd, inv, len(tg), len(bg)


if __name__ == "__main__":
    text, fwd, inv, ntop, nbot = emit()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = os.path.join(root, "paper_1902_05234_b200", "csrc", "aes_bs_sbox.inc")
    if "--check" in sys.argv:
        sys.exit(0 if open(out).read() == text else 1)
    open(out, "w").write(text)
    print(f"forward S-box: {fwd} gates; inverse S-box: {inv} gates (top {ntop} XOR, bottom {nbot} XOR); wrote {out}")
