#!/usr/bin/env python
"""Generate paper_1902_05234_b200/csrc/aes_bs_sbox.inc: bitsliced AES S-box and
inverse S-box circuits for the hybrid kernel's bitsliced warps.

Product-side code generator (it never touches oracle/): the S-box is rebuilt
here from its definition (GF(2^8) inverse, then the FIPS-197 5.1.1 affine map;
PAPER.md:280 only says "a 256-byte look-up table").

* Forward S-box: the Boyar-Peralta depth-16 circuit (top linear layer,
  shared GF(2^4)-tower inversion core, bottom linear layer; 128 gates,
  34 AND).  Checked here on all 256 inputs.  Its two linear layers are then
  re-synthesised (seeded random-tie-break Paar, FWD_RELIN) for a smaller LUT
  cover.
* Both netlists are then covered by 3-input LUTs (one LOP3 each; cut
  enumeration + iterated local search, seeded), cutting the instruction count
  per S-box evaluation by about a third.
* Inverse S-box: the same inversion core; the top layer is composed with the
  inverse affine map U = A^-1 (Y ^ 0x63) and the bottom layer with A^-1
  (S = A inv(U) ^ 0x63  =>  inv(U) = A^-1 (S ^ 0x63)), both linear layers
  re-synthesised with a greedy common-pair (Paar) XOR heuristic.  Checked here
  on all 256 inputs.

Bit convention of the emitted code: x[b] holds bit b (b = 0 is the LSB) of a
byte in every bit lane of the 32-bit words; BP's U0 is the MSB, i.e. x[7].
Run: python tools/gen_bitslice.py  (rewrites the .inc, prints gate counts; ~1 min)
     python tools/gen_bitslice.py --check  (evaluates the committed .inc exhaustively)
"""
import os
import random
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


def rpaar(rows, nin, prefix, rnd):
    """paar() with random tie-breaking among the most frequent pairs (and now and
    then a runner-up pair) -- a seeded, deterministic source of alternative XOR
    networks for the same linear layer, to be scored by the LUT mapper."""
    sig = [f"in{i}" for i in range(nin)]
    rows = [set(i for i in range(nin) if r >> i & 1) for r in rows]
    gates = []
    while True:
        cands = {}
        for r in rows:
            s_ = sorted(r)
            for i in range(len(s_)):
                for j in range(i + 1, len(s_)):
                    cands[(s_[i], s_[j])] = cands.get((s_[i], s_[j]), 0) + 1
        if not cands:
            break
        mx = max(cands.values())
        if mx < 2:
            break
        best = rnd.choice([k for k, c in cands.items() if c == mx or (c == mx - 1 and rnd.random() < 0.15 and mx > 2)])
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
    for r in rows:
        s_ = sorted(r)
        rnd.shuffle(s_)
        cur = sig[s_[0]]
        for k in s_[1:]:
            name = f"{prefix}{len(gates)}"
            gates.append((name, cur, sig[k]))
            cur = name
        outs.append(cur)
    return gates, outs


def forward_relin_nodes(g, rnd):
    """BP's nonlinear core (M1..M63) with its two linear layers re-synthesised by
    rpaar: the 21 core inputs T_k as XORs of U, and S (before the XNOR
    constants) as XORs of M46..M63.  Same function as BP's netlist."""
    U = [f"U{i}" for i in range(8)]
    core_start = next(d for d, a, op, b in g if op == "x")
    top = forms(g, U, core_start)
    core = [x for x in g if x[0].startswith("M")]
    core_names = {x[0] for x in core}
    core_in = sorted({s_ for _, a, _, b in core for s_ in (a, b) if s_ not in core_names and s_.startswith("T")},
                     key=lambda s_: int(s_[1:]))
    Mout = [f"M{i}" for i in range(46, 64)]
    Lf = {m: 1 << i for i, m in enumerate(Mout)}
    for d, a, op, b in g:
        if d[0] in "LS":
            Lf[d] = Lf[a] ^ Lf[b]
    sops = {d: op for d, a, op, b in g if d.startswith("S")}
    nodes = [(u, "IN", []) for u in U]
    ren = {f"in{i}": U[i] for i in range(8)}
    tg, tout = rpaar([top[t] for t in core_in], 8, "t", rnd)
    for n_, a, b in tg:
        nodes.append((n_, "XOR", [ren.get(a, a), ren.get(b, b)]))
    for i, t in enumerate(core_in):
        nodes.append((t, "BUF", [ren.get(tout[i], tout[i])]))
    nodes += [(d, "XOR" if op == "+" else "AND", [a, b]) for d, a, op, b in core]
    bg, bout = rpaar([Lf[f"S{j}"] for j in range(8)], 18, "b", rnd)
    ren2 = {f"in{k}": Mout[k] for k in range(18)}
    for n_, a, b in bg:
        nodes.append((n_, "XOR", [ren2.get(a, a), ren2.get(b, b)]))
    outs = []
    for j in range(8):
        o = ren2.get(bout[j], bout[j])
        if sops[f"S{j}"] == "#":
            nodes.append((f"SO{j}", "NOT", [o]))
            outs.append(f"SO{j}")
        else:
            outs.append(o)
    return nodes, outs, U


# The linear-layer syntheses chosen by search (tools: seeded rpaar draws, each
# scored by lut_map; the best of 4 x 40 draws): (seed, draw index).
FWD_RELIN = (3, 31)   # 79 LOP3 (BP's own layers: 82)
INV_RELIN = (1, 23)   # 81 LOP3 (deterministic paar: 83)


def inverse_circuit(g, synth=None):
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
    synth = synth or paar
    tg, tout = synth(rows, 8, "t")
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
    bg, bout = synth(out_rows, 18, "b")
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


# ---- uniform netlists: [(name, op, [fanins])], op in IN / XOR / AND / XNOR / NOT ----
def forward_nodes(g):
    nodes = [(f"U{i}", "IN", []) for i in range(8)]
    for d, a, op, b in g:
        nodes.append((d, {"+": "XOR", "x": "AND", "#": "XNOR"}[op], [a, b]))
    return nodes, [f"S{i}" for i in range(8)], [f"U{i}" for i in range(8)]


def inverse_nodes(core_in, consts, tg, tout, core, bg, bout):
    nodes = [(f"in{k}", "IN", []) for k in range(8)]
    nodes += [(n, "XOR", [a, b]) for n, a, b in tg]
    for i, s_ in enumerate(core_in):
        nodes.append((s_, "NOT" if consts[i] else "BUF", [tout[i]]))
    nodes += [(d, "XOR" if op == "+" else "AND", [a, b]) for d, a, op, b in core]
    ren = {f"in{k}": f"M{46 + k}" for k in range(18)}
    nodes += [("b" + n[1:] if False else n, "XOR", [ren.get(a, a), ren.get(b, b)]) for n, a, b in bg]
    outs = [ren.get(o, o) for o in bout]
    return nodes, outs, [f"in{k}" for k in range(8)]


def eval_nodes(nodes, env):
    v = dict(env)
    for n, op, fi in nodes:
        if op == "IN":
            continue
        x = [v[f] for f in fi]
        v[n] = {"XOR": lambda: x[0] ^ x[1], "AND": lambda: x[0] & x[1], "XNOR": lambda: ~(x[0] ^ x[1]),
                "NOT": lambda: ~x[0], "BUF": lambda: x[0]}[op]()
    return v


def lut_map(nodes, outputs, K=3, iters=1500, seed=5):
    """Cover the netlist with K-input LUTs (LOP3 = any 3-input function):
    enumerate every K-feasible cut of every node, start from the area-flow
    choice, then iterated local search (seeded, deterministic): single-node
    cut changes that shrink the cover (ties accepted at random), restarted from
    random perturbations of the best cover found.  Returns {node: cut} for the
    nodes implemented as LUTs."""
    rnd = random.Random(seed)
    kind = {n: op for n, op, _ in nodes}
    fanin = {n: fi for n, _, fi in nodes}
    order = [n for n, _, _ in nodes]
    cuts = {}
    for n in order:
        if kind[n] == "IN":
            cuts[n] = [frozenset([n])]
            continue
        cs = {frozenset([n])}
        fi = fanin[n]
        if len(fi) == 1:
            cs.update(cuts[fi[0]])
        else:
            for c1 in cuts[fi[0]]:
                for c2 in cuts[fi[1]]:
                    u = c1 | c2
                    if len(u) <= K:
                        cs.add(u)
        cuts[n] = sorted(cs, key=lambda c: (len(c), sorted(c)))
    opts = {n: [c for c in cuts[n] if c != frozenset([n])] for n in order if kind[n] != "IN"}
    gates = list(opts)
    fanout = {n: 0 for n in order}
    for n in order:
        for f in fanin[n]:
            fanout[f] += 1
    af, choice = {}, {}
    for n in order:
        if kind[n] == "IN":
            af[n] = 0.0
            continue
        af[n], choice[n] = min(((1.0 + sum(af[u] / max(1, fanout[u]) for u in c), c) for c in opts[n]),
                               key=lambda t: (t[0], len(t[1]), sorted(t[1])))

    def cover(ch):
        need, seen = list(outputs), set()
        while need:
            v = need.pop()
            if v in seen or kind[v] == "IN":
                continue
            seen.add(v)
            need.extend(sorted(ch[v]))
        return seen

    def local(ch):
        cur = cover(ch)
        improved = True
        while improved:
            improved = False
            for n in gates:
                if n not in cur:
                    continue
                for c in opts[n]:
                    if c == ch[n]:
                        continue
                    old = ch[n]
                    ch[n] = c
                    cand = cover(ch)
                    if len(cand) < len(cur):
                        cur, improved = cand, True
                    elif len(cand) == len(cur) and rnd.random() < 0.3:
                        cur = cand
                    else:
                        ch[n] = old
        return cur

    best_cov = local(choice)
    best = dict(choice)
    for _ in range(iters):
        ch = dict(best)
        for _ in range(rnd.randint(1, 6)):
            n = rnd.choice(gates)
            ch[n] = rnd.choice(opts[n])
        cov = local(ch)
        if len(cov) <= len(best_cov):
            best_cov, best = cov, ch
    return {n: best[n] for n in order if n in best_cov}


def lut_imm(nodes, n, leaves):
    """LOP3 immediate of node n over leaves (a, b, c) = (0xF0, 0xCC, 0xAA)."""
    env = {}
    pats = (0xF0, 0xCC, 0xAA)
    for i, l in enumerate(leaves):
        env[l] = pats[i]
    sub = []
    need, seen = [n], set()
    fanin = {m: fi for m, _, fi in nodes}
    while need:
        v = need.pop()
        if v in seen or v in env:
            continue
        seen.add(v)
        need.extend(fanin[v])
    sub = [x for x in nodes if x[0] in seen]
    return eval_nodes(sub, env)[n] & 0xFF


def emit_lut_fn(fname, nodes, outputs, inputs, in_bit):
    m = lut_map(nodes, outputs)
    order = [n for n, _, _ in nodes]
    ind = "    "
    L = ["template <class W>", f"__host__ __device__ __forceinline__ constexpr void {fname}(W (&x)[8]) {{"]
    for i, nm in enumerate(inputs):
        L.append(f"{ind}const W {nm} = x[{in_bit(i)}];")
    luts = []
    for n in order:
        if n not in m:
            continue
        leaves = sorted(m[n], key=order.index)
        imm = lut_imm(nodes, n, leaves)
        args = leaves + [leaves[0]] * (3 - len(leaves))
        luts.append((n, imm, args))
        L.append(f"{ind}const W {n} = bs_lop3<0x{imm:02X}>({', '.join(args)});")
    for i, o in enumerate(outputs):
        L.append(f"{ind}x[{in_bit(i)}] = {o};")
    L.append("}")
    return L, luts


def check_luts(luts, inputs, outputs, table):
    for x in range(256):
        v = {nm: -((x >> (7 - i)) & 1) & 0xFF for i, nm in enumerate(inputs)}   # 0x00 / 0xFF lanes
        for n, imm, (a, b, c) in luts:
            r = 0
            for i in range(8):
                if imm >> i & 1:
                    r |= (v[a] if i & 4 else ~v[a]) & (v[b] if i & 2 else ~v[b]) & (v[c] if i & 1 else ~v[c])
            v[n] = r & 0xFF
        y = sum((v[o] & 1) << (7 - i) for i, o in enumerate(outputs))
        assert y == table[x], (x, y, table[x])


def ngates(nodes):
    """2-input gates + inverters of a netlist (inputs and buffers excluded)."""
    return sum(1 for _, op, _ in nodes if op not in ("IN", "BUF"))


def emit():
    g = netlist()
    S_tab, _ = sbox_table()
    for x in range(256):
        v = run(g, {f"U{i}": (x >> (7 - i)) & 1 for i in range(8)})
        assert sum(v[f"S{i}"] << (7 - i) for i in range(8)) == S_tab[x]
    rnd = random.Random(INV_RELIN[0])
    for _ in range(INV_RELIN[1] + 1):
        inv = inverse_circuit(g, lambda rows, nin, prefix: rpaar(rows, nin, prefix, rnd))
    check_inverse(*inv)
    inv_tab = [0] * 256
    for a in range(256):
        inv_tab[S_tab[a]] = a
    rnd = random.Random(FWD_RELIN[0])
    for _ in range(FWD_RELIN[1] + 1):
        fn, fo, fi = forward_relin_nodes(g, rnd)
    for x in range(256):                    # the re-synthesised forward netlist is still S
        v = eval_nodes(fn, {fi[i]: -((x >> (7 - i)) & 1) & 0xFF for i in range(8)})
        assert sum((v[o] & 1) << (7 - i) for i, o in enumerate(fo)) == S_tab[x]
    iv, io, ii = inverse_nodes(*inv)
    Lf, lf = emit_lut_fn("bs_sbox", fn, fo, fi, lambda i: 7 - i)
    Li, li = emit_lut_fn("bs_inv_sbox", iv, io, ii, lambda i: 7 - i)
    check_luts(lf, fi, fo, S_tab)
    check_luts(li, ii, io, inv_tab)
    L = ["// aes_bs_sbox.inc -- GENERATED by tools/gen_bitslice.py; do not edit.",
         "// Bitsliced S-box / inverse S-box over 32 independent bytes per word:",
         "// x[b] = bit b (b = 0: LSB) of the byte in every bit lane.  Forward: the",
         "// Boyar-Peralta depth-16 circuit's nonlinear core with re-synthesised linear",
         "// layers; inverse: the same GF(2^4)-tower inversion core with the inverse",
         "// affine map folded into re-synthesised linear layers.",
         "// Both netlists are covered by 3-input LUTs (one LOP3 each, bs_lop3<imm>).",
         f"// Forward: {ngates(fn)} gates -> {len(lf)} LOP3; inverse: {ngates(iv)} gates -> {len(li)} LOP3.",
         "// Both checked on all 256 inputs by the generator and by static_asserts in",
         "// aes_bitslice.cuh."]
    L += Lf + [""] + Li
    return "\n".join(L) + "\n", ngates(fn), len(lf), ngates(iv), len(li)


def check_include(path):
    """Evaluate the committed .inc's two functions on all 256 inputs (fast; no search)."""
    import re
    S_tab, _ = sbox_table()
    inv_tab = [0] * 256
    for a in range(256):
        inv_tab[S_tab[a]] = a
    text = open(path).read()
    fns = re.findall(r"void (bs_\w+)\(W \(&x\)\[8\]\) \{(.*?)\n\}", text, re.S)
    assert [f for f, _ in fns] == ["bs_sbox", "bs_inv_sbox"], [f for f, _ in fns]
    for fname, body in fns:
        table = S_tab if fname == "bs_sbox" else inv_tab
        for x in range(256):
            v = {}
            for line in body.strip().splitlines():
                line = line.strip()
                m = re.match(r"const W (\w+) = x\[(\d)\];", line)
                if m:
                    v[m.group(1)] = -((x >> int(m.group(2))) & 1) & 0xFF
                    continue
                m = re.match(r"const W (\w+) = bs_lop3<0x([0-9A-F]{2})>\((\w+), (\w+), (\w+)\);", line)
                if m:
                    imm, a, b, c = int(m.group(2), 16), v[m.group(3)], v[m.group(4)], v[m.group(5)]
                    r = 0
                    for i in range(8):
                        if imm >> i & 1:
                            r |= (a if i & 4 else ~a) & (b if i & 2 else ~b) & (c if i & 1 else ~c)
                    v[m.group(1)] = r & 0xFF
                    continue
                m = re.match(r"x\[(\d)\] = (\w+);", line)
                assert m, line
                v["out%s" % m.group(1)] = v[m.group(2)]
            y = sum((v["out%d" % b] & 1) << b for b in range(8))
            assert y == table[x], (fname, x, y, table[x])
    return len(re.findall(r"bs_lop3<", text))


if __name__ == "__main__":
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = os.path.join(root, "paper_1902_05234_b200", "csrc", "aes_bs_sbox.inc")
    if "--check" in sys.argv:      # the committed circuits, on all 256 inputs each
        print(f"{out}: {check_include(out)} LOP3, both functions exhaustive-checked")
        sys.exit(0)
    text, fwd, fl, inv, il = emit()
    open(out, "w").write(text)
    print(f"forward S-box: {fwd} gates -> {fl} LOP3; inverse S-box: {inv} gates -> {il} LOP3; wrote {out}")
