#!/usr/bin/env python
"""Per-block instruction counts of the hybrid kernel, read from its SASS
(cuobjdump of the in-tree libaes_b200.so), per pipe: the inputs of the joint
shared-memory + ALU roofline that bench.py reports as `roofline_hybrid`.

For hybrid_kernel<NR, DEC>:
  * T-table loop (2 blocks per trip): LDS, ALU-pipe (PRMT/LOP3/ISETP/IADD3/
    LEA/SHF/...), FMA-pipe (IMAD*) instructions per block;
  * bitsliced pass (8 blocks per thread): the outer body plus (NR-1) x the
    round loop, per block.
Writes profiles/r02_sass_counts.json (or --out).  Runs on CPU (no GPU)."""
import argparse
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1902_05234_b200", "libaes_b200.so")
ALU = {"LOP3", "PRMT", "ISETP", "IADD3", "LEA", "SHF", "VIADD", "POPC", "FLO", "SEL", "MOV", "IABS", "P2R", "R2P",
       "PLOP3", "BMSK", "SGXT", "LOP", "VIMNMX"}
FMA = {"IMAD", "IMUL", "FFMA", "FMUL", "FADD", "HFMA2"}


def functions(sass):
    out = {}
    for part in re.split(r"\n\s+Function : ", sass)[1:]:
        out[part.split("\n")[0].strip()] = part
    return out


def instrs(body):
    return [(int(m.group(1), 16), re.sub(r"^@!?U?P\w+\s+", "", m.group(2)), m.group(0))
            for m in re.finditer(r"/\*([0-9a-f]{4,})\*/\s+((?:@!?U?P\w+\s+)?[A-Z0-9_.]+)[^\n]*", body)]


def loops(ins):
    res = []
    for a, op, full in ins:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", full.split("BRA", 1)[1])
            if t and int(t.group(1), 16) < a and a - int(t.group(1), 16) > 0x400:
                res.append((int(t.group(1), 16), a))
    return res


def classify(ops):
    c = {"total": 0, "lds": 0, "alu": 0, "fma": 0, "other": 0}
    for op in ops:
        base = op.split(".")[0]
        c["total"] += 1
        if base == "LDS":
            c["lds"] += 1
        elif base in ALU:
            c["alu"] += 1
        elif base in FMA:
            c["fma"] += 1
        else:
            c["other"] += 1
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sass_counts.json"))
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    res = {"source": "cuobjdump -sass paper_1902_05234_b200/libaes_b200.so (tools/sass_counts.py)",
           "note": "per 16-byte block; ALU = alu-pipe ops, FMA = fma-pipe ops (IMAD*), LDS = lookups (LDS + LDS.U8)"}
    for name, body in functions(sass).items():
        m = re.search(r"hybrid_kernelILi(\d+)ELb([01])ELi0E", name)   # MODE 0 = ECB
        if not m:
            continue
        nr, dec = int(m.group(1)), m.group(2) == "1"
        ins = instrs(body)
        lp = sorted(loops(ins), key=lambda t: t[1] - t[0])
        # the T loop contains LDS; of the rest, the smaller is the round loop, the larger the pass loop
        tl = [x for x in lp if any(o.startswith("LDS") for b, o, _ in ins if x[0] <= b <= x[1]) and
              sum(1 for b, o, _ in ins if x[0] <= b <= x[1] and o.startswith("LDS")) > 100]
        bl = [x for x in lp if x not in tl]
        t_ops = [o for b, o, _ in ins if tl[0][0] <= b <= tl[0][1]]
        rnd = [o for b, o, _ in ins if bl[0][0] <= b <= bl[0][1]]
        outer = [o for b, o, _ in ins if bl[-1][0] <= b <= bl[-1][1]]
        T = {k: v / 2 for k, v in classify(t_ops).items()}
        r, o = classify(rnd), classify(outer)
        B = {k: ((o[k] - r[k]) + (nr - 1) * r[k]) / 8 for k in o}
        res[f"nr{nr}_{'dec' if dec else 'enc'}"] = {"t_table_per_block": T, "bitsliced_per_block": B}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
