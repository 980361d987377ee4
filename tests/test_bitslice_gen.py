"""CPU checks of the bitsliced S-box circuits used by the hybrid kernel's
lookup-free warps (paper_1902_05234_b200/csrc/aes_bs_sbox.inc).

The generator rebuilds both circuits, evaluates them on all 256 inputs against
an S-box it derives from the definition (GF(2^8) inverse + affine map, FIPS-197
5.1.1; PAPER.md:280 names only "a 256-byte look-up table"); the committed .inc
(its LOP3 cover) is parsed and evaluated on all 256 inputs.  (The .inc is also static_assert-checked
against the product's own tables and FIPS-197 App. C when it is compiled.)
Here the S-box the generator derives is additionally pinned to the oracle's."""
import os
import subprocess
import sys

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def test_committed_lut_circuits_exhaustive():
    """Parse the committed aes_bs_sbox.inc and evaluate its LOP3 networks on all
    256 inputs against S and Si."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_bitslice.py"), "--check"])
    assert r.returncode == 0


def test_generator_sbox_matches_oracle_and_circuits_evaluate():
    import gen_bitslice as g
    S, _ = g.sbox_table()
    assert S == list(oracle.sbox_table())
    inv_o = list(oracle.inv_sbox_table())
    net = g.netlist()
    for x in range(256):
        v = g.run(net, {f"U{i}": (x >> (7 - i)) & 1 for i in range(8)})
        assert sum(v[f"S{i}"] << (7 - i) for i in range(8)) == S[x]
    core_in, consts, tg, tout, core, bg, bout = g.inverse_circuit(net)
    g.check_inverse(core_in, consts, tg, tout, core, bg, bout)   # against the generator's own inverse table
    S_inv = [0] * 256
    for a in range(256):
        S_inv[S[a]] = a
    assert S_inv == inv_o
