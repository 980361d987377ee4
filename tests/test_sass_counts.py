"""The per-block instruction counts behind bench.py's roofline_hybrid
(profiles/r02_sass_counts.json) must match the SASS of the library as built:
re-derive them with tools/sass_counts.py (cuobjdump, CPU only) and compare, and
check what the hybrid design relies on -- 16*Nr lookups per T-table block and
no shared-memory lookups in the bitsliced warps."""
import json
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_committed_sass_counts_match_the_build(tmp_path):
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not found")
    import __graft_entry__
    __graft_entry__.build()
    out = tmp_path / "counts.json"
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_counts.py"), "--out", str(out)], check=True,
                   capture_output=True)
    got = json.load(open(out))
    want = json.load(open(os.path.join(ROOT, "profiles", "r02_sass_counts.json")))
    for k in ("nr10_enc", "nr10_dec", "nr12_enc", "nr12_dec", "nr14_enc", "nr14_dec"):
        assert got[k] == want[k], f"{k}: rerun python tools/sass_counts.py"
        nr = int(k[2:4])
        assert got[k]["t_table_per_block"]["lds"] == 16 * nr
        assert got[k]["bitsliced_per_block"]["lds"] < 1          # only the queue read, amortised over a pass
