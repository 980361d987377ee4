"""Every C ABI entry point is documented in DESIGN.md's boundary table, and
every golden fixture names its source."""
import os
import re

from conftest import ROOT


def test_every_abi_function_is_in_design_md():
    hdr = open(os.path.join(ROOT, "include", "aes_b200.h")).read()
    design = open(os.path.join(ROOT, "DESIGN.md")).read()
    for name in set(re.findall(r"\b(aes_[a-z0-9_]+)\s*\(", hdr)):
        stem = name.replace("_create", "").replace("_run", "").replace("_destroy", "")
        assert name in design or stem in design, name


def test_golden_fixtures_cite_their_source():
    gdir = os.path.join(ROOT, "tests", "golden")
    for f in os.listdir(gdir):
        if f.endswith(".txt"):
            head = open(os.path.join(gdir, f)).read(600)
            assert head.startswith("#"), f
            assert any(w in head for w in ("PAPER.md", "FIPS-197", "SP 800-38A", "make_samples.py")), f
