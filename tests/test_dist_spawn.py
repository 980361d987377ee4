"""The multi-process entry point without an external launcher:
``respawn_under_torchrun`` starts N ranks under torch.distributed.run when the
caller was not launched by torchrun, and ``require_world`` refuses a run whose
WORLD_SIZE differs from --gpus.  CPU only (gloo)."""
import json
import os
import subprocess
import sys
import textwrap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = textwrap.dedent("""
    import json, os, sys
    sys.path.insert(0, {root!r})
    from paper_1902_05234_b200 import dist as pdist
    rc = pdist.respawn_under_torchrun(int(sys.argv[1]), [os.path.abspath(__file__), *sys.argv[1:]])
    if rc is not None:
        sys.exit(rc)
    pdist.require_world(int(sys.argv[1]))
    r, w, _ = pdist.init(backend="gloo")
    total = pdist.sum_over_ranks(1.0 + r)
    devs = pdist.gather_objects(f"rank{{r}}")
    if r == 0:
        print(json.dumps({{"world": w, "sum": total, "ranks": devs, "backend": pdist.backend_name()}}), flush=True)
    pdist.barrier()
    pdist.finalize()
""")


def _run(tmp_path, n, env_extra=None):
    script = tmp_path / "child.py"
    script.write_text(CHILD.format(root=ROOT))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, str(script), str(n)], capture_output=True, text=True, timeout=300,
                          env=env)


def test_respawn_starts_n_ranks(tmp_path):
    for n in (2, 3):
        r = _run(tmp_path, n)
        assert r.returncode == 0, r.stderr[-3000:]
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        assert len(line) == 1, r.stdout                  # rank 0 only; the parent prints nothing
        d = json.loads(line[0])
        assert d["world"] == n and d["sum"] == n * (n + 1) / 2
        assert d["ranks"] == [f"rank{i}" for i in range(n)] and d["backend"] == "gloo"


def test_single_process_needs_no_launcher(tmp_path):
    r = _run(tmp_path, 1)
    assert r.returncode == 0, r.stderr[-3000:]
    assert json.loads(r.stdout.strip().splitlines()[-1])["world"] == 1


def test_world_mismatch_refused(tmp_path):
    r = _run(tmp_path, 2, {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "refusing to run" in r.stderr


def test_bench_refuses_world_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900, env=env)
    assert r.returncode != 0 and "refusing to run" in r.stderr
