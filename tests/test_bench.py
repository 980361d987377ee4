"""bench.py contract: the JSON line's keys, on CPU (--impl reference) and on
the GPU (our arm at N=1, and the N=2 code path with two gloo ranks sharing
one GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_reference_arm_on_cpu():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--ref-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "Gbps"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_bench_our_arm_n1():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--bytes-per-gpu",
                        str(64 << 20), "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d) and {"roofline", "roofline_lds", "clocks", "gpu_launches"} <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 100 and d["gpu_launches"] == 6
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.2
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * (64 << 20)
    assert d["cpu_baseline"]["kind"] == "oracle"


@pytest.mark.gpu
def test_bench_n2_code_path_with_gloo_on_one_gpu():
    """Driver-style launch: torchrun --nproc-per-node 2 ... bench.py --gpus 2."""
    env = dict(os.environ, AES_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--bytes-per-gpu", str(32 << 20), "--cpu-seconds", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["config"]["global_bytes"] == 2 * (32 << 20)
    assert d["cpu_baseline"]["kind"] == "oracle" and d["gpu_launches"] == 6
    assert d["ranks"]["world"] == 2 and len(d["ranks"]["devices"]) == 2


@pytest.mark.gpu
def test_bench_gpus_2_without_torchrun_spawns_its_ranks():
    """`python bench.py --gpus 2` with no launcher re-launches itself with two
    ranks (here both on the one GPU of the test box, gloo): n_gpus 2, twice
    the bytes, cpu_baseline from rank 0."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["AES_BENCH_BACKEND"] = "gloo"
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--bytes-per-gpu", str(32 << 20), "--cpu-seconds", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_bytes"] == 2 * (32 << 20)
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["ranks"]["world"] == 2 and d["ranks"]["backend"] == "gloo"
    assert d["ranks"]["kernel_ms_min"] <= d["ranks"]["kernel_ms_max"]


def test_reference_arm_flags_relabel_on_cpu():
    """--keybits / --dir / --seed reach the reference arm: metric and workload
    are relabelled, the oracle runs that direction on that stream."""
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--ref-seconds", "1", "--keybits", "256", "--dir", "dec", "--seed", "7"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["metric"].startswith("AES-256 ECB decrypt Gbps") and d["config"]["keybits"] == 256
    assert "AES-256 ECB decrypt," in d["config"]["workload"] and "seed 7" in d["data"]
    assert "decrypt" in d["cpu_baseline"]["sample"] and "+" not in d["cpu_baseline"]["sample"]


@pytest.mark.gpu
@pytest.mark.parametrize("flags,keybits,passes", [
    (["--keybits", "256", "--dir", "dec", "--variant", "smem_repl"], 256, 1),
    (["--keybits", "192", "--dir", "enc", "--variant", "hybrid", "--seed", "12345"], 192, 1),
    (["--variant", "smem_repl", "--spt", "2"], 128, 2),
])
def test_bench_flags(flags, keybits, passes):
    """SURVEY.md 5 "Config / flags": --keybits/--dir/--variant/--spt/--seed on
    our arm, parity-gated (the golden samples on the sampled stream in the same
    kernel configuration, the round trip on the --seed stream)."""
    nbytes = 32 << 20
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--bytes-per-gpu", str(nbytes),
                        "--no-cpu", *flags], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert "error" not in d and d["value"] > 100
    assert d["config"]["keybits"] == keybits and d["metric"].startswith(f"AES-{keybits} ECB")
    assert d["e2e"]["h2d_bytes_per_step"] == passes * nbytes
    if "--variant" in flags:
        assert d["config"]["variant"].startswith(flags[flags.index("--variant") + 1])
    if "--seed" in flags:
        assert d["config"]["seed"] == 12345


def test_hybrid_ceiling_solves_both_resource_equations():
    """roofline_hybrid: the T-table / bitsliced block mix saturates the L1 data
    path (32 lane-slots/clk/SM) and the ALU pipe (64 lane-ops/clk/SM) at once,
    with the per-block counts of profiles/r02_sass_counts.json; the joint
    ceiling lies above the T-table-only one (32 / (L_T + 8) blocks/clk/SM)."""
    sys.path.insert(0, ROOT)
    import bench
    for dom, key in (("encrypt", "nr10_enc"), ("decrypt", "nr10_dec")):
        h = bench._hybrid_ceiling(dom, {"sm_mhz": 1965.0}, 148)
        c = json.load(open(os.path.join(ROOT, "profiles", "r02_sass_counts.json")))[key]
        LT, AT = c["t_table_per_block"]["lds"], c["t_table_per_block"]["alu"]
        AB = c["bitsliced_per_block"]["alu"]
        tot = h["peak_blocks_per_clk_per_sm"]
        t, b = tot * h["t_share"], tot * (1 - h["t_share"])
        assert abs((LT + 8) * t + 8 * b - 32) < 1e-9 and abs(AT * t + AB * b - 64) < 1e-9
        assert 0 < b < t and tot > 32 / (LT + 8)
        assert abs(h["peak_GBps_payload"] - 16 * tot * 148 * 1.965e9 / 1e9) < 1e-6
