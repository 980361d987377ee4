"""Multi-GPU plumbing for the ECB path.

ECB blocks are independent (Eq 1; Table 1 "Suitable",
PAPER.md:153,161), so a buffer of n blocks is split into N contiguous shards,
one per rank/GPU, with NO collective on the data path.  torch.distributed is
used only to start, align (barrier) and time the ranks (MAX of elapsed
times, SUM of counts).  Works with the nccl backend on GPUs and gloo on CPU.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys


def shard_range(nblocks: int, rank: int, world: int) -> tuple[int, int]:
    """Rank r of N owns global blocks [r*n//N, (r+1)*n//N)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return nblocks * rank // world, nblocks * (rank + 1) // world


def env_rank_world() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def respawn_under_torchrun(nproc: int, argv: list[str] | None = None) -> int | None:
    """One process per GPU without an external launcher: when ``nproc`` > 1 and
    this process was not started by torchrun (no WORLD_SIZE in the env), run
    ``python -m torch.distributed.run --nnodes=1 --nproc-per-node nproc
    --master-addr 127.0.0.1 --master-port <free> <argv>`` and return its exit
    code (the children print; this parent prints nothing).  Returns None when
    no re-launch is needed (nproc == 1, or already under torchrun)."""
    if nproc <= 1 or "WORLD_SIZE" in os.environ:
        return None
    argv = list(sys.argv if argv is None else argv)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", *argv]
    print("[dist] launching " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def require_world(expected: int) -> None:
    """Exit non-zero unless the process group has exactly ``expected`` ranks
    (a silent 1-rank run labelled N GPUs is the failure this guards)."""
    _, world, _ = env_rank_world()
    if world != expected:
        raise SystemExit(f"[dist] --gpus {expected} but WORLD_SIZE={world}: refusing to run "
                         "(launch under torchrun with --nproc-per-node matching --gpus, or without torchrun "
                         "and let the script spawn its ranks)")


def init(backend: str | None = None):
    """Initialise the default process group from torchrun's env (if WORLD_SIZE>1)."""
    import torch
    import torch.distributed as dist
    rank, world, local = env_rank_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            if world > torch.cuda.device_count():
                raise SystemExit(f"[dist] {world} ranks but {torch.cuda.device_count()} visible GPU(s): NCCL needs "
                                 "one GPU per rank (for a harness run on fewer GPUs set AES_BENCH_BACKEND=gloo)")
            local = local % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def _reduce(value: float, op, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    if dist.get_backend() == "nccl":      # NCCL reduces device tensors only
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    else:
        dev = "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def min_over_ranks(value: float, device=None) -> float:
    import torch.distributed as dist
    return _reduce(value, dist.ReduceOp.MIN, device)


def gather_objects(obj) -> list:
    """all_gather_object over the default group ([obj] when not distributed)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def max_over_ranks(value: float, device=None) -> float:
    import torch.distributed as dist
    return _reduce(value, dist.ReduceOp.MAX, device)


def sum_over_ranks(value: float, device=None) -> float:
    import torch.distributed as dist
    return _reduce(value, dist.ReduceOp.SUM, device)


def barrier(device=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        if dist.get_backend() == "nccl" and device is not None:
            dist.barrier(device_ids=[device.index if hasattr(device, "index") else int(device)])
        else:
            dist.barrier()


def backend_name() -> str | None:
    import torch.distributed as dist
    return dist.get_backend() if dist.is_available() and dist.is_initialized() else None


def finalize():
    """Destroy the default process group if this module created one."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()
