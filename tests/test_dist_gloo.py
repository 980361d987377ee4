"""N>1 host logic on CPU: world_size-2 gloo process group.

Checks the shard partition (contiguous, disjoint, covering, global block
indices), that per-rank ECB over shards reproduces the single-process output
byte for byte (sharding invariance), and the MAX/SUM scalar
reductions the bench uses for timing.  The per-shard cipher here is the
oracle (no GPU on this box); the GPU kernel's sharding invariance follows from
its parity with the oracle on arbitrary global offsets (test_gpu_parity).
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1902_05234_b200.dist import shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import oracle
    import synth
    from paper_1902_05234_b200 import dist as pdist
    r, w, _ = pdist.init(backend="gloo")
    assert (r, w) == (rank, world)
    b0, b1 = pdist.shard_range(n, r, w)
    key = synth.key(128)
    ct = oracle.encrypt(key, synth.blocks(b0, b1 - b0))
    mx = pdist.max_over_ranks(float(10 + r))
    sm = pdist.sum_over_ranks(float(b1 - b0))
    pdist.barrier()
    q.put((r, b0, b1, ct.tobytes(), mx, sm))
    dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (0, 1, 7, 1000, 2**32):
        for world in (1, 2, 3, 8):
            prev = 0
            for r in range(world):
                a, b = shard_range(n, r, world)
                assert a == prev and b >= a
                prev = b
            assert prev == n
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharding_invariance(world):
    import oracle
    import synth
    n = 1001
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    whole = oracle.encrypt(synth.key(128), synth.blocks(0, n)).tobytes()
    assert b"".join(r[3] for r in res) == whole
    assert [r[1:3] for r in res] == [shard_range(n, r, world) for r in range(world)]
    assert all(r[4] == 10.0 + world - 1 for r in res)   # MAX over ranks
    assert all(r[5] == float(n) for r in res)           # SUM over ranks
