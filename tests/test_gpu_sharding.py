"""Sharding invariance of the CUDA path ("the concatenated
output must be byte-identical across N"; Eq 1; Table 1,
PAPER.md:153/161).  World 2 and 3 gloo ranks share the test box's GPU; rank r
fills its contiguous global shard [r*n/N, (r+1)*n/N) of the splitmix64 stream
on the device and ciphers it through the C ABI (aes_ecb_encrypt, and CTR with
block_offset = the shard's first block).  Rank 0 gathers the shards; the
concatenation must equal the N = 1 CUDA output byte for byte, and the oracle
on every block."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle
import synth

N_BLOCKS = 1_000_003          # 16 MB: several trips of the persistent grid + ragged shards
IV = bytes.fromhex("f0f1f2f3f4f5f6f7f8f9fafbfcfdfeff")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import paper_1902_05234_b200 as aes
    from paper_1902_05234_b200 import dist as pdist
    r, w, _ = pdist.init(backend="gloo")
    torch.cuda.set_device(0)
    b0, b1 = pdist.shard_range(N_BLOCKS, r, w)
    key = synth.key(128)
    rk = aes.expand_key(key)
    x = torch.empty(16 * (b1 - b0), dtype=torch.uint8, device="cuda")
    synth.fill_device(x, first_block=b0)
    ct = aes.ecb_encrypt(rk, x)
    ks = aes.ctr_xcrypt(rk, IV, x, block_offset=b0)
    torch.cuda.synchronize()
    shards = pdist.gather_objects((r, b0, b1, ct.cpu().numpy().tobytes(), ks.cpu().numpy().tobytes()))
    if r == 0:
        q.put(shards)
    pdist.barrier()
    pdist.finalize()


@pytest.mark.parametrize("world", [2, 3])
def test_cuda_path_sharding_invariance(world):
    import __graft_entry__
    __graft_entry__.build()
    import paper_1902_05234_b200 as aes
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    shards = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    shards.sort()
    from paper_1902_05234_b200.dist import shard_range
    assert [s[1:3] for s in shards] == [shard_range(N_BLOCKS, r, world) for r in range(world)]
    ecb_cat = b"".join(s[3] for s in shards)
    ctr_cat = b"".join(s[4] for s in shards)
    # the N = 1 CUDA output
    key = synth.key(128)
    rk = aes.expand_key(key)
    x = torch.empty(16 * N_BLOCKS, dtype=torch.uint8, device="cuda")
    synth.fill_device(x)
    one_ecb = aes.ecb_encrypt(rk, x).cpu().numpy().tobytes()
    one_ctr = aes.ctr_xcrypt(rk, IV, x).cpu().numpy().tobytes()
    assert ecb_cat == one_ecb
    assert ctr_cat == one_ctr
    # and the oracle on every block
    host = synth.blocks(0, N_BLOCKS)
    want = oracle.encrypt(key, host, nthreads=os.cpu_count() or 4)
    got = np.frombuffer(ecb_cat, np.uint8)
    bad = np.nonzero((got.reshape(-1, 16) != want.reshape(-1, 16)).any(axis=1))[0]
    assert not len(bad), f"first mismatching block {int(bad[0])}"
    wctr = oracle.ctr(key, IV, host, nthreads=os.cpu_count() or 4)
    assert np.array_equal(np.frombuffer(ctr_cat, np.uint8), wctr)
