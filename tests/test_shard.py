"""N>1 host logic on CPU: text ownership ranges, halo, clipping and the
rank-ordered gather, over a real world_size-2 gloo process group.

The per-span search here is the CPU restatement (a stand-in for the GPU
engine, which needs a device); the logic under test is shard.py's.  The
GPU version of the same flow is tests/test_gpu_parity.py::test_sharded_spans.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from pyoracle import as_pairs

from paper_1405_5483_b200 import shard


def test_ownership_and_spans():
    for n in (0, 1, 100, 4096, 4097, 1 << 20, 12345678):
        for world in (1, 2, 3, 8):
            b = shard.ownership(n, world)
            assert b[0] == 0 and b[-1] == n and all(x <= y for x, y in zip(b, b[1:]))
            if n > shard.ALIGN * world:
                assert all(x % shard.ALIGN == 0 for x in b[1:-1])
            for g in range(world):
                lo, hi = shard.read_span(n, b, g, 32)
                assert lo == b[g] and hi <= n and (hi >= b[g + 1] or b[g + 1] == b[g])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, text, pats, out_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    from pyoracle import Port
    port_ = Port()
    maxlen = max(len(p) for p in pats)
    res = shard.sharded_search(lambda lo, hi: port_.naive(text[lo:hi], pats), text.size, maxlen, world, rank)
    if rank == 0:
        np.savez(out_path, offs=res[0], pids=res[1])
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_equals_whole_text(tmp_path, port, world):
    rng = np.random.default_rng(8)
    n = 3 * shard.ALIGN * world + 777
    text = (rng.integers(0, 4, n) + 65).astype(np.uint8)
    pats = [text[s:s + L].tobytes() for s, L in ((10, 40), (n // 2 - 5, 33), (shard.ALIGN * 3 - 20, 64))]
    pats += [(rng.integers(0, 4, 6) + 65).astype(np.uint8).tobytes() for _ in range(5)]
    # plant occurrences straddling every ownership boundary
    b = shard.ownership(n, world)
    for x in b[1:-1]:
        text[x - 20:x + 20] = np.frombuffer(pats[0], dtype=np.uint8)
    out = str(tmp_path / "res.npz")
    mp.start_processes(_worker, args=(world, _free_port(), text, pats, out), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    want = port.naive(text, pats)
    assert as_pairs(got["offs"], got["pids"]) == as_pairs(*want)
    assert len(want[0]) > 0
