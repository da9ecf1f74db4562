"""The N > 1 bench path runs independent replicas (the north star keeps the
path on one GPU: no data-path collective).  Its only cross-rank step is the
max-over-ranks timing reduction; exercised here with world_size 2 over gloo,
each rank running the (CPU) oracle on its own replica."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    import time

    import torch.distributed as dist

    import bench
    from oracle.pyoracle import Oracle
    from paper_1204_1533_b200 import CONFIGS

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cfg = CONFIGS[1]
    case, U = cfg.build(n=4)
    o = Oracle(case, cfg.physics)
    t0 = time.perf_counter()
    R = o.residual(U)
    ms = (time.perf_counter() - t0) * 1e3 + rank  # distinct per rank
    ms_max = bench.max_over_ranks(ms, "cpu")
    val = bench.replica_throughput(R.size, world, ms_max)
    out.put((rank, ms, ms_max, val, float(np.abs(R).max())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ms_max = max(r[1] for r in res)
    for r in res:
        assert r[2] == pytest.approx(ms_max)
        assert r[3] == pytest.approx(2 * (16 * 25 * 4) / (ms_max * 1e-3) / 1e9)
    assert res[0][4] == res[1][4]  # identical replicas
