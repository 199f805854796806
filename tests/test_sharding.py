"""Multi-rank host logic on CPU: world_size 2 over gloo (127.0.0.1).

Each rank codes its shard of a BASELINE workload with the CPU oracle (no GPU
here) and the shards are gathered to rank 0; the gathered arrays must equal
one oracle run over the whole batch -- the property the GPU shards rely on
(signals are independent, the dictionary is replicated)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1511_05174_b200.sharding import shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 100, 100_000):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, out_path):
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, repo)
    sys.path.insert(0, os.path.join(repo, "oracle"))
    import torch.distributed as dist

    import oracle as O
    from paper_1511_05174_b200 import workloads as W
    from paper_1511_05174_b200.sharding import gather_solutions, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(total, rank, world)
    d = W.dictionaries(0)
    ys = W.signals(0, a, b)
    res = O.omp_many_arrays(d.high_t, ys, 8, rel_tol=W.REL_TOL)
    res["flag"] = res["flag"].astype(np.uint8)
    full = gather_solutions(res, total)
    if rank == 0:
        np.savez(out_path, **full)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_equals_single_run(tmp_path):
    import oracle as O
    from paper_1511_05174_b200 import workloads as W

    total, world = 301, 2
    out = str(tmp_path / "gathered.npz")
    mp.spawn(_worker, args=(world, _free_port(), total, out), nprocs=world, join=True)
    got = np.load(out)
    d = W.dictionaries(0)
    ref = O.omp_many_arrays(d.high_t, W.signals(0, 0, total), 8, rel_tol=W.REL_TOL)
    for k in ("counts", "sel", "alpha", "rnorm", "scans"):
        assert np.array_equal(got[k], ref[k]), k
