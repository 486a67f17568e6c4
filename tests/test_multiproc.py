"""N > 1 host path on CPU: world_size-2 gloo process group, contiguous shards
(batch.hpp:61-70), results gathered and compared bit-for-bit with a
single-process solve (G-invariance).  The solve function here is the CPU
oracle (test-only injection); on GPU boxes it is Solver.solve_batch."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2106_14995_b200.shard import partition


def test_partition_matches_reference_rule():
    assert partition(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert partition(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    assert partition(0, 2) == [(0, 0), (0, 0)]
    with pytest.raises(ValueError):
        partition(5, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from oracle import pyoracle as po
    from paper_2106_14995_b200 import synth
    from paper_2106_14995_b200.shard import solve_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b = synth.branch(1001, 6, seed=2)
    out = solve_sharded(b, rank, world, lambda sb: po.solve_batch(sb, impl="oracle"))
    if rank == 0:
        q.put({k: v for k, v in out.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_equals_single_process():
    from oracle import pyoracle as po
    from paper_2106_14995_b200 import synth

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = po.solve_batch(synth.branch(1001, 6, seed=2), impl="oracle")
    for k, v in got.items():
        assert np.array_equal(v, getattr(ref, k)), k
