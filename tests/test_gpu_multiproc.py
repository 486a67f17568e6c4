"""The product's N > 1 paths with real processes on the GPU: two ranks share
cuda:0 (only one GPU is available to these runs) under a gloo group, each
solving its shard on the device.  The sharded TRON solve (shard.solve_sharded
over Solver.solve_batch, batch.hpp:61-70 partitions) must equal the oracle
bit for bit, and the sharded ADMM (ShardedAdmm: equal branch chunks, all-
gather of the branch solutions, max-allreduce of the residuals and failure
flag) must reproduce the single-process trajectory bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _solve_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2106_14995_b200 import Solver, synth
    from paper_2106_14995_b200.shard import solve_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = Solver((0,))
    b = synth.branch(40001, 6, seed=7)  # 20,001 problems per rank: ranked launches on each
    out = solve_sharded(b, rank, world, s.solve_batch)
    s.close()
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def _spawn(target, world, *args, timeout=300):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=timeout)
    for p in procs:
        p.join(timeout=timeout)
        assert p.exitcode == 0
    return got


def test_two_ranks_sharded_solve_on_the_gpu_equals_oracle():
    from conftest import FIELDS
    from oracle import pyoracle as po
    from paper_2106_14995_b200 import synth

    got = _spawn(_solve_worker, 2)
    ref = po.solve_batch(synth.branch(40001, 6, seed=7), impl="oracle", workers=os.cpu_count() or 8)
    for k in FIELDS:
        a, b = got[k], getattr(ref, k)
        if a.dtype.kind == "f":
            assert np.array_equal(a.view(np.int64), b.view(np.int64)), k
        else:
            assert np.array_equal(a, b), k


def _admm_grid():
    from paper_2106_14995_b200 import synth

    return synth.grid(300, 450, 90, seed=9, shunt_frac=0.3, rate=(0.05, 0.6))


def _admm_worker(rank, world, port, q, line_limits):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_2106_14995_b200.admm import AdmmOptions, ShardedAdmm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sa = ShardedAdmm(_admm_grid(), rank, world, 0, AdmmOptions(line_limits=line_limits), record_times=True)
    hist = [sa.step() for _ in range(8)]
    times = sa.partition_times()
    x = sa.x.cpu().numpy().copy()
    if rank == 0:
        q.put((hist, x, times))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("line_limits", [False, True])
def test_two_ranks_sharded_admm_on_the_gpu_equals_one_process(line_limits):
    from paper_2106_14995_b200.admm import BRANCH_X, AdmmOptions, AdmmSolver

    hist, x, times = _spawn(_admm_worker, 2, line_limits)
    a = AdmmSolver(_admm_grid(), AdmmOptions(line_limits=line_limits))
    try:
        ref = [a.step() for _ in range(8)]
        xr = a.get(BRANCH_X)
    finally:
        a.close()
    assert hist == ref  # residual trajectory, bit for bit
    n = xr.shape[0]
    assert np.array_equal(x[:n].view(np.int64), np.asarray(xr).view(np.int64))
    assert len(times) == 8 and all(len(r) == 2 and min(r) > 0 for r in times)
