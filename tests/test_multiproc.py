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


def _admm_worker(rank, world, port, q, line_limits=False):
    """One rank of the sharded ADMM scheme (paper_2106_14995_b200/admm.py
    ShardedAdmm) with the CPU oracle as the compute backend and gloo as the
    collective: equal branch chunks, in-place all-gather of the branch
    solutions, bus update on every rank, max-allreduce of the residuals."""
    import ctypes as C
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from oracle import pyoracle as po
    from paper_2106_14995_b200 import synth
    from paper_2106_14995_b200.shard import partition

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2106_14995_b200.admm import AdmmOptions

    g = synth.grid(150, 210, 40, seed=9, shunt_frac=0.3, rate=(0.05, 0.6))
    opts = AdmmOptions(line_limits=line_limits)
    D = opts.branch_dim
    a = po.OracleAdmm(g, opts)
    lib = a.lib
    lib.orc_admm_solve_components.argtypes = [C.c_void_p, C.c_int64, C.c_int64]
    lib.orc_admm_x.argtypes = [C.c_void_p]
    lib.orc_admm_x.restype = C.POINTER(C.c_double)
    lib.orc_admm_update_consensus.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double),
                                              C.POINTER(C.c_double)]
    chunk = (g.n_branch + world - 1) // world
    lo, hi = min(g.n_branch, rank * chunk), min(g.n_branch, (rank + 1) * chunk)
    blo, bhi = partition(g.n_bus, world)[rank]
    xs = np.ctypeslib.as_array(lib.orc_admm_x(a._h), shape=(g.n_branch * D,))
    buf = torch.zeros(chunk * world * D, dtype=torch.float64)
    hist = []
    for _ in range(12):
        assert lib.orc_admm_solve_components(a._h, lo, hi) == 0
        buf[: g.n_branch * D] = torch.from_numpy(xs)
        dist.all_gather_into_tensor(buf, buf[rank * chunk * D:(rank + 1) * chunk * D].clone())
        xs[:] = buf[: g.n_branch * D].numpy()
        p, d = C.c_double(), C.c_double()
        lib.orc_admm_update_consensus(a._h, blo, bhi, C.byref(p), C.byref(d))
        r = torch.tensor([p.value, d.value], dtype=torch.float64)
        dist.all_reduce(r, op=dist.ReduceOp.MAX)
        hist.append(tuple(r.tolist()))
    if rank == 0:
        q.put(hist)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("line_limits", [False, True])
def test_gloo_world2_sharded_admm_equals_single_process(line_limits):
    from oracle import pyoracle as po
    from paper_2106_14995_b200 import synth
    from paper_2106_14995_b200.admm import AdmmOptions

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_admm_worker, args=(r, 2, port, q, line_limits)) for r in range(2)]
    for p in procs:
        p.start()
    hist = q.get(timeout=180)
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    a = po.OracleAdmm(synth.grid(150, 210, 40, seed=9, shunt_frac=0.3, rate=(0.05, 0.6)),
                      AdmmOptions(line_limits=line_limits))
    ref = [a.step() for _ in range(12)]
    assert hist == ref
