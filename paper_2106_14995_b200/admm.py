"""Device-resident component ADMM for AC-OPF over the C ABI
(tb_admm_*), with the batched TRON kernel as its branch stage.

Single GPU:      AdmmSolver(grid).run(iters)
One process per GPU (torchrun): ShardedAdmm(grid, rank, world, device) —
branches sharded in equal chunks; per iteration one NCCL all-gather of the
branch solutions (the consensus exchange: exact, no arithmetic) and one
max-allreduce of the two residuals.  Every process then holds bit-identical
state, equal to the single-GPU run and to the CPU oracle.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _lib as L
from .tron import SolverError, TronConfig

GEN_P, GEN_Q, GEN_PT, GEN_QT, GEN_LP, GEN_LQ, BUS_WT, BUS_TT = range(8)
BRANCH_X, BRANCH_PARAMS, BRANCH_STATUS, COST = 8, 9, 10, 11
AUGLAG_ROUNDS, LINE_VIOL, STAGE_TIMES = 12, 13, 14
TB_E_PROBLEM = 4


@dataclass
class Grid:
    """Network in per unit (SPEC.md:325 NetworkCase minus parsing)."""

    bus_pd: np.ndarray
    bus_qd: np.ndarray
    bus_gsh: np.ndarray
    bus_bsh: np.ndarray
    bus_vmin: np.ndarray
    bus_vmax: np.ndarray
    gen_bus: np.ndarray
    gen_c2: np.ndarray
    gen_c1: np.ndarray
    gen_pmin: np.ndarray
    gen_pmax: np.ndarray
    gen_qmin: np.ndarray
    gen_qmax: np.ndarray
    br_from: np.ndarray
    br_to: np.ndarray
    br_coef: np.ndarray  # [n_branch, 8]
    br_smax2: Optional[np.ndarray] = None  # [n_branch] line limit s-bar^2 (per unit^2); None = unlimited

    @property
    def n_bus(self):
        return len(self.bus_pd)

    @property
    def n_gen(self):
        return len(self.gen_bus)

    @property
    def n_branch(self):
        return len(self.br_from)

    def to_c(self):
        """tb_admm_grid pointing at contiguous copies (kept alive by the return)."""
        keep = {}
        g = GridC()
        g.n_bus, g.n_gen, g.n_branch = self.n_bus, self.n_gen, self.n_branch
        for name, _ in GridC._fields_[3:]:
            a = getattr(self, name)
            if a is None:  # optional arrays (br_smax2)
                setattr(g, name, None)
                continue
            a = np.ascontiguousarray(a, dtype=np.int32 if name in ("gen_bus", "br_from", "br_to") else np.float64)
            keep[name] = a
            setattr(g, name, a.ctypes.data)
        return g, keep


class GridC(C.Structure):
    _fields_ = [("n_bus", C.c_int32), ("n_gen", C.c_int32), ("n_branch", C.c_int32)] + [
        (n, C.c_void_p) for n in ("bus_pd", "bus_qd", "bus_gsh", "bus_bsh", "bus_vmin", "bus_vmax", "gen_bus",
                                  "gen_c2", "gen_c1", "gen_pmin", "gen_pmax", "gen_qmin", "gen_qmax", "br_from",
                                  "br_to", "br_coef", "br_smax2")]


class OptionsC(C.Structure):
    _fields_ = [("rho_pq", C.c_double), ("rho_va", C.c_double), ("shard_rank", C.c_int32),
                ("shard_count", C.c_int32), ("tron", L.TronConfigC), ("line_limits", C.c_int32),
                ("auglag_max_iter", C.c_int32), ("auglag_xi0", C.c_double), ("auglag_xi_max", C.c_double),
                ("auglag_eta0", C.c_double), ("auglag_feas_tol", C.c_double), ("branch_form", C.c_int32)]


@dataclass
class AdmmOptions:
    rho_pq: float = 10.0  # SPEC.md:426 rho0
    rho_va: float = 40.0  # 4 rho0
    tron: TronConfig = field(default_factory=TronConfig)
    # line limits (tb_admm_options): d = 6 branch subproblems + an augmented-
    # Lagrangian loop per ADMM iteration
    line_limits: bool = False
    auglag_max_iter: int = 20
    auglag_xi0: float = 10.0
    auglag_xi_max: float = 1e8
    auglag_eta0: float = 0.1
    auglag_feas_tol: float = 1e-6
    # d = 4 branch stage kernel form: "auto" (thread per branch, fused with the
    # generator updates) or "warp" (warp per branch); identical results
    branch_form: str = "auto"

    @property
    def branch_dim(self) -> int:
        return 6 if self.line_limits else 4

    def to_c(self, rank=0, world=1) -> OptionsC:
        o = OptionsC()
        o.rho_pq, o.rho_va, o.shard_rank, o.shard_count = self.rho_pq, self.rho_va, rank, world
        o.tron = self.tron.to_c()
        o.line_limits = 1 if self.line_limits else 0
        o.auglag_max_iter = self.auglag_max_iter
        o.auglag_xi0, o.auglag_xi_max = self.auglag_xi0, self.auglag_xi_max
        o.auglag_eta0, o.auglag_feas_tol = self.auglag_eta0, self.auglag_feas_tol
        o.branch_form = {"auto": 0, "warp": 1}[self.branch_form]
        return o


_SIG = {
    "tb_admm_create": (C.c_int, [C.POINTER(GridC), C.POINTER(OptionsC), C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "tb_admm_destroy": (C.c_int, [C.c_void_p]),
    "tb_admm_solve_components": (C.c_int, [C.c_void_p, C.c_void_p]),
    "tb_admm_branch_solution": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tb_admm_update_consensus": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "tb_admm_step": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "tb_admm_run": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_void_p,
                              C.POINTER(C.c_int32)]),
    "tb_admm_branch_errors": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "tb_admm_get": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "tb_admm_last_error": (C.c_char_p, []),
    "tb_admm_options_default": (None, [C.POINTER(OptionsC)]),
}


def _lib():
    lib = L.load()
    for n, (res, args) in _SIG.items():
        fn = getattr(lib, n)
        fn.restype, fn.argtypes = res, args
    return lib


class AdmmSolver:
    """One GPU (or one shard of a multi-process run)."""

    def __init__(self, grid: Grid, options: AdmmOptions = None, device: int = 0, rank: int = 0, world: int = 1,
                 x_buffer_ptr: Optional[int] = None):
        self.lib = _lib()
        self.grid = grid
        self.options = options or AdmmOptions()
        g, self._keep = grid.to_c()
        o = self.options.to_c(rank, world)
        h = C.c_void_p()
        if self.lib.tb_admm_create(C.byref(g), C.byref(o), device, C.c_void_p(x_buffer_ptr or 0), C.byref(h)) != 0:
            raise SolverError(self.lib.tb_admm_last_error().decode())
        self._h = h
        self.history: List[Tuple[float, float]] = []

    def close(self):
        if getattr(self, "_h", None):
            self.lib.tb_admm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise _admm_error(rc, self.lib.tb_admm_last_error().decode())

    def step(self) -> Tuple[float, float]:
        """One ADMM iteration (single process): returns (primal, dual).  A
        branch solve that ends where the reference throws raises its
        exception type (solver failures propagate)."""
        p, d = C.c_double(), C.c_double()
        self._check(self.lib.tb_admm_step(self._h, C.byref(p), C.byref(d)))
        self.history.append((p.value, d.value))
        return p.value, d.value

    def run(self, max_iter: int, tol_primal: float = 0.0, tol_dual: float = 0.0, check_every: int = 16):
        """admm_solve until both residuals <= tol or
        max_iter, without a host round trip per iteration (tb_admm_run: one
        CUDA graph per iteration, device stop flag, host poll every
        `check_every` iterations).  Single shard only."""
        if max_iter <= 0:
            return self.history
        hist = np.zeros((max_iter, 2))
        it = C.c_int32()
        rc = self.lib.tb_admm_run(self._h, max_iter, tol_primal, tol_dual, check_every, hist.ctypes.data, C.byref(it))
        self.history.extend((float(p), float(d)) for p, d in hist[:it.value])
        self._check(rc)
        return self.history

    def stage_times(self) -> Tuple[float, float]:
        """Device seconds of the latest iteration's (components, consensus)
        stages -- the per-partition batch time of SPEC.md:408."""
        out = np.zeros(2)
        self._check(self.lib.tb_admm_get(self._h, STAGE_TIMES, out.ctypes.data))
        return float(out[0]), float(out[1])

    def branch_errors(self) -> Tuple[int, int]:
        """(first failed branch since the last call or -1, its status)."""
        i, st = C.c_int64(), C.c_int32()
        self._check(self.lib.tb_admm_branch_errors(self._h, C.byref(i), C.byref(st)))
        return i.value, st.value

    # phases for the multi-process path
    def solve_components(self, stream: int = 0):
        self._check(self.lib.tb_admm_solve_components(self._h, C.c_void_p(stream or 0)))

    def branch_solution(self):
        x, lo, hi = C.c_void_p(), C.c_int64(), C.c_int64()
        self._check(self.lib.tb_admm_branch_solution(self._h, C.byref(x), C.byref(lo), C.byref(hi)))
        return x.value, lo.value, hi.value

    def update_consensus(self, stream: int = 0, res3_dev_ptr: int = 0):
        """res3_dev_ptr: 3 device doubles (primal, dual, first failed branch or -1)."""
        self._check(self.lib.tb_admm_update_consensus(self._h, C.c_void_p(stream or 0), C.c_void_p(res3_dev_ptr)))

    def get(self, what: int) -> np.ndarray:
        g = self.grid
        if what in (COST, LINE_VIOL):
            out = np.zeros(1)
        elif what == AUGLAG_ROUNDS:
            out = np.zeros(1, np.int64)
        elif what in (BRANCH_X,):
            out = np.zeros((g.n_branch, self.options.branch_dim))
        elif what == BRANCH_PARAMS:
            out = np.zeros((g.n_branch, 36))
        elif what == BRANCH_STATUS:
            out = np.zeros(g.n_branch, np.int32)
        elif what == STAGE_TIMES:
            out = np.zeros(2)
        elif what in (BUS_WT, BUS_TT):
            out = np.zeros(g.n_bus)
        else:
            out = np.zeros(g.n_gen)
        self._check(self.lib.tb_admm_get(self._h, what, out.ctypes.data))
        return out


def branch_bounds(grid: Grid, dim: int = 4):
    """The branch subproblems' bounds (v in [v_min, v_max] of
    the end buses, theta in [-2 pi, 2 pi]; dim 6 adds the slacks s in
    [-s-bar^2, 0]) -- the same boxes tb_admm_create builds."""
    n = grid.n_branch
    lo = np.stack([grid.bus_vmin[grid.br_from], grid.bus_vmin[grid.br_to], np.full(n, -2 * np.pi),
                   np.full(n, -2 * np.pi)], 1)
    up = np.stack([grid.bus_vmax[grid.br_from], grid.bus_vmax[grid.br_to], np.full(n, 2 * np.pi),
                   np.full(n, 2 * np.pi)], 1)
    if dim == 6:
        sm = grid.br_smax2 if grid.br_smax2 is not None else np.full(n, np.inf)
        lo = np.concatenate([lo, -np.stack([sm, sm], 1)], 1)
        up = np.concatenate([up, np.zeros((n, 2))], 1)
    return lo, up


def partition_stage_times(solver, x, params, lower, upper, parts, device=0):
    """Per-partition batch times of one branch stage (SPEC.md:408 history,
    PAPER.md:689-703): each partition's share of the branch subproblems
    (`parts`: a list of index arrays, e.g. contiguous even ranges as in
    batch.hpp:61-70) solved alone on the device from the same warm starts
    and multipliers the stage used; its kernel time is what one GPU of a
    len(parts)-GPU run spends on the stage.  `solver`: a tron.Solver."""
    import torch

    from .tron import ProblemBatch, Solver as _S

    dev = torch.device("cuda", device)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    dim = x.shape[1]
    X, P, Lo, Up = t(x), t(params), t(lower), t(upper)
    out = []
    for idx in parts:
        i = torch.as_tensor(np.asarray(idx, dtype=np.int64), device=dev)
        sub = ProblemBatch(3, dim, Lo[i].contiguous(), Up[i].contiguous(), P[i].contiguous(), X[i].contiguous())
        res = _S.alloc_result(len(idx), dim, device=True)
        solver.solve_batch(sub, out=res)  # warm-up launch of the same share
        solver.solve_batch(sub, out=res)
        out.append(res.kernel_time)
    return out


def _admm_error(rc: int, msg: str) -> Exception:
    """The reference's exception type for a failed branch solve (batch.hpp:75-76
    rethrows it out of solve_batch, and admm_solve propagates it)."""
    from .tron import EvaluationError, SingularFactorError

    if rc == TB_E_PROBLEM:
        if "EvaluationError" in msg:
            return EvaluationError(msg)
        if "SingularFactorError" in msg:
            return SingularFactorError(msg)
        return ValueError(msg)
    return SolverError(msg)


class ShardedAdmm:
    """One process per GPU under torch.distributed (NCCL): the C5 path."""

    def __init__(self, grid: Grid, rank: int, world: int, device: int, options: AdmmOptions = None,
                 record_times: bool = False):
        import torch

        self.torch = torch
        self.dev = torch.device("cuda", device)
        chunk = (grid.n_branch + world - 1) // world
        self.chunk, self.rank, self.world = chunk, rank, world
        dim = (options or AdmmOptions()).branch_dim
        # the branch-solution buffer the all-gather writes into (caller-owned)
        self.x = torch.zeros((chunk * world, dim), dtype=torch.float64, device=self.dev)
        self.res = torch.zeros(3, dtype=torch.float64, device=self.dev)
        self.solver = AdmmSolver(grid, options, device, rank, world, x_buffer_ptr=self.x.data_ptr())
        self.history: List[Tuple[float, float]] = []
        # per-iteration device time of this shard's branch stage (generators +
        # branch TRON), read back lazily: partition_times() all-gathers them
        self.record_times = record_times
        self._ev: List[tuple] = []

    def step(self) -> Tuple[float, float]:
        import torch.distributed as dist

        cs = self.torch.cuda.current_stream(self.dev)
        st = cs.cuda_stream
        st = st if st != 0 else 1  # cudaStreamLegacy
        if self.record_times:
            e0, e1 = self.torch.cuda.Event(enable_timing=True), self.torch.cuda.Event(enable_timing=True)
            e0.record(cs)
        self.solver.solve_components(st)
        if self.record_times:
            e1.record(cs)
            self._ev.append((e0, e1))
        if self.world > 1:  # consensus exchange: in-place all-gather of the branch solutions
            mine = self.x[self.rank * self.chunk:(self.rank + 1) * self.chunk]
            self._all_gather(self.x, mine)
        self.solver.update_consensus(st, self.res.data_ptr())
        if self.world > 1:
            self._all_reduce_max(self.res)
        p, d, bad = self.res.tolist()
        self.history.append((p, d))
        if bad >= 0:  # a failed branch solve propagates (from every rank)
            b = int(bad)
            lo, hi = self.rank * self.chunk, (self.rank + 1) * self.chunk
            st_ = int(self.solver.get(BRANCH_STATUS)[b]) if lo <= b < hi else -1
            raise SolverError(f"ADMM branch stage: branch {b} failed with status {st_}")
        return p, d

    # NCCL moves the device buffers directly (the GPU path); other backends
    # (gloo: several ranks sharing one GPU in the tests) go through host copies
    # of the same bytes, so the trajectory is identical either way
    def _nccl(self) -> bool:
        import torch.distributed as dist

        return dist.get_backend() == "nccl"

    def _all_gather(self, out, mine):
        import torch.distributed as dist

        if self._nccl():
            dist.all_gather_into_tensor(out, mine)
            return
        h = mine.cpu()
        ho = self.torch.empty((out.shape[0],) + tuple(out.shape[1:]), dtype=out.dtype)
        dist.all_gather_into_tensor(ho, h)
        out.copy_(ho)

    def _all_reduce_max(self, t):
        import torch.distributed as dist

        if self._nccl():
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX)
        t.copy_(h)

    def partition_times(self) -> List[List[float]]:
        """[iteration][rank] seconds of the branch stage of every recorded
        iteration (SPEC.md:408 per-partition batch times; feed imbalance())."""
        import torch.distributed as dist

        self.torch.cuda.synchronize(self.dev)
        mine = self.torch.tensor([1e-3 * a.elapsed_time(b) for a, b in self._ev], dtype=torch_f64(self.torch),
                                 device=self.dev)
        if self.world == 1:
            return [[t] for t in mine.tolist()]
        if not self._nccl():
            mine = mine.cpu()
        allt = [self.torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(allt, mine)
        return [list(r) for r in zip(*[a.tolist() for a in allt])]


def torch_f64(torch):
    return torch.float64
