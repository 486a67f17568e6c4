"""Python mirror of the reference solver API (tronbatch::solve_batch & co.)
over the C ABI.  Names, argument meaning and error behaviour follow
/root/reference/proj/include/tronbatch/{tron,batch}.hpp:

  TronConfig     tron.hpp:54-81   (validate() raises ValueError = std::invalid_argument)
  SolveStatus    tron.hpp:83
  SolveReport    tron.hpp:94-103
  BatchResult    batch.hpp:17-22
  solve_batch    batch.hpp:27-78  (workers -> devices; raises the reference's
                                   exception types when a problem would throw)
  imbalance      batch.hpp:80-111

Problems are described as a `ProblemBatch` (family id + bounds + parameters),
the device-side replacement for a std::vector of BoundedProblem callbacks.
Arrays may be numpy arrays (host, TB_MEM_HOST) or CUDA tensors exposing
`data_ptr()` (TB_MEM_DEVICE); results come back in the same memory space.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L


# ---------------------------------------------------------------- exceptions
class FactorizationError(RuntimeError):
    """dense.hpp:15-18"""


class SingularFactorError(RuntimeError):
    """dense.hpp:21-24"""


class EvaluationError(RuntimeError):
    """tron.hpp:21-24"""


class SolverError(RuntimeError):
    """CUDA / library failure (no reference equivalent)."""


class SolveStatus(enum.IntEnum):
    """tron.hpp:83, plus the device extensions of include/tb_capi.h."""

    Converged = 0
    IterLimit = 1
    FactorizationFailed = 2
    EvaluationError = 3
    ZeroDirection = 4
    SingularFactor = 5
    InvalidBounds = 6


class Family(enum.IntEnum):
    HS45 = L.TB_FAMILY_HS45
    BOXQP = L.TB_FAMILY_BOXQP
    NCVX = L.TB_FAMILY_NCVX
    BRANCH = L.TB_FAMILY_BRANCH


class KernelForm(enum.IntEnum):
    """tb_capi.h TB_FORM_*: which device kernel form solves a batch.  Every
    form returns the same bits; AUTO routes by family, dimension and size."""

    AUTO = 0
    WARP = 1    # one warp per problem (d <= 32)
    THREAD = 3  # one thread per problem (d = 4)
    BLOCK = 4   # 32 / 64 / 128 threads per problem, persistent (d >= 9)


class LaunchOrder(enum.IntEnum):
    """tb_capi.h TB_ORDER_*: which problems of a batch start first.  Results
    never depend on it; START_PG launches the problems in descending
    projected-gradient norm at their clipped start points (long solves
    first), AUTO where that was measured to pay, INDEX never."""

    AUTO = 0
    INDEX = 1
    START_PG = 2
    CALLER = 3  # the caller sorted the batch (its own cost model): one launch in index order


@dataclass
class TronConfig:
    """tron.hpp:54-81, same defaults."""

    tol_pg: float = 1e-6
    delta0: Optional[float] = None
    max_iter: int = 200
    cg_tol: float = 0.1
    eta0: float = 1e-4
    sigma1: float = 0.25
    sigma2: float = 0.5
    sigma3: float = 4.0
    mu0: float = 1e-2
    mu1: float = 1.0
    interp_factor: float = 0.5
    delta_max: float = 1e10

    def to_c(self) -> L.TronConfigC:
        c = L.TronConfigC()
        c.tol_pg = self.tol_pg
        c.has_delta0 = 0 if self.delta0 is None else 1
        c.delta0 = 0.0 if self.delta0 is None else float(self.delta0)
        c.max_iter = int(self.max_iter)
        for k in ("cg_tol", "eta0", "sigma1", "sigma2", "sigma3", "mu0", "mu1", "interp_factor", "delta_max"):
            setattr(c, k, float(getattr(self, k)))
        return c

    def validate(self) -> None:
        c = self.to_c()
        if L.load().tb_config_validate(C.byref(c)) != L.TB_OK:
            raise ValueError(L.last_error())


@dataclass
class SolveReport:
    """tron.hpp:94-103"""

    x_star: np.ndarray
    f_star: float
    pg_norm: float
    status: SolveStatus
    iterations: int
    cg_iterations: int
    f_evals: int
    wall_time: float


@dataclass
class ProblemBatch:
    """A batch of same-family problems: the device form of
    std::vector<P> problems (batch.hpp:28).  Arrays are [count, dim] and
    [count, nparams]."""

    family: int
    dim: int
    lower: object
    upper: object
    params: object = None
    x0: object = None  # default starting points (e.g. hs45 default_start)

    @property
    def count(self) -> int:
        return int(self.lower.shape[0])


@dataclass
class BatchResult:
    """batch.hpp:17-22 in structure-of-arrays form."""

    x_star: object
    f_star: object
    pg_norm: object
    status: object
    iterations: object
    cg_iterations: object
    f_evals: object
    per_problem_time: object
    flops: object
    partition_times: List[float] = field(default_factory=list)
    batch_wall_time: float = 0.0
    kernel_time: float = 0.0

    @property
    def reports(self) -> List[SolveReport]:
        def host(a):
            return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)

        xs, fs, ps, st, it, cg, fe, wt = map(
            host,
            (self.x_star, self.f_star, self.pg_norm, self.status, self.iterations,
             self.cg_iterations, self.f_evals, self.per_problem_time),
        )
        return [
            SolveReport(xs[i].copy(), float(fs[i]), float(ps[i]), SolveStatus(int(st[i])), int(it[i]),
                        int(cg[i]), int(fe[i]), float(wt[i]))
            for i in range(xs.shape[0])
        ]


def _is_device(a) -> bool:
    return a is not None and hasattr(a, "data_ptr") and getattr(a, "is_cuda", False)


def _ptr(a) -> int:
    if a is None:
        return 0
    if _is_device(a):
        assert a.is_contiguous(), "device arrays must be contiguous"
        return a.data_ptr()
    assert isinstance(a, np.ndarray) and a.flags["C_CONTIGUOUS"], "host arrays must be C-contiguous numpy"
    return a.ctypes.data


def _host_f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Solver:
    """Owns a tb_context (device streams + workspace).  `devices` plays the
    role of solve_batch's `workers`: contiguous even partitions per device."""

    def __init__(self, devices: Sequence[int] = (0,), fast_forward=True,
                 form: "KernelForm" = KernelForm.AUTO, order: "LaunchOrder" = LaunchOrder.AUTO):
        self._lib = L.load()
        arr = (C.c_int32 * len(devices))(*devices)
        ctx = C.c_void_p()
        if self._lib.tb_context_create(arr, len(devices), C.byref(ctx)) != L.TB_OK:
            raise SolverError(L.last_error())
        self._ctx = ctx
        self.devices = list(devices)
        ff = int(fast_forward) if not isinstance(fast_forward, bool) else (1 if fast_forward else 0)
        if self._lib.tb_context_set_mode(self._ctx, 0, ff) != L.TB_OK:
            raise SolverError(L.last_error())
        self.set_form(form)
        self.set_order(order)

    def set_order(self, order: "LaunchOrder") -> None:
        """Launch order of later solves (TB_ORDER_*; results are identical)."""
        if int(order) == 0 and not hasattr(self._lib, "tb_context_set_order"):
            self.order = LaunchOrder.AUTO  # older library build (A/B experiments)
            return
        if self._lib.tb_context_set_order(self._ctx, int(order)) != L.TB_OK:
            raise ValueError(L.last_error())
        self.order = LaunchOrder(int(order))

    def set_form(self, form: "KernelForm") -> None:
        """Kernel form of later solves (TB_FORM_*; results are identical)."""
        if int(form) == 0 and not hasattr(self._lib, "tb_context_set_form"):
            self.form = KernelForm.AUTO  # older library build (A/B experiments)
            return
        if self._lib.tb_context_set_form(self._ctx, int(form)) != L.TB_OK:
            raise ValueError(L.last_error())
        self.form = KernelForm(int(form))

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            self._lib.tb_context_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve_batch(self, problems: ProblemBatch, x0s=None, cfg: TronConfig = TronConfig(),
                    out: Optional[BatchResult] = None, stream=None, count_flops: bool = False) -> BatchResult:
        """batch.hpp:27-78.  x0s defaults to problems.x0.  count_flops selects
        the kernel variant that also counts algorithmic flops per problem
        (out.flops); results are identical either way."""
        x0s = problems.x0 if x0s is None else x0s
        if x0s is None:
            raise ValueError("solve_batch: no starting points")
        dev = _is_device(problems.lower)
        n, N = int(problems.dim), problems.count
        # every input array must live where `lower` lives (a host pointer
        # passed as device memory would fault and poison the CUDA context)
        for name, arr in (("x0s", x0s), ("upper", problems.upper), ("params", problems.params)):
            if arr is None:
                continue
            if _is_device(arr) != dev:
                raise ValueError(f"solve_batch: {name} is in {'device' if _is_device(arr) else 'host'} memory "
                                 f"but lower is in {'device' if dev else 'host'} memory")
            if dev and arr.device != problems.lower.device:
                raise ValueError(f"solve_batch: {name} is on {arr.device}, lower on {problems.lower.device}")
        if not dev:
            x0s = _host_f64(x0s)
            lower, upper = _host_f64(problems.lower), _host_f64(problems.upper)
            params = None if problems.params is None else _host_f64(problems.params)
        else:
            lower, upper, params = problems.lower, problems.upper, problems.params
        if tuple(x0s.shape) != (N, n) or tuple(lower.shape) != (N, n) or tuple(upper.shape) != (N, n):
            raise ValueError("solve_batch: problems and x0s length mismatch")
        stride = int(params.shape[1]) if params is not None and N > 0 else 0

        b = L.ProblemBatchC()
        b.family, b.dim, b.count = int(problems.family), n, N
        b.x0, b.lower, b.upper, b.params = _ptr(x0s), _ptr(lower), _ptr(upper), _ptr(params)
        b.params_stride = stride
        b.memspace = L.TB_MEM_DEVICE if dev else L.TB_MEM_HOST

        if out is None:
            out = self.alloc_result(N, n, device=dev)
        r = L.BatchResultC()
        r.x_star, r.f_star, r.pg_norm = _ptr(out.x_star), _ptr(out.f_star), _ptr(out.pg_norm)
        r.status, r.iterations = _ptr(out.status), _ptr(out.iterations)
        r.cg_iterations, r.f_evals = _ptr(out.cg_iterations), _ptr(out.f_evals)
        r.wall_time, r.flops = _ptr(out.per_problem_time), (_ptr(out.flops) if count_flops else 0)
        r.memspace = L.TB_MEM_DEVICE if _is_device(out.status) else L.TB_MEM_HOST
        c = cfg.to_c()
        if stream is not None:
            # 0 is the legacy default stream (torch's default): pass it as
            # cudaStreamLegacy (0x1); NULL would select the context stream
            h = int(stream) if int(stream) != 0 else 1
            rc = self._lib.tb_solve_batch_async(self._ctx, C.byref(b), C.byref(c), C.byref(r), C.c_void_p(h))
            if rc != L.TB_OK:
                _raise(rc)
            return out
        rc = self._lib.tb_solve_batch(self._ctx, C.byref(b), C.byref(c), C.byref(r))
        out.partition_times = [r.partition_times[k] for k in range(r.n_partitions)]
        out.batch_wall_time = r.batch_wall_time
        out.kernel_time = r.kernel_time
        if rc != L.TB_OK:
            _raise(rc)
        return out

    @staticmethod
    def alloc_result(N: int, n: int, device: bool = False) -> BatchResult:
        if device:
            import torch

            dv = torch.device("cuda", torch.cuda.current_device())
            f64 = dict(dtype=torch.float64, device=dv)
            return BatchResult(
                torch.empty((N, n), **f64), torch.empty(N, **f64), torch.empty(N, **f64),
                torch.empty(N, dtype=torch.int32, device=dv), torch.empty(N, dtype=torch.int32, device=dv),
                torch.empty(N, dtype=torch.int64, device=dv), torch.empty(N, dtype=torch.int64, device=dv),
                torch.empty(N, **f64), torch.empty(N, dtype=torch.int64, device=dv),
            )
        return BatchResult(
            np.empty((N, n)), np.empty(N), np.empty(N), np.empty(N, np.int32), np.empty(N, np.int32),
            np.empty(N, np.int64), np.empty(N, np.int64), np.empty(N), np.empty(N, np.int64),
        )


def _raise(rc: int) -> None:
    msg = L.last_error()
    if rc == L.TB_E_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == L.TB_E_PROBLEM:
        if "EvaluationError" in msg:
            raise EvaluationError(msg)
        if "SingularFactorError" in msg:
            raise SingularFactorError(msg)
        raise ValueError(msg)  # std::invalid_argument from trqsol / bounds
    raise SolverError(msg)


_default: Optional[Solver] = None


def default_solver() -> Solver:
    global _default
    if _default is None:
        _default = Solver((0,))
    return _default


def solve_batch(problems: ProblemBatch, x0s=None, cfg: TronConfig = TronConfig(),
                devices: Optional[Sequence[int]] = None) -> BatchResult:
    """tronbatch::solve_batch (batch.hpp:27-29); `devices` replaces `workers`."""
    if devices is None:
        return default_solver().solve_batch(problems, x0s, cfg)
    s = Solver(devices)
    try:
        return s.solve_batch(problems, x0s, cfg)
    finally:
        s.close()


@dataclass
class ImbalanceStats:
    """batch.hpp:80-85"""

    nu_per_iter: List[float]
    nu_max: float
    nu_min: float
    nu_mean: float


def imbalance(times_per_iter: Sequence[Sequence[float]]) -> ImbalanceStats:
    """batch.hpp:87-111: nu_k = (t_max/t_mean - 1) * 100."""
    if len(times_per_iter) == 0:
        raise ValueError("imbalance: need at least one iteration")
    t = np.ascontiguousarray(times_per_iter, dtype=np.float64)
    if t.ndim != 2:
        raise ValueError("imbalance: ragged partition times")
    k, p = t.shape
    nu = np.empty(k)
    mx, mn, me = C.c_double(), C.c_double(), C.c_double()
    dp = C.POINTER(C.c_double)
    rc = L.load().tb_imbalance(t.ctypes.data_as(dp), k, p, nu.ctypes.data_as(dp), C.byref(mx), C.byref(mn), C.byref(me))
    if rc != L.TB_OK:
        raise ValueError(L.last_error())
    return ImbalanceStats(nu.tolist(), mx.value, mn.value, me.value)


def family_nparams(family: int, dim: int) -> int:
    return int(L.load().tb_family_nparams(int(family), int(dim)))
