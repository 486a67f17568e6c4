"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers:

  oracle/build/liboracle.so  the plain-C restatement (tron_oracle.c)
  oracle/_ref/libtronref.so  the reference headers compiled unmodified

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtronref.so")
REF_TESTS = os.path.join(HERE, "_ref", "ref_unit_tests")
ORACLE_TESTS = os.path.join(HERE, "build", "oracle_unit_tests")

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int32)
lp = C.POINTER(C.c_int64)


def build(ref: bool = True) -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _p(a, t=dp):
    return None if a is None else a.ctypes.data_as(t)


def config_c(cfg=None):
    """TronConfig (python dataclass or None) -> tb_tron_config."""
    from paper_2106_14995_b200._lib import TronConfigC

    c = TronConfigC()
    c.tol_pg, c.has_delta0, c.delta0, c.max_iter = 1e-6, 0, 0.0, 200
    c.cg_tol, c.eta0, c.sigma1, c.sigma2, c.sigma3 = 0.1, 1e-4, 0.25, 0.5, 4.0
    c.mu0, c.mu1, c.interp_factor, c.delta_max = 1e-2, 1.0, 0.5, 1e10
    if cfg is not None:
        c = cfg.to_c()
    return c


class _Lib:
    def __init__(self, path, prefix):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} not built (make -C oracle{' ref' if prefix == 'ref' else ''})")
        self.lib = C.CDLL(path)
        self.prefix = prefix

    def fn(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")


_oracle = None
_ref = None


def oracle_lib() -> _Lib:
    global _oracle
    if _oracle is None:
        _oracle = _Lib(ORACLE_SO, "orc")
    return _oracle


def ref_lib() -> _Lib:
    global _ref
    if _ref is None:
        _ref = _Lib(REF_SO, "ref")
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class Result:
    def __init__(self, N, n):
        self.x_star = np.zeros((N, n))
        self.f_star = np.zeros(N)
        self.pg_norm = np.zeros(N)
        self.status = np.zeros(N, np.int32)
        self.iterations = np.zeros(N, np.int32)
        self.cg_iterations = np.zeros(N, np.int64)
        self.f_evals = np.zeros(N, np.int64)
        self.flops = np.zeros(N, np.int64)
        self.executed = np.zeros(N, np.int32)
        self.ff_iter = np.zeros(N, np.int32)
        self.per_problem_time = np.zeros(N)
        self.batch_wall_time = 0.0
        self.rc = 0


def _arrays(batch, x0):
    x0 = np.ascontiguousarray(batch.x0 if x0 is None else x0, dtype=np.float64)
    lo = np.ascontiguousarray(batch.lower, dtype=np.float64)
    up = np.ascontiguousarray(batch.upper, dtype=np.float64)
    prm = None if batch.params is None else np.ascontiguousarray(batch.params, dtype=np.float64)
    stride = 0 if prm is None else prm.shape[1]
    return x0, lo, up, prm, stride


def set_fast_forward(on: bool) -> None:
    """Opt-in replay-skip of zero-change fixed points in the C restatement."""
    oracle_lib().fn("set_fast_forward")(1 if on else 0)


def solve_batch(batch, x0=None, cfg=None, workers=1, impl="oracle") -> Result:
    """solve_batch on the CPU: impl="oracle" (C restatement) or "ref"
    (reference headers).  Returns arrays + rc (0 or the status the reference
    threw)."""
    x0, lo, up, prm, stride = _arrays(batch, x0)
    N, n = x0.shape
    r = Result(N, n)
    c = config_c(cfg)
    wall = C.c_double()
    if impl == "oracle":
        # solve() validates first (tron.hpp:457 -> :70-80, std::invalid_argument)
        v = oracle_lib().fn("config_validate")
        v.restype = C.c_int
        msg = C.c_char_p()
        if v(C.byref(c), C.byref(msg)):
            raise ValueError(msg.value.decode())
        f = oracle_lib().fn("solve_batch")
        f.restype = C.c_int
        r.rc = f(int(batch.family), n, C.c_int64(N), _p(x0), _p(lo), _p(up), _p(prm), C.c_int64(stride),
                 C.byref(c), int(workers), _p(r.x_star), _p(r.f_star), _p(r.pg_norm), _p(r.status, ip),
                 _p(r.iterations, ip), _p(r.cg_iterations, lp), _p(r.f_evals, lp), _p(r.flops, lp),
                 _p(r.executed, ip), _p(r.ff_iter, ip), C.byref(wall))
    else:
        f = ref_lib().fn("solve_batch")
        f.restype = C.c_int
        parts = np.zeros(max(1, workers))
        r.rc = f(int(batch.family), n, C.c_int64(N), _p(x0), _p(lo), _p(up), _p(prm), C.c_int64(stride),
                 C.byref(c), int(workers), _p(r.x_star), _p(r.f_star), _p(r.pg_norm), _p(r.status, ip),
                 _p(r.iterations, ip), _p(r.cg_iterations, lp), _p(r.f_evals, lp), _p(r.per_problem_time),
                 _p(parts), C.byref(wall))
        r.partition_times = parts
    r.batch_wall_time = wall.value
    return r


def family_eval(family, n, x, params=None):
    f = oracle_lib().fn("family_eval")
    fv = C.c_double()
    g = np.zeros(n)
    H = np.zeros(n * n)
    x = np.ascontiguousarray(x, dtype=np.float64)
    prm = None if params is None else np.ascontiguousarray(params, dtype=np.float64)
    f(int(family), n, _p(x), _p(prm), C.byref(fv), _p(g), _p(H))
    return fv.value, g, H.reshape(n, n).T.copy()  # col-major -> [i, j]


def last_error(impl="ref") -> str:
    if impl == "ref":
        f = ref_lib().fn("last_error")
        f.restype = C.c_char_p
        return f().decode()
    return ""


def run_unit_tests(which="oracle"):
    """Run the reference's own Catch2 tests (shim) against the C restatement
    (which="oracle") or the reference headers (which="ref")."""
    exe = ORACLE_TESTS if which == "oracle" else REF_TESTS
    p = subprocess.run([exe], capture_output=True, text=True)
    return p.returncode, p.stdout


class OracleAdmm:
    """CPU ADMM oracle (oracle/admm_oracle.c): same closed forms as the
    device (csrc/tb_admm.h), branch stage through the C TRON restatement."""

    def __init__(self, grid, options=None, workers=1):
        from paper_2106_14995_b200.admm import AdmmOptions

        self.lib = oracle_lib().lib
        self.grid = grid
        g, self._keep = grid.to_c()
        options = options or AdmmOptions()
        self.dim = options.branch_dim
        o = options.to_c(0, 1)
        h = C.c_void_p()
        self.lib.orc_admm_create.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        assert self.lib.orc_admm_create(C.addressof(g), C.addressof(o), int(workers), C.byref(h)) == 0
        self._g, self._o = g, o
        self._h = h
        self.history = []

    def step(self):
        p, d = C.c_double(), C.c_double()
        self.lib.orc_admm_step.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        rc = self.lib.orc_admm_step(self._h, C.byref(p), C.byref(d))
        assert rc == 0, f"TRON error status {rc} in the branch stage"
        self.history.append((p.value, d.value))
        return p.value, d.value

    def get(self, what):
        from paper_2106_14995_b200 import admm as A

        g = self.grid
        shapes = {A.BRANCH_X: ((g.n_branch, self.dim), np.float64), A.BRANCH_PARAMS: ((g.n_branch, 36), np.float64),
                  A.BRANCH_STATUS: ((g.n_branch,), np.int32), A.BUS_WT: ((g.n_bus,), np.float64),
                  A.BUS_TT: ((g.n_bus,), np.float64), A.COST: ((1,), np.float64),
                  A.AUGLAG_ROUNDS: ((1,), np.int64), A.LINE_VIOL: ((1,), np.float64)}
        shape, dt = shapes.get(what, ((g.n_gen,), np.float64))
        out = np.zeros(shape, dt)
        self.lib.orc_admm_get.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        assert self.lib.orc_admm_get(self._h, int(what), out.ctypes.data) == 0
        return out

    def close(self):
        if self._h:
            self.lib.orc_admm_destroy.argtypes = [C.c_void_p]
            self.lib.orc_admm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def admm_gen_p(c2, c1, lam, rho, ptil, pmin, pmax):
    f = oracle_lib().lib.orc_admm_gen_p
    f.restype = C.c_double
    f.argtypes = [C.c_double] * 7
    return f(c2, c1, lam, rho, ptil, pmin, pmax)
