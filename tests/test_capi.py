"""The C-ABI library: it loads, exports every symbol include/tb_capi.h
declares, mirrors the reference's config defaults/validation, and the product
package never touches the oracle.  No GPU compute here."""
import ctypes as C
import os
import re

import pytest

from paper_2106_14995_b200 import TronConfig, _lib, family_nparams

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "tb_capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), n
    from paper_2106_14995_b200 import admm

    bound = set(_lib.SIGNATURES) | set(admm._SIG)
    assert set(names) == bound, f"ctypes signatures must cover the header exactly: {set(names) ^ bound}"


def test_config_defaults_match_reference():
    """tron.hpp:54-68 defaults through tb_config_default."""
    c = _lib.TronConfigC()
    _lib.load().tb_config_default(C.byref(c))
    d = TronConfig()
    assert (c.tol_pg, c.has_delta0, c.max_iter, c.cg_tol, c.eta0) == (d.tol_pg, 0, d.max_iter, d.cg_tol, d.eta0)
    assert (c.sigma1, c.sigma2, c.sigma3, c.mu0, c.mu1, c.interp_factor, c.delta_max) == (
        0.25, 0.5, 4.0, 1e-2, 1.0, 0.5, 1e10)


def test_validate_uses_reference_messages():
    with pytest.raises(ValueError, match="TronConfig: need 0 < sigma1 < sigma2 < 1 < sigma3"):
        TronConfig(sigma2=1.5).validate()
    with pytest.raises(ValueError, match="TronConfig: max_iter must be >= 1"):
        TronConfig(max_iter=0).validate()


@pytest.mark.parametrize("bad", [dict(tol_pg=0.0), dict(delta0=-1.0), dict(eta0=1.0), dict(mu0=0.0),
                                 dict(interp_factor=1.0), dict(max_iter=0), dict(sigma1=0.6)])
def test_oracle_and_product_reject_the_same_configs(bad):
    """The oracle's solve_batch validates first like solve() (tron.hpp:457),
    with the messages the product raises (tb_config_validate)."""
    from oracle import pyoracle as po
    from paper_2106_14995_b200 import synth

    cfg = TronConfig(**bad)
    with pytest.raises(ValueError) as prod:
        cfg.validate()
    with pytest.raises(ValueError) as orc:
        po.solve_batch(synth.boxqp(2, 3), cfg=cfg, impl="oracle")
    assert str(orc.value) == str(prod.value)


def test_family_nparams():
    assert family_nparams(0, 8) == 0
    assert family_nparams(1, 4) == 20
    assert family_nparams(2, 4) == 22  # C1 ncvx P = 22
    assert family_nparams(3, 6) == 36
    assert family_nparams(3, 5) == -1
    assert family_nparams(9, 4) == -1


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2106_14995_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|pyoracle|tron_oracle|libtronref|liboracle",
                                     s, flags=re.M), f


def test_solver_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2106_14995_b200 import Solver, SolverError

    with pytest.raises(SolverError):
        Solver((0,))


def test_python_enums_match_the_header():
    """KernelForm / LaunchOrder mirror the header's TB_FORM_* / TB_ORDER_*."""
    from paper_2106_14995_b200 import KernelForm, LaunchOrder

    src = open(os.path.join(ROOT, "include", "tb_capi.h")).read()
    defs = {k: int(v) for k, v in re.findall(r"#define\s+(TB_(?:FORM|ORDER)_[A-Z_]+)\s+(\d+)", src)}
    forms = {k[len("TB_FORM_"):]: v for k, v in defs.items() if k.startswith("TB_FORM_")}
    orders = {k[len("TB_ORDER_"):]: v for k, v in defs.items() if k.startswith("TB_ORDER_")}
    assert forms == {m.name: int(m) for m in KernelForm}
    assert orders == {m.name: int(m) for m in LaunchOrder}
