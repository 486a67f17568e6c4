"""MATPOWER parsing (SPEC.md acopf-admm `parse_matpower` / `branch_params`),
ADMM acceptance 6(b) on case9, and the CLI's usage / exit-code contract
(SPEC.md `cli`).  The GPU tests run the device ADMM on case9 against the
oracle and drive the CLI end to end."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2106_14995_b200 import admm as A
from paper_2106_14995_b200 import matpower, synth

HERE = os.path.dirname(os.path.abspath(__file__))
CASE9 = os.path.join(HERE, "data", "case9.m")
ROOT = os.path.dirname(HERE)


def _text():
    return open(CASE9).read()


def test_case9_counts_and_per_unit():
    c = matpower.load(CASE9)
    g = c.grid
    assert (g.n_bus, g.n_gen, g.n_branch) == (9, 3, 9)  # SPEC example
    assert c.base_mva == 100.0
    assert np.allclose(g.bus_pd[[4, 6, 8]], [0.9, 1.0, 1.25]) and np.allclose(g.bus_qd[[4, 6, 8]], [0.3, 0.35, 0.5])
    assert np.allclose(g.gen_pmax, [2.5, 3.0, 2.7]) and np.allclose(g.gen_pmin, 0.1)
    # per-unit cost (cost_scale = 1/baseMVA): c2 * base, c1 unchanged
    assert np.allclose(g.gen_c2, [11.0, 8.5, 12.25]) and np.allclose(g.gen_c1, [5.0, 1.2, 1.0])
    assert np.allclose(g.br_smax2, (np.array([250, 250, 150, 300, 150, 250, 250, 250, 250]) / 100.0) ** 2)
    assert list(g.br_from) == [0, 3, 4, 2, 5, 6, 7, 7, 8] and list(g.br_to) == [3, 4, 5, 5, 6, 7, 1, 8, 3]


def test_branch_params_match_complex_pi_model_with_tap_and_shift():
    """SPEC branch_params example: flows from the 8 coefficients equal the
    direct complex pi-model S = V (Y V)* (tap 1.05, shift 10 deg)."""
    txt = _text().replace("\t4\t5\t0.017\t0.092\t0.158\t250\t250\t250\t0\t0\t1",
                          "\t4\t5\t0.017\t0.092\t0.158\t250\t250\t250\t1.05\t10\t1")
    c = matpower.parse(txt)
    cf = c.grid.br_coef[1]
    r, x, bc, tap, sh = 0.017, 0.092, 0.158, 1.05, np.deg2rad(10.0)
    ys = 1.0 / complex(r, x)
    t = tap * np.exp(1j * sh)
    Yff, Yft, Ytf, Ytt = (ys + 0.5j * bc) / (tap * tap), -ys / np.conj(t), -ys / t, ys + 0.5j * bc
    rng = np.random.default_rng(1)
    for _ in range(20):
        vi, vj = rng.uniform(0.9, 1.1, 2)
        ti, tj = rng.uniform(-0.3, 0.3, 2)
        Vi, Vj = vi * np.exp(1j * ti), vj * np.exp(1j * tj)
        Sij = Vi * np.conj(Yff * Vi + Yft * Vj)
        Sji = Vj * np.conj(Ytf * Vi + Ytt * Vj)
        f = synth.branch_flows(cf, vi, vj, ti, tj)
        assert np.allclose(f, [Sij.real, Sij.imag, Sji.real, Sji.imag], atol=1e-12)


def test_status_filters_and_tap_default():
    txt = _text().replace("\t2\t163\t6.54\t300\t-300\t1.025\t100\t1\t", "\t2\t163\t6.54\t300\t-300\t1.025\t100\t0\t")
    txt = txt.replace("\t8\t9\t0.032\t0.161\t0.306\t250\t250\t250\t0\t0\t1", "\t8\t9\t0.032\t0.161\t0.306\t250\t250\t250\t0\t0\t0")
    c = matpower.parse(txt)
    assert c.grid.n_gen == 2 and list(c.gen_rows) == [0, 2]
    assert c.grid.n_branch == 8 and 7 not in list(c.branch_rows)
    # ratio 0 -> tap 1: the coefficients equal an explicit tap of 1
    c1 = matpower.parse(_text().replace("\t1\t4\t0\t0.0576\t0\t250\t250\t250\t0\t", "\t1\t4\t0\t0.0576\t0\t250\t250\t250\t1\t"))
    assert np.array_equal(c1.grid.br_coef[0], matpower.load(CASE9).grid.br_coef[0])


@pytest.mark.parametrize("edit,msg", [
    (lambda t: t.replace("mpc.branch = [", "mpc.notbranch = ["), "mpc.branch"),
    (lambda t: t.replace("\t5\t1\t90\t30", "\t5\t1\tninety\t30"), "malformed row"),
    (lambda t: t.replace("\t8\t2\t0\t0.0625", "\t8\t22\t0\t0.0625"), "bus 22"),
    (lambda t: t.replace("\t3\t6\t0\t0.0586", "\t3\t6\t0\t0"), "zero impedance"),
    (lambda t: t.replace("\t2\t1500\t0\t3\t0.11\t5\t150", "\t1\t1500\t0\t2\t0\t0\t100\t500"), "polynomial"),
    (lambda t: t.replace("mpc.baseMVA = 100;", ""), "mpc.baseMVA"),
])
def test_parse_errors(edit, msg):
    with pytest.raises(matpower.MatpowerError, match=msg):
        matpower.parse(edit(_text()))


def test_malformed_row_reports_line_number():
    txt = _text().replace("\t7\t1\t100\t35", "\t7\t1\t1O0\t35")
    line = next(k for k, l in enumerate(txt.split("\n"), 1) if "1O0" in l)
    with pytest.raises(matpower.MatpowerError, match=f"line {line}:"):
        matpower.parse(txt)


def _case9_nlp(case):
    """Independent full AC-OPF NLP of case9 (scipy SLSQP, polar form, 24 vars)."""
    from scipy.optimize import minimize

    g = case.grid
    nb, ng, nl = g.n_bus, g.n_gen, g.n_branch

    def flows(z):
        v, th = z[2 * ng:2 * ng + nb], z[2 * ng + nb:]
        return synth.branch_flows(g.br_coef, v[g.br_from], v[g.br_to], th[g.br_from], th[g.br_to])

    def balance(z):
        pg, qg = z[:ng], z[ng:2 * ng]
        v = z[2 * ng:2 * ng + nb]
        f = flows(z)
        P = -g.bus_pd - g.bus_gsh * v * v
        Q = -g.bus_qd + g.bus_bsh * v * v
        np.add.at(P, g.gen_bus, pg)
        np.add.at(Q, g.gen_bus, qg)
        np.add.at(P, g.br_from, -f[:, 0])
        np.add.at(Q, g.br_from, -f[:, 1])
        np.add.at(P, g.br_to, -f[:, 2])
        np.add.at(Q, g.br_to, -f[:, 3])
        return np.concatenate([P, Q])

    z0 = np.concatenate([0.5 * (g.gen_pmin + g.gen_pmax), np.zeros(ng), np.ones(nb), np.zeros(nb)])
    bounds = ([(lo, hi) for lo, hi in zip(g.gen_pmin, g.gen_pmax)] + [(lo, hi) for lo, hi in zip(g.gen_qmin, g.gen_qmax)]
              + [(lo, hi) for lo, hi in zip(g.bus_vmin, g.bus_vmax)] + [(-np.pi, np.pi)] * nb)
    cons = [{"type": "eq", "fun": balance}, {"type": "eq", "fun": lambda z: z[2 * ng + nb]}]
    res = minimize(lambda z: case.cost(z[:ng]), z0, bounds=bounds, constraints=cons, method="SLSQP",
                   options={"ftol": 1e-12, "maxiter": 1000})
    assert res.success, res.message
    return res.fun


def test_case9_admm_acceptance_6b():
    """SPEC acceptance 6(b): case9 reaches primal <= 1e-4 within 5000
    iterations with generation cost within 1 % of the full-NLP oracle."""
    case = matpower.load(CASE9)
    a = po.OracleAdmm(case.grid)
    for k in range(5000):
        p, d = a.step()
        if p <= 1e-4 and d <= 1e-3:
            break
    assert p <= 1e-4, (k, p, d)
    cost = case.cost(a.get(A.GEN_P))
    nlp = _case9_nlp(case)
    assert abs(cost - nlp) <= 0.01 * nlp, (cost, nlp)
    assert abs(cost - 5296.69) <= 1.0  # MATPOWER's runopf optimum for case9


def _cli(*args, cwd=ROOT):
    return subprocess.run([sys.executable, "-m", "paper_2106_14995_b200", *args], capture_output=True, text=True,
                          cwd=cwd, timeout=600)


@pytest.mark.parametrize("args", [["--mode", "bench", "--n", "65"], ["--mode", "admm", "--case", "/nonexistent.m"],
                                  ["--bogus"], ["--mode", "admm"]])
def test_cli_usage_errors_exit_2(args, tmp_path):
    r = _cli(*args, "--out", str(tmp_path))
    assert r.returncode == 2 and "error:" in r.stderr


def test_cli_parse_error_exit_2(tmp_path):
    bad = tmp_path / "bad.m"
    bad.write_text(_text().replace("mpc.gen = [", "mpc.generators = ["))
    r = _cli("--mode", "admm", "--case", str(bad), "--out", str(tmp_path))
    assert r.returncode == 2 and "mpc.gen" in r.stderr


# ------------------------------------------------------------ device
@pytest.mark.gpu
def test_device_admm_case9_bitwise_and_converged():
    case = matpower.load(CASE9)
    dev, cpu = A.AdmmSolver(case.grid), po.OracleAdmm(case.grid)
    for k in range(5000):
        rd = dev.step()
        assert rd == cpu.step(), k
        if rd[0] <= 1e-4 and rd[1] <= 1e-3:
            break
    assert rd[0] <= 1e-4
    assert abs(case.cost(dev.get(A.GEN_P)) - 5296.69) <= 1.0


@pytest.mark.gpu
def test_cli_bench_and_admm(tmp_path):
    r = _cli("--mode", "bench", "--n", "8", "--batch", "100", "--out", str(tmp_path))
    assert r.returncode == 0, r.stderr
    rows = open(tmp_path / "bench.csv").read().strip().split("\n")
    assert len(rows) == 101 and rows[0].startswith("problem,status")
    assert all(row.split(",")[1] == "0" and float(row.split(",")[3]) == 120.0 - 40320.0 for row in rows[1:])
    s = json.load(open(tmp_path / "bench.json"))
    assert s["failures"] == 0 and s["batch"] == 100
    r = _cli("--mode", "bench", "--n", "8", "--batch", "0", "--out", str(tmp_path / "empty"))
    assert r.returncode == 0
    r = _cli("--mode", "admm", "--case", CASE9, "--out", str(tmp_path / "a"), "--workers", "2")
    assert r.returncode == 0, r.stderr
    s = json.load(open(tmp_path / "a" / "admm.json"))
    assert s["status"] == "converged" and abs(s["objective"] - 5296.69) <= 1.0 and "imbalance" in s
    assert s["imbalance"]["partitions"] == 2 and s["imbalance"]["iterations"] == s["iterations"]
    hdr = open(tmp_path / "a" / "admm.csv").readline().strip().split(",")
    assert hdr[-3:] == ["stage_time_s", "batch_time_p0", "batch_time_p1"]
    r = _cli("--mode", "admm", "--case", CASE9, "--max-iter", "1", "--out", str(tmp_path / "b"))
    assert r.returncode == 1
    assert len(open(tmp_path / "b" / "admm.csv").read().strip().split("\n")) == 2
