"""Randomized bitwise parity fuzz (GPU vs the CPU oracle): families, dims
1..128, TronConfig variants, bound patterns (infinite, l == u, starts outside
the box), kernel forms and launch orders.  python scripts/fuzz_parity.py [seconds] [seed]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import pyoracle as po  # noqa: E402
from paper_2106_14995_b200 import KernelForm, LaunchOrder, ProblemBatch, Solver, TronConfig, synth  # noqa: E402

FIELDS = ("x_star", "f_star", "pg_norm", "status", "iterations", "cg_iterations", "f_evals")
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
s = Solver((0,))
t_end = time.time() + budget
cases = fails = 0
while time.time() < t_end:
    fam = rng.choice(["ncvx", "boxqp", "hs45", "branch"], p=[0.45, 0.3, 0.1, 0.15])
    if fam == "branch":
        d = int(rng.choice([4, 6]))
        # FUZZ_BIG=1: also batches past one wave (AUTO ranks them; the d = 4 thread form from 16,384)
        n = int(rng.integers(1, 3000 if not os.environ.get("FUZZ_BIG") or rng.random() < 0.7 else 24000))
    else:
        d = int(rng.choice([rng.integers(1, 21), rng.integers(21, 65), rng.integers(65, 129)], p=[0.6, 0.3, 0.1]))
        n = int(rng.integers(1, 400 if d <= 20 else (48 if d <= 64 else 8)))
    seed = int(rng.integers(0, 1 << 30))
    b = synth.make(fam, n, d, seed) if fam != "hs45" else synth.hs45(n, min(d, 64))
    d = b.dim
    x0 = b.x0.copy()
    if fam != "hs45" and rng.random() < 0.5:  # bound patterns
        m = rng.random(b.lower.shape)
        b.lower[m < 0.05] = -np.inf
        b.upper[m > 0.95] = np.inf
        eq = (m > 0.45) & (m < 0.48)
        b.upper[eq] = b.lower[eq]  # fixed variables (never free: strict inequalities)
    if rng.random() < 0.3:
        x0 = x0 * rng.uniform(1.5, 6.0)  # starts outside the box (projected)
    if fam == "boxqp" and rng.random() < 0.25:  # extreme scales: quotients outside the Markstein range
        hs, cs = 10.0 ** rng.uniform(-300, 250), 10.0 ** rng.uniform(-250, 250)
        xs = 10.0 ** rng.uniform(-250, 250)
        b.params[:, :d * d] *= hs
        b.params[:, d * d:] *= cs
        b.lower *= xs
        b.upper *= xs
        x0 = x0 * xs
    kw = {}
    r = rng.random()
    if r < 0.15:
        kw = dict(max_iter=int(rng.integers(1, 6)))
    elif r < 0.3:
        kw = dict(delta0=float(rng.uniform(0.01, 3.0)))
    elif r < 0.45:
        kw = dict(cg_tol=float(rng.uniform(0.01, 0.9)), mu0=float(rng.uniform(0.001, 0.5)),
                  interp_factor=float(rng.uniform(0.1, 0.9)))
    elif r < 0.55:
        kw = dict(tol_pg=float(10.0 ** rng.uniform(-300, -3)))
    cfg = TronConfig(**kw)
    # kernel form: AUTO routing, or a forced form where it exists for d
    forms = [KernelForm.AUTO, KernelForm.WARP] + ([KernelForm.THREAD] if d == 4 and fam in ("ncvx", "branch") else []) \
        + ([KernelForm.BLOCK] if d >= 9 and fam != "branch" else [])
    form = forms[int(rng.integers(0, len(forms)))]
    s.set_form(form)
    order = list(LaunchOrder)[int(rng.integers(0, len(LaunchOrder)))]  # START_PG ranks at any size
    s.set_order(order)
    try:
        counted = bool(rng.random() < 0.2) and form != KernelForm.THREAD  # the thread form does not count
        res = s.solve_batch(b, x0, cfg=cfg, count_flops=counted)
        err = None
    except Exception as e:  # the reference would have thrown: compare with the oracle's rc
        res, err = None, e
    ref = po.solve_batch(b, x0, cfg=cfg, impl="oracle", workers=8)
    cases += 1
    ok = True
    if res is None:
        ok = ref.rc != 0
    else:
        if counted and not np.array_equal(np.asarray(res.flops), ref.flops):
            ok = False
            print(f"MISMATCH {fam} d={d} n={n} seed={seed} cfg={kw} form={form.name} order={order.name} field flops", flush=True)
        for k in FIELDS:
            a, c = np.asarray(getattr(res, k)), getattr(ref, k)
            if a.dtype.kind == "f":
                eq = (a.view(np.int64) == c.view(np.int64)) | (np.isnan(a) & np.isnan(c))
            else:
                eq = a == c
            if not eq.all():
                ok = False
                print(f"MISMATCH {fam} d={d} n={n} seed={seed} cfg={kw} form={form.name} order={order.name} field {k}", flush=True)
                break
    if not ok:
        fails += 1
        if res is None:
            print(f"MISMATCH {fam} d={d} n={n} seed={seed} cfg={kw}: device raised {err!r}, oracle rc {ref.rc}")
print(f"fuzz: {cases} cases, {fails} mismatches", flush=True)
sys.exit(1 if fails else 0)
