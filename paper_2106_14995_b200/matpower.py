"""MATPOWER case files -> admm.Grid (SPEC.md acopf-admm `parse_matpower`,
`branch_params`).

    grid = matpower.load("case9.m")            # or parse(text)
    hist = admm.AdmmSolver(grid).run(1000)

Host-side plumbing, no path arithmetic: the blocks `mpc.baseMVA`, `mpc.bus`,
`mpc.gen`, `mpc.branch`, `mpc.gencost` are read (whitespace / semicolon rows,
`%` comments, `...` continuations), powers are converted to per unit (divide by
baseMVA), out-of-service generators and branches and isolated buses (type 4)
are dropped, tap 0 defaults to 1, phase shifts go from degrees to radians,
and rateA becomes the line limit s-bar^2 = (rateA / baseMVA)^2 (0 = unlimited)
used when `AdmmOptions(line_limits=True)`.  Polynomial gencost (model 2) of
degree <= 2 is supported; piecewise-linear cost (model 1) is a parse error
(SPEC.md: "piecewise-linear cost -> parse error").

Generator costs with powers in per unit are c2 * baseMVA^2, c1 * baseMVA
(and c0, reported separately) in $/h, times `cost_scale`.  The default
cost_scale = 1 / baseMVA gives the per-unit cost (c1 stays the marginal cost
in $/MWh), which matches the per-unit ADMM penalties rho0 = 10 / 40; rescaling
the objective does not move the optimum.  `Case.cost` reports $/h.  (case9:
361 ADMM iterations to primal 1e-4, cost 5296.69 $/h = MATPOWER's runopf
optimum; with cost_scale = 1 the consensus needs far more iterations.)
"""
from __future__ import annotations

import math
import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from .admm import Grid
from .synth import pi_model


class MatpowerError(ValueError):
    """Parse error: missing block, malformed row or dangling reference (with
    the line number where it applies)."""


_BLOCK = re.compile(r"mpc\.(\w+)\s*=\s*", re.M)


@dataclass
class Case:
    """NetworkCase (SPEC.md acopf-admm) in per unit plus the id maps."""

    base_mva: float
    grid: Grid
    bus_ids: np.ndarray          # original bus number of each kept bus
    gen_rows: np.ndarray         # row index in mpc.gen of each kept generator
    branch_rows: np.ndarray      # row index in mpc.branch of each kept branch
    gen_c0: np.ndarray           # constant cost terms ($/h, times cost_scale)
    cost_scale: float = 1.0
    meta: Dict[str, object] = field(default_factory=dict)

    def cost(self, gen_p: np.ndarray) -> float:
        """Total generation cost in $/h at per-unit dispatch gen_p (c0 included)."""
        g = self.grid
        return float(np.sum(g.gen_c2 * gen_p * gen_p + g.gen_c1 * gen_p + self.gen_c0) / self.cost_scale)


def _strip(text: str) -> List[str]:
    out = []
    for line in text.split("\n"):
        k = line.find("%")
        out.append(line if k < 0 else line[:k])
    return out


def _blocks(text: str):
    """{name: (value_text, first_line_number)} for every `mpc.<name> = ...;`."""
    lines = _strip(text)
    src = "\n".join(lines).replace("...\n", " ")
    res = {}
    for m in _BLOCK.finditer(src):
        name = m.group(1)
        start = m.end()
        line_no = src.count("\n", 0, start) + 1
        if src[start:start + 1] == "[":
            end = src.find("]", start)
            if end < 0:
                raise MatpowerError(f"line {line_no}: mpc.{name}: unterminated matrix")
            res[name] = (src[start + 1:end], line_no)
        else:
            end = src.find(";", start)
            end = len(src) if end < 0 else end
            res[name] = (src[start:end], line_no)
    return res


def _matrix(name: str, blocks, min_cols: int) -> np.ndarray:
    if name not in blocks:
        raise MatpowerError(f"missing block mpc.{name}")
    body, line0 = blocks[name]
    rows = []
    line = line0
    for chunk in re.split(r"(;|\n)", body):
        if chunk == "\n":
            line += 1
            continue
        if chunk == ";":
            continue
        toks = chunk.replace(",", " ").split()
        if not toks:
            continue
        try:
            vals = [float(t) for t in toks]
        except ValueError:
            raise MatpowerError(f"line {line}: mpc.{name}: malformed row {chunk.strip()!r}") from None
        if len(vals) < min_cols:
            raise MatpowerError(f"line {line}: mpc.{name}: row has {len(vals)} columns, need >= {min_cols}")
        rows.append(vals)
    if not rows:
        return np.zeros((0, min_cols))
    width = max(len(r) for r in rows)
    return np.array([r + [0.0] * (width - len(r)) for r in rows])


def parse(text: str, cost_scale: Optional[float] = None) -> Case:
    blocks = _blocks(text)
    if "baseMVA" not in blocks:
        raise MatpowerError("missing block mpc.baseMVA")
    try:
        base = float(blocks["baseMVA"][0].strip())
    except ValueError:
        raise MatpowerError(f"line {blocks['baseMVA'][1]}: mpc.baseMVA: not a number") from None
    if not (base > 0.0):
        raise MatpowerError("mpc.baseMVA must be > 0")
    if cost_scale is None:
        cost_scale = 1.0 / base
    bus = _matrix("bus", blocks, 13)
    gen = _matrix("gen", blocks, 10)
    branch = _matrix("branch", blocks, 11)
    gencost = _matrix("gencost", blocks, 4)

    keep_bus = bus[:, 1] != 4
    ids = bus[keep_bus, 0].astype(np.int64)
    index = {int(b): k for k, b in enumerate(ids)}
    if len(index) != len(ids):
        raise MatpowerError("mpc.bus: duplicate bus number")
    b = bus[keep_bus]
    if np.any(b[:, 12] > b[:, 11]):
        raise MatpowerError("mpc.bus: Vmin > Vmax")

    def ref(v, what, row):
        k = index.get(int(v))
        if k is None:
            raise MatpowerError(f"{what} row {row + 1}: bus {int(v)} does not exist (or is isolated)")
        return k

    # generators in service (status column 8), with their cost rows
    if gencost.shape[0] < gen.shape[0]:
        raise MatpowerError("mpc.gencost: fewer rows than mpc.gen")
    g_rows = [r for r in range(gen.shape[0]) if gen[r, 7] > 0]
    c2 = np.zeros(len(g_rows))
    c1 = np.zeros(len(g_rows))
    c0 = np.zeros(len(g_rows))
    gbus = np.zeros(len(g_rows), np.int32)
    for k, r in enumerate(g_rows):
        gbus[k] = ref(gen[r, 0], "mpc.gen", r)
        model, ncost = int(gencost[r, 0]), int(gencost[r, 3])
        if model != 2:
            raise MatpowerError(f"mpc.gencost row {r + 1}: only polynomial cost (model 2) is supported")
        if ncost < 1 or ncost > 3:
            raise MatpowerError(f"mpc.gencost row {r + 1}: polynomial degree {ncost - 1} > 2 is not supported")
        coef = list(gencost[r, 4:4 + ncost])
        coef = [0.0] * (3 - ncost) + coef  # (c2, c1, c0)
        c2[k] = coef[0] * base * base * cost_scale
        c1[k] = coef[1] * base * cost_scale
        c0[k] = coef[2] * cost_scale
    pmax, pmin = gen[g_rows, 8] / base, gen[g_rows, 9] / base
    qmax, qmin = gen[g_rows, 3] / base, gen[g_rows, 4] / base
    if np.any(pmin > pmax) or np.any(qmin > qmax):
        raise MatpowerError("mpc.gen: Pmin > Pmax or Qmin > Qmax")

    # branches in service (status column 10)
    l_rows = [r for r in range(branch.shape[0]) if branch[r, 10] > 0]
    frm = np.array([ref(branch[r, 0], "mpc.branch", r) for r in l_rows], np.int32)
    to = np.array([ref(branch[r, 1], "mpc.branch", r) for r in l_rows], np.int32)
    br = branch[l_rows]
    r_, x_ = br[:, 2], br[:, 3]
    if np.any(r_ * r_ + x_ * x_ == 0.0):
        bad = l_rows[int(np.argmax(r_ * r_ + x_ * x_ == 0.0))]
        raise MatpowerError(f"mpc.branch row {bad + 1}: zero impedance")
    tap = np.where(br[:, 8] == 0.0, 1.0, br[:, 8])
    shift = br[:, 9] * (math.pi / 180.0)
    coef = pi_model(r_, x_, br[:, 4], tap, shift)
    rate = br[:, 5] / base
    smax2 = np.where(rate > 0.0, rate * rate, np.inf)

    grid = Grid(bus_pd=b[:, 2] / base, bus_qd=b[:, 3] / base, bus_gsh=b[:, 4] / base, bus_bsh=b[:, 5] / base,
                bus_vmin=b[:, 12].copy(), bus_vmax=b[:, 11].copy(), gen_bus=gbus, gen_c2=c2, gen_c1=c1,
                gen_pmin=pmin, gen_pmax=pmax, gen_qmin=qmin, gen_qmax=qmax, br_from=frm, br_to=to,
                br_coef=np.ascontiguousarray(coef), br_smax2=smax2)
    return Case(base, grid, ids, np.array(g_rows, np.int64), np.array(l_rows, np.int64), c0, cost_scale,
                {"n_bus_file": int(bus.shape[0]), "n_gen_file": int(gen.shape[0]),
                 "n_branch_file": int(branch.shape[0])})


def load(path: str, cost_scale: Optional[float] = None) -> Case:
    with open(path) as f:
        return parse(f.read(), cost_scale)
