"""Small invocations of every kernel form and the ADMM stages for
compute-sanitizer (scripts/sanitize.sh): warp form D = 4 / 6 / 8 / 16 / 32,
thread form, block kernel D = 32 / 64 / 128 (flop-counting variants too),
ranked launches (launch-order kernels), ADMM step / graph run / line limits.  Host buffers only (no torch import)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_14995_b200 import KernelForm, LaunchOrder, Solver, synth  # noqa: E402
from paper_2106_14995_b200 import admm as A  # noqa: E402

n = int(os.environ.get("SAN_N", 48))
s = Solver((0,))
for fam, d in (("ncvx", 3), ("ncvx", 6), ("ncvx", 8), ("ncvx", 12), ("ncvx", 24), ("branch", 4), ("branch", 6),
               ("hs45", 8), ("boxqp", 5)):
    b = synth.make(fam, n, d)
    s.solve_batch(b)
    s.solve_batch(b, count_flops=True)
s.set_form(KernelForm.THREAD)
s.solve_batch(synth.ncvx(n, 4))
s.solve_batch(synth.branch(n, 4))
s.set_form(KernelForm.AUTO)
for d in (40, 100):
    b = synth.ncvx(max(8, n // 4), d)
    s.solve_batch(b)
    s.solve_batch(b, count_flops=True)
# ranked launches (tron_order.cu): warp, thread and block forms, host and pageable paths
s.set_order(LaunchOrder.START_PG)
for fam, d in (("branch", 6), ("ncvx", 8), ("ncvx", 24)):
    s.solve_batch(synth.make(fam, n, d))
s.set_form(KernelForm.THREAD)
s.solve_batch(synth.branch(n, 4))
s.set_form(KernelForm.AUTO)
s.set_order(LaunchOrder.CALLER)
s.solve_batch(synth.branch(n, 6))
s.close()
g = synth.grid(40, 60, 12, seed=3)
a = A.AdmmSolver(g)
for _ in range(2):
    a.step()
a.run(3)
a.close()
ll = A.AdmmSolver(g, A.AdmmOptions(line_limits=True))
ll.step()
ll.close()
w = A.AdmmSolver(g, A.AdmmOptions(branch_form="warp"))
w.step()
w.close()
print("sanitize driver done")
