"""Full solve() (precondition, factor, Lipschitz estimate, warm start, solver,
verification; solvers.hpp:645-720) on C3, device against the CPU oracle.
python tools/solve_parity_probe.py [kind] [precondition 0/1] [warm_start 0/1]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_01745_b200 as so
from oracle import oracle as orc
kind = sys.argv[1] if len(sys.argv) > 1 else "nama"
pre = len(sys.argv) > 2 and sys.argv[2] == "1"
ws = len(sys.argv) > 3 and sys.argv[3] == "1"
prob = so.gen_random_instance(1, 50, 20, 20, [8, 8, 8, 2])
po = orc.Problem.from_flat(prob.flat())
cfg = dict(precondition=pre, warm_start=ws, nama_parallel_linesearch=kind == "nama")
t = time.time()
rep = so.solve(prob, so.SolverConfig(**cfg), kind)
tg = time.time() - t
t = time.time()
orep = orc.solve(po, orc.SolverConfig(**cfg), so.api.KINDS[kind])
tc = time.time() - t
print(f"{kind} precondition={pre} warm_start={ws}: GPU {rep.iterations} it {rep.status} wall_ms {rep.wall_ms:.2f} "
      f"(call {tg:.2f} s) verified {rep.verified} | CPU {orep['iterations']} it status {orep['status']} "
      f"wall_ms {orep['wall_ms']:.0f} (call {tc:.1f} s) verified {orep['verified']}")
yo = orep["y"]
print("  y gap", np.abs(rep.y - yo).max(), "bound", 10 * 5e-4 * (1 + np.abs(yo).max()),
      "| L", rep.lipschitz_estimate, orep["lipschitz_estimate"],
      "| dual_grad", rep.stats.dual_grad_calls, orep["dual_grad_calls"])
