"""Small emulated multi-rank solve for debugging (used under compute-sanitizer)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import paper_1511_03703_b200 as ep  # noqa: E402

n, s, nranks = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ctx = ep.Context(0)
kl = ep.KlField(3, 1.0, 0.1, 1.0)
y = torch.full((3, s), 0.25, dtype=torch.float64, device="cuda")
d = ep.Dist(ctx, n, s, nranks, kl=kl)
d.assemble(y)
torch.cuda.synchronize()
print("assembled", flush=True)
it, st = d.solve(ep.SolverConfig(tol=1e-7, max_iterations=50, flavour=ep.CG_COUPLED, dot_mode=ep.DOT_CANONICAL,
                                 check_every=2))
print("solved", it, st, flush=True)
