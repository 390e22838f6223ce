"""Serial-order dot and CG at growing sizes vs the C oracle (debug aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1511_03703_b200 as ep  # noqa: E402
from oracles import DOT_SERIAL, Oracle, pack_group  # noqa: E402

O = Oracle()
ctx = ep.Context(0)
rng = np.random.default_rng(0)
for rows in (70001, 274625):
    u, v = rng.uniform(-1, 1, (rows, 32)), rng.uniform(-1, 1, (rows, 32))
    lanes, _ = ep.dot_lanes(ctx, 32, torch.as_tensor(u).cuda(), torch.as_tensor(v).cuda(), ep.DOT_SERIAL)
    ref = O.dot_lanes(32, u, v, DOT_SERIAL)
    print("dot rows", rows, "equal:", lanes == list(ref), flush=True)
    uu = torch.as_tensor(u).cuda()
    lanes, _ = ep.dot_lanes(ctx, 32, uu, uu, ep.DOT_SERIAL)
    print("dot u.u rows", rows, "equal:", lanes == list(O.dot_lanes(32, u, u, DOT_SERIAL)), flush=True)
for n in (8, 16, 32, 64):
    for fused in (0, 1):
        ctx.set_option(ep.OPT_FUSED_DIRECTION, fused)
        s = 32
        y = torch.as_tensor(pack_group(O.draw_samples(0, s, 3), s)).cuda()
        p = ep.Problem(ctx, n, s, ep.KlField(3, 1.0, 0.1, 1.0))
        p.assemble(y)
        it, _, st = p.solve(ep.SolverConfig(tol=1e-6, max_iterations=3000, flavour=ep.CG_UNCOUPLED,
                                            dot_mode=ep.DOT_SERIAL), raise_on_failure=False)
        print("n", n, "fused", fused, "iters", max(it), "status", sorted(set(st)), flush=True)
        p.close()
