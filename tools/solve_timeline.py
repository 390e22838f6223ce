"""Where does a solve's time go?  Times Problem.solve at 64^3/s=32 (canonical,
uncoupled) with GPU events and host wall clock for several check_every values,
and with/without history collection.

    python tools/solve_timeline.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1511_03703_b200 as ep  # noqa: E402

n, s = 64, 32
ctx = ep.Context(0)
y = ep.pack_sample_group(ep.draw_samples(0, s, 3), s, 0).cuda()
p = ep.Problem(ctx, n, s, ep.KlField(3, 1.0, 0.1, 1.0))
p.assemble(y)
st = torch.cuda.current_stream()
for ce in (4, 16, 64):
    for maxit in (10000, 400):
        cfg = ep.SolverConfig(tol=1e-6, max_iterations=maxit, flavour=ep.CG_UNCOUPLED,
                              dot_mode=ep.DOT_CANONICAL, check_every=ce)
        p.solve(cfg)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        t0 = time.perf_counter()
        a.record(st)
        it, _, _ = p.solve(cfg)
        b.record(st)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(f"check_every={ce:3d} maxit={maxit:5d}: gpu {a.elapsed_time(b):8.2f} ms  host {1e3*(t1-t0):8.2f} ms  "
              f"iters {max(it)}  gpu/iter {a.elapsed_time(b)/max(it):.4f}", flush=True)
launches0 = ctx.launches
cfg = ep.SolverConfig(tol=1e-6, max_iterations=400, flavour=ep.CG_UNCOUPLED, dot_mode=ep.DOT_CANONICAL)
p.solve(cfg)
print("launches per solve:", ctx.launches - launches0)
