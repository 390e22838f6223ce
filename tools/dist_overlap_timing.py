"""Slab solve time on ONE GPU with 1/2/4 emulated ranks (all ranks in one
process, stream-ordered): the cost of splitting each rank's SpMV into the
interior launch (overlapped with the halo copies on the side stream) and the
boundary launch. One JSON line per rank count."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1511_03703_b200 as ep  # noqa: E402


def main(n=128, s=32):
    ctx = ep.Context(0)
    kl = ep.KlField(3, 1.0, 0.1, 1.0)
    y = ep.pack_sample_group(ep.draw_samples(0, s, 3), s, 0).cuda()
    cfg = ep.SolverConfig(tol=1e-6, max_iterations=20000, flavour=ep.CG_UNCOUPLED, dot_mode=ep.DOT_CANONICAL)
    x0 = None
    for nranks in (1, 2, 4):
        d = ep.Dist(ctx, n, s, nranks, kl=kl)
        d.assemble(y)
        d.solve(cfg)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it, _ = d.solve(cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        x = d.solution().cpu()
        same = True if x0 is None else bool(torch.equal(x.view(torch.int64), x0.view(torch.int64)))
        x0 = x if x0 is None else x0
        print(json.dumps({"overlap": os.environ.get("ENPROP_DIST_OVERLAP", "1"), "n": n, "s": s, "nranks": nranks, "iters_max": max(it), "solve_s": round(dt, 4),
                          "ms_per_iter": round(dt * 1e3 / max(it), 4), "stages": d.stages(),
                          "bitwise_vs_1": same}), flush=True)
        d.close()
    ctx.close()


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
