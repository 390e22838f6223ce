"""Staged vs warp-per-tile CG SpMV on one configuration: iteration counts and
solution bits must agree (ep_staged.cu is bitwise interchangeable).
    python tools/staged_check.py [--n 32] [--s 16] [--m 3] [--sigma 0.1]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1511_03703_b200 as ep  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--s", type=int, default=16)
    ap.add_argument("--m", type=int, default=3)
    ap.add_argument("--sigma", type=float, default=0.1)
    args = ap.parse_args()
    ctx = ep.Context(0)
    y = ep.pack_sample_group(ep.draw_samples(0, args.s, args.m), args.s, 0).cuda()
    p = ep.Problem(ctx, args.n, args.s, ep.KlField(args.m, 1.0, args.sigma, 1.0))
    p.assemble(y)
    for flavour in (ep.CG_COUPLED, ep.CG_UNCOUPLED):
        cfg = ep.SolverConfig(tol=1e-6, max_iterations=20000, flavour=flavour, dot_mode=ep.DOT_CANONICAL)
        out = {}
        for var in (-1, 2):
            ctx.set_option(ep.OPT_SPMV_VARIANT, var)
            it, hist, _ = p.solve(cfg)
            out[var] = (it, p.solution.clone())
        ctx.set_option(ep.OPT_SPMV_VARIANT, -1)
        same = torch.equal(out[-1][1].view(torch.int64), out[2][1].view(torch.int64))
        print({"flavour": "coupled" if flavour == ep.CG_COUPLED else "uncoupled",
               "staged_iters": out[-1][0], "warp_iters": out[2][0], "bitwise_equal": same})


if __name__ == "__main__":
    main()
