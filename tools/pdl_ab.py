"""Same-process A/B of programmatic dependent launch (ENPROP_OPT_PDL) on whole
canonical uncoupled solves at 64^3 (no per-kernel events in the timed region).
    python tools/pdl_ab.py [--n 64] [--s 32] [--rounds 4]"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1511_03703_b200 as ep  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--s", type=int, default=32)
    ap.add_argument("--rounds", type=int, default=4)
    args = ap.parse_args()
    ctx = ep.Context(0)
    y = ep.pack_sample_group(ep.draw_samples(0, args.s, 3), args.s, 0).cuda()
    p = ep.Problem(ctx, args.n, args.s, ep.KlField(3, 1.0, 0.1, 1.0))
    p.assemble(y)
    cfg = ep.SolverConfig(tol=1e-6, max_iterations=10000, flavour=ep.CG_UNCOUPLED, dot_mode=ep.DOT_CANONICAL)
    st = torch.cuda.current_stream()
    res = {0: [], 1: []}
    for pdl in (0, 1):
        ctx.set_option(ep.OPT_PDL, pdl)
        p.solve(cfg)
    for _ in range(args.rounds):
        for pdl in (0, 1):
            ctx.set_option(ep.OPT_PDL, pdl)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record(st)
            it, _, _ = p.solve(cfg)
            b.record(st)
            torch.cuda.synchronize()
            res[pdl].append(a.elapsed_time(b) / max(it))
    ctx.set_option(ep.OPT_PDL, 1)
    print({k: round(statistics.median(v), 4) for k, v in res.items()}, "ms per iteration (solve / max iterations)")


if __name__ == "__main__":
    main()
