"""Aggregate samples/s with G sample groups solved concurrently (one context /
stream / problem per group, one host thread each) at 64^3, s=32.

    python tools/concurrency_bench.py [--dot canonical|serial] [--groups 1,2,3,4]
"""
import argparse
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1511_03703_b200 as ep  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dot", default="canonical")
    ap.add_argument("--groups", default="1,2,3,4")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--torch-streams", action="store_true", help="bench.py's setup: torch streams, 3 shared y")
    ap.add_argument("--pdl", type=int, default=0)
    args = ap.parse_args()
    n, s = args.n, 32
    Gmax = max(int(g) for g in args.groups.split(","))
    pool = ep.draw_samples(0, s * Gmax * (args.rounds + 1), 3)
    workers = []
    shared = [ep.pack_sample_group(pool, s, s * g).cuda() for g in range(3)]
    for g in range(Gmax):
        ctx = ep.Context(0, use_torch_stream=False)
        if args.torch_streams:
            stream = torch.cuda.Stream()
            ctx.set_stream(stream.cuda_stream)
            ctx._keep = stream
        ctx.set_option(ep.OPT_PDL, args.pdl)
        p = ep.Problem(ctx, n, s, ep.KlField(3, 1.0, 0.1, 1.0))
        if args.torch_streams:
            ys = [shared[g % 3] for r in range(args.rounds + 1)]
        else:
            ys = [ep.pack_sample_group(pool, s, s * (r * Gmax + g)).cuda() for r in range(args.rounds + 1)]
        workers.append((ctx, p, ys))
    torch.cuda.synchronize()
    mode = ep.DOT_CANONICAL if args.dot == "canonical" else ep.DOT_SERIAL
    cfg = ep.SolverConfig(tol=1e-6, max_iterations=10000, flavour=ep.CG_UNCOUPLED, dot_mode=mode)

    def run(w, rounds, out, idx):
        ctx, p, ys = w
        its = []
        for r in range(rounds):
            p.assemble(ys[r])
            it, _, _ = p.solve(cfg)
            its.append(max(it))
        ctx.synchronize()
        out[idx] = its

    for G in [int(g) for g in args.groups.split(",")]:
        out = [None] * G
        # warm-up
        th = [threading.Thread(target=run, args=(workers[g], 1, out, g)) for g in range(G)]
        [t.start() for t in th]
        [t.join() for t in th]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th = [threading.Thread(target=run, args=(workers[g], args.rounds, out, g)) for g in range(G)]
        [t.start() for t in th]
        [t.join() for t in th]
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        samples = G * args.rounds * s
        print(f"dot={args.dot} G={G}: {samples / dt:8.1f} samples/s  ({dt / args.rounds * 1e3:.1f} ms per round of {G} groups) iters={[o[0] for o in out]}", flush=True)


if __name__ == "__main__":
    main()
