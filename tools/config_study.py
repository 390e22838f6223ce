"""BASELINE.json configs beyond the bench headline, measured on one B200:

  cfg1  32^3, m=3, sigma=0.1, s=16, tol 1e-6 (the reference's CPU case)
  cfg2  64^3, m=3, sigma=0.1, tol 1e-6, s in {1,4,8,16,32}: samples/s, coupled and uncoupled
  cfg5  128^3, m=10, sigma=0.25, s=32, tol 1e-6: coupled vs uncoupled iterations and samples/s
  cfg4  256^3, m=3, sigma=0.1, s=32, tol 1e-6 on ONE GPU through the device-resident
        problem (symmetric storage, staged SpMV); the slab path is bench.py --workload dd

Each line: one sample group (seed 0, group 0) assembled + solved on the device,
timed with CUDA events (one stream; no inter-group concurrency), canonical dot
order unless --dot serial.  Prints JSON lines.

    python tools/config_study.py [--which 1,2,5] [--dot canonical|serial]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1511_03703_b200 as ep  # noqa: E402


def solve_line(ctx, O, n, s, m, sigma, flavour, dot, reps=2, tag=""):
    y = ep.pack_sample_group(ep.draw_samples(0, s, m), s, 0).cuda()
    p = ep.Problem(ctx, n, s, ep.KlField(m, 1.0, sigma, 1.0))
    cfg = ep.SolverConfig(tol=1e-6, max_iterations=20000, flavour=flavour,
                          dot_mode=ep.DOT_CANONICAL if dot == "canonical" else ep.DOT_SERIAL)
    p.assemble(y)
    p.solve(cfg)  # warm-up
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    a.record(st)
    for _ in range(reps):
        p.assemble(y)
        it, _, status = p.solve(cfg)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    its = it if isinstance(it, list) else [it]
    out = {"config": tag, "mesh": n, "s": s, "m": m, "sigma": sigma,
           "cg": "coupled" if flavour == ep.CG_COUPLED else "uncoupled", "dot_order": dot,
           "iterations_max": max(its), "iterations_min": min(its), "ms_per_group": round(ms, 2),
           "samples_per_s": round(s / (ms / 1e3), 2), "status": sorted(set(status))}
    p.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="1,2,5")
    ap.add_argument("--dot", default="canonical")
    args = ap.parse_args()
    which = set(args.which.split(","))
    ctx = ep.Context(0)
    if "1" in which:
        for fl in (ep.CG_COUPLED, ep.CG_UNCOUPLED):
            print(json.dumps(solve_line(ctx, O, 32, 16, 3, 0.1, fl, args.dot, tag="cfg1")), flush=True)
    if "2" in which:
        for s in (1, 4, 8, 16, 32):
            for fl in (ep.CG_COUPLED, ep.CG_UNCOUPLED):
                print(json.dumps(solve_line(ctx, O, 64, s, 3, 0.1, fl, args.dot, tag="cfg2")), flush=True)
    if "4" in which:
        print(json.dumps(solve_line(ctx, O, 256, 32, 3, 0.1, ep.CG_UNCOUPLED, args.dot, reps=1, tag="cfg4-1gpu")),
              flush=True)
    if "5" in which:
        for fl in (ep.CG_COUPLED, ep.CG_UNCOUPLED):
            print(json.dumps(solve_line(ctx, O, 128, 32, 10, 0.25, fl, args.dot, reps=1, tag="cfg5")), flush=True)


if __name__ == "__main__":
    main()
