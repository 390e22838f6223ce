"""Kernel-level timing of the CG step pieces at a given mesh / ensemble width
(CUDA events on the library's stream).  Used to choose kernel variants; the
official numbers come from bench.py.

    python tools/kernel_bench.py [--n 64] [--s 32] [--steps 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1511_03703_b200 as ep  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--s", type=int, default=32)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--spmv-only", action="store_true")
    ap.add_argument("--sym", type=int, default=1, help="symmetric storage for the CG problems")
    ap.add_argument("--modes", default="canonical,serial")
    ap.add_argument("--variant", type=int, default=-1, help="CG SpMV variant (-1 auto)")
    ap.add_argument("--ab", default="", help="comma list of SpMV variants timed alternately (CG SpMV kernel only)")
    ap.add_argument("--ab-rounds", type=int, default=5)
    ap.add_argument("--fused", default="1,0", help="fused-direction settings to time")
    ap.add_argument("--pdl", type=int, default=0, help="programmatic dependent launch (ENPROP_OPT_PDL)")
    args = ap.parse_args()
    n, s = args.n, args.s
    ctx = ep.Context(0)
    ctx.set_option(ep.OPT_SPMV_VARIANT, args.variant)
    ctx.set_option(ep.OPT_PDL, args.pdl)
    y = ep.pack_sample_group(ep.draw_samples(0, s, 3), s, 0).cuda()
    ctx.set_option(ep.OPT_SYMMETRIC_STORAGE, 0)
    pfull = ep.Problem(ctx, n, s, ep.KlField(3, 1.0, 0.1, 1.0))
    ctx.set_option(ep.OPT_SYMMETRIC_STORAGE, args.sym)
    p = ep.Problem(ctx, n, s, ep.KlField(3, 1.0, 0.1, 1.0)) if args.sym else pfull
    st = torch.cuda.current_stream()
    out = {"n": n, "s": s, "sym": args.sym}
    # assembly
    p.assemble(y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record(st)
    for _ in range(3):
        p.assemble(y)
    b.record(st)
    torch.cuda.synchronize()
    out["assemble_ms"] = a.elapsed_time(b) / 3
    # plain spmv on the assembled matrix
    pfull.assemble(y)
    vals_full = pfull.values
    x = torch.rand((p.rows, s), dtype=torch.float64, device="cuda")
    z = torch.empty_like(x)
    nnz, rows = p.nnz, p.rows
    for pipe in (1, 0):
        ctx.set_option(ep.OPT_SPMV_PIPELINE, pipe)
        for _ in range(3):
            ep.spmv(ctx, s, p.row_map, p.col_entry, vals_full, x, z)
        torch.cuda.synchronize()
        a.record(st)
        for _ in range(10):
            ep.spmv(ctx, s, p.row_map, p.col_entry, vals_full, x, z)
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        out[f"spmv_pipe{pipe}_ms"] = round(ms, 4)
        out[f"spmv_pipe{pipe}_gbs"] = round((nnz * (8 * s + 4) + 4 * (rows + 1) + 16 * s * rows) / (ms / 1e3) / 1e9, 1)
    ctx.set_option(ep.OPT_SPMV_PIPELINE, 0)
    if args.spmv_only:
        print(json.dumps(out, indent=1))
        return
    if args.ab:
        # same process, same box: alternate the variants, median SpMV kernel time
        import statistics
        cfg = ep.SolverConfig(tol=1e-6, max_iterations=10000, flavour=ep.CG_UNCOUPLED,
                              dot_mode=ep.DOT_CANONICAL)
        vs = [int(v) for v in args.ab.split(",")]
        res = {v: [] for v in vs}
        for v in vs:
            ctx.set_option(ep.OPT_SPMV_VARIANT, v)
            p.solve(cfg)
        for _ in range(args.ab_rounds):
            for v in vs:
                ctx.set_option(ep.OPT_SPMV_VARIANT, v)
                ctx.profile(1)
                p.solve(cfg)
                sp_ms, sp_n = ctx.profile(0)
                res[v].append(sp_ms / max(sp_n, 1))
        out["ab_spmv_kernel_ms"] = {v: round(statistics.median(r), 4) for v, r in res.items()}
        out["ab_all"] = {v: [round(t, 4) for t in r] for v, r in res.items()}
        print(json.dumps(out, indent=1))
        return
    modes = {"canonical": ep.DOT_CANONICAL, "serial": ep.DOT_SERIAL}
    for mode_name in args.modes.split(","):
        mode = modes[mode_name]
        for fused in (int(v) for v in args.fused.split(",")):
            ctx.set_option(ep.OPT_FUSED_DIRECTION, fused)
            cfg = ep.SolverConfig(tol=1e-6, max_iterations=10000, flavour=ep.CG_UNCOUPLED, dot_mode=mode)
            p.solve(cfg)
            torch.cuda.synchronize()
            ctx.profile(1)
            a.record(st)
            its = []
            for _ in range(args.steps):
                it, _, _ = p.solve(cfg)
                its.append(max(it))
            b.record(st)
            torch.cuda.synchronize()
            det = ctx.profile_detail()
            sp_ms, sp_n = ctx.profile(0)
            ms = a.elapsed_time(b) / args.steps
            key = f"{mode_name}_fused{fused}"
            out[key] = {"solve_ms": round(ms, 3), "iters": its, "ms_per_iter": round(ms / its[-1], 4),
                        "spmv_kernel_ms": round(sp_ms / max(sp_n, 1), 4),
                        "per_iter_ms": {k: round(v / max(det["iterations"], 1), 4)
                                        for k, v in det.items()
                                        if k not in ("iterations", "solve", "init", "loop", "early_exit")},
                        "counted_iterations": det["iterations"],
                        "per_solve_ms": {k: round(det[k] / args.steps, 3)
                                         for k in ("solve", "init", "loop", "early_exit")}}
            if mode_name == "serial" and args.steps > 1:
                pass
    ctx.set_option(ep.OPT_FUSED_DIRECTION, 0)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
