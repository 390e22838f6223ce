"""Serial (reference-order) dot and CG timing: the chain kernel (ep_chain.cu)
per call at 64^3 rows for each width, and serial-order solve throughput at
several concurrency levels (bench.py --dot serial).

    python tools/serial_ab.py [--groups 8,12,16] [--steps 1]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def chain_times(rows=274625, reps=5):
    import torch
    import paper_1511_03703_b200 as ep
    ctx = ep.Context(0)
    out = {}
    for s in (1, 4, 8, 16, 32):
        u = torch.rand((rows, s), dtype=torch.float64, device="cuda")
        v = torch.rand((rows, s), dtype=torch.float64, device="cuda")
        res = {}
        for name, a, b in (("square", u, u), ("product", u, v)):
            ep.dot_lanes(ctx, s, a, b, ep.DOT_SERIAL)
            ts = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                ep.dot_lanes(ctx, s, a, b, ep.DOT_SERIAL)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[name] = round(min(ts), 4)
        out[str(s)] = res
    return out


def phase_times(s=32, n=64, dot="serial"):
    """Per-iteration phase times (CUDA events) of one single-stream solve."""
    import torch
    import paper_1511_03703_b200 as ep
    ctx = ep.Context(0)
    p = ep.Problem(ctx, n, s, ep.KlField(3, 1.0, 0.1, 1.0))
    y = ep.pack_sample_group(ep.draw_samples(0, s, 3), s, 0).cuda()
    cfg = ep.SolverConfig(tol=1e-6, max_iterations=10000, flavour=ep.CG_UNCOUPLED,
                          dot_mode=ep.DOT_SERIAL if dot == "serial" else ep.DOT_CANONICAL)
    p.assemble(y)
    p.solve(cfg)
    ctx.profile(1)
    p.assemble(y)
    it, _, _ = p.solve(cfg)
    det = ctx.profile_detail()
    ctx.profile(0)
    nit = max(det["iterations"], 1)
    p.close()
    return {"s": s, "dot": dot, "iters": max(it), "solve_ms": round(det["solve"], 3),
            **{k: round(det[k] / nit, 4) for k in ("direction", "spmv_kernel", "fin_pq", "update", "fin_rr", "iteration")}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", default="8,12,16")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--skip-chain", action="store_true")
    ap.add_argument("--staged", default="0,1", help="ENPROP_STAGED_SERIAL values to compare")
    a = ap.parse_args()
    if not a.skip_chain:
        print(json.dumps({"chain_ms_incl_host_alloc": chain_times()}), flush=True)
        for s in (1, 32):
            print(json.dumps(phase_times(s)), flush=True)
        print(json.dumps(phase_times(32, dot="canonical")), flush=True)
    for g, st in [(g, st) for st in a.staged.split(",") for g in a.groups.split(",")]:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--dot", "serial", "--groups", g,
               "--steps", str(a.steps), "--warmup", "1", "--skip-spmv", "--skip-cpu", "--profile-only"]
        r = subprocess.run(cmd, capture_output=True, text=True, env=dict(os.environ, ENPROP_STAGED_SERIAL=st))
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-2000:]
        try:
            d = json.loads(line)
            d["samples_per_s"] = round(int(g) * 32 * a.steps / (d["ms"] / 1e3), 2)
            d["groups"] = int(g)
            d["staged_serial"] = st
            d.pop("iters", None)
            print(json.dumps(d), flush=True)
        except ValueError:
            print(line, flush=True)


if __name__ == "__main__":
    main()
