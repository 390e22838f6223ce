"""The CUDA-IPC slab transport at full cfg-4 size on one GPU: a 256^3, s = 32
ensemble solved (canonical order, uncoupled, tol 1e-6) by 1 rank, then by 2
and 4 real processes exchanging halos and per-plane sums through exported
buffers and interprocess events. Per-slab SHA-256 of the solution and the
iteration counts must equal the 1-rank run (the canonical order is defined per
mesh plane). One JSON line per rank count; wall times include process start,
assembly and the solve (ranks share one GPU here, so they show function at
scale, not NVLink speed)."""
import hashlib
import json
import multiprocessing as mp
import sys
import time
import uuid

N, S, M = 256, 32, 3


def planes(nranks):
    Np = N + 1
    base, extra = Np // nranks, Np % nranks
    out, k0 = [], 0
    for r in range(nranks):
        k1 = k0 + base + (1 if r < extra else 0)
        out.append((k0, k1))
        k0 = k1
    return out


def run_rank(job, nranks, rank, q, split):
    import torch

    sys.path.insert(0, ".")
    import paper_1511_03703_b200 as ep
    try:
        t0 = time.perf_counter()
        ctx = ep.Context(0)
        kl = ep.KlField(M, 1.0, 0.1, 1.0)
        d = ep.Dist(ctx, N, S, nranks, rank, kl=kl, ipc_job=job)
        y = ep.pack_sample_group(ep.draw_samples(0, S, M), S, 0).cuda()
        d.assemble(y)
        cfg = ep.SolverConfig(tol=1e-6, max_iterations=20000, flavour=ep.CG_UNCOUPLED, dot_mode=ep.DOT_CANONICAL)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        it, st = d.solve(cfg)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        (rk, rb, rows, x), = d.local()
        plane = (N + 1) ** 2
        hashes = []  # per slab of `split` (the rank count being checked), in row order
        for k0, k1 in split:
            lo, hi = max(k0 * plane, rb), min(k1 * plane, rb + rows)
            if lo < hi:
                hashes.append((k0, hashlib.sha256(x[lo - rb:hi - rb].cpu().numpy().tobytes()).hexdigest()))
        q.put({"rank": rank, "iters_max": max(it), "iters": it, "status_ok": all(v == 0 for v in st),
               "stages": d.stages(), "hashes": hashes, "solve_s": round(t2 - t1, 3), "total_s": round(t2 - t0, 3)})
        d.close()
        ctx.close()
    except Exception as e:
        q.put({"rank": rank, "error": repr(e)})


def run(nranks, split):
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    job = uuid.uuid4().hex[:16]
    procs = [mpc.Process(target=run_rank, args=(job, nranks, r, q, split)) for r in range(nranks)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=1800) for _ in range(nranks)], key=lambda r: r["rank"])
    for p in procs:
        p.join(timeout=120)
    return res


def main():
    out = {}
    for nranks in (2, 4):
        split = planes(nranks)
        one = run(1, split)[0]
        many = run(nranks, split)
        errs = [r.get("error") for r in [one] + many if r.get("error")]
        if errs:
            print(json.dumps({"nranks": nranks, "errors": errs}), flush=True)
            continue
        h1 = dict(one["hashes"])
        hn = dict(kv for r in many for kv in r["hashes"])
        line = {"mesh": N, "s": S, "nranks": nranks, "transport": "CUDA IPC, ranks sharing one B200",
                "iterations_equal": all(r["iters"] == one["iters"] for r in many),
                "solution_bitwise_per_slab": h1 == hn, "iters_max": one["iters_max"],
                "one_rank_solve_s": one["solve_s"], "ranks_solve_s": [r["solve_s"] for r in many],
                "interior_stages": [r["stages"] for r in many]}
        out[nranks] = line
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
