"""Benchmark: sample solves/s (assembly + Dirichlet + CG) at ensemble s=32 on the
64^3 hex mesh (BASELINE.json configs[1], "cfg 2"), plus the ensemble SpMV HBM
GB/s on the 128^3 matrix (configs[2], "cfg 3") in the same run.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one sample group of s=32 samples: assemble the ensemble matrix with
the fused Dirichlet elimination, then solve A x = -residual with uncoupled
(per-sample) identity-preconditioned CG to tol 1e-6, all on the device.  With
N>1 (torchrun, one process per GPU) every rank solves its own sample groups
(groups are independent units: weak scaling, no data-path collective).

--impl reference times the reference's own CPU path (oracle/_ref: the unmodified
proj/ sources) on the host cores for the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

N_MESH, S, M_TERMS, SIGMA, TOL = 64, 32, 3, 0.1, 1e-6
SPMV_MESH = 128
# Coupled CG iteration count of sample group 0 at 64^3, s=32 (seed 0): measured
# by the reference itself and reproduced bitwise by the GPU's
# serial-order coupled solve (tests/test_gpu_parity.py).
REF_COUPLED_ITERS_64 = 168


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def spmv_bytes(nnz, rows, s):
    """Algorithmic bytes of one ensemble SpMV: values + cols +
    row_map + x once + z once."""
    return nnz * (8 * s + 4) + 4 * (rows + 1) + 16 * s * rows


def cg_spmv_bytes(nnz, nnz_stored, rows, s):
    """Algorithmic bytes of one CG SpMV launch (k_cg_spmv_staged / k_cg_spmv_warp):
    the stored value slots once (symmetric storage: diagonal + upper), column
    indices, the slot map (symmetric storage only), row_map, the direction
    vector gathered once and q written once. The transposed re-reads of the
    upper slots are not algorithmic bytes."""
    sym = nnz_stored < nnz
    return nnz_stored * 8 * s + nnz * (8 if sym else 4) + 4 * (rows + 1) + 16 * s * rows


def direction_bytes(rows, s):
    """k_cg_direction: read r, p_old, x; write p_new, x."""
    return 5 * 8 * s * rows


def measured_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full capture (profiles/*/traffic.json), else None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "traffic.json")), reverse=True):
        try:
            with open(path) as fh:
                d = json.load(fh)
            if kernel in d:
                return d[kernel]
        except (OSError, ValueError):
            pass
    return None


# --------------------------------------------------------------------------- ours
class GroupWorker:
    """One sample-group lane of the step: its own context, torch stream and
    device-resident problem (graph, KL tables, matrix, CG workspace)."""

    def __init__(self, ep, torch, device, kl):
        self.stream = torch.cuda.Stream(device=device)
        self.ctx = ep.Context(device, use_torch_stream=False)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.prob = ep.Problem(self.ctx, N_MESH, S, kl)


def run_groups(torch, workers, jobs, cfg, host=False):
    """Solve jobs[i] (lists of device or host sample tensors) on workers[i]
    concurrently (one host thread each; ctypes releases the GIL).  Returns the
    per-worker max iteration counts and lane statuses."""
    import threading
    out = [None] * len(workers)

    def run(i):
        w = workers[i]
        its, sts = [], []
        for item in jobs[i]:
            if host:
                y_host, x_host = item
                it, st, rc = w.prob.solve_host(y_host, x_host, cfg)
            else:
                w.prob.assemble(item)
                it, _, st = w.prob.solve(cfg)
            its.append(max(it))
            sts.extend(st)
        out[i] = (its, sts)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(workers))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return out


def timed_round(torch, workers, jobs, cfg):
    """Device time of one concurrent round: a start event on the main stream,
    every worker stream waits on it, and the end event waits on every worker."""
    main = torch.cuda.current_stream()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(main)
    for w in workers:
        w.stream.wait_event(start)
    res = run_groups(torch, workers, jobs, cfg)
    for w in workers:
        ev = torch.cuda.Event()
        ev.record(w.stream)
        main.wait_event(ev)
    end.record(main)
    torch.cuda.synchronize()
    return start.elapsed_time(end), res


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1511_03703_b200 as ep
    from oracles import Oracle, pack_group

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    G = args.groups
    O = Oracle()  # only to draw the reference's samples (samples.cpp:7-18)
    rounds = args.warmup + args.steps
    # rank r, round k, worker i solves sample group ((r * rounds + k) * G + i)
    pool = O.draw_samples(0, S * G * rounds * world, M_TERMS)
    group_of = lambda k, i: (rank * rounds + k) * G + i  # noqa: E731
    kl = ep.KlField(M_TERMS, 1.0, SIGMA, 1.0)
    workers = [GroupWorker(ep, torch, local, kl) for _ in range(G)]
    ys = {(k, i): torch.as_tensor(pack_group(pool, S, group_of(k, i))).cuda()
          for k in range(rounds) for i in range(G)}
    cfg = ep.SolverConfig(tol=TOL, max_iterations=10000, flavour=ep.CG_UNCOUPLED,
                          dot_mode=ep.DOT_CANONICAL if args.dot == "canonical" else ep.DOT_SERIAL)

    for k in range(args.warmup):
        timed_round(torch, workers, [[ys[(k, i)]] for i in range(G)], cfg)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = sum(w.ctx.launches for w in workers)
    jobs = [[ys[(args.warmup + k, i)] for k in range(args.steps)] for i in range(G)]
    ms, res = timed_round(torch, workers, jobs, cfg)
    launches = sum(w.ctx.launches for w in workers) - launches0
    clk = clocks.stop()
    iters = [r[0] for r in res]
    assert all(v == 0 for r in res for v in r[1]), "a lane did not converge"
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    samples = args.steps * G * S * world
    value = samples / (ms / 1e3)
    if args.profile_only:
        print(json.dumps({"profile_only": True, "ms": ms, "iters": iters}), flush=True)
        return

    # ---- e2e: the reference-facing C-ABI call with HOST buffers (pinned); the
    # H2D of y and the D2H of the solution are inside the timed region
    x_host = [torch.empty((workers[0].prob.rows, S), dtype=torch.float64).pin_memory() for _ in range(G)]
    hjobs = [[(torch.as_tensor(pack_group(pool, S, group_of(args.warmup + k, i))).contiguous().pin_memory(),
               x_host[i]) for k in range(args.steps)] for i in range(G)]
    run_groups(torch, workers, [[j[0]] for j in hjobs], cfg, host=True)  # warm
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run_groups(torch, workers, hjobs, cfg, host=True)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": round(samples / e2e_s, 3), "unit": "samples/s",
           "h2d_bytes_per_step": G * M_TERMS * S * 8, "d2h_bytes_per_step": G * workers[0].prob.rows * S * 8,
           "api": "enprop_problem_solve_host (C ABI; pinned host y in, x out; G groups concurrently)"}

    # ---- roofline of the dominant kernel, from a single-stream solve of the same
    # workload (kernels of concurrent streams overlap, so they are timed alone)
    hbm, peak_kind = peaks()
    w0 = workers[0]
    w0.ctx.profile(1)
    w0.prob.assemble(ys[(args.warmup, 0)])
    w0.prob.solve(cfg)
    det = w0.ctx.profile_detail()
    spmv_ms, spmv_n = w0.ctx.profile(0)
    nnz, nnz_st, rows = w0.prob.nnz, w0.prob.nnz_stored, w0.prob.rows
    avg_spmv_ms = spmv_ms / max(spmv_n, 1)
    nit = max(det["iterations"], 1)
    byt = cg_spmv_bytes(nnz, nnz_st, rows, S)
    achieved = byt / (avg_spmv_ms / 1e3) / 1e9
    it_ms = det["iteration"] / nit
    # the library's auto choice (ep_capi.cu enprop_problem_solve): the staged
    # kernel for symmetric storage + canonical dots at s in {4, 16, 32}
    if nnz_st < nnz and args.dot == "canonical" and S in (4, 16, 32):
        kname = f"k_cg_spmv_staged<{S},true>"
    else:
        kname = "k_cg_spmv_warp<32,true,true,2>" if nnz_st < nnz else "k_cg_spmv_warp<32,true,false,0>"
    dir_ms = det["direction"] / nit
    it_bytes = byt + direction_bytes(rows, S) + 3 * 8 * S * rows  # + update (r, q -> r)
    roofline = {"bound": "hbm", "kernel": kname,
                "achieved": round(achieved, 1), "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": measured_traffic(kname),
                "bytes_per_launch": byt, "avg_launch_ms": round(avg_spmv_ms, 4),
                "launches_timed": spmv_n,
                "share_of_iteration": round(avg_spmv_ms / it_ms, 3) if it_ms else None,
                "per_iteration_ms": {k: round(det[k] / nit, 4) for k in
                                     ("direction", "spmv_kernel", "fin_pq", "update", "fin_rr", "iteration")},
                "direction": {"kernel": "k_cg_direction<32>", "bytes": direction_bytes(rows, S),
                              "achieved": round(direction_bytes(rows, S) / (dir_ms / 1e3) / 1e9, 1) if dir_ms else None},
                "iteration_bytes": it_bytes,
                "iteration_gbs": round(it_bytes / (it_ms / 1e3) / 1e9, 1) if it_ms else None,
                "timing": "CUDA events on the solve's stream, single-stream solve"}

    extra = {}
    if rank == 0 and not args.skip_serial and args.dot == "canonical":
        extra["serial_order"] = bench_serial(torch, ep, workers, ys, args, cfg)
    spmv_obj = None
    if rank == 0 and not args.skip_spmv:
        for w in workers:
            w.prob.close()
        spmv_obj = bench_spmv(ep.Context(local), ep, torch, pack_group, O, hbm, peak_kind)
    if rank == 0 and world == 1 and not args.skip_spmv:
        extra["halo_model"] = bench_halo_model(ep, torch)
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        cpu = cpu_baseline_sample()

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    line = {
        "metric": "sample solves/sec (assembly+CG) at ensemble s=32",
        "value": round(value, 3), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2: 64^3 Q1 hex mesh, KL m=3 sigma=0.1 L=1, s=32; per sample group: "
                               "assembly + fused Dirichlet + uncoupled identity-PCG to tol 1e-6 "
                               "(per-sample stopping); samples draw_samples(seed=0)",
                   "step": f"{G} sample groups of s=32 solved concurrently (one stream each)",
                   "mesh": N_MESH, "ensemble_size": S, "groups_per_step": G, "cg": "uncoupled",
                   "dot_order": args.dot, "cg_iterations_max": iters,
                   "l2": "inputs larger than L2 (matrix 1.84 GB per group)",
                   "parallelism": f"sample groups x {world} GPU(s)"},
        "e2e": e2e, "roofline": roofline, "gpu_launches": int(launches), "clocks": clk,
    }
    line.update(extra)
    if spmv_obj:
        line["spmv_cfg3"] = spmv_obj
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def run_dd(args):
    """cfg 4: ONE ensemble (s=32) on an n^3 mesh (default 256^3) domain-decomposed
    into z-slabs over the N ranks (NCCL halo of p + all-gathered per-plane dot
    sums); a step = assemble + Dirichlet + uncoupled CG to 1e-6.
    Strong scaling: the work per step is fixed as N grows."""
    import torch
    import torch.distributed as dist

    import paper_1511_03703_b200 as ep
    from oracles import Oracle, pack_group

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    nccl_id = None
    if world > 1:
        dist.init_process_group("gloo")  # host plumbing only: broadcast the NCCL id, barrier, max
        obj = [ep.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    n = args.dd_mesh
    ctx = ep.Context(local)
    kl = ep.KlField(M_TERMS, 1.0, SIGMA, 1.0)
    d = ep.Dist(ctx, n, S, world, rank, nccl_id, kl=kl)
    O = Oracle()
    pool = O.draw_samples(0, S * (args.warmup + args.steps), M_TERMS)
    ys = [torch.as_tensor(pack_group(pool, S, g)).cuda() for g in range(args.warmup + args.steps)]
    cfg = ep.SolverConfig(tol=TOL, max_iterations=20000, flavour=ep.CG_UNCOUPLED, dot_mode=ep.DOT_CANONICAL)
    for g in range(args.warmup):
        d.assemble(ys[g])
        d.solve(cfg)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    launches0 = ctx.launches
    e0.record(st)
    iters = []
    for k in range(args.steps):
        d.assemble(ys[args.warmup + k])
        it, status = d.solve(cfg)
        iters.append(max(it))
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    launches = ctx.launches - launches0
    if world > 1:
        t = [None] * world
        dist.all_gather_object(t, ms)
        ms = max(t)
        dist.barrier()
    if rank == 0:
        samples = args.steps * S
        print(json.dumps({
            "metric": "sample solves/sec (assembly+CG) at ensemble s=32", "value": round(samples / (ms / 1e3), 3),
            "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg4: {n}^3 mesh domain-decomposed into z-slabs over {world} GPU(s); "
                                   "NCCL halo of p + all-gathered per-plane dot sums; s=32, KL m=3 "
                                   "sigma=0.1, uncoupled CG tol 1e-6, canonical dot order",
                       "mesh": n, "ensemble_size": S, "cg_iterations_max": iters,
                       "parallelism": f"domain decomposition x {world}"},
            "gpu_launches": int(launches), "clocks": clk}), flush=True)
    d.close()
    if world > 1:
        dist.destroy_process_group()


def bench_serial(torch, ep, workers, ys, args, cfg):
    """Throughput in the reference's own (serial) dot order, which reproduces
    pcg_solve bit for bit; its chains are latency-bound, so more sample groups
    run concurrently (workers reused round-robin) to fill the GPU."""
    import dataclasses
    scfg = dataclasses.replace(cfg, dot_mode=ep.DOT_SERIAL)
    G2 = args.serial_groups
    kl = workers[0].prob.kl
    extra = [GroupWorker(ep, torch, torch.cuda.current_device(), kl) for _ in range(max(0, G2 - len(workers)))]
    pool = (workers + extra)[:G2]
    jobs = [[ys[(args.warmup + (i % args.steps), i % len(workers))]] for i in range(G2)]
    ms, res = timed_round(torch, pool, jobs, scfg)
    for w in extra:
        w.prob.close()
    samples = G2 * S
    return {"value": round(samples / (ms / 1e3), 3), "unit": "samples/s", "groups": G2,
            "cg_iterations_max": [r[0] for r in res],
            "note": "DOT_SERIAL: the reference's reduction order, bitwise equal to its pcg_solve per sample"}


def time_queued(torch, fn, reps, stream):
    """Per-launch CUDA-event times of reps back-to-back launches of fn queued on
    stream with no host synchronisation in between, so the host's launch
    overhead overlaps the previous launch instead of being timed (a sync per
    rep leaves the GPU idle while the next launch is issued: ~20 us, 10-15% of a
    0.2 ms s = 1 SpMV). Returns the list of milliseconds."""
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def bench_spmv(ctx, ep, torch, pack_group, O, hbm, peak_kind, reps=20):
    """cfg 3: enprop_spmv on the assembled + Dirichlet 128^3 matrix, s = 32, x
    uniform in [-1, 1); CUDA events on the context's (torch's current) stream."""
    n, s = SPMV_MESH, S
    y = torch.as_tensor(pack_group(O.draw_samples(0, s, M_TERMS), s)).cuda()
    p = ep.Problem(ctx, n, s, ep.KlField(M_TERMS, 1.0, SIGMA, 1.0))
    p.assemble(y)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((p.rows, s), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    z = torch.empty_like(x)
    rm, ce, vals = p.row_map, p.col_entry, p.values
    for _ in range(3):
        ep.spmv(ctx, s, rm, ce, vals, x, z)
    stream = torch.cuda.current_stream()
    times = time_queued(torch, lambda: ep.spmv(ctx, s, rm, ce, vals, x, z), reps, stream)
    best = min(times)
    med = statistics.median(times)
    byt = spmv_bytes(p.nnz, p.rows, s)
    out = {"metric": "ensemble SpMV HBM GB/s (128^3 27-pt matrix, s=32, fp64)",
           "value": round(byt / (med / 1e3) / 1e9, 1), "unit": "GB/s", "best_gbs": round(byt / (best / 1e3) / 1e9, 1),
           "median_ms": round(med, 4), "best_ms": round(best, 4), "bytes": byt,
           "gflops": round(2 * p.nnz * s / (med / 1e3) / 1e9, 1),
           "roofline": {"bound": "hbm", "kernel": "k_spmv<32>", "achieved": round(byt / (med / 1e3) / 1e9, 1),
                        "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                        "frac": round(byt / (med / 1e3) / 1e9 / hbm, 4), "traffic": None},
           "l2": "matrix 14.6 GB >> L2", "reps": reps}
    out["layouts"] = bench_spmv_layouts(ctx, ep, torch, p, x, z, byt, med, reps=max(5, reps // 4))
    p.close()
    del vals, x, z
    out["widths"] = bench_spmv_widths(ctx, ep, torch, pack_group, O, hbm, n, out["value"])
    return out


def bench_spmv_widths(ctx, ep, torch, pack_group, O, hbm, n, gbs32, reps=10):
    """Ensemble SpMV GB/s at s = 1, 4, 8, 16 on the same 128^3 matrix family (s <= 16: k_spmv_small)
    (north_star: throughput at ensemble sizes 1/4/8/16/32); s = 32 is cfg 3."""
    res = {}
    stream = torch.cuda.current_stream()
    for s in (1, 4, 8, 16):
        y = torch.as_tensor(pack_group(O.draw_samples(0, s, M_TERMS), s)).cuda()
        p = ep.Problem(ctx, n, s, ep.KlField(M_TERMS, 1.0, SIGMA, 1.0))
        p.assemble(y)
        vals = p.values
        g = torch.Generator(device="cuda").manual_seed(0)
        x = torch.rand((p.rows, s), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        z = torch.empty_like(x)
        for _ in range(3):
            ep.spmv(ctx, s, p.row_map, p.col_entry, vals, x, z)
        ts = time_queued(torch, lambda: ep.spmv(ctx, s, p.row_map, p.col_entry, vals, x, z), reps, stream)
        med = statistics.median(ts)
        byt = spmv_bytes(p.nnz, p.rows, s)
        res[str(s)] = {"ms": round(med, 4), "gbs": round(byt / (med / 1e3) / 1e9, 1),
                       "frac": round(byt / (med / 1e3) / 1e9 / hbm, 4),
                       "kernel": f"k_spmv_small<{s},64>" if s <= 16 else f"k_spmv<{s}>"}
        p.close()
        del vals, x, z
    res["32"] = {"gbs": gbs32, "frac": round(gbs32 / hbm, 4), "kernel": "k_spmv<32>"}
    return res


def bench_spmv_layouts(ctx, ep, torch, p, x, z, byt, commuted_ms, reps=5):
    """The paper's SpMV layout comparison (bench.cpp:73-238, acceptance.cpp:377-408)
    on the same matrix: commuted = ensemble layout (enprop_spmv); outer =
    sample-major OuterEnsembleMatrix (enprop_spmv_outer); scalar = s back-to-back
    s = 1 products over the shared graph. Gate: outer and scalar equal the
    commuted product bitwise. Median of reps, CUDA events."""
    s = S
    rm, ce = p.row_map, p.col_entry
    vo = p.values.t().contiguous()          # [s][nnz]
    xo = x.t().contiguous()                 # [s][rows]
    zo = torch.empty_like(xo)
    zs = torch.empty_like(xo)
    stream = torch.cuda.current_stream()

    def timed(fn):
        fn()
        return statistics.median(time_queued(torch, fn, reps, stream))

    def scalar():
        for e in range(s):
            ep.spmv(ctx, 1, rm, ce, vo[e], xo[e], zs[e])

    outer_ms = timed(lambda: ep.spmv_outer(ctx, s, rm, ce, vo, xo, zo))
    scalar_ms = timed(scalar)
    gate = bool(torch.equal(zo.view(torch.int64), z.t().contiguous().view(torch.int64)) and
                torch.equal(zs.view(torch.int64), zo.view(torch.int64)))
    del vo
    gbs = lambda ms: round(byt / (ms / 1e3) / 1e9, 1)
    return {"commuted": {"ms": round(commuted_ms, 4), "gbs": gbs(commuted_ms), "kernel": "k_spmv<32>"},
            "outer": {"ms": round(outer_ms, 4), "gbs": gbs(outer_ms), "kernel": "k_spmv_outer"},
            "scalar": {"ms": round(scalar_ms, 4), "gbs": gbs(scalar_ms), "kernel": "32 x k_spmv_small<1,64>"},
            "speedup_commuted_vs_scalar": round(scalar_ms / commuted_ms, 3),
            "speedup_commuted_vs_outer": round(outer_ms / commuted_ms, 3),
            "gate_bitwise": gate}


def bench_halo_model(ep, torch, n=128, nranks=2, reps=50):
    """T(s) = a + b*s fitted (enprop_fit_halo_model =
    halo.cpp:156-181) to the slab solver's MEASURED halo exchange (one plane of
    s values per neighbour, 128^3 mesh) at s = 1..32, and predicted_speedup
    (halo.cpp:183-188). On one GPU the transport is the emulated one (device
    copies inside HBM); NVLink needs two GPUs."""
    ctx = ep.Context(0)
    samples = []
    for s in (1, 2, 4, 8, 16, 32):
        d = ep.Dist(ctx, n, s, nranks=nranks, kl=ep.KlField(M_TERMS, 1.0, SIGMA, 1.0))
        samples.append((s, d.time_halo(reps)))
        del d
        torch.cuda.synchronize()
    a, b, rss = ep.fit_halo_model(samples)
    return {"transport": f"emulated ({nranks} ranks on one GPU: device-to-device copies)",
            "mesh": n, "plane_bytes_per_component": (n + 1) ** 2 * 8,
            "measured_us": {str(s): round(t * 1e6, 3) for s, t in samples},
            "fit": {"a_us": round(a * 1e6, 4), "b_us_per_component": round(b * 1e6, 5),
                    "rss": rss},
            "predicted_speedup": {str(s): round(ep.predicted_speedup(a, b, s), 3) for s in (4, 16, 32)}}


def cpu_baseline_sample(max_cg=10):
    """The reference's own ensemble path (coupled pcg_solve<Ensemble<32>>, the
    reference's fused method, bench.cpp:356-362 with IdentityPreconditioner) on one
    host core: full assembly + Dirichlet, then max_cg CG iterations timed and
    scaled to the full solve's iteration count."""
    from oracles import RefLib
    import ctypes as C
    import numpy as np
    R = RefLib()
    times = np.zeros(3)
    its = np.zeros(S, np.int32)
    rc = R.lib.ref_time_group(S, 1, N_MESH, M_TERMS, 1.0, SIGMA, 1.0, 0, 0, TOL, max_cg,
                              times.ctypes.data_as(C.POINTER(C.c_double)),
                              its.ctypes.data_as(C.POINTER(C.c_int)))
    if rc not in (0, 2):
        return None
    t_asm, t_cg, ran = times
    per_it = t_cg / max(ran, 1)
    total = t_asm + per_it * REF_COUPLED_ITERS_64
    return {"value": round(S / total, 4), "unit": "samples/s", "cores": 1, "kind": "reference",
            "sample": f"reference assemble<Ensemble<32>>+apply_dirichlet (full, {t_asm:.2f}s) + "
                      f"{int(ran)} pcg_solve iterations ({per_it:.3f}s/it) scaled to the full "
                      f"{REF_COUPLED_ITERS_64}-iteration coupled solve; 64^3, s=32, 1 core"}


# ---------------------------------------------------------------------- reference
def run_reference(args):
    """The reference CPU path (oracle/_ref, unmodified proj/ sources) on all host
    cores: P worker processes each solve a different sample group with the
    reference's ensemble method; each step is a bounded sample (full assembly +
    `max_cg` CG iterations scaled to the full coupled iteration count)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    try:
        import psutil
        mem_gb = psutil.virtual_memory().available / 1e9
    except Exception:
        mem_gb = 16.0
    procs = max(1, min(cores, int(mem_gb // 4), 16))
    max_cg = 4
    ctx = mp.get_context("spawn")
    vals = []
    for k in range(args.warmup + args.steps):
        with ctx.Pool(procs) as pool:
            t0 = time.perf_counter()
            res = pool.map(_ref_worker, [(g, max_cg) for g in range(procs)])
            wall = time.perf_counter() - t0
        # each process: assembly + full solve extrapolated from its per-iteration time
        per_proc = [r for r in res if r is not None]
        if not per_proc:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref failed"}))
            return
        total_s = max(t_asm + per_it * REF_COUPLED_ITERS_64 for (t_asm, per_it) in per_proc)
        if k >= args.warmup:
            vals.append(len(per_proc) * S / total_s)
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": "sample solves/sec (assembly+CG) at ensemble s=32",
            "value": round(value, 4), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2: 64^3 Q1 hex mesh, KL m=3 sigma=0.1, s=32, reference "
                                   "assemble<Ensemble<32>> + apply_dirichlet + pcg_solve<Ensemble<32>> "
                                   "(IdentityPreconditioner, tol 1e-6)", "processes": procs},
            "cpu_baseline": {"value": round(value, 4), "unit": "samples/s", "cores": procs,
                             "kind": "reference",
                             "sample": f"{procs} processes x one s=32 group: full assembly + "
                                       f"{max_cg} CG iterations scaled to {REF_COUPLED_ITERS_64}"},
            "e2e": {"value": round(value, 4), "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _ref_worker(a):
    g, max_cg = a
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import ctypes as C
    import numpy as np
    from oracles import RefLib
    R = RefLib()
    times = np.zeros(3)
    its = np.zeros(S, np.int32)
    rc = R.lib.ref_time_group(S, 1, N_MESH, M_TERMS, 1.0, SIGMA, 1.0, 0, g, TOL, max_cg,
                              times.ctypes.data_as(C.POINTER(C.c_double)),
                              its.ctypes.data_as(C.POINTER(C.c_int)))
    if rc not in (0, 2):
        return None
    return times[0], times[1] / max(times[2], 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dot", choices=["canonical", "serial"], default="canonical")
    ap.add_argument("--skip-spmv", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-serial", action="store_true")
    ap.add_argument("--serial-groups", type=int, default=8)
    ap.add_argument("--workload", choices=["groups", "dd"], default="groups",
                    help="groups: cfg 2 sample groups (default); dd: cfg 4 domain decomposition")
    ap.add_argument("--dd-mesh", type=int, default=256)
    ap.add_argument("--groups", type=int, default=3,
                    help="sample groups solved concurrently per step (one stream each)")
    ap.add_argument("--profile-only", action="store_true",
                    help="warm-up + timed steps only (for ncu launch lists)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "dd":
        run_dd(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
