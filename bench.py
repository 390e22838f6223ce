"""Benchmark: sample solves/s (assembly + Dirichlet + CG) at ensemble s=32 on the
64^3 hex mesh (BASELINE.json configs[1], "cfg 2"), plus the ensemble SpMV HBM
GB/s on the 128^3 matrix (configs[2], "cfg 3") and the other configs' keys in
the same run.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = G sample groups of s=32 samples solved concurrently, one stream each:
per group, assemble the ensemble matrix with the fused Dirichlet elimination,
then solve A x = -residual with uncoupled (per-sample) identity-preconditioned
CG to tol 1e-6, all on the device.  The headline runs the reference's own dot
order (ENPROP_DOT_SERIAL): every sample's solution, iteration count and
residual history are bitwise the reference's s x pcg_solve<double>
(src/bench.cpp:340-349; tests/test_gpu_cfg.py pins it at this very size).  The
fast fixed-tree order (DOT_CANONICAL) is reported beside it with its
iteration / solution deltas against the reference.  With N>1 (torchrun, one
process per GPU) every rank solves its own sample groups (independent units:
weak scaling, no data-path collective).

--impl reference times the reference's own CPU path (oracle/_ref: the unmodified
proj/ sources) on all host cores for the same workload and flavour.
"""
import os

# Every sample group runs on its own stream; CUDA multiplexes streams onto
# CUDA_DEVICE_MAX_CONNECTIONS hardware queues (default 8), and a long
# serial-order chain kernel would block the other groups sharing its queue.
# Must be set before the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import argparse  # noqa: E402
import json  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_MESH, S, M_TERMS, SIGMA, TOL = 64, 32, 3, 0.1, 1e-6
SPMV_MESH = 128
# Reference uncoupled iteration counts of sample group 0 at cfg 2 (64^3, s=32,
# seed 0): s x pcg_solve<double> run by the reference itself
# (tests/golden/make_cfg2.py -> tests/golden/cfg2_64_s32.npz); the GPU's serial
# order reproduces them bitwise (tests/test_gpu_cfg.py).
CFG2_FIXTURE = os.path.join(ROOT, "tests", "golden", "cfg2_64_s32.npz")
# scalar CG iterations per sample in the reference arm's bounded sample
# (extrapolation checked against a full solve: tests/ref_extrapolation.py)
REF_SAMPLE_ITERS = 6


def cfg2_fixture():
    import numpy as np
    try:
        return dict(np.load(CFG2_FIXTURE))
    except OSError:
        return None


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


def cg_spmv_bytes(nnz, nnz_stored, rows, s, products=False):
    """Algorithmic bytes of one CG SpMV launch (k_cg_spmv_staged / k_cg_spmv_warp,
    DESIGN.md §3): the stored value slots once (symmetric storage: diagonal +
    upper), column indices, the slot map (symmetric storage only), row_map, the
    direction vector gathered once and q written once; in the serial order also
    the p*q products written for the chain kernel. The transposed re-reads of
    the upper slots are not algorithmic bytes."""
    sym = nnz_stored < nnz
    b = nnz_stored * 8 * s + nnz * (8 if sym else 4) + 4 * (rows + 1) + 16 * s * rows
    return b + (8 * s * rows if products else 0)


def direction_bytes(rows, s):
    """k_cg_direction: read r, p_old, x; write p_new, x."""
    return 5 * 8 * s * rows


def measured_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full capture (profiles/*/traffic.json, newest
    round first), else None."""
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

    def __init__(self, ep, torch, device, kl, n=N_MESH, s=S):
        self.stream = torch.cuda.Stream(device=device)
        self.ctx = ep.Context(device, use_torch_stream=False)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.prob = ep.Problem(self.ctx, n, s, kl)

    def close(self):
        self.prob.close()
        self.ctx.close()


def run_groups(torch, workers, jobs, cfg, host=False):
    """Solve jobs[i] (lists of device or host sample tensors) on workers[i]
    concurrently (one host thread each; ctypes releases the GIL).  Returns the
    per-worker (max iteration counts, lane statuses, per-lane iterations)."""
    out = [None] * len(workers)

    def run(i):
        w = workers[i]
        its, sts, lanes = [], [], []
        for item in jobs[i]:
            if host:
                y_host, x_host = item
                it, st, rc = w.prob.solve_host(y_host, x_host, cfg)  # lists (one per lane)
            else:
                w.prob.assemble(item)
                it, _, st = w.prob.solve(cfg)
            it = list(it) if isinstance(it, (list, tuple)) else [it]  # coupled: one count
            its.append(max(it))
            sts.extend(st)
            lanes.append(it)
        out[i] = (its, sts, lanes)

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


def solver_cfg(ep, dot, flavour=None, maxit=10000):
    return ep.SolverConfig(tol=TOL, max_iterations=maxit,
                           flavour=ep.CG_UNCOUPLED if flavour is None else flavour,
                           dot_mode=ep.DOT_CANONICAL if dot == "canonical" else ep.DOT_SERIAL)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1511_03703_b200 as ep

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    G = args.groups
    rounds = args.warmup + args.steps
    # rank r, round k, worker i solves sample group ((r * rounds + k) * G + i);
    # samples: the library's draw_samples / pack_sample_group (samples.cpp:7-18)
    pool = ep.draw_samples(0, S * G * rounds * world, M_TERMS)
    group_of = lambda k, i: (rank * rounds + k) * G + i  # noqa: E731
    kl = ep.KlField(M_TERMS, 1.0, SIGMA, 1.0)
    workers = [GroupWorker(ep, torch, local, kl) for _ in range(G)]
    ys = {(k, i): ep.pack_sample_group(pool, S, S * group_of(k, i)).cuda()
          for k in range(rounds) for i in range(G)}
    cfg = solver_cfg(ep, args.dot)

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
    hjobs = [[(ep.pack_sample_group(pool, S, S * group_of(args.warmup + k, i)).contiguous().pin_memory(),
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

    hbm, peak_kind = peaks()
    w0 = workers[0]
    roofline = bench_roofline(ep, w0, ys[(args.warmup, 0)], cfg, args.dot, hbm, peak_kind)
    extra = {}
    if rank == 0:
        extra["parity"] = bench_parity(ep, torch, w0, ys[(0, 0)], args.dot)
    if rank == 0 and not args.skip_canonical:
        extra["canonical_order"] = bench_canonical(ep, torch, workers, ys, args, extra["parity"])
    if rank == 0 and not args.skip_asm:
        extra["assembly"] = bench_assembly(ep, torch, w0, ys[(0, 0)], hbm, peak_kind)
    for w in workers:
        w.close()
    del workers
    torch.cuda.empty_cache()
    if rank == 0 and not args.skip_widths:
        extra["widths"] = bench_widths(ep, torch, local, pool, kl)
    spmv_obj = None
    if rank == 0 and not args.skip_spmv:
        spmv_obj = bench_spmv(ep.Context(local), ep, torch, pool, hbm, peak_kind)
    if rank == 0 and world == 1 and not args.skip_spmv:
        extra["halo_model"] = bench_halo_model(ep, torch)
    if rank == 0 and world == 1 and not args.skip_configs:
        extra["cfg5"] = bench_cfg5(ep, torch, local)
        extra["cfg4_one_gpu"] = bench_cfg4_one_gpu(ep, torch, local)
        extra["multigrid_newton"] = bench_multigrid(ep, torch, local)
    if not args.skip_dd:  # every rank takes part (strong scaling of one 256^3 ensemble)
        try:
            dd = bench_cfg4_dd(ep, torch, dist, local, rank, world, args.dd_mesh)
        except Exception as e:  # never lose the headline line to this extra (peers time out too)
            dd = {"mesh": args.dd_mesh, "ranks": world, "error": repr(e)[:300]}
            torch.cuda.empty_cache()
        if rank == 0:
            extra["cfg4_dd"] = dd
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        cpu = cpu_baseline_sample()

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    order = ("serial (the reference's own order: bitwise its s x pcg_solve<double> per sample)"
             if args.dot == "serial" else "canonical (fixed tree; bitwise the C restatement)")
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
                   "dot_order": order, "cg_iterations_max": iters,
                   "l2": "inputs larger than L2 (matrix 0.96 GB stored per group, 24 GB per step)",
                   "parallelism": f"sample groups x {world} GPU(s)",
                   "hw_queues": os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS")},
        "e2e": e2e, "roofline": roofline, "gpu_launches": int(launches), "clocks": clk,
    }
    line.update(extra)
    if spmv_obj:
        line["spmv_cfg3"] = spmv_obj
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def bench_roofline(ep, w, y, cfg, dot, hbm, peak_kind):
    """Dominant HBM kernel of the benchmarked mode from a single-stream solve
    (CUDA events on the solve's stream; kernels of concurrent streams overlap,
    so they are timed alone): k_cg_spmv_staged<32, tiles> -- in the serial order
    it also writes the p*q products the chain kernel sums."""
    w.ctx.profile(1)
    w.prob.assemble(y)
    w.prob.solve(cfg)
    det = w.ctx.profile_detail()
    spmv_ms, spmv_n = w.ctx.profile(0)
    p = w.prob
    nnz, nnz_st, rows = p.nnz, p.nnz_stored, p.rows
    serial = dot == "serial"
    avg_spmv_ms = spmv_ms / max(spmv_n, 1)
    nit = max(det["iterations"], 1)
    byt = cg_spmv_bytes(nnz, nnz_st, rows, S, products=serial)
    achieved = byt / (avg_spmv_ms / 1e3) / 1e9
    it_ms = det["iteration"] / nit
    kname = f"k_cg_spmv_staged<{S},{'false' if serial else 'true'}>"
    dir_ms = det["direction"] / nit
    it_bytes = byt + direction_bytes(rows, S) + 3 * 8 * S * rows  # + update (r, q -> r)
    out = {"bound": "hbm", "kernel": kname,
           "achieved": round(achieved, 1), "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
           "frac": round(achieved / hbm, 4), "frac_of_8000_spec": round(achieved / 8000.0, 4),
           "traffic": measured_traffic(kname),
           "bytes_per_launch": byt, "avg_launch_ms": round(avg_spmv_ms, 4), "launches_timed": spmv_n,
           "share_of_iteration_hbm_work": round(avg_spmv_ms / (avg_spmv_ms + det["direction"] / nit + det["update"] / nit), 3),
           "per_iteration_ms": {k: round(det[k] / nit, 4) for k in
                                ("direction", "spmv_kernel", "fin_pq", "update", "fin_rr", "iteration")},
           "direction": {"kernel": f"k_cg_direction<{S}>", "bytes": direction_bytes(rows, S),
                         "achieved": round(direction_bytes(rows, S) / (dir_ms / 1e3) / 1e9, 1) if dir_ms else None},
           "timing": "CUDA events on the solve's stream, single-stream solve"}
    if serial:
        # the two reference-order dot chains (k_chain): latency-bound, one
        # dependent DADD per row (8.0 cycles measured, tools/microbench/chain_bench.cu)
        clk = _sm_clock_mhz()
        pq, rr = det["fin_pq"] / nit, det["fin_rr"] / nit
        out["chain"] = {"kernel": "k_chain<32, given | square>", "pq_ms": round(pq, 4), "rr_ms": round(rr, 4),
                        "rows": rows, "floor_ms_at_8_cycles": round(rows * 8.0 / (clk * 1e3), 4) if clk else None,
                        "sm_mhz": clk,
                        "note": "latency-bound chains overlap other sample groups' HBM work (one CTA each)"}
    else:
        out["iteration_bytes"] = it_bytes
        out["iteration_gbs"] = round(it_bytes / (it_ms / 1e3) / 1e9, 1) if it_ms else None
    return out


def _sm_clock_mhz():
    try:
        r = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True, timeout=10)
        return float(r.stdout.strip().splitlines()[0])
    except Exception:
        return None


def bench_parity(ep, torch, w, y, dot):
    """Group 0 of cfg 2 solved in both orders on the device: the serial order
    against the reference's fixture (tests/golden/cfg2_64_s32.npz: the reference's
    own s x pcg_solve<double>; iterations and solution hashes), and the
    canonical order's deltas against it (north_star: identical uncoupled
    iteration counts, solutions within 1e-12 relative)."""
    import hashlib
    import numpy as np
    fx = cfg2_fixture()
    out = {}
    sol = {}
    for order in ("serial", "canonical"):
        w.prob.assemble(y)
        it, hist, st = w.prob.solve(solver_cfg(ep, order))
        torch.cuda.synchronize()
        x = w.prob.solution.cpu().numpy().copy()
        sol[order] = (np.array(it), x)
    its_s, xs = sol["serial"]
    its_c, xc = sol["canonical"]
    if fx is not None:
        shas = [hashlib.sha256(np.ascontiguousarray(xs[:, e]).tobytes()).hexdigest() for e in range(S)]
        out["serial_vs_reference"] = {
            "iterations_equal": bool((its_s == fx["ref_iterations"]).all()),
            "solutions_bitwise": bool(all(a == b for a, b in zip(shas, fx["ref_x_sha"]))),
            "reference_iterations": fx["ref_iterations"].tolist(),
            "fixture": "tests/golden/cfg2_64_s32.npz (reference run by tests/golden/make_cfg2.py)"}
    num = np.abs(xc - xs).max(axis=0)
    den = np.abs(xs).max(axis=0)
    out["canonical_vs_reference"] = {
        "max_iter_delta": int(np.abs(its_c - its_s).max()), "lanes_with_other_count": int((its_c != its_s).sum()),
        "max_rel_x": float((num / den).max()), "tolerance_north_star": 1e-12,
        "within_north_star": bool((its_c == its_s).all() and (num / den).max() <= 1e-12),
        "note": "reference = the serial order, bitwise the reference (serial_vs_reference)"}
    return out


def bench_canonical(ep, torch, workers, ys, args, parity):
    """The fast fixed-tree order (DOT_CANONICAL, staged SpMV with the fused p.q
    finalize) on the same workload; NOT reference-identical (parity deltas in
    canonical_vs_reference)."""
    G = len(workers)
    cfg = solver_cfg(ep, "canonical")
    timed_round(torch, workers, [[ys[(0, i)]] for i in range(G)], cfg)
    steps = max(1, min(args.steps, 3))
    jobs = [[ys[(args.warmup + k, i)] for k in range(steps)] for i in range(G)]
    ms, res = timed_round(torch, workers, jobs, cfg)
    return {"value": round(steps * G * S / (ms / 1e3), 3), "unit": "samples/s", "groups": G, "steps": steps,
            "cg_iterations_max": [r[0] for r in res],
            "deltas": parity.get("canonical_vs_reference")}


def bench_assembly(ep, torch, w, y, hbm, peak_kind, reps=5):
    """Assembly + fused Dirichlet (k_assemble) at 64^3, s=32: HBM fraction
    (bytes: stored value slots + residual written) and FP64
    fraction (cells * s * (1536 + 16m) non-FMA flops) against
    the measured DGEMM rate / 2 (one DMUL or DADD per FMA slot)."""
    p = w.prob
    st = torch.cuda.Stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    w.prob.assemble(y)
    torch.cuda.synchronize()
    for a, b in ev:
        a.record(w.stream)
        p.assemble(y)
        b.record(w.stream)
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ev)
    byt = 8 * S * p.nnz_stored + 8 * S * p.rows
    flops = N_MESH ** 3 * S * (1536 + 16 * M_TERMS)
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    with torch.cuda.stream(st):
        torch.mm(a, a)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            torch.mm(a, a)
        e1.record(st)
    torch.cuda.synchronize()
    dgemm = 3 * 2 * 8192 ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12
    del a
    gbs = byt / (ms / 1e3) / 1e9
    tf = flops / (ms / 1e3) / 1e12
    return {"kernel": "k_assemble<32> (node-centric gather + fused Dirichlet)", "ms": round(ms, 4),
            "hbm": {"bytes": byt, "achieved": round(gbs, 1), "peak": hbm, "peak_kind": peak_kind,
                    "frac": round(gbs / hbm, 4)},
            "fp64": {"flops": flops, "achieved_tflops": round(tf, 3),
                     "peak_tflops": round(dgemm / 2, 3),
                     "peak_kind": "measured: torch.mm fp64 8192^3 (cuBLAS DGEMM) / 2 (non-FMA ops)",
                     "frac": round(tf / (dgemm / 2), 4)}}


WIDTH_GROUPS = {1: 32, 4: 32, 8: 32, 16: 24}  # one stream each, <= the 32 hardware queues


def bench_widths(ep, torch, device, pool, kl):
    """cfg 2 at s = 1, 4, 8, 16 (north_star: throughput at ensemble sizes
    1/4/8/16/32): WIDTH_GROUPS[s] concurrent groups per width (narrow groups
    are latency-bound, so more of them fit), one round, both dot orders (the
    serial order is bitwise the reference at every width)."""
    out = {}
    for s, groups in WIDTH_GROUPS.items():
        ws = [GroupWorker(ep, torch, device, kl, s=s) for _ in range(groups)]
        ys = [ep.pack_sample_group(pool, s, s * i).cuda() for i in range(groups)]
        res = {}
        for dot in ("serial", "canonical"):
            cfg = solver_cfg(ep, dot)
            timed_round(torch, ws, [[ys[i]] for i in range(groups)], cfg)
            ms, r = timed_round(torch, ws, [[ys[i]] for i in range(groups)], cfg)
            res[dot] = round(groups * s / (ms / 1e3), 2)
        res["groups"] = groups
        out[str(s)] = res
        for w in ws:
            w.close()
    return out


def bench_cfg5(ep, torch, device):
    """cfg 5: 128^3, KL m=10, sigma=0.25, s=32: coupled vs uncoupled CG
    iterations and samples/s (one group, canonical order; single stream)."""
    kl = ep.KlField(10, 1.0, 0.25, 1.0)
    w = GroupWorker(ep, torch, device, kl, n=128)
    y = ep.pack_sample_group(ep.draw_samples(0, S, 10), S, 0).cuda()
    out = {"mesh": 128, "num_terms": 10, "sigma": 0.25, "dot_order": "canonical"}
    for name, fl in (("coupled", ep.CG_COUPLED), ("uncoupled", ep.CG_UNCOUPLED)):
        cfg = solver_cfg(ep, "canonical", flavour=fl, maxit=20000)
        ms, res = timed_round(torch, [w], [[y]], cfg)
        it = res[0][2][0]
        out[name] = {"iterations": it if fl == ep.CG_UNCOUPLED else it[0],  # per lane / coupled
                     "samples_per_s": round(S / (ms / 1e3), 3), "ms": round(ms, 1)}
    w.close()
    return out


def bench_multigrid(ep, torch, device, n=32):
    """f4 and f3 measured where the reference's multigrid is practical (its
    dense-LU coarse level): cfg 1's mesh, s = 32, KL m = 3,
    sigma = 0.1, the reference's serial dot order (bitwise its MG-PCG and
    newton_solve: tests/test_gpu_mg.py). Host-driven solves, so wall times
    with the device synchronised on both sides."""
    s = S
    ctx = ep.Context(device)
    kl = ep.KlField(M_TERMS, 1.0, SIGMA, 1.0)
    y = ep.pack_sample_group(ep.draw_samples(0, s, M_TERMS), s, 0).cuda()

    def wall(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3, r

    out = {"mesh": n, "s": s, "dot_order": "serial (bitwise the reference)"}
    p = ep.Problem(ctx, n, s, kl)
    p.assemble(y)
    vals, b = p.values, (-p.residual).contiguous()
    cfg = ep.SolverConfig(tol=TOL, max_iterations=10000, flavour=ep.CG_COUPLED, dot_mode=ep.DOT_SERIAL)
    h = ep.MgHierarchy(ctx, s, p.row_map, p.col_entry, vals)  # warm-up build
    h.close()
    ms_build, h = wall(lambda: ep.MgHierarchy(ctx, s, p.row_map, p.col_entry, vals))
    rows, _ = h.describe()
    h.pcg(b, cfg)  # warm-up
    ms_mg, res = wall(lambda: h.pcg(b, cfg))
    p.solve(cfg)
    ms_id, (it_id, _, _) = wall(lambda: p.solve(cfg))
    out["mg_pcg_coupled"] = {"levels_rows": rows, "build_ms": round(ms_build, 1), "solve_ms": round(ms_mg, 1),
                             "iterations": res.iterations}
    out["identity_cg_coupled"] = {"solve_ms": round(ms_id, 1), "iterations": it_id}
    h.close()
    del vals
    p.close()
    q = ep.Problem(ctx, n, s, kl, coeffs=ep.PdeCoefficients(0.0, 1.0))
    nopt = ep.NewtonOptions(tol=1e-8, max_iterations=20,
                            linear=ep.SolverConfig(tol=1e-8, max_iterations=1000, dot_mode=ep.DOT_SERIAL))
    ms_nmg, r_mg = wall(lambda: q.newton(y, nopt, multigrid=ep.MgOptions()))  # (hierarchy rebuilt per step)
    ms_nid, r_id = wall(lambda: q.newton(y, nopt))
    out["newton_beta1"] = {
        "multigrid": {"ms": round(ms_nmg, 1), "steps": r_mg.iterations, "cg_iterations": r_mg.total_cg_iterations},
        "identity": {"ms": round(ms_nid, 1), "steps": r_id.iterations, "cg_iterations": r_id.total_cg_iterations}}
    q.close()
    ctx.close()
    return out


def bench_cfg4_one_gpu(ep, torch, device):
    """cfg 4 on one GPU: 256^3, s=32, one group (assembly + uncoupled CG,
    canonical order, staged SpMV): the 1-GPU baseline of the slab run."""
    kl = ep.KlField(M_TERMS, 1.0, SIGMA, 1.0)
    w = GroupWorker(ep, torch, device, kl, n=256)
    y = ep.pack_sample_group(ep.draw_samples(0, S, M_TERMS), S, 0).cuda()
    cfg = solver_cfg(ep, "canonical", maxit=20000)
    ms, res = timed_round(torch, [w], [[y]], cfg)
    w.close()
    return {"mesh": 256, "samples_per_s": round(S / (ms / 1e3), 3), "ms": round(ms, 1),
            "cg_iterations_max": res[0][0], "dot_order": "canonical",
            "note": "serial order at 256^3: a dot chain is 17M dependent DADDs (~72 ms); one group cannot hide it"}


def bench_cfg4_dd(ep, torch, dist, local, rank, world, n, steps=1):
    """cfg 4 (north_star: 1 -> 8 GPUs on 256^3): ONE s=32 ensemble on the n^3
    mesh split into z-slabs over the `world` ranks of this job (partition.cpp
    rule), halo of p and all-gathered per-plane dot sums over the CUDA-IPC
    transport (NVLink P2P between GPUs; the in-process transport at 1 rank);
    canonical order, so every rank count gives the one-GPU bits. Strong
    scaling: samples/s of the whole job; device time, max over ranks."""
    import uuid
    job = None
    if world > 1:
        obj = [uuid.uuid4().hex[:16] if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        job = obj[0]
    ctx = ep.Context(local)
    kl = ep.KlField(M_TERMS, 1.0, SIGMA, 1.0)
    d = ep.Dist(ctx, n, S, world, rank, kl=kl, ipc_job=job)
    pool = ep.draw_samples(0, S * (steps + 1), M_TERMS)
    cfg = solver_cfg(ep, "canonical", maxit=20000)
    d.assemble(ep.pack_sample_group(pool, S, 0).cuda())  # warm-up solve
    d.solve(cfg)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record(st)
    iters = []
    for k in range(steps):
        d.assemble(ep.pack_sample_group(pool, S, S * (k + 1)).cuda())
        it, status = d.solve(cfg)
        iters.append(max(it))
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    d.close()
    ctx.close()
    return {"mesh": n, "ranks": world, "samples_per_s": round(steps * S / (ms / 1e3), 3), "ms": round(ms, 1),
            "cg_iterations_max": iters, "dot_order": "canonical",
            "transport": "CUDA IPC (NVLink P2P)" if world > 1 else "single rank",
            "scaling": "strong (one ensemble per step split over the ranks)"}


def time_queued(torch, fn, reps, stream):
    """Per-launch CUDA-event times of reps back-to-back launches of fn queued on
    stream with no host synchronisation in between, so the host's launch
    overhead overlaps the previous launch instead of being timed. Returns the
    list of milliseconds."""
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def bench_spmv(ctx, ep, torch, pool, hbm, peak_kind, reps=20):
    """cfg 3: enprop_spmv on the assembled + Dirichlet 128^3 matrix, s = 32, x
    uniform in [-1, 1); CUDA events on the context's (torch's current) stream."""
    n, s = SPMV_MESH, S
    y = ep.pack_sample_group(pool, s, 0).cuda()
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
                        "frac": round(byt / (med / 1e3) / 1e9 / hbm, 4),
                        "frac_of_8000_spec": round(byt / (med / 1e3) / 1e9 / 8000.0, 4),
                        "traffic": measured_traffic("k_spmv<32>")},
           "l2": "matrix 14.6 GB >> L2", "reps": reps}
    out["layouts"] = bench_spmv_layouts(ctx, ep, torch, p, x, z, byt, med, reps=max(5, reps // 4))
    p.close()
    del vals, x, z
    out["widths"] = bench_spmv_widths(ctx, ep, torch, pool, hbm, n, out["value"])
    return out


def bench_spmv_widths(ctx, ep, torch, pool, hbm, n, gbs32, reps=10):
    """Ensemble SpMV GB/s at s = 1, 4, 8, 16 on the same 128^3 matrix family (s <= 16: k_spmv_small)
    (north_star: throughput at ensemble sizes 1/4/8/16/32); s = 32 is cfg 3."""
    res = {}
    stream = torch.cuda.current_stream()
    for s in (1, 4, 8, 16):
        y = ep.pack_sample_group(pool, s, 0).cuda()
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
    gbs = lambda ms: round(byt / (ms / 1e3) / 1e9, 1)  # noqa: E731
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
    d = ep.Dist(ctx, n, 32, nranks=3, kl=ep.KlField(M_TERMS, 1.0, SIGMA, 1.0))
    trace, elapsed = d.exchange_trace()  # halo.cpp:140-150 record order, measured times
    d.close()
    return {"transport": f"emulated ({nranks} ranks on one GPU: device-to-device copies)",
            "trace_s32_3ranks": {"records": [{"rank": r[0], "neighbor": r[1], "bytes": r[2],
                                              "time_us": round(r[3] * 1e6, 3)} for r in trace],
                                 "elapsed_us": round(elapsed * 1e6, 3)},
            "mesh": n, "plane_bytes_per_component": (n + 1) ** 2 * 8,
            "measured_us": {str(s): round(t * 1e6, 3) for s, t in samples},
            "fit": {"a_us": round(a * 1e6, 4), "b_us_per_component": round(b * 1e6, 5),
                    "rss": rss},
            "predicted_speedup": {str(s): round(ep.predicted_speedup(a, b, s), 3) for s in (4, 16, 32)}}


# ---------------------------------------------------------------- CPU reference
def host_facts():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        import psutil
        mem_gb = psutil.virtual_memory().total / 1e9
        avail_gb = psutil.virtual_memory().available / 1e9
    except Exception:
        mem_gb = avail_gb = None
    return {"cpu_model": model, "nproc": os.cpu_count(), "ram_gb": round(mem_gb, 1) if mem_gb else None,
            "ram_available_gb": round(avail_gb, 1) if avail_gb else None}


def ref_uncoupled_iterations():
    """Total scalar CG iterations of the reference's uncoupled cfg-2 solve of
    group 0 (sum over the 32 samples; the fixture's own run)."""
    fx = cfg2_fixture()
    if fx is None:
        return None
    return int(fx["ref_iterations"].sum())


def ref_group_sample(group, max_cg, cores_note=""):
    """One reference group: assemble<Ensemble<32>> + apply_dirichlet in full,
    then s x pcg_solve<double> on extract_component for max_cg iterations each
    (the uncoupled flavour, bench.cpp:340-349); returns (fixed seconds:
    assembly + Dirichlet + the s component extractions, seconds per scalar
    CG iteration)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import ctypes as C
    import numpy as np
    from oracles import RefLib
    R = RefLib()
    times = np.zeros(4)
    its = np.zeros(S, np.int32)
    rc = R.lib.ref_time_group(S, 0, N_MESH, M_TERMS, 1.0, SIGMA, 1.0, 0, group, TOL, max_cg,
                              times.ctypes.data_as(C.POINTER(C.c_double)),
                              its.ctypes.data_as(C.POINTER(C.c_int)))
    if rc not in (0, 2):
        return None
    # the s extractions are a fixed cost of the solve (each reads the whole
    # ensemble matrix), not a per-iteration one
    return float(times[0]) + float(times[3]), (float(times[1]) - float(times[3])) / max(float(times[2]), 1.0)


def cpu_baseline_sample(max_cg=REF_SAMPLE_ITERS):
    """The reference's own uncoupled path on one host core (same flavour as the
    GPU arm): full assembly + Dirichlet, max_cg scalar CG iterations per sample,
    scaled to the reference's total iteration count of the full solve."""
    total_it = ref_uncoupled_iterations()
    r = ref_group_sample(0, max_cg)
    if r is None or total_it is None:
        return None
    t_asm, per_it = r
    total = t_asm + per_it * total_it
    return {"value": round(S / total, 4), "unit": "samples/s", "cores": 1, "kind": "reference",
            "sample": f"reference assemble<Ensemble<32>>+apply_dirichlet+32 extract_component (full, {t_asm:.2f}s) "
                      f"+ 32 x {max_cg} pcg_solve<double> iterations ({per_it * 1e3:.2f} ms/it) "
                      f"scaled to the reference's {total_it} scalar iterations of the full uncoupled solve; "
                      f"64^3, s=32, 1 core",
            "host": host_facts()}


def run_reference(args):
    """The reference CPU path (oracle/_ref, unmodified proj/ sources) on all host
    cores: P = nproc worker processes (capped only by RAM, ~4 GB each) each
    solve a different sample group with the reference's uncoupled method (s x
    pcg_solve<double>, as the GPU arm); each step is a bounded sample (full
    assembly + max_cg scalar iterations per sample) scaled to the reference's
    own total iteration count (tests/golden/cfg2_64_s32.npz; the scaling is
    checked against a full solve in profiles/round2/ref_extrapolation.json)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    facts = host_facts()
    cores = facts["nproc"] or 1
    avail = facts["ram_available_gb"] or 16.0
    procs = max(1, min(cores, int(avail // 4)))
    total_it = ref_uncoupled_iterations()
    if total_it is None:
        print(json.dumps({"impl": "reference", "unavailable": "tests/golden/cfg2_64_s32.npz missing"}))
        return
    max_cg = REF_SAMPLE_ITERS
    ctx = mp.get_context("spawn")
    vals = []
    with ctx.Pool(procs) as pool:
        for k in range(args.warmup + args.steps):
            res = pool.map(_ref_worker, [(k * procs + g, max_cg) for g in range(procs)])
            per_proc = [r for r in res if r is not None]
            if not per_proc:
                print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref failed"}))
                return
            total_s = max(t_asm + per_it * total_it for (t_asm, per_it) in per_proc)
            if k >= args.warmup:
                vals.append(len(per_proc) * S / total_s)
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": "sample solves/sec (assembly+CG) at ensemble s=32",
            "value": round(value, 4), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2: 64^3 Q1 hex mesh, KL m=3 sigma=0.1, s=32; reference "
                                   "assemble<Ensemble<32>> + apply_dirichlet + uncoupled s x pcg_solve<double> "
                                   "(extract_component, IdentityPreconditioner, tol 1e-6) -- the GPU arm's flavour",
                       "processes": procs, "host": facts},
            "cpu_baseline": {"value": round(value, 4), "unit": "samples/s", "cores": procs,
                             "kind": "reference",
                             "sample": f"{procs} processes (nproc {cores}, RAM-capped at ~4 GB each) x one s=32 "
                                       f"group: full assembly + 32 x {max_cg} scalar CG iterations, scaled to the "
                                       f"reference's {total_it} iterations of the full uncoupled solve"},
            "e2e": {"value": round(value, 4), "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _ref_worker(a):
    g, max_cg = a
    return ref_group_sample(g, max_cg)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dot", choices=["canonical", "serial"], default="serial")
    ap.add_argument("--skip-spmv", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-canonical", action="store_true")
    ap.add_argument("--skip-asm", action="store_true")
    ap.add_argument("--skip-widths", action="store_true")
    ap.add_argument("--skip-configs", action="store_true", help="skip cfg 4 (one GPU) and cfg 5")
    ap.add_argument("--skip-dd", action="store_true", help="skip the cfg 4 slab solve over the job's ranks")
    ap.add_argument("--workload", choices=["groups", "dd"], default="groups",
                    help="groups: cfg 2 sample groups (default); dd: cfg 4 domain decomposition")
    ap.add_argument("--dd-mesh", type=int, default=256)
    ap.add_argument("--groups", type=int, default=24,
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


def run_dd(args):
    """cfg 4: ONE ensemble (s=32) on an n^3 mesh (default 256^3) domain-decomposed
    into z-slabs over the N ranks (NCCL halo of p + all-gathered per-plane dot
    sums); a step = assemble + Dirichlet + uncoupled CG to 1e-6.
    Strong scaling: the work per step is fixed as N grows."""
    import torch
    import torch.distributed as dist

    import paper_1511_03703_b200 as ep

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
    pool = ep.draw_samples(0, S * (args.warmup + args.steps), M_TERMS)
    ys = [ep.pack_sample_group(pool, S, S * g).cuda() for g in range(args.warmup + args.steps)]
    cfg = solver_cfg(ep, "canonical", maxit=20000)
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


if __name__ == "__main__":
    main()
