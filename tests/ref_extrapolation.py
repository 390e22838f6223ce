"""Check bench.py's reference-arm extrapolation once (a measurement script kept
under tests/ because it runs the reference, oracle/_ref; not collected by
pytest): the reference's uncoupled
cfg-2 solve of group 0 (assemble<Ensemble<32>> + apply_dirichlet + 32 x
pcg_solve<double> on extract_component, tol 1e-6) timed in full on one host
core, against the bounded sample bench.py uses (full assembly + 2 scalar
iterations per sample, scaled to the reference's total iteration count).
The extraction (extract_component, a strided read of the whole ensemble matrix
per sample) is timed separately and counted once per sample, not per iteration.
Writes profiles/round2/ref_extrapolation.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402


def main():
    total_it = bench.ref_uncoupled_iterations()
    t0 = time.perf_counter()
    full = bench.ref_group_sample(0, 10000)  # runs to convergence: (t_asm, s per iteration)
    wall = time.perf_counter() - t0
    t_asm_full, per_it_full = full
    full_s = t_asm_full + per_it_full * total_it
    samp = bench.ref_group_sample(0, bench.REF_SAMPLE_ITERS)
    extrap_s = samp[0] + samp[1] * total_it
    out = {"workload": "cfg2 group 0: 64^3, s=32, uncoupled (32 x pcg_solve<double>), 1 core",
           "host": bench.host_facts(), "total_scalar_iterations": total_it,
           "full_solve_s": round(full_s, 3), "full_wall_s": round(wall, 3),
           "extrapolated_s": round(extrap_s, 3), "ratio_extrapolated_over_full": round(extrap_s / full_s, 4),
           "sample": f"full assembly + 32 extractions + 32 x {bench.REF_SAMPLE_ITERS} scalar iterations, "
                     "per-iteration time x total iterations"}
    os.makedirs(os.path.join(ROOT, "profiles", "round2"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "round2", "ref_extrapolation.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
