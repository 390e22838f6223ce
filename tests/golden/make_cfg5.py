"""Reference fixtures at the BASELINE cfg-5 size (128^3 mesh, s = 32, KL
m = 10, sigma = 0.25, seed 0, group 0, tol 1e-6): tests/golden/cfg5_128_s32.npz.

Run here (where /root/reference exists; ~30 GB of RAM, ~25 min on 8 cores):
    make -C oracle && python tests/golden/make_cfg5.py [--canonical]
It records, for the group's ensemble system assembled by the UNMODIFIED
reference (assemble<Ensemble<32>> + apply_dirichlet, oracle/_ref):
  * the reference's uncoupled solve -- s x pcg_solve<double> on the extracted
    components (src/bench.cpp:340-349): per sample the iteration count,
    residual history and SHA-256 of the solution bytes;
  * the reference's coupled solve pcg_solve<Ensemble<32>>: iterations, history,
    solution SHA-256;
  * with --canonical only: the C restatement's canonical-order solves
    (oracle/enprop_oracle.c, DOT_CANONICAL, segments = mesh planes), coupled
    and uncoupled. The restatement takes ~37 s per iteration at this size
    (~3 h per solve), so the committed fixture omits them. cfg 2 pins the
    canonical order at full size;
  * SHA-256 of the assembled values / residual (the restatement's assembly is
    checked equal to the reference's here).
Solutions (550 MB each) are not committed; hashes pin them. The solves run in
forked workers sharing the assembled values.
"""
import hashlib
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracles import CG_COUPLED, CG_UNCOUPLED, DOT_CANONICAL, Oracle, RefLib, pack_group  # noqa: E402

N, S, M, SIGMA, TOL, MAXIT, HMAX = 128, 32, 10, 0.25, 1e-6, 10000, 1000
G = {}  # assembled system, inherited by the forked workers


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def task(job):
    kind, e = job
    rm, ce, vals, b = G["rm"], G["ce"], G["vals"], G["b"]
    t0 = time.perf_counter()
    if kind == "ref_scalar":
        out = RefLib().pcg(1, rm, ce, np.ascontiguousarray(vals[:, e]), np.ascontiguousarray(b[:, e]), TOL, MAXIT,
                           scalar=True)
        assert out["status"] == 0, out["status"]
        r = dict(it=[int(out["iterations"])], hist=[out["history"]], x=[sha(out["x"])])
    elif kind == "ref_coupled":
        out = RefLib().pcg(S, rm, ce, vals, b, TOL, MAXIT)
        assert out["status"] == 0, out["status"]
        r = dict(it=[int(out["iterations"])], hist=[out["history"]], x=[sha(out["x"])])
    else:
        fl = CG_COUPLED if kind == "canon_coupled" else CG_UNCOUPLED
        oc = Oracle().pcg(S, rm, ce, vals, b, TOL, MAXIT, flavour=fl, mode=DOT_CANONICAL, seg=(N + 1) ** 2)
        assert oc["status"] == 0, oc["status"]
        lanes = S if fl == CG_UNCOUPLED else 1
        r = dict(it=[int(v) for v in oc["iterations"]],
                 hist=[oc["history"][:oc["hist_len"][l], l] for l in range(lanes)],
                 x=[sha(np.ascontiguousarray(oc["x"][:, e2])) for e2 in range(S)])
    print(f"{kind} {e}: iterations {r['it'][:4]} ({time.perf_counter() - t0:.0f} s)", flush=True)
    return kind, e, r


def main():
    R, O = RefLib(), Oracle()
    y = pack_group(R.draw_samples(0, S, M), S)
    t0 = time.perf_counter()
    vals, res = R.assemble(S, N, M, y, sigma=SIGMA, dirichlet=True)
    t_asm = time.perf_counter() - t0
    vsha, rsha = sha(vals), sha(res)
    ov, orr = O.assemble(S, N, O.kl(M, 1.0, SIGMA, 1.0), y, dirichlet=True)
    assert sha(ov) == vsha and sha(orr) == rsha, "oracle assembly != reference assembly"
    del ov, orr
    rm, ce = R.graph(N)
    G.update(rm=rm, ce=ce, vals=vals, b=-res)
    print(f"assembly {t_asm:.1f} s; solving", flush=True)
    canonical = "--canonical" in sys.argv[1:]
    jobs = [("ref_coupled", 0)] + ([("canon_coupled", 0), ("canon_uncoupled", 0)] if canonical else [])
    jobs += [("ref_scalar", e) for e in range(S)]
    with mp.get_context("fork").Pool(min(os.cpu_count() or 1, 8)) as pool:
        done = pool.map(task, jobs, chunksize=1)
    out = {(k, e): r for k, e, r in done}

    def hist_rows(hs):
        h = np.full((len(hs), HMAX), np.nan)
        for i, v in enumerate(hs):
            h[i, :len(v)] = v[:HMAX]
        return h

    ref_it = np.array([out[("ref_scalar", e)]["it"][0] for e in range(S)], np.int32)
    extra = {}
    if canonical:
        extra = dict(canon_iterations=np.array(out[("canon_uncoupled", 0)]["it"], np.int32),
                     canon_x_sha=np.array(out[("canon_uncoupled", 0)]["x"]),
                     canon_coupled_iterations=np.array(out[("canon_coupled", 0)]["it"], np.int32),
                     canon_coupled_x_sha=np.array(out[("canon_coupled", 0)]["x"]))
    np.savez_compressed(
        os.path.join(HERE, "cfg5_128_s32.npz"),
        ref_iterations=ref_it,
        ref_history=hist_rows([out[("ref_scalar", e)]["hist"][0][:ref_it[e] + 1] for e in range(S)]),
        ref_x_sha=np.array([out[("ref_scalar", e)]["x"][0] for e in range(S)]),
        ref_coupled_iterations=np.array(out[("ref_coupled", 0)]["it"], np.int32),
        ref_coupled_history=hist_rows([out[("ref_coupled", 0)]["hist"][0][:out[("ref_coupled", 0)]["it"][0] + 1]]),
        ref_coupled_x_sha=np.array(out[("ref_coupled", 0)]["x"]),
        values_sha=np.array([vsha]), residual_sha=np.array([rsha]), ref_seconds=np.array([t_asm]),
        config=np.array([N, S, M]), sigma=np.array([SIGMA]), tol=np.array([TOL]), **extra)
    print("iterations ref", ref_it.tolist())
    print("coupled ref", out[("ref_coupled", 0)]["it"])


if __name__ == "__main__":
    main()
