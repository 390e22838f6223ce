"""Reference fixtures at the BASELINE cfg-2 size (64^3 mesh, s = 32, KL m = 3,
sigma = 0.1, seed 0, group 0, tol 1e-6): tests/golden/cfg2_64_s32.npz.

Run here (where /root/reference exists):
    make -C oracle && python tests/golden/make_cfg2.py
It records, per sample e of the group:
  * the UNMODIFIED reference's uncoupled solve -- s x pcg_solve<double> on the
    extracted components (src/bench.cpp:340-349) of the reference's own
    assemble<Ensemble<32>> + apply_dirichlet system (oracle/_ref) -- its
    iteration count, residual history and the SHA-256 of the solution bytes;
  * the same for the C restatement's canonical-order uncoupled solve
    (oracle/enprop_oracle.c, DOT_CANONICAL, segments = mesh planes), the order
    of ENPROP_DOT_CANONICAL;
  * SHA-256 of the reference's assembled values / residual and wall times
    (assembly, the full uncoupled solve) that pin bench.py's extrapolated
    reference timing (bench.py run_reference).
The solution vectors themselves (70 MB) are not committed; hashes pin them.
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracles import CG_UNCOUPLED, DOT_CANONICAL, Oracle, RefLib, pack_group  # noqa: E402

N, S, M, SIGMA, TOL, MAXIT = 64, 32, 3, 0.1, 1e-6, 10000


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    R, O = RefLib(), Oracle()
    y = pack_group(R.draw_samples(0, S, M), S)
    t0 = time.perf_counter()
    vals, res = R.assemble(S, N, M, y, sigma=SIGMA, dirichlet=True)
    t_asm = time.perf_counter() - t0
    rm, ce = R.graph(N)
    b = -res
    rows = len(rm) - 1
    its = np.zeros(S, np.int32)
    hist = np.full((S, 400), np.nan)
    xs = []
    t0 = time.perf_counter()
    for e in range(S):
        v = np.ascontiguousarray(vals[:, e])
        be = np.ascontiguousarray(b[:, e])
        out = R.pcg(1, rm, ce, v, be, TOL, MAXIT, scalar=True)
        assert out["status"] == 0, out["status"]
        its[e] = out["iterations"]
        hl = len(out["history"])
        hist[e, :hl] = out["history"]
        xs.append(sha(out["x"].reshape(rows)))
        print(f"ref sample {e}: {its[e]} iterations", flush=True)
    t_solve = time.perf_counter() - t0
    # canonical order (C restatement), uncoupled, segments = planes
    f = O.kl(M, 1.0, SIGMA, 1.0)
    ov, orr = O.assemble(S, N, f, y, dirichlet=True)
    assert sha(ov) == sha(vals) and sha(orr) == sha(res), "oracle assembly != reference assembly"
    t0 = time.perf_counter()
    oc = O.pcg(S, rm, ce, ov, -orr, TOL, MAXIT, flavour=CG_UNCOUPLED, mode=DOT_CANONICAL, seg=(N + 1) ** 2)
    t_canon = time.perf_counter() - t0
    chist = np.full((S, 400), np.nan)
    for e in range(S):
        hl = oc["hist_len"][e]
        chist[e, :hl] = oc["history"][:hl, e]
    np.savez_compressed(
        os.path.join(HERE, "cfg2_64_s32.npz"),
        ref_iterations=its, ref_history=hist, ref_x_sha=np.array(xs),
        canon_iterations=oc["iterations"].astype(np.int32), canon_history=chist,
        canon_x_sha=np.array([sha(np.ascontiguousarray(oc["x"][:, e])) for e in range(S)]),
        values_sha=np.array([sha(vals)]), residual_sha=np.array([sha(res)]),
        ref_seconds=np.array([t_asm, t_solve]), canon_seconds=np.array([t_canon]),
        config=np.array([N, S, M, 0, 0]), sigma=np.array([SIGMA]), tol=np.array([TOL]))
    print(f"assembly {t_asm:.2f} s, reference uncoupled solve {t_solve:.1f} s, canonical oracle {t_canon:.1f} s")
    print("iterations ref", its.tolist())
    print("iterations canonical", oc["iterations"].tolist())


if __name__ == "__main__":
    main()
