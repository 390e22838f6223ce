"""Regenerate tests/golden/reference_golden.npz from the UNMODIFIED reference.

Run here (where /root/reference exists):  make -C oracle && python tests/golden/make_golden.py
The reference is executed through oracle/_ref/libenprop_ref.so (oracle/ref_capi.cpp
forwards to proj/include/enprop templates).  The fixtures are small on purpose;
they pin the oracle and the GPU path on boxes without /root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracles import RefLib, pack_group  # noqa: E402


def main():
    R = RefLib()
    g = {}
    # mesh.cpp:13-55
    for n in (1, 2, 3):
        rm, ce = R.graph(n)
        g[f"graph{n}_row_map"], g[f"graph{n}_col_entry"] = rm, ce
    g["entry_of_pair2"] = R.entry_of_pair(2)
    # samples.cpp:7-18
    g["samples_seed0"] = R.draw_samples(0, 8, 5)
    g["samples_seed515"] = R.draw_samples(515, 4, 5)
    # kl.cpp:41-89
    for m, sig in ((5, 0.2), (10, 0.25)):
        d = R.kl_describe(m, 1.0, sig, 1.0)
        for k, v in d.items():
            g[f"kl{m}_{k}"] = v
    # fem.hpp:115-243 — linear (bench path) and nonlinear with u
    n, s, m = 3, 2, 5
    y = pack_group(R.draw_samples(7, s, m), s)
    g["asm_y"] = y
    v, r = R.assemble(s, n, m, y, sigma=0.2, dirichlet=True)
    g["asm_lin_values"], g["asm_lin_residual"] = v, r
    rng = np.random.default_rng(11)
    u = rng.uniform(-1, 1, ((n + 1) ** 3, s))
    g["asm_u"] = u
    v, r = R.assemble(s, n, m, y, sigma=0.2, u=u, alpha=0.3, beta=0.7, velocity=(1.0, 0.5, -0.25),
                      dirichlet=False)
    g["asm_nl_values"], g["asm_nl_residual"] = v, r
    v, r = R.assemble(s, n, m, y, sigma=0.2, u=u, alpha=0.3, beta=0.7, velocity=(1.0, 0.5, -0.25),
                      dirichlet=True)
    g["asm_nld_values"], g["asm_nld_residual"] = v, r
    # kernels.hpp:15-26 on the assembled matrix, random x
    rm, ce = R.graph(n)
    x = rng.uniform(-1, 1, ((n + 1) ** 3, s))
    g["spmv_x"] = x
    g["spmv_z"] = R.spmv(s, rm, ce, g["asm_lin_values"], x)
    g["dot_uv"] = np.array([R.dot(s, x, g["spmv_z"])])
    # pcg.hpp:52-103 on the n=4 bench problem, s=2, m=3, tol 1e-6
    n, s, m = 4, 2, 3
    y = pack_group(R.draw_samples(0, s, m), s)
    v, r = R.assemble(s, n, m, y)
    b = -r
    rm, ce = R.graph(n)
    g["cg_values"], g["cg_b"] = v, b
    res = R.pcg(s, rm, ce, v, b, 1e-6, 1000)
    g["cg_coupled_x"], g["cg_coupled_hist"] = res["x"], res["history"]
    g["cg_coupled_it"] = np.array([res["iterations"]])
    un = R.pcg_uncoupled(s, rm, ce, v, b, 1e-6, 1000)
    g["cg_uncoupled_x"] = np.stack([u_["x"][:, 0] for u_ in un], axis=1)
    g["cg_uncoupled_it"] = np.array([u_["iterations"] for u_ in un])
    for e, u_ in enumerate(un):
        g[f"cg_uncoupled_hist{e}"] = u_["history"]
    out = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(out, **g)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
