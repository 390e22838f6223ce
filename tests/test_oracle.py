"""CPU tests: the C oracle (oracle/enprop_oracle.c) is pinned to the reference.

1. against the committed golden vectors made by the unmodified reference
   (tests/golden/make_golden.py) — runs anywhere;
2. against the reference itself (oracle/_ref/libenprop_ref.so, built from
   /root/reference sources by oracle/Makefile) on more cases, when present.
"""
import os

import numpy as np
import pytest

from oracles import (CG_COUPLED, CG_UNCOUPLED, DOT_CANONICAL, DOT_SERIAL, REF_SO, TILE_ROWS, Oracle,
                     RefLib, bits, pack_group)

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))
O = Oracle()
HAVE_REF = os.path.exists(REF_SO)
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and (bits(a.astype(np.float64)) == bits(b.astype(np.float64))).all()


# ----------------------------------------------------------------- golden vectors
@pytest.mark.parametrize("n", [1, 2, 3])
def test_graph_golden(n):
    rm, ce = O.graph(n)
    assert (rm == GOLD[f"graph{n}_row_map"]).all()
    assert (ce == GOLD[f"graph{n}_col_entry"]).all()


def test_graph_known_answers():
    # test_mesh_fem.cpp:103-114: interior rows 27 entries, corner rows 8
    rm, ce = O.graph(4)
    N = 5
    interior = 2 + N * (2 + N * 2)
    assert rm[interior + 1] - rm[interior] == 27
    assert rm[1] - rm[0] == 8
    # columns strictly increasing in every row (crs.hpp:64-65)
    for r in range(N ** 3):
        row = ce[rm[r]:rm[r + 1]]
        assert (np.diff(row) > 0).all()


def test_samples_golden():
    assert same(O.draw_samples(0, 8, 5), GOLD["samples_seed0"])
    assert same(O.draw_samples(515, 4, 5), GOLD["samples_seed515"])


@pytest.mark.parametrize("m,sig", [(5, 0.2), (10, 0.25)])
def test_kl_golden(m, sig):
    f = O.kl(m, 1.0, sig, 1.0)
    assert same(np.array(f.axis_freq[:m]), GOLD[f"kl{m}_axis_freq"])
    assert same(np.array(f.axis_eig[:m]), GOLD[f"kl{m}_axis_eig"])
    assert same(np.array(f.axis_invnorm[:m]), GOLD[f"kl{m}_axis_invnorm"])
    assert same(np.array(f.mode_eig[:m]), GOLD[f"kl{m}_mode_eig"])
    axes = np.array([[f.mode_axes[i][k] for k in range(3)] for i in range(m)])
    assert (axes == GOLD[f"kl{m}_mode_axes"]).all()


def test_assembly_golden_linear():
    f = O.kl(5, 1.0, 0.2, 1.0)
    v, r = O.assemble(2, 3, f, GOLD["asm_y"], dirichlet=True)
    assert same(v, GOLD["asm_lin_values"]) and same(r, GOLD["asm_lin_residual"])


@pytest.mark.parametrize("dirichlet", [False, True])
def test_assembly_golden_nonlinear(dirichlet):
    f = O.kl(5, 1.0, 0.2, 1.0)
    v, r = O.assemble(2, 3, f, GOLD["asm_y"], u=GOLD["asm_u"], alpha=0.3, beta=0.7,
                      velocity=(1.0, 0.5, -0.25), dirichlet=dirichlet)
    tag = "nld" if dirichlet else "nl"
    assert same(v, GOLD[f"asm_{tag}_values"]) and same(r, GOLD[f"asm_{tag}_residual"])


def test_spmv_dot_golden():
    rm, ce = O.graph(3)
    z = O.spmv(2, rm, ce, GOLD["asm_lin_values"], GOLD["spmv_x"])
    assert same(z, GOLD["spmv_z"])
    assert O.dot(2, GOLD["spmv_x"], z) == GOLD["dot_uv"][0]


def test_pcg_golden_coupled_and_uncoupled():
    rm, ce = O.graph(4)
    v, b = GOLD["cg_values"], GOLD["cg_b"]
    c = O.pcg(2, rm, ce, v, b, 1e-6, 1000, flavour=CG_COUPLED, mode=DOT_SERIAL)
    assert c["status"] == 0 and c["iterations"][0] == GOLD["cg_coupled_it"][0]
    assert same(c["x"], GOLD["cg_coupled_x"])
    assert same(c["history"][:c["hist_len"][0], 0], GOLD["cg_coupled_hist"])
    u = O.pcg(2, rm, ce, v, b, 1e-6, 1000, flavour=CG_UNCOUPLED, mode=DOT_SERIAL)
    assert (u["iterations"] == GOLD["cg_uncoupled_it"]).all()
    assert same(u["x"], GOLD["cg_uncoupled_x"])
    for e in range(2):
        assert same(u["history"][:u["hist_len"][e], e], GOLD[f"cg_uncoupled_hist{e}"])


# --------------------------------------------------------- canonical order itself
def fold(t):
    t = t.copy()
    h = len(t) // 2
    while h >= 1:
        t[:h] = t[:h] + t[h:2 * h]
        h //= 2
    return t[0]


def canonical_lane(u, v, seg, e):
    """The canonical order in numpy: tiles of TILE_ROWS rows,
    blocks of 16 tiles, both stride-halving folds with +0.0 padding; segment
    and total sums sequential."""
    n = u.shape[0]
    total = 0.0
    for r0 in range(0, n, seg):
        r1 = min(r0 + seg, n)
        sg = 0.0
        for b0 in range(r0, r1, 16 * TILE_ROWS):
            blk = np.zeros(16)
            for k in range(16):
                t0 = b0 + k * TILE_ROWS
                if t0 >= r1:
                    continue
                t = np.zeros(TILE_ROWS)
                m = min(TILE_ROWS, r1 - t0)
                t[:m] = u[t0:t0 + m, e] * v[t0:t0 + m, e]
                blk[k] = fold(t)
            sg = sg + fold(blk)
        total = total + sg
    return total


def test_canonical_dot_definition():
    """The canonical order restated in numpy agrees with the C oracle."""
    rng = np.random.default_rng(5)
    for n, seg in ((1, 7), (200, 64), (1000, 137), (4225, 4225), (9000, 4225)):
        u = rng.uniform(-1, 1, (n, 4))
        v = rng.uniform(-1, 1, (n, 4))
        lanes = O.dot_lanes(4, u, v, DOT_CANONICAL, TILE_ROWS, seg)
        for e in range(4):
            assert canonical_lane(u, v, seg, e) == lanes[e]


def test_serial_dot_is_sequential():
    rng = np.random.default_rng(6)
    u = rng.uniform(-1, 1, (333, 2))
    v = rng.uniform(-1, 1, (333, 2))
    lanes = O.dot_lanes(2, u, v, DOT_SERIAL)
    for e in range(2):
        acc = 0.0
        for r in range(333):
            acc = acc + u[r, e] * v[r, e]
        assert acc == lanes[e]


# -------------------------------------------------------- against the reference
@needs_ref
@pytest.mark.parametrize("s", [1, 2, 4, 8, 16, 32])
def test_oracle_matches_reference_assembly(s):
    R = RefLib()
    n, m = 3, 5
    rng = np.random.default_rng(100 + s)
    y = rng.uniform(-1, 1, (m, s))
    u = rng.uniform(-1, 1, ((n + 1) ** 3, s))
    f = O.kl(m, 1.0, 0.2, 1.0)
    for kw in (dict(), dict(u=u, alpha=0.25, beta=0.5)):
        for d in (False, True):
            v1, r1 = O.assemble(s, n, f, y, dirichlet=d, **kw)
            v2, r2 = R.assemble(s, n, m, y, sigma=0.2, dirichlet=d, **kw)
            assert same(v1, v2) and same(r1, r2)


@needs_ref
def test_oracle_matches_reference_graph_and_pairs():
    R = RefLib()
    for n in (4, 7, 16):
        a, b = O.graph(n), R.graph(n)
        assert (a[0] == b[0]).all() and (a[1] == b[1]).all()


@needs_ref
@pytest.mark.parametrize("s", [1, 4, 16])
def test_oracle_matches_reference_cg(s):
    R = RefLib()
    n, m = 6, 3
    y = pack_group(R.draw_samples(0, s, m), s)
    v, r = R.assemble(s, n, m, y)
    b = -r
    rm, ce = R.graph(n)
    ref = R.pcg(s, rm, ce, v, b, 1e-8, 1000)
    o = O.pcg(s, rm, ce, v, b, 1e-8, 1000)
    assert o["iterations"][0] == ref["iterations"]
    assert same(o["x"], ref["x"])
    assert same(o["history"][:o["hist_len"][0], 0], ref["history"])
    un = R.pcg_uncoupled(s, rm, ce, v, b, 1e-8, 1000)
    ou = O.pcg(s, rm, ce, v, b, 1e-8, 1000, flavour=CG_UNCOUPLED)
    for e in range(s):
        assert ou["iterations"][e] == un[e]["iterations"]
        assert same(ou["x"][:, e], un[e]["x"][:, 0])


@needs_ref
def test_oracle_matches_reference_cg_failures():
    R = RefLib()
    # iteration exhaustion carries the history (test_pcg.cpp:164-179)
    rng = np.random.default_rng(3)
    n = 40
    A = np.diag(np.linspace(1, 100, n))
    rm = np.arange(n + 1, dtype=np.int32)
    ce = np.arange(n, dtype=np.int32)
    vals = np.ascontiguousarray(np.diag(A)).reshape(n, 1)
    b = rng.uniform(-1, 1, (n, 1))
    ref = R.pcg(1, rm, ce, vals, b, 1e-15, 2, scalar=True)
    o = O.pcg(1, rm, ce, vals, b, 1e-15, 2)
    assert ref["status"] == 2 and o["status"] == 2
    assert len(ref["history"]) == 3 and o["hist_len"][0] == 3
    assert same(o["history"][:3, 0], ref["history"])
    # indefinite operator (test_pcg.cpp:181-190)
    vals2 = np.array([[1.0], [-1.0]])
    rm2 = np.array([0, 1, 2], np.int32)
    ce2 = np.array([0, 1], np.int32)
    b2 = np.array([[0.0], [1.0]])
    assert R.pcg(1, rm2, ce2, vals2, b2, 1e-8, 100, scalar=True)["status"] == 3
    assert O.pcg(1, rm2, ce2, vals2, b2, 1e-8, 100)["status"] == 3


def _random_crs(rng, rows, cols, density):
    """testutil::random_crs (tests/oracles.hpp:25-34): per-coordinate Bernoulli."""
    mask = rng.uniform(0, 1, (rows, cols)) < density
    rm = np.zeros(rows + 1, np.int32)
    rm[1:] = np.cumsum(mask.sum(axis=1))
    return rm, np.nonzero(mask)[1].astype(np.int32)


@needs_ref
@pytest.mark.parametrize("s", [1, 3, 4, 32])
def test_spmv_outer_oracle_equals_reference(s):
    """or_spmv_outer (the C restatement of kernels.hpp:38-56) == the reference's
    spmv_outer bitwise, and each component == the scalar spmv of that component
    (test_kernels.cpp:127-143)."""
    R = RefLib()
    rng = np.random.default_rng(3 + s)
    for trial in range(10):
        rows, cols = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        rm, ce = _random_crs(rng, rows, cols, 0.15)
        nnz = len(ce)
        vals = rng.uniform(-1, 1, (s, nnz))
        x = rng.uniform(-1, 1, (s, cols))
        zr = R.spmv_outer(s, rm, ce, vals, x, cols)
        zo = O.spmv_outer(s, rm, ce, vals, x, cols)
        assert same(zr, zo)
        for e in range(s):
            ze = R.spmv(1, rm, ce, np.ascontiguousarray(vals[e][:, None]), np.ascontiguousarray(x[e][:, None]), cols)
            assert same(ze[:, 0], zr[e])


@needs_ref
def test_newton_identity_oracle_properties():
    """The reference-composed Newton (fem.hpp:265-302 with the identity
    preconditioner, oracle/ref_capi.cpp) on test_mesh_fem.cpp:240-258's
    reaction-diffusion case: 2..6 steps, residual down by 1e-8, iterate in the
    boundary band; and one step on the linear problem with the exact 1 - x
    profile (test_mesh_fem.cpp:220-237)."""
    R = RefLib()
    y = O.draw_samples(19, 1, 5).reshape(5, 1)
    rc, u, its, cg, norms = R.newton_identity(1, 4, 5, y, sigma=0.2, beta=1.0)
    assert rc == 0 and 2 <= its <= 6 and cg > 0
    assert norms[-1] < 1e-8 * norms[0]
    assert (u > -0.05).all() and (u < 1.05).all()
    for n in (2, 4):
        rc, u, its, cg, norms = R.newton_identity(1, n, 1, np.zeros((1, 1)), sigma=0.0, lin_tol=1e-13)
        assert rc == 0 and its == 1
        N = n + 1
        x = (np.arange(N ** 3) % N) / n
        assert np.abs(u[:, 0] - (1 - x)).max() < 1e-10
