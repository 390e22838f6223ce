"""GPU parity: the CUDA path (through the C ABI) against the reference.

Checkers: oracle/_ref/libenprop_ref.so (the unmodified reference, prebuilt) and
oracle/liboracle.so (the C restatement, itself pinned in test_oracle.py).
Bar: graph/indices bit-exact; assembly, Dirichlet, SpMV, axpby bitwise;
dots and CG bitwise in the reference's serial order, and bitwise against the
restatement in the canonical order. Cases mirror the reference suites
(test_kernels.cpp, test_mesh_fem.cpp, test_pcg.cpp, acceptance.cpp:46-115).
"""
import math

import numpy as np
import pytest
import torch

import paper_1511_03703_b200 as ep
from oracles import (CG_COUPLED, CG_UNCOUPLED, DOT_CANONICAL, DOT_SERIAL, TILE_ROWS, Oracle, RefLib,
                     bits, pack_group)

pytestmark = pytest.mark.gpu
WIDTHS = (1, 2, 4, 8, 16, 32)
O = Oracle()


@pytest.fixture(scope="module")
def R():
    return RefLib()


@pytest.fixture(scope="module")
def ctx():
    c = ep.Context(0)
    yield c
    c.close()


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def same(a, b):
    a, b = np.ascontiguousarray(a, dtype=np.float64), np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and (bits(a) == bits(b)).all()


def random_crs(rng, rows, cols, density):
    """testutil::random_crs (tests/oracles.hpp:25-34): per-coordinate Bernoulli."""
    mask = rng.uniform(0, 1, (rows, cols)) < density
    rm = np.zeros(rows + 1, np.int32)
    rm[1:] = np.cumsum(mask.sum(axis=1))
    ce = np.nonzero(mask)[1].astype(np.int32)
    return rm, ce


# ------------------------------------------------------------------ mesh graph
@pytest.mark.parametrize("n", [1, 2, 3, 8, 17, 64])
def test_node_graph_bit_exact(ctx, n):
    rm, ce = ep.build_node_graph(ctx, n)
    orm, oce = O.graph(n)
    assert (host(rm) == orm).all() and (host(ce) == oce).all()


# ------------------------------------------------------------------- assembly
@pytest.mark.parametrize("s", WIDTHS)
@pytest.mark.parametrize("n", [1, 3, 8])
def test_assembly_linear_dirichlet_bitwise(ctx, R, s, n):
    m = 5
    y = pack_group(R.draw_samples(515, s, m), s)
    rm, _ = ep.build_node_graph(ctx, n)
    kl = ep.KlField(m, 1.0, 0.1, 1.0)
    v, r = ep.assemble(ctx, s, n, kl, dev(y), rm, bc=ep.DirichletBc())
    rv, rr = R.assemble(s, n, m, y, sigma=0.1, dirichlet=True)
    assert same(host(v), rv) and same(host(r), rr)


@pytest.mark.parametrize("s", WIDTHS)
def test_assembly_nonlinear_with_u_bitwise(ctx, R, s):
    """acceptance.cpp:86-115: alpha, beta != 0 and a random iterate u."""
    n, m = 3, 5
    rng = np.random.default_rng(200 + s)
    y = rng.uniform(-1, 1, (m, s))
    u = rng.uniform(-1, 1, ((n + 1) ** 3, s))
    rm, ce = ep.build_node_graph(ctx, n)
    kl = ep.KlField(m, 1.0, 0.2, 1.0)
    co = ep.PdeCoefficients(0.3, 0.7, (1.0, 0.5, -0.25))
    for d in (False, True):
        v, r = ep.assemble(ctx, s, n, kl, dev(y), rm, coeffs=co, u=dev(u),
                           bc=ep.DirichletBc() if d else None)
        rv, rr = R.assemble(s, n, m, y, sigma=0.2, u=u, alpha=0.3, beta=0.7,
                            velocity=(1.0, 0.5, -0.25), dirichlet=d)
        assert same(host(v), rv), f"values differ (dirichlet={d})"
        assert same(host(r), rr), f"residual differs (dirichlet={d})"


@pytest.mark.parametrize("s", [1, 4, 32])
def test_apply_dirichlet_standalone_equals_fused(ctx, R, s):
    n, m = 4, 3
    rng = np.random.default_rng(7)
    y = rng.uniform(-1, 1, (m, s))
    u = rng.uniform(-1, 1, ((n + 1) ** 3, s))
    rm, ce = ep.build_node_graph(ctx, n)
    kl = ep.KlField(m, 1.0, 0.25, 1.0)
    bc = ep.DirichletBc(0.75, -0.5)
    v, r = ep.assemble(ctx, s, n, kl, dev(y), rm, u=dev(u))
    ep.apply_dirichlet(ctx, s, n, bc, rm, ce, v, r, u=dev(u))
    rv, rr = R.assemble(s, n, m, y, sigma=0.25, u=u, dirichlet=True, bc=(0.75, -0.5))
    assert same(host(v), rv) and same(host(r), rr)


def test_assembly_rejects_mismatched_lengths(ctx):
    rm, _ = ep.build_node_graph(ctx, 2)
    kl = ep.KlField(1, 1.0, 0.0, 1.0)
    with pytest.raises(ValueError):
        ep.assemble(ctx, 1, 2, kl, dev(np.zeros(2)), rm)
    with pytest.raises(ValueError):
        ep.assemble(ctx, 1, 2, kl, dev(np.zeros(1)), rm, u=dev(np.zeros(5)))


@pytest.mark.parametrize("s", [4, 32])
def test_ensemble_assembly_is_per_sample_scalar_assembly(ctx, s):
    """test_mesh_fem.cpp:260-294 / bench.cpp:250-269 at a mid size: each
    component of the fused assembly equals the s=1 assembly of that sample."""
    n, m = 24, 3
    rng = np.random.default_rng(31)
    y = rng.uniform(-1, 1, (m, s))
    rm, _ = ep.build_node_graph(ctx, n)
    kl = ep.KlField(m, 1.0, 0.1, 1.0)
    v, r = ep.assemble(ctx, s, n, kl, dev(y), rm, bc=ep.DirichletBc())
    vh, rh = host(v), host(r)
    for e in (0, s // 2, s - 1):
        v1, r1 = ep.assemble(ctx, 1, n, kl, dev(y[:, e:e + 1]), rm, bc=ep.DirichletBc())
        assert same(vh[:, e:e + 1], host(v1)) and same(rh[:, e:e + 1], host(r1))


def test_assembled_matrix_is_exactly_symmetric(ctx):
    """a_ij == a_ji bitwise (G_qij == G_qji; Dirichlet keeps symmetry)."""
    n, s = 12, 8
    rm, ce = ep.build_node_graph(ctx, n)
    y = np.random.default_rng(2).uniform(-1, 1, (3, s))
    v, _ = ep.assemble(ctx, s, n, ep.KlField(3, 1.0, 0.1, 1.0), dev(y), rm, bc=ep.DirichletBc())
    rmh, ceh, vh = host(rm), host(ce), host(v)
    rows = np.repeat(np.arange(len(rmh) - 1), np.diff(rmh))
    key = {(int(a), int(b)): k for k, (a, b) in enumerate(zip(rows, ceh))}
    t = np.array([key[(int(b), int(a))] for a, b in zip(rows, ceh)])
    assert same(vh, vh[t])


# ------------------------------------------------------------------------ SpMV
@pytest.mark.parametrize("s", WIDTHS)
def test_spmv_random_crs_bitwise(ctx, R, s):
    """test_kernels.cpp:120-125 / acceptance.cpp:46-66: random shapes, empty rows."""
    rng = np.random.default_rng(771420 + s)
    for trial in range(12):
        rows, cols = int(rng.integers(1, 61)), int(rng.integers(1, 61))
        rm, ce = random_crs(rng, rows, cols, 0.15)
        vals = rng.uniform(-1, 1, (len(ce), s))
        x = rng.uniform(-1, 1, (cols, s))
        z = ep.spmv(ctx, s, dev(rm, torch.int32), dev(ce, torch.int32), dev(vals), dev(x),
                    num_cols=cols)
        assert same(host(z), R.spmv(s, rm, ce, vals, x, cols=cols))


@pytest.mark.parametrize("s", WIDTHS)
def test_spmv_crs_200_bitwise(ctx, R, s):
    rng = np.random.default_rng(515 + s)
    rm, ce = random_crs(rng, 200, 200, 0.05)
    vals = rng.uniform(-1, 1, (len(ce), s))
    x = rng.uniform(-1, 1, (200, s))
    z = ep.spmv(ctx, s, dev(rm, torch.int32), dev(ce, torch.int32), dev(vals), dev(x))
    assert same(host(z), R.spmv(s, rm, ce, vals, x))


@pytest.mark.parametrize("s", WIDTHS)
def test_spmv_mesh_matrix_bitwise(ctx, R, s):
    n, m = 16, 3
    y = pack_group(R.draw_samples(0, s, m), s)
    rm, ce = ep.build_node_graph(ctx, n)
    v, _ = ep.assemble(ctx, s, n, ep.KlField(m, 1.0, 0.1, 1.0), dev(y), rm, bc=ep.DirichletBc())
    x = np.random.default_rng(9).uniform(-1, 1, ((n + 1) ** 3, s))
    z = ep.spmv(ctx, s, rm, ce, v, dev(x))
    assert same(host(z), O.spmv(s, host(rm), host(ce), host(v), x))


@pytest.mark.parametrize("s", WIDTHS)
def test_spmv_dense_rows_bitwise(ctx, R, s):
    """Row blocks whose entries exceed the kernels' shared-memory staging
    capacity (100-entry rows) take the direct-read path: still bitwise."""
    rng = np.random.default_rng(4242 + s)
    rows, cols = 300, 100
    rm, ce = random_crs(rng, rows, cols, 1.0)
    vals = rng.uniform(-1, 1, (len(ce), s))
    x = rng.uniform(-1, 1, (cols, s))
    z = ep.spmv(ctx, s, dev(rm, torch.int32), dev(ce, torch.int32), dev(vals), dev(x), num_cols=cols)
    assert same(host(z), R.spmv(s, rm, ce, vals, x, cols=cols))


@pytest.mark.parametrize("mode", ["0", "2"])
def test_spmv_small_staging_modes_bitwise(mode):
    """The narrow-ensemble SpMV's A/B staging modes (ENPROP_SMALL_STAGE, read
    once per process; default 1 is covered above) stay bitwise: the SpMV
    parity cases rerun in a child process with the mode set."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, ENPROP_SMALL_STAGE=mode)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.join(here, "test_gpu_parity.py"),
                        "-k", "spmv and bitwise and not staging_modes"],
                       env=env, cwd=os.path.dirname(here), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    # the mode under test is the one that launches, at every width
    # and register cap it is routed with (no silent fallback to mode 1)
    probe = ("import paper_1511_03703_b200 as ep, json; "
             "print(json.dumps([ep.spmv_small_config(s) for s in (1, 2, 4, 8, 16)]))")
    for regs in ("", "0", "32", "48", "64"):
        env2 = dict(env, ENPROP_SMALL_REGS=regs)
        out = subprocess.run([sys.executable, "-c", probe], env=env2, cwd=os.path.dirname(here),
                             capture_output=True, text=True, timeout=120)
        import json
        cfgs = json.loads(out.stdout.strip().splitlines()[-1])
        assert all(c["stage_mode"] == int(mode) for c in cfgs), (regs, cfgs)


def test_spmv_rejects_bad_length(ctx):
    rm = dev(np.array([0, 1, 2, 3], np.int32), torch.int32)
    ce = dev(np.array([0, 1, 2], np.int32), torch.int32)
    with pytest.raises(ValueError):
        ep.spmv(ctx, 1, rm, ce, dev(np.ones(3)), dev(np.ones(2)))


# ------------------------------------------------------------- dots and axpby
@pytest.mark.parametrize("s", WIDTHS)
def test_dot_serial_equals_reference(ctx, R, s):
    """test_kernels.cpp:146-160: coupled dot exact."""
    rng = np.random.default_rng(40 + s)
    for n in (1, 17, 100, 5000, 70001):
        u, v = rng.uniform(-1, 1, (n, s)), rng.uniform(-1, 1, (n, s))
        lanes, coupled = ep.dot_lanes(ctx, s, dev(u), dev(v), ep.DOT_SERIAL)
        assert coupled == R.dot(s, u, v)
        assert lanes == list(O.dot_lanes(s, u, v, DOT_SERIAL))
        # operands 8 bytes off a 16-byte boundary take the register-chain
        # fallback (k_fin_serial) instead of the TMA-fed k_chain: same bits
        ub = torch.zeros(n * s + 1, dtype=torch.float64, device="cuda")
        ub[1:] = dev(u).reshape(-1)
        lanes2, coupled2 = ep.dot_lanes(ctx, s, ub[1:].view(n, s), dev(v), ep.DOT_SERIAL)
        assert ub[1:].data_ptr() % 16 == 8
        assert coupled2 == coupled and lanes2 == lanes


@pytest.mark.parametrize("s", WIDTHS)
def test_dot_canonical_equals_restatement(ctx, s):
    rng = np.random.default_rng(60 + s)
    for n, seg in ((1, 4096), (300, 64), (4225, 4225), (70001, 4225), (70001, 70001), (70001, 300)):
        u, v = rng.uniform(-1, 1, (n, s)), rng.uniform(-1, 1, (n, s))
        lanes, coupled = ep.dot_lanes(ctx, s, dev(u), dev(v), ep.DOT_CANONICAL, seg)
        assert lanes == list(O.dot_lanes(s, u, v, DOT_CANONICAL, TILE_ROWS, seg))
        assert coupled == O.dot(s, u, v, DOT_CANONICAL, TILE_ROWS, seg)
    z = np.zeros((10, s))
    assert ep.norm2(ctx, s, dev(z)) == 0.0


@pytest.mark.parametrize("s", [1, 3 - 1, 8, 32])
def test_axpby_both_coefficient_kinds(ctx, R, s):
    """test_kernels.cpp:169-192."""
    rng = np.random.default_rng(s)
    x, y0 = rng.uniform(-1, 1, (50, s)), rng.uniform(-1, 1, (50, s))
    y = dev(y0)
    ep.axpby(ctx, s, 2.5, dev(x), -0.75, y)
    assert same(host(y), R.axpby(s, 2.5, x, -0.75, y0))
    a, b = list(rng.uniform(-1, 1, s)), list(rng.uniform(-1, 1, s))
    y = dev(y0)
    ep.axpby(ctx, s, a, dev(x), b, y)
    assert same(host(y), R.axpby(s, a, x, b, y0, per_lane=True))


# -------------------------------------------------------------------------- CG
def mesh_system(R, s, n, m=3, sigma=0.1, seed=0):
    y = pack_group(R.draw_samples(seed, s, m), s)
    v, r = R.assemble(s, n, m, y, sigma=sigma)
    rm, ce = R.graph(n)
    return rm, ce, v, -r


@pytest.mark.parametrize("s", WIDTHS)
def test_cg_coupled_serial_is_reference_bitwise(ctx, R, s):
    n = 8
    rm, ce, v, b = mesh_system(R, s, n)
    cfg = ep.SolverConfig(tol=1e-8, max_iterations=1000, flavour=ep.CG_COUPLED, dot_mode=ep.DOT_SERIAL)
    res = ep.pcg_solve(ctx, s, dev(rm, torch.int32), dev(ce, torch.int32), dev(v), dev(b), cfg)
    ref = R.pcg(s, rm, ce, v, b, 1e-8, 1000)
    assert res.iterations == ref["iterations"]
    assert same(np.array(res.residual_history), ref["history"])
    assert same(host(res.solution), ref["x"])


@pytest.mark.parametrize("s", WIDTHS)
def test_cg_uncoupled_serial_is_per_sample_reference_bitwise(ctx, R, s):
    """Uncoupled = s x pcg_solve<double> on extracted components (bench.cpp:340-349):
    identical iteration counts and bitwise solutions per sample."""
    n = 8
    rm, ce, v, b = mesh_system(R, s, n, m=10, sigma=0.25, seed=4)
    cfg = ep.SolverConfig(tol=1e-6, max_iterations=1000, flavour=ep.CG_UNCOUPLED, dot_mode=ep.DOT_SERIAL)
    res = ep.pcg_solve(ctx, s, dev(rm, torch.int32), dev(ce, torch.int32), dev(v), dev(b), cfg)
    ref = R.pcg_uncoupled(s, rm, ce, v, b, 1e-6, 1000)
    x = host(res.solution)
    for e in range(s):
        assert res.iterations[e] == ref[e]["iterations"]
        assert same(np.array(res.residual_history[e]), ref[e]["history"])
        assert same(x[:, e], ref[e]["x"][:, 0])


@pytest.mark.parametrize("s", WIDTHS)
@pytest.mark.parametrize("flavour", [CG_COUPLED, CG_UNCOUPLED])
def test_cg_canonical_is_restatement_bitwise(ctx, R, s, flavour):
    n = 10
    seg = (n + 1) ** 2
    rm, ce, v, b = mesh_system(R, s, n, seed=2)
    cfg = ep.SolverConfig(tol=1e-7, max_iterations=1000, flavour=flavour, dot_mode=ep.DOT_CANONICAL,
                          seg_rows=seg)
    res = ep.pcg_solve(ctx, s, dev(rm, torch.int32), dev(ce, torch.int32), dev(v), dev(b), cfg)
    o = O.pcg(s, rm, ce, v, b, 1e-7, 1000, flavour=flavour, mode=DOT_CANONICAL, seg=seg)
    x = host(res.solution)
    assert same(x, o["x"])
    if flavour == CG_COUPLED:
        assert res.iterations == o["iterations"][0]
    else:
        assert list(res.iterations) == list(o["iterations"])
    # and within tolerance-level of the reference's serial-order solve
    ref = R.pcg(s, rm, ce, v, b, 1e-7, 1000)
    rel = np.abs(x - ref["x"]).max() / np.abs(ref["x"]).max()
    assert rel < 1e-4


def test_cg_identical_components_replicate_scalar(ctx, R):
    """test_pcg.cpp:101-121."""
    rng = np.random.default_rng(31)
    n = 40
    A = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1, n):
            if rng.uniform() < 0.15:
                A[i, j] = A[j, i] = rng.uniform(-1, 1)
    np.fill_diagonal(A, np.abs(A).sum(axis=1) + 1.0)
    rm = np.zeros(n + 1, np.int32)
    rm[1:] = np.cumsum((A != 0).sum(axis=1))
    ce = np.nonzero(A)[1].astype(np.int32)
    vals1 = A[A != 0].reshape(-1, 1)
    b1 = rng.uniform(-1, 1, (n, 1))
    scalar = R.pcg(1, rm, ce, vals1, b1, 1e-11, 1000, scalar=True)
    vals2 = np.repeat(vals1, 2, axis=1)
    b2 = np.repeat(b1, 2, axis=1)
    res = ep.pcg_solve(ctx, 2, dev(rm, torch.int32), dev(ce, torch.int32), dev(vals2), dev(b2),
                       ep.SolverConfig(tol=1e-11))
    assert res.iterations == scalar["iterations"]
    assert np.abs(host(res.solution) - b2 * 0 - scalar["x"]).max() < 1e-9


def test_cg_exhaustion_raises_with_history(ctx):
    """test_pcg.cpp:164-179."""
    rng = np.random.default_rng(3)
    n = 50
    rm = np.arange(n + 1, dtype=np.int32)
    ce = np.arange(n, dtype=np.int32)
    vals = np.linspace(1, 100, n).reshape(n, 1)
    b = rng.uniform(-1, 1, (n, 1))
    with pytest.raises(ep.SolverError) as ex:
        ep.pcg_solve(ctx, 1, dev(rm, torch.int32), dev(ce, torch.int32), dev(vals), dev(b),
                     ep.SolverConfig(tol=1e-15, max_iterations=2))
    assert len(ex.value.history()) == 3 and ex.value.history()[0] == 1.0


def test_cg_indefinite_raises(ctx):
    """test_pcg.cpp:181-190."""
    rm = np.array([0, 1, 2], np.int32)
    ce = np.array([0, 1], np.int32)
    with pytest.raises(ep.SolverError) as ex:
        ep.pcg_solve(ctx, 1, dev(rm, torch.int32), dev(ce, torch.int32), dev(np.array([[1.0], [-1.0]])),
                     dev(np.array([[0.0], [1.0]])))
    assert len(ex.value.history()) >= 1


def test_cg_zero_rhs_and_diagonal(ctx):
    """test_pcg.cpp:36-58."""
    rm = np.arange(6, dtype=np.int32)
    ce = np.arange(5, dtype=np.int32)
    res = ep.pcg_solve(ctx, 1, dev(rm, torch.int32), dev(ce, torch.int32), dev(np.ones((5, 1))),
                       dev(np.zeros((5, 1))))
    assert res.iterations == 0 and res.residual_history == [0.0]
    assert (host(res.solution) == 0).all()
    rm = np.arange(4, dtype=np.int32)
    ce = np.arange(3, dtype=np.int32)
    res = ep.pcg_solve(ctx, 1, dev(rm, torch.int32), dev(ce, torch.int32),
                       dev(np.array([[1.0], [2.0], [3.0]])), dev(np.ones((3, 1))),
                       ep.SolverConfig(tol=1e-12))
    assert res.iterations <= 3
    assert np.allclose(host(res.solution)[:, 0], [1.0, 0.5, 1.0 / 3.0], rtol=1e-12)
    assert len(res.residual_history) == res.iterations + 1 and res.residual_history[0] == 1.0


def test_cg_uncoupled_lane_with_zero_rhs(ctx, R):
    n, s = 5, 4
    rm, ce, v, b = mesh_system(R, s, n)
    b = b.copy()
    b[:, 2] = 0.0
    res = ep.pcg_solve(ctx, s, dev(rm, torch.int32), dev(ce, torch.int32), dev(v), dev(b),
                       ep.SolverConfig(tol=1e-8, flavour=ep.CG_UNCOUPLED))
    ref = R.pcg_uncoupled(s, rm, ce, v, b, 1e-8, 1000)
    assert res.iterations[2] == 0 and res.residual_history[2] == [0.0]
    x = host(res.solution)
    for e in range(s):
        assert same(x[:, e], ref[e]["x"][:, 0])


def test_cg_rejects_bad_rhs_length(ctx):
    rm = dev(np.arange(5, dtype=np.int32), torch.int32)
    ce = dev(np.arange(4, dtype=np.int32), torch.int32)
    with pytest.raises(ValueError):
        ep.pcg_solve(ctx, 1, rm, ce, dev(np.ones(4)), dev(np.ones(3)))


# -------------------------------------------------------- device-resident path
@pytest.mark.parametrize("s", [1, 8, 32])
def test_problem_end_to_end_matches_reference(ctx, R, s):
    n, m = 8, 3
    y = pack_group(R.draw_samples(0, s, m), s)
    p = ep.Problem(ctx, n, s, ep.KlField(m, 1.0, 0.1, 1.0))
    p.assemble(dev(y))
    it, hist, st = p.solve(ep.SolverConfig(tol=1e-6, flavour=ep.CG_UNCOUPLED, dot_mode=ep.DOT_SERIAL))
    rm, ce, v, b = mesh_system(R, s, n)
    assert same(host(p.values), v)
    ref = R.pcg_uncoupled(s, rm, ce, v, b, 1e-6, 1000)
    x = host(p.solution)
    for e in range(s):
        assert it[e] == ref[e]["iterations"]
        assert same(x[:, e], ref[e]["x"][:, 0])
    # the host entry point gives the same answer
    xh = torch.empty(((n + 1) ** 3, s), dtype=torch.float64).pin_memory()
    it2, st2, rc = p.solve_host(torch.as_tensor(y).contiguous(), xh,
                                ep.SolverConfig(tol=1e-6, flavour=ep.CG_UNCOUPLED))
    assert rc == 0 and it2 == list(it) and same(xh.numpy(), x)
    p.close()


@pytest.mark.slow
def test_bench_config_64_cubed_properties(ctx):
    """cfg 2 at full size (64^3, s=32): per-sample bitwise assembly vs s=1 runs,
    uncoupled canonical CG converges every lane and the true residual agrees."""
    n, s, m = 64, 32, 3
    samples = O.draw_samples(0, s, m)
    y = pack_group(samples, s)
    p = ep.Problem(ctx, n, s, ep.KlField(m, 1.0, 0.1, 1.0))
    p.assemble(dev(y))
    it, hist, st = p.solve(ep.SolverConfig(tol=1e-6, max_iterations=10000, flavour=ep.CG_UNCOUPLED,
                                           dot_mode=ep.DOT_CANONICAL))
    assert all(x == 0 for x in st)
    assert 80 < max(it) < 250
    b = -p.residual.clone()
    x = p.solution.clone()
    ax = ep.spmv(ctx, s, p.row_map, p.col_entry, p.values, x)
    rel = torch.linalg.norm(b - ax, dim=0) / torch.linalg.norm(b, dim=0)
    assert float(rel.max()) < 2e-6
    p1 = ep.Problem(ctx, n, 1, ep.KlField(m, 1.0, 0.1, 1.0))
    for e in (0, 31):
        p1.assemble(dev(y[:, e:e + 1]))
        assert same(host(p1.values), host(p.values)[:, e:e + 1])
    p1.close()
    p.close()


@pytest.mark.parametrize("mode", [DOT_SERIAL, DOT_CANONICAL])
@pytest.mark.parametrize("s", [1, 8, 32])
def test_cg_split_direction_option_is_bitwise_neutral(ctx, R, mode, s):
    n = 9
    rm, ce, v, b = mesh_system(R, s, n, seed=5)
    cfg = ep.SolverConfig(tol=1e-8, flavour=ep.CG_UNCOUPLED, dot_mode=mode, seg_rows=(n + 1) ** 2)
    args = (ctx, s, dev(rm, torch.int32), dev(ce, torch.int32), dev(v), dev(b), cfg)
    a = ep.pcg_solve(*args)
    ctx.set_option(ep.OPT_FUSED_DIRECTION, 1)
    try:
        c = ep.pcg_solve(*args)
    finally:
        ctx.set_option(ep.OPT_FUSED_DIRECTION, 0)
    assert a.iterations == c.iterations and same(host(a.solution), host(c.solution))


@pytest.mark.parametrize("mode", [DOT_SERIAL, DOT_CANONICAL])
@pytest.mark.parametrize("s", [1, 4, 32])
def test_symmetric_storage_is_bitwise_neutral(ctx, R, mode, s):
    """ENPROP_OPT_SYMMETRIC_STORAGE: diagonal + upper values only, lower entries
    read from their transposed slots; same operator, same bits."""
    n, m = 9, 3
    y = dev(pack_group(R.draw_samples(3, s, m), s))
    kl = ep.KlField(m, 1.0, 0.2, 1.0)
    cfg = ep.SolverConfig(tol=1e-8, flavour=ep.CG_UNCOUPLED, dot_mode=mode)
    ctx.set_option(ep.OPT_SYMMETRIC_STORAGE, 2)  # every width (default: s >= 4)
    try:
        ps = ep.Problem(ctx, n, s, kl)
    finally:
        ctx.set_option(ep.OPT_SYMMETRIC_STORAGE, 1)
    ctx.set_option(ep.OPT_SYMMETRIC_STORAGE, 0)
    try:
        pf = ep.Problem(ctx, n, s, kl)
    finally:
        ctx.set_option(ep.OPT_SYMMETRIC_STORAGE, 1)
    N = n + 1
    assert ps.nnz_stored == (ps.nnz + N ** 3) // 2 and pf.nnz_stored == pf.nnz
    for p in (ps, pf):
        p.assemble(y)
    assert same(host(ps.values), host(pf.values))
    a = ps.solve(cfg)
    b = pf.solve(cfg)
    assert a[0] == b[0]
    assert same(host(ps.solution), host(pf.solution))
    rv, _ = R.assemble(s, n, m, host(y), sigma=0.2)
    assert same(host(ps.values), rv)
    ps.close()
    pf.close()


@pytest.mark.parametrize("mode", [DOT_SERIAL, DOT_CANONICAL])
@pytest.mark.parametrize("s,n,seg", [(32, 7, 0), (32, 12, 0), (32, 23, 0), (16, 8, 0), (16, 19, 0),
                                     (32, 12, 1000), (16, 12, 77), (4, 17, 0), (4, 30, 0), (4, 9, 50)])
def test_staged_spmv_is_bitwise_equal_to_warp_kernel(ctx, mode, s, n, seg):
    """The stage-pipelined CG SpMV (ep_staged.cu; auto-selected for structured
    problems with symmetric storage at s in {16, 32}) gives the same bits as the
    warp-per-tile kernel: solution, iteration counts and residual histories,
    coupled and uncoupled, for plane-aligned and arbitrary canonical segments."""
    m = 3
    y = dev(pack_group(O.draw_samples(11, s, m), s))
    kl = ep.KlField(m, 1.0, 0.25, 1.0)
    p = ep.Problem(ctx, n, s, kl)
    p.assemble(y)
    for flavour in (ep.CG_UNCOUPLED, ep.CG_COUPLED):
        cfg = ep.SolverConfig(tol=1e-9, flavour=flavour, dot_mode=mode, seg_rows=seg)
        a = p.solve(cfg)
        xa = host(p.solution).copy()
        ctx.set_option(ep.OPT_SPMV_VARIANT, 2)
        try:
            b = p.solve(cfg)
        finally:
            ctx.set_option(ep.OPT_SPMV_VARIANT, -1)
        assert a[0] == b[0]
        assert a[1] == b[1]  # residual histories
        assert same(xa, host(p.solution))
    p.close()


# ------------------------------------------------- sample-major (outer) layout
@pytest.mark.parametrize("s", [1, 3, 4, 32])
def test_spmv_outer_random_crs_bitwise(ctx, R, s):
    """enprop_spmv_outer == the reference's spmv_outer (kernels.hpp:38-56)
    bitwise on random CRS (empty rows, rectangular) and a long-row matrix that
    exceeds the staging capacity (direct-read path)."""
    rng = np.random.default_rng(40 + s)
    shapes = [(int(rng.integers(1, 300)), int(rng.integers(1, 300)), 0.05) for _ in range(6)]
    shapes.append((130, 200, 0.9))  # ~180 entries per row: > 28 * 128 per block
    for rows, cols, dens in shapes:
        rm, ce = random_crs(rng, rows, cols, dens)
        vals = rng.uniform(-1, 1, (s, len(ce)))
        x = rng.uniform(-1, 1, (s, cols))
        z = ep.spmv_outer(ctx, s, dev(rm, torch.int32), dev(ce, torch.int32), dev(vals), dev(x), num_cols=cols)
        assert same(host(z), R.spmv_outer(s, rm, ce, vals, x, cols))


def test_spmv_outer_mesh_matrix_equals_ensemble_layout(ctx, R):
    """On the assembled mesh matrix (16^3, s = 8): the sample-major product of the
    transposed values equals the ensemble-layout product transposed, bitwise."""
    s, n = 8, 16
    rm, ce, v, _ = mesh_system(R, s, n)
    x = np.random.default_rng(1).uniform(-1, 1, (len(rm) - 1, s))
    zc = ep.spmv(ctx, s, dev(rm, torch.int32), dev(ce, torch.int32), dev(v), dev(x))
    zo = ep.spmv_outer(ctx, s, dev(rm, torch.int32), dev(ce, torch.int32), dev(np.ascontiguousarray(v.T)),
                       dev(np.ascontiguousarray(x.T)))
    assert same(host(zo), host(zc).T)


def test_spmv_outer_rejects_bad_lengths(ctx):
    rm = dev(np.arange(5, dtype=np.int32), torch.int32)
    ce = dev(np.arange(4, dtype=np.int32), torch.int32)
    with pytest.raises(ValueError):
        ep.spmv_outer(ctx, 2, rm, ce, dev(np.ones(8)), dev(np.ones(7)))
    with pytest.raises(ValueError):
        ep.spmv_outer(ctx, 2, rm, ce, dev(np.ones(7)), dev(np.ones(8)))


# ---------------------------------------------------------------- Newton (f.3)
@pytest.mark.parametrize("s", [1, 4, 32])
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_newton_matches_reference_composition_bitwise(ctx, R, s, beta):
    """enprop_problem_newton == newton_solve (fem.hpp:265-302) composed from the
    reference's assemble / apply_dirichlet / norm2 / pcg_solve(Identity) / axpby
    (oracle/ref_capi.cpp), serial dots, coupled CG: iterate, Newton steps, total
    CG iterations and residual norms bitwise (reaction term on and off;
    symmetric storage stays valid with the reaction term)."""
    n, m = 5, 5
    y = pack_group(R.draw_samples(19, s, m), s)
    coeffs = ep.PdeCoefficients(0.0, beta)
    p = ep.Problem(ctx, n, s, ep.KlField(m, 1.0, 0.2, 1.0), coeffs=coeffs)
    opt = ep.NewtonOptions(tol=1e-8, max_iterations=20,
                           linear=ep.SolverConfig(tol=1e-10, max_iterations=1000, dot_mode=DOT_SERIAL))
    res = p.newton(dev(y), opt)
    rc, u, its, cg, norms = R.newton_identity(s, n, m, y, sigma=0.2, beta=beta, lin_tol=1e-10)
    assert rc == 0
    assert res.iterations == its and res.total_cg_iterations == cg
    assert same(np.array(res.residual_norms), np.array(norms))
    assert same(host(p.solution), u)
    assert its == (1 if beta == 0.0 else its) and (beta == 0.0 or its >= 2)
    p.close()


def test_newton_exhaustion_raises_with_norms(ctx, R):
    n, m, s = 4, 5, 2
    y = pack_group(R.draw_samples(19, s, m), s)
    p = ep.Problem(ctx, n, s, ep.KlField(m, 1.0, 0.2, 1.0), coeffs=ep.PdeCoefficients(0.0, 1.0))
    opt = ep.NewtonOptions(tol=1e-30, max_iterations=2,
                           linear=ep.SolverConfig(tol=1e-10, dot_mode=DOT_SERIAL))
    with pytest.raises(ep.SolverError) as e:
        p.newton(dev(y), opt)
    assert len(e.value.history()) == 3  # norms before steps 0, 1, 2
    p.close()


@pytest.mark.parametrize("variant", [-1, 2])
def test_problem_canonical_cg_equals_restatement_straddling_stages(ctx, R, variant):
    """30^3, s = 16: a plane is 61 canonical tiles (60 full + 1 row), so the
    staged kernel's two-tile stages straddle planes with a one-row first tile,
    and each CTA cycles its stage rings several times. Both SpMV kernels must
    reproduce the C restatement of canonical CG bitwise (coupled)."""
    n, s, m = 30, 16, 3
    N = n + 1
    rm, ce, v, b = mesh_system(R, s, n)
    y = pack_group(R.draw_samples(0, s, m), s)
    p = ep.Problem(ctx, n, s, ep.KlField(m, 1.0, 0.1, 1.0))
    p.assemble(dev(y))
    cfg = ep.SolverConfig(tol=1e-6, max_iterations=1000, flavour=CG_COUPLED, dot_mode=DOT_CANONICAL)
    ctx.set_option(ep.OPT_SPMV_VARIANT, variant)
    try:
        it, _, _ = p.solve(cfg)
    finally:
        ctx.set_option(ep.OPT_SPMV_VARIANT, -1)
    o = O.pcg(s, rm, ce, v, b, 1e-6, 1000, flavour=CG_COUPLED, mode=DOT_CANONICAL, seg=N * N)
    assert it == o["iterations"][0]
    assert same(host(p.solution), o["x"])
    p.close()
