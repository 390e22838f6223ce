"""GPU parity of the multigrid preconditioner against the
UNMODIFIED reference (oracle/_ref: multigrid.hpp / multigrid.cpp through
ref_capi.cpp): hierarchy shape and eigenvalue estimates, one V-cycle, and
pcg_solve with MgPreconditioner (solution, iterations, residual history) bit
for bit; uncoupled = s x the reference's scalar MG-PCG on extracted
components (bench.cpp:322-330). Sizes stay <= 24^3: the reference's own host
setup and dense coarse LU are the limit."""
import numpy as np
import pytest
import torch

import paper_1511_03703_b200 as ep
from oracles import CG_COUPLED, CG_UNCOUPLED, DOT_SERIAL, RefLib, bits, pack_group

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    return RefLib()


@pytest.fixture(scope="module")
def ctx():
    c = ep.Context(0)
    yield c
    c.close()


def same(a, b):
    a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and (bits(a) == bits(b)).all()


def system(R, n, s, m=3, sigma=0.1, seed=0):
    y = pack_group(R.draw_samples(seed, s, m), s)
    v, r = R.assemble(s, n, m, y, sigma=sigma)
    rm, ce = R.graph(n)
    return rm, ce, v, -r


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def hierarchy(ctx, s, rm, ce, v, opts):
    return ep.MgHierarchy(ctx, s, dev(rm, torch.int32), dev(ce, torch.int32), dev(v), ep.MgOptions(*opts))


OPTS = [(500, 2, 30.0, 1.1, 40), (100, 3, 20.0, 1.2, 25)]


@pytest.mark.parametrize("n,s", [(8, 4), (16, 4), (12, 32)])
@pytest.mark.parametrize("opts", OPTS)
def test_hierarchy_matches_reference(ctx, R, n, s, opts):
    rm, ce, v, b = system(R, n, s)
    h = hierarchy(ctx, s, rm, ce, v, opts)
    rows, lm = h.describe()
    rrows, rlm = R.mg_describe(s, rm, ce, v, opts)
    assert rows == list(rrows)
    assert same(np.array(lm).reshape(-1, s) if lm else np.zeros((0, s)), rlm)
    h.close()


@pytest.mark.parametrize("n,s", [(8, 4), (16, 4), (12, 32), (16, 1)])
def test_vcycle_is_reference_bitwise(ctx, R, n, s):
    rm, ce, v, b = system(R, n, s)
    h = hierarchy(ctx, s, rm, ce, v, OPTS[0])
    rng = np.random.default_rng(5)
    x0 = rng.uniform(-1, 1, b.shape)
    x = dev(x0)
    h.vcycle(dev(b), x)
    torch.cuda.synchronize()
    assert same(x.cpu().numpy(), R.mg_vcycle(s, rm, ce, v, b, x0, OPTS[0], scalar=(s == 1)))
    h.close()


@pytest.mark.parametrize("n,s", [(8, 4), (16, 4), (12, 32), (24, 1)])
@pytest.mark.parametrize("opts", OPTS)
def test_mg_pcg_coupled_is_reference_bitwise(ctx, R, n, s, opts):
    rm, ce, v, b = system(R, n, s)
    h = hierarchy(ctx, s, rm, ce, v, opts)
    cfg = ep.SolverConfig(tol=1e-8, max_iterations=200, flavour=CG_COUPLED, dot_mode=DOT_SERIAL)
    res = h.pcg(dev(b), cfg)
    o = R.mg_pcg(s, rm, ce, v, b, 1e-8, 200, opts, scalar=(s == 1))
    assert o["status"] == 0
    assert res.iterations == o["iterations"]
    assert same(np.array(res.residual_history), o["history"])
    assert same(res.solution.cpu().numpy(), o["x"])
    h.close()


def test_mg_pcg_uncoupled_is_per_sample_reference(ctx, R):
    n, s = 12, 4
    rm, ce, v, b = system(R, n, s, sigma=0.25, seed=3)
    h = hierarchy(ctx, s, rm, ce, v, OPTS[0])
    cfg = ep.SolverConfig(tol=1e-9, max_iterations=200, flavour=CG_UNCOUPLED, dot_mode=DOT_SERIAL)
    res = h.pcg(dev(b), cfg)
    x = res.solution.cpu().numpy()
    for e in range(s):
        o = R.mg_pcg(1, rm, ce, np.ascontiguousarray(v[:, e]), np.ascontiguousarray(b[:, e]), 1e-9, 200,
                     OPTS[0], scalar=True)
        assert res.iterations[e] == o["iterations"]
        assert same(np.array(res.residual_history[e]), o["history"])
        assert same(x[:, e], o["x"][:, 0])
    h.close()


def test_mg_pcg_exhaustion_and_invalid(ctx, R):
    rm, ce, v, b = system(R, 8, 4)
    h = hierarchy(ctx, 4, rm, ce, v, OPTS[0])
    with pytest.raises(ep.SolverError) as e:
        h.pcg(dev(b), ep.SolverConfig(tol=1e-15, max_iterations=2, flavour=CG_COUPLED, dot_mode=DOT_SERIAL))
    assert len(e.value.history()) == 3
    with pytest.raises(ValueError):  # the multigrid solve uses the reference's order
        h.pcg(dev(b), ep.SolverConfig(dot_mode=ep.DOT_CANONICAL))
    h.close()


@pytest.mark.parametrize("s,n,beta", [(4, 8, 0.0), (4, 8, 0.7), (1, 10, 0.7), (32, 6, 0.5)])
def test_newton_multigrid_is_the_reference_newton_solve(ctx, R, s, n, beta):
    """f3 as the reference runs it: newton_solve (fem.hpp:265-302) with each
    step's hierarchy and MG-preconditioned coupled CG -- iterate, steps, CG
    total and residual norms bitwise equal to the reference's own function."""
    m = 3
    y = pack_group(R.draw_samples(7, s, m), s)
    opts = (100, 2, 30.0, 1.1, 40)
    o = R.newton_mg(s, n, m, y, beta=beta, tol=1e-8, lin_tol=1e-10, opts=opts, scalar=(s == 1))
    assert o["status"] == 0
    p = ep.Problem(ctx, n, s, ep.KlField(m, 1.0, 0.1, 1.0), ep.PdeCoefficients(0.0, beta))
    lin = ep.SolverConfig(tol=1e-10, max_iterations=1000, flavour=CG_COUPLED, dot_mode=DOT_SERIAL)
    res = p.newton(dev(y), ep.NewtonOptions(tol=1e-8, max_iterations=20, linear=lin), multigrid=ep.MgOptions(*opts))
    assert res.iterations == o["iterations"]
    assert res.total_cg_iterations == o["total_cg"]
    assert same(np.array(res.residual_norms), o["norms"])
    assert same(p.solution.cpu().numpy(), o["u"])
    p.close()
