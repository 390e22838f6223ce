"""Slab domain decomposition on one GPU with the in-process
transport: any rank count gives the one-GPU canonical solve bit for bit
(the canonical reduction is defined per mesh plane, independent of the
partition), and the partition follows partition.cpp:31-72."""
import numpy as np
import pytest
import torch

import paper_1511_03703_b200 as ep
from oracles import CG_COUPLED, CG_UNCOUPLED, DOT_CANONICAL, Oracle, RefLib, bits, pack_group

pytestmark = pytest.mark.gpu
O = Oracle()


@pytest.fixture(scope="module")
def ctx():
    c = ep.Context(0)
    yield c
    c.close()


def same(a, b):
    a, b = np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and (bits(a) == bits(b)).all()


@pytest.mark.parametrize("s", [1, 4, 8, 16, 32])  # 4, 16, 32: symmetric storage + the staged SpMV per slab
@pytest.mark.parametrize("flavour", [CG_COUPLED, CG_UNCOUPLED])
@pytest.mark.parametrize("nranks", [1, 2, 3, 5, 11])
def test_emulated_ranks_equal_one_gpu_bitwise(ctx, s, flavour, nranks):
    n, m = 10, 3
    y = torch.as_tensor(pack_group(O.draw_samples(0, s, m), s)).cuda()
    kl = ep.KlField(m, 1.0, 0.1, 1.0)
    cfg = ep.SolverConfig(tol=1e-7, max_iterations=2000, flavour=flavour, dot_mode=ep.DOT_CANONICAL)
    p = ep.Problem(ctx, n, s, kl)
    p.assemble(y)
    it1, _, _ = p.solve(cfg)
    x1 = p.solution.cpu().numpy()
    d = ep.Dist(ctx, n, s, nranks, kl=kl)
    d.assemble(y)
    it2, st2 = d.solve(cfg)
    x2 = d.solution().cpu().numpy()
    assert it1 == it2
    assert same(x1, x2)
    assert all(v == 0 for v in st2)
    p.close()
    d.close()


@pytest.mark.parametrize("s", [1, 4, 32])
@pytest.mark.parametrize("alpha,beta", [(0.0, 1.0), (0.4, 1.0)])  # staged slabs at s = 4, 32 / full storage
@pytest.mark.parametrize("nranks", [2, 3, 5])
def test_dist_newton_equals_one_gpu_bitwise(ctx, s, alpha, beta, nranks):
    """Newton over the slabs (f3 with Alg. 2's u halo): every step imports the
    neighbours' boundary planes of u before assembling, so residual norms,
    steps, CG iterations and the iterate equal the one-GPU Newton (canonical
    order) bit for bit."""
    n, m = 9, 3
    y = torch.as_tensor(pack_group(O.draw_samples(5, s, m), s)).cuda()
    kl = ep.KlField(m, 1.0, 0.2, 1.0)
    coeffs = ep.PdeCoefficients(alpha, beta)
    opt = ep.NewtonOptions(tol=1e-9, max_iterations=20,
                           linear=ep.SolverConfig(tol=1e-10, max_iterations=2000, dot_mode=ep.DOT_CANONICAL))
    p = ep.Problem(ctx, n, s, kl, coeffs=coeffs)
    r1 = p.newton(y, opt)
    u1 = p.solution.cpu().numpy()
    d = ep.Dist(ctx, n, s, nranks, kl=kl, coeffs=coeffs)
    r2 = d.newton(y, opt)
    u2 = d.solution().cpu().numpy()
    assert r1.iterations >= 2  # the nonlinear term is live: more than one step
    assert (r1.iterations, r1.total_cg_iterations) == (r2.iterations, r2.total_cg_iterations)
    assert same(np.array(r1.residual_norms), np.array(r2.residual_norms))
    assert same(u1, u2)
    p.close()
    d.close()


def test_dist_newton_rejects_serial_order(ctx):
    d = ep.Dist(ctx, 3, 4, 2, kl=ep.KlField(3, 1.0, 0.1, 1.0), coeffs=ep.PdeCoefficients(0.0, 1.0))
    with pytest.raises(ValueError):
        d.newton(torch.zeros((3, 4), dtype=torch.float64, device="cuda"),
                 ep.NewtonOptions(linear=ep.SolverConfig(dot_mode=ep.DOT_SERIAL)))
    d.close()


def test_halo_overlap_splits_interior_stages(ctx):
    """Staged slabs order their interior stages (no ghost plane read) first; the
    iteration runs them while the halo is in flight. Ranks with >= 3 planes have
    some, a lone rank (no ghosts) runs every stage in one launch (0 interior),
    and unstaged widths report none."""
    n = 10  # 11 planes
    kl = ep.KlField(3, 1.0, 0.1, 1.0)
    d = ep.Dist(ctx, n, 32, 3, kl=kl)  # 4 + 4 + 3 planes
    for (interior, total), (_, rb, rows, _) in zip(d.stages(), d.local()):
        assert 0 < interior < total
    d.close()
    d = ep.Dist(ctx, n, 32, 1, kl=kl)
    (interior, total), = d.stages()
    assert interior == 0 and total > 0
    d.close()
    d = ep.Dist(ctx, n, 8, 3, kl=kl)
    assert all(st == (0, 0) for st in d.stages())
    d.close()


@pytest.mark.parametrize("s", [4, 32])
def test_nccl_single_rank_job_equals_emulated_bitwise(ctx, s):
    """The NCCL transport (libnccl.so.2 loaded at run time, unique id, comm
    init, per-plane sums all-gathered by ncclAllGather, comm destroy) as a
    1-rank job on this GPU -- NCCL refuses two ranks on one device, so this
    is the part of the NCCL path one GPU can run. Bitwise the emulated solve."""
    n, m = 10, 3
    y = torch.as_tensor(pack_group(O.draw_samples(0, s, m), s)).cuda()
    kl = ep.KlField(m, 1.0, 0.1, 1.0)
    cfg = ep.SolverConfig(tol=1e-7, max_iterations=2000, flavour=CG_UNCOUPLED, dot_mode=ep.DOT_CANONICAL)
    d1 = ep.Dist(ctx, n, s, 1, kl=kl)
    d1.assemble(y)
    it1, _ = d1.solve(cfg)
    x1 = d1.solution().cpu().numpy()
    d1.close()
    d2 = ep.Dist(ctx, n, s, 1, 0, nccl_id=ep.nccl_unique_id(), kl=kl)
    d2.assemble(y)
    it2, st2 = d2.solve(cfg)
    x2 = d2.solution().cpu().numpy()
    assert it1 == it2 and all(v == 0 for v in st2)
    assert same(x1, x2)
    d2.close()


def test_partition_matches_reference_rule(ctx):
    R = RefLib()
    n = 10
    for nranks in (2, 3, 4, 7):
        d = ep.Dist(ctx, n, 1, nranks, kl=ep.KlField(1, 1.0, 0.0, 1.0))
        got = sorted((rb // (n + 1) ** 2, rows // (n + 1) ** 2) for (_, rb, rows, _) in d.local())
        ref = R.partition(n, nranks)  # x-plane ranges; we split z-planes by the same rule
        assert got == [tuple(r) for r in ref]
        d.close()


def test_dist_rejects_serial_order_and_too_many_ranks(ctx):
    with pytest.raises(ValueError):
        ep.Dist(ctx, 3, 4, 5)
    d = ep.Dist(ctx, 3, 4, 2, kl=ep.KlField(3, 1.0, 0.1, 1.0))
    d.assemble(torch.zeros((3, 4), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        d.solve(ep.SolverConfig(dot_mode=ep.DOT_SERIAL))
    d.close()


def test_time_halo_measures_the_exchange(ctx):
    """enprop_dist_time_halo: the solver's own halo exchange, timed; larger
    ensembles move more bytes (one plane of s values per neighbour)."""
    times = {}
    for s in (1, 32):
        d = ep.Dist(ctx, 24, s, nranks=3, kl=ep.KlField(3, 1.0, 0.1, 1.0))
        times[s] = d.time_halo(20)
        assert 0 < times[s] < 1e-3  # a few microseconds of device copies
    a, b, rss = ep.fit_halo_model([(1, times[1]), (32, times[32])])
    assert rss == 0.0 or rss < 1e-18  # two points: an exact line
    assert a + b * 32 == pytest.approx(times[32], rel=1e-9, abs=1e-15)


def test_exchange_trace_records_the_measured_exchange(ctx, tmp_path):
    """Dist.exchange_trace (f2): one record per message in the reference's order
    (sender rank, lower link before upper: partition.cpp:59-72), one plane of s
    values each, the sender's cumulative measured time; exported as the
    reference's CSV."""
    n, s = 10, 4
    d = ep.Dist(ctx, n, s, nranks=3, kl=ep.KlField(3, 1.0, 0.1, 1.0))
    recs, elapsed = d.exchange_trace()
    assert [(r[0], r[1]) for r in recs] == [(0, 1), (1, 0), (1, 2), (2, 1)]
    assert all(r[2] == (n + 1) ** 2 * s * 8 for r in recs)
    assert all(r[3] > 0 for r in recs)
    assert recs[2][3] > recs[1][3]  # rank 1's clock accumulates over its two messages
    assert elapsed == max(r[3] for r in recs)
    path = tmp_path / "trace.csv"
    ep.write_exchange_trace_csv(str(path), recs)
    lines = path.read_text().splitlines()
    assert lines[0] == "rank,neighbor,bytes,virtual_time" and len(lines) == 5
    d.close()
