"""Slab domain decomposition over REAL rank processes: 2 and 3
processes on one GPU exchange halos and per-plane dot sums through the CUDA-IPC
transport (exported buffers + interprocess events; no kernel waits on another
rank). Their solution, iteration counts and statuses equal the one-GPU
canonical solve bit for bit -- the property the reference states for its own
distributed SpMV (test_halo.cpp:248-281) and that the canonical order extends
to the whole CG solve."""
import multiprocessing as mp
import os
import uuid

import numpy as np
import pytest
import torch

import paper_1511_03703_b200 as ep
from oracles import bits

pytestmark = pytest.mark.gpu


def _newton_cfg():
    return ep.NewtonOptions(tol=1e-9, max_iterations=20,
                            linear=ep.SolverConfig(tol=1e-10, max_iterations=2000, dot_mode=ep.DOT_CANONICAL))


def _rank_newton(job, nranks, rank, n, s, q):
    """Two back-to-back linear solves (their per-plane sum buffers are reused
    across solves), then Newton with the u halo over the IPC transport."""
    import torch  # noqa: F811  (fresh process)

    import paper_1511_03703_b200 as ep  # noqa: F811
    try:
        ctx = ep.Context(0)
        kl = ep.KlField(3, 1.0, 0.2, 1.0)
        d = ep.Dist(ctx, n, s, nranks, rank, kl=kl, coeffs=ep.PdeCoefficients(0.0, 1.0), ipc_job=job)
        y = ep.pack_sample_group(ep.draw_samples(5, s, 3), s, 0).cuda()
        d.assemble(y)
        cfg = ep.SolverConfig(tol=1e-7, max_iterations=2000, flavour=ep.CG_UNCOUPLED, dot_mode=ep.DOT_CANONICAL)
        its = [d.solve(cfg)[0] for _ in range(2)]
        res = d.newton(y, _newton_cfg())
        (rk, rb, rows, x), = d.local()
        q.put((rank, rb, x.cpu().numpy().copy(), (its, res.iterations, res.total_cg_iterations,
                                                     res.residual_norms), None, None))
        d.close()
        ctx.close()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, None, None, None, repr(e)))


def _rank_main(job, nranks, rank, n, s, flavour, q):
    import torch  # noqa: F811  (fresh process)

    import paper_1511_03703_b200 as ep  # noqa: F811
    try:
        ctx = ep.Context(0)
        kl = ep.KlField(3, 1.0, 0.1, 1.0)
        d = ep.Dist(ctx, n, s, nranks, rank, kl=kl, ipc_job=job)
        y = ep.pack_sample_group(ep.draw_samples(0, s, 3), s, 0).cuda()
        d.assemble(y)
        cfg = ep.SolverConfig(tol=1e-7, max_iterations=2000, flavour=flavour, dot_mode=ep.DOT_CANONICAL)
        it, st = d.solve(cfg)
        (rk, rb, rows, x), = d.local()
        q.put((rank, rb, x.cpu().numpy().copy(), it, st, None))
        d.close()
        ctx.close()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, None, None, None, repr(e)))


@pytest.mark.parametrize("nranks,s,flavour", [(2, 32, ep.CG_UNCOUPLED), (3, 4, ep.CG_COUPLED)])
def test_ipc_ranks_equal_one_gpu_bitwise(nranks, s, flavour):
    n = 10
    kl = ep.KlField(3, 1.0, 0.1, 1.0)
    ctx = ep.Context(0)
    p = ep.Problem(ctx, n, s, kl)
    p.assemble(ep.pack_sample_group(ep.draw_samples(0, s, 3), s, 0).cuda())
    cfg = ep.SolverConfig(tol=1e-7, max_iterations=2000, flavour=flavour, dot_mode=ep.DOT_CANONICAL)
    it1, _, _ = p.solve(cfg)
    x1 = p.solution.cpu().numpy().copy()
    p.close()
    ctx.close()

    job = uuid.uuid4().hex[:16]
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=_rank_main, args=(job, nranks, r, n, s, flavour, q)) for r in range(nranks)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(nranks)]
    for pr in procs:
        pr.join(timeout=60)
    errs = [r[5] for r in res if r[5]]
    assert not errs, errs
    res.sort(key=lambda r: r[1])
    x2 = np.concatenate([r[2] for r in res], axis=0)
    assert all(r[3] == it1 for r in res)  # every rank took the same decisions
    assert all(all(v == 0 for v in r[4]) for r in res)
    assert (bits(x1) == bits(x2)).all()
    assert not os.path.exists(f"/dev/shm/enprop_b200_{job}")  # board removed


def test_ipc_newton_and_repeated_solves_equal_one_gpu_bitwise():
    n, s, nranks = 10, 4, 2
    ctx = ep.Context(0)
    kl = ep.KlField(3, 1.0, 0.2, 1.0)
    p = ep.Problem(ctx, n, s, kl, coeffs=ep.PdeCoefficients(0.0, 1.0))
    y = ep.pack_sample_group(ep.draw_samples(5, s, 3), s, 0).cuda()
    p.assemble(y)
    cfg = ep.SolverConfig(tol=1e-7, max_iterations=2000, flavour=ep.CG_UNCOUPLED, dot_mode=ep.DOT_CANONICAL)
    it1, _, _ = p.solve(cfg)
    r1 = p.newton(y, _newton_cfg())
    u1 = p.solution.cpu().numpy().copy()
    p.close()
    ctx.close()

    job = uuid.uuid4().hex[:16]
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=_rank_newton, args=(job, nranks, r, n, s, q)) for r in range(nranks)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(nranks)]
    for pr in procs:
        pr.join(timeout=60)
    errs = [r[5] for r in res if r[5]]
    assert not errs, errs
    res.sort(key=lambda r: r[1])
    for r in res:
        its, steps, cg, norms = r[3]
        assert its == [it1, it1]
        assert (steps, cg) == (r1.iterations, r1.total_cg_iterations)
        assert (bits(np.array(norms)) == bits(np.array(r1.residual_norms))).all()
    u2 = np.concatenate([r[2] for r in res], axis=0)
    assert (bits(u1) == bits(u2)).all()
