"""CPU, world_size 2 and 3 (torch.distributed gloo): the multi-rank protocol of
the slab-decomposed solve (paper_1511_03703_b200/csrc/ep_dist.cu)
restated in numpy and checked against the single-process C oracle.

Each rank owns the z-planes partition.cpp:31-72 gives it, holds its rows of the
assembled CRS with columns renumbered into the ghost-extended layout
[lo ghost plane | owned planes | hi ghost plane], exchanges one ghost plane with
each neighbour per SpMV (send/recv), and all-gathers its per-plane canonical
dot sums; totals are summed in global plane order.  The result must equal the
one-process canonical CG of the C oracle bit for bit (solution and iteration
counts), for coupled and uncoupled CG.

The distributed Newton (enprop_dist_newton, f3 with Alg. 2's u halo) is
restated the same way: each step imports the neighbours' boundary planes of u,
assembles the owned rows from u known only on [lo ghost | owned | hi ghost],
forms the coupled canonical residual norm from all-gathered plane sums, and
solves by the protocol's CG. Norms, steps and u equal the one-process Newton
composed from the oracle's pieces (canonical order) bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

TILE = 16


def plane_range(N, P, r):
    base, extra = N // P, N % P
    k0 = r * base + min(r, extra)
    return k0, k0 + base + (1 if r < extra else 0)


def fold(t):
    h = t.shape[0] // 2
    while h >= 1:
        t[:h] = t[:h] + t[h:2 * h]
        h //= 2
    return t[0]


def plane_sums(u, v, plane, s):
    """Canonical per-segment (plane) sums of the owned rows:
    tiles of 16 rows and blocks of 16 tiles folded by stride halving (+0.0
    padding), then 0.0 + block_0 + block_1 + ... per plane."""
    nplanes = u.shape[0] // plane
    out = np.zeros((nplanes, s))
    for k in range(nplanes):
        r0, r1 = k * plane, (k + 1) * plane
        seg = np.zeros(s)
        for b0 in range(r0, r1, 16 * TILE):
            blk = np.zeros((16, s))
            for j in range(16):
                t0 = b0 + j * TILE
                if t0 >= r1:
                    continue
                t = np.zeros((TILE, s))
                m = min(TILE, r1 - t0)
                t[:m] = u[t0:t0 + m] * v[t0:t0 + m]
                blk[j] = fold(t)
            seg = seg + fold(blk)
        out[k] = seg
    return out


def spmv(rm, ce, vals, xe, s):
    z = np.zeros((len(rm) - 1, s))
    for row in range(len(rm) - 1):
        acc = np.zeros(s)
        for k in range(rm[row], rm[row + 1]):
            acc = acc + vals[k] * xe[ce[k]]
        z[row] = acc
    return z


def worker(rank, world, port, n, s, flavour, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracles import Oracle, pack_group
    O = Oracle()
    N, plane = n + 1, (n + 1) ** 2
    y = pack_group(O.draw_samples(0, s, 3), s)
    vals_g, res_g = O.assemble(s, n, O.kl(3, 1.0, 0.1, 1.0), y, dirichlet=True)
    rm_g, ce_g = O.graph(n)
    k0, k1 = plane_range(N, world, rank)
    rb, re_ = k0 * plane, k1 * plane
    lo = plane if k0 > 0 else 0
    hi = plane if k1 < N else 0
    ext_begin = rb - lo
    rm = (rm_g[rb:re_ + 1] - rm_g[rb]).astype(np.int64)
    ce = (ce_g[rm_g[rb]:rm_g[re_]] - ext_begin).astype(np.int64)
    vals = vals_g[rm_g[rb]:rm_g[re_]]
    rows = re_ - rb
    maxplanes = (N + world - 1) // world
    b = -res_g[rb:re_]

    def total(u, v):
        ps = np.zeros((maxplanes, s))
        ps[:k1 - k0] = plane_sums(u, v, plane, s)
        bufs = [torch.zeros((maxplanes, s), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(bufs, torch.from_numpy(ps))
        acc = np.zeros(s)
        for q in range(world):
            a, c = plane_range(N, world, q)
            for k in range(c - a):
                acc = acc + bufs[q].numpy()[k]
        return acc

    def halo(p_own):
        pe = np.zeros((lo + rows + hi, s))
        pe[lo:lo + rows] = p_own
        reqs = []
        lo_buf = torch.zeros((plane, s), dtype=torch.float64)
        hi_buf = torch.zeros((plane, s), dtype=torch.float64)
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(p_own[:plane])), rank - 1))
            reqs.append(dist.irecv(lo_buf, rank - 1))
        if rank + 1 < world:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(p_own[rows - plane:])), rank + 1))
            reqs.append(dist.irecv(hi_buf, rank + 1))
        for r_ in reqs:
            r_.wait()
        if lo:
            pe[:plane] = lo_buf.numpy()
        if hi:
            pe[lo + rows:] = hi_buf.numpy()
        return pe

    # CG (pcg.hpp:52-103), canonical totals; coupled: one decision for all lanes
    coupled = flavour == 0
    red = (lambda d: np.full(s, sum_left(d))) if coupled else (lambda d: d)

    def sum_left(d):
        acc = 0.0
        for e in range(s):
            acc = acc + d[e]
        return acc

    tol, maxit = 1e-8, 500
    x = np.zeros((rows, s))
    r = b.copy()
    dd = red(total(b, b))
    bnorm = np.sqrt(dd)
    rz = dd.copy()
    active = (np.sqrt(dd) / bnorm >= tol)
    iters = np.zeros(s, int)
    p = r.copy()
    it = 0
    while active.any() and it < maxit:
        q = spmv(rm, ce, vals, halo(p), s)
        pq = red(total(p, q))
        alpha = rz / pq
        a = np.where(active, alpha, 0.0)
        x = np.where(active, a * p + x, x)
        r = np.where(active, (-a) * q + r, r)
        rr = red(total(r, r))
        beta = rr / rz
        rz = np.where(active, rr, rz)
        it += 1
        rel = np.sqrt(rr) / bnorm
        done_now = active & (rel < tol)
        iters[done_now] = it
        active = active & ~done_now
        p = np.where(active, r + beta * p, p)
    xs = [None] * world
    dist.all_gather_object(xs, (rb, x))
    if rank == 0:
        xg = np.concatenate([v for _, v in sorted(xs, key=lambda t: t[0])])
        out.put((xg, iters.tolist()))
    dist.barrier()
    dist.destroy_process_group()


def newton_worker(rank, world, port, n, s, beta, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from oracles import Oracle, pack_group
    O = Oracle()
    N, plane = n + 1, (n + 1) ** 2
    f = O.kl(3, 1.0, 0.2, 1.0)
    y = pack_group(O.draw_samples(5, s, 3), s)
    rm_g, ce_g = O.graph(n)
    k0, k1 = plane_range(N, world, rank)
    rb, re_ = k0 * plane, k1 * plane
    lo = plane if k0 > 0 else 0
    hi = plane if k1 < N else 0
    ext_begin = rb - lo
    rm = (rm_g[rb:re_ + 1] - rm_g[rb]).astype(np.int64)
    ce = (ce_g[rm_g[rb]:rm_g[re_]] - ext_begin).astype(np.int64)
    rows = re_ - rb
    maxplanes = (N + world - 1) // world

    def total(u, v):
        ps = np.zeros((maxplanes, s))
        ps[:k1 - k0] = plane_sums(u, v, plane, s)
        bufs = [torch.zeros((maxplanes, s), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(bufs, torch.from_numpy(ps))
        acc = np.zeros(s)
        for q in range(world):
            a, c = plane_range(N, world, q)
            for k in range(c - a):
                acc = acc + bufs[q].numpy()[k]
        return acc

    def coupled(d):
        acc = 0.0
        for e in range(s):
            acc = acc + d[e]
        return acc

    def halo(own):
        pe = np.zeros((lo + rows + hi, s))
        pe[lo:lo + rows] = own
        reqs = []
        lo_buf = torch.zeros((plane, s), dtype=torch.float64)
        hi_buf = torch.zeros((plane, s), dtype=torch.float64)
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(own[:plane])), rank - 1))
            reqs.append(dist.irecv(lo_buf, rank - 1))
        if rank + 1 < world:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(own[rows - plane:])), rank + 1))
            reqs.append(dist.irecv(hi_buf, rank + 1))
        for r_ in reqs:
            r_.wait()
        if lo:
            pe[:plane] = lo_buf.numpy()
        if hi:
            pe[lo + rows:] = hi_buf.numpy()
        return pe

    def cg(vals, b, tol=1e-10, maxit=1000):  # coupled, canonical totals (pcg.hpp:52-103)
        x = np.zeros((rows, s))
        r = b.copy()
        dd = coupled(total(b, b))
        bnorm = np.sqrt(dd)
        if bnorm == 0.0:
            return x
        rz = dd
        p = r.copy()
        for it in range(maxit):
            q = spmv(rm, ce, vals, halo(p), s)
            alpha = rz / coupled(total(p, q))
            x = alpha * p + x
            r = (-alpha) * q + r
            rr = coupled(total(r, r))
            beta_ = rr / rz
            rz = rr
            if np.sqrt(rr) / bnorm < tol:
                break
            p = r + beta_ * p
        return x

    u = np.zeros((rows, s))
    norms, steps, tol = [], 0, 1e-9
    for step in range(21):
        ue = halo(u)  # Alg. 2: import the neighbours' boundary planes of u
        uf = np.zeros(((n + 1) ** 3, s))
        uf[ext_begin:ext_begin + lo + rows + hi] = ue
        vals_g, res_g = O.assemble(s, n, f, y, u=uf, beta=beta, dirichlet=True)
        vals, res = vals_g[rm_g[rb]:rm_g[re_]], res_g[rb:re_]
        norm = np.sqrt(coupled(total(res, res)))
        norms.append(norm)
        if step == 0 and norm == 0.0:
            break
        if step > 0 and norm < tol * norms[0]:
            steps = step
            break
        du = cg(vals, -res)
        u = 1.0 * du + 1.0 * u  # axpby(1.0, du, 1.0, u) (fem.hpp:300)
    us = [None] * world
    dist.all_gather_object(us, (rb, u))
    if rank == 0:
        ug = np.concatenate([v for _, v in sorted(us, key=lambda t: t[0])])
        out.put((ug, norms, steps))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_newton_protocol_equals_single_process_newton(world):
    from oracles import CG_COUPLED, DOT_CANONICAL, Oracle, bits, pack_group
    n, s, beta = 4, 2, 1.0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=newton_worker, args=(r, world, port, n, s, beta, q)) for r in range(world)]
    for p in procs:
        p.start()
    ug, norms, steps = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the one-process Newton from the oracle's pieces, canonical order (segments = planes)
    O = Oracle()
    f = O.kl(3, 1.0, 0.2, 1.0)
    y = pack_group(O.draw_samples(5, s, 3), s)
    rm, ce = O.graph(n)
    seg = (n + 1) ** 2
    u = np.zeros(((n + 1) ** 3, s))
    rn, rsteps = [], 0
    for step in range(21):
        vals, res = O.assemble(s, n, f, y, u=u, beta=beta, dirichlet=True)
        norm = np.sqrt(O.dot(s, res, res, DOT_CANONICAL, TILE, seg))
        rn.append(norm)
        if step > 0 and norm < 1e-9 * rn[0]:
            rsteps = step
            break
        du = O.pcg(s, rm, ce, vals, -res, 1e-10, 1000, flavour=CG_COUPLED, mode=DOT_CANONICAL, tile=TILE,
                   seg=seg)["x"]
        u = 1.0 * du + 1.0 * u
    assert rsteps >= 2 and steps == rsteps
    assert (bits(np.array(norms)) == bits(np.array(rn))).all()
    assert (bits(ug) == bits(u)).all()


def free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("flavour", [0, 1])
def test_slab_protocol_equals_single_process_canonical_cg(world, flavour):
    from oracles import DOT_CANONICAL, Oracle, bits, pack_group
    n, s = 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, n, s, flavour, q)) for r in range(world)]
    for p in procs:
        p.start()
    xg, iters = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    O = Oracle()
    y = pack_group(O.draw_samples(0, s, 3), s)
    vals, res = O.assemble(s, n, O.kl(3, 1.0, 0.1, 1.0), y, dirichlet=True)
    rm, ce = O.graph(n)
    ref = O.pcg(s, rm, ce, vals, -res, 1e-8, 500, flavour=flavour, mode=DOT_CANONICAL, tile=TILE,
                seg=(n + 1) ** 2)
    assert (bits(xg) == bits(ref["x"])).all()
    if flavour == 1:
        assert iters == list(ref["iterations"])
    else:
        assert iters[0] == ref["iterations"][0]
