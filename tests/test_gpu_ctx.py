"""GPU tests of the context-level C ABI a non-torch caller uses: device
allocation and stream-ordered copies (enprop_malloc / enprop_free /
enprop_memcpy_h2d / enprop_memcpy_d2h), the context stream, the launch
counter and the CG profiling counters (enprop_ctx_profile / _detail)."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_1511_03703_b200 as ep
from oracles import CG_UNCOUPLED, DOT_SERIAL, Oracle, pack_group

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = ep.Context(0)
    yield c
    c.close()


def test_malloc_copies_roundtrip(ctx):
    L = ep.lib()
    L.enprop_malloc.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]
    L.enprop_free.argtypes = [C.c_void_p, C.c_void_p]
    L.enprop_memcpy_h2d.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]
    L.enprop_memcpy_d2h.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]
    L.enprop_ctx_stream.argtypes = [C.c_void_p]
    L.enprop_ctx_stream.restype = C.c_void_p
    src = np.random.default_rng(3).uniform(-1, 1, 4097)
    out = np.zeros_like(src)
    d = C.c_void_p()
    assert L.enprop_malloc(ctx.h, src.nbytes, C.byref(d)) == 0 and d.value
    assert L.enprop_memcpy_h2d(ctx.h, d, src.ctypes.data, src.nbytes) == 0
    assert L.enprop_memcpy_d2h(ctx.h, out.ctypes.data, d, src.nbytes) == 0
    assert (out.view(np.uint64) == src.view(np.uint64)).all()
    assert L.enprop_free(ctx.h, d) == 0
    # the Python Context runs on torch's current stream (the null handle for
    # torch's default stream)
    assert (L.enprop_ctx_stream(ctx.h) or 0) == torch.cuda.current_stream().cuda_stream


def test_launch_counter_and_profile(ctx):
    """The launch counter grows with the solve; the profiling counters see
    every CG iteration of the solve (the serial order: direction, SpMV, two
    chains and the update per iteration) with positive phase times."""
    s, n = 4, 10
    p = ep.Problem(ctx, n, s, ep.KlField(3, 1.0, 0.1, 1.0))
    p.assemble(torch.as_tensor(pack_group(Oracle().draw_samples(0, s, 3), s)).cuda())
    cfg = ep.SolverConfig(tol=1e-7, max_iterations=2000, flavour=CG_UNCOUPLED, dot_mode=DOT_SERIAL)
    before = ctx.launches
    ctx.profile(1)
    it, _, _ = p.solve(cfg)
    det = ctx.profile_detail()
    ms, launches = ctx.profile(0)
    assert ctx.launches > before
    assert det["iterations"] == max(it)
    assert det["solve"] > 0 and det["spmv_kernel"] > 0 and det["iteration"] > 0
    assert launches == det["iterations"] and ms > 0
    p.close()
