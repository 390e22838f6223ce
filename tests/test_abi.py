"""CPU tests of the drop-in boundary: the C-ABI library loads and exports every
symbol include/enprop_b200.h declares; host-only entry points work without a
GPU; device entry points fail loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest
import torch

import paper_1511_03703_b200 as ep
from oracles import Oracle, bits

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "enprop_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(enprop_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    names = declared_functions()
    for required in ("enprop_spmv", "enprop_assemble", "enprop_apply_dirichlet", "enprop_cg",
                     "enprop_dot", "enprop_axpby", "enprop_build_node_graph",
                     "enprop_problem_solve_host"):
        assert required in names


def test_library_exports_every_declared_symbol():
    L = ep.lib()
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, f"not exported: {missing}"


def test_abi_version_and_nnz():
    L = ep.lib()
    assert L.enprop_abi_version() == 1
    for n in (1, 2, 16, 64, 128, 256):
        assert ep.mesh_nnz(n) == (3 * (n + 1) - 2) ** 3
    assert ep.mesh_nnz(0) == 0


def test_kl_describe_host_is_bitwise_reference_order():
    """enprop_kl_describe runs the library's host restatement of kl.cpp:41-89."""
    O = Oracle()
    for m, sig in ((1, 0.0), (3, 0.1), (5, 0.2), (10, 0.25)):
        d = ep.kl_describe(ep.KlField(m, 1.0, sig, 1.0))
        f = O.kl(m, 1.0, sig, 1.0)
        assert bits(np.array(d["axis_freq"])).tolist() == bits(np.array(f.axis_freq[:m])).tolist()
        assert bits(np.array(d["mode_eig"])).tolist() == bits(np.array(f.mode_eig[:m])).tolist()
        assert d["mode_axes"] == [[f.mode_axes[i][k] for k in range(3)] for i in range(m)]
    with pytest.raises(ValueError):
        ep.kl_describe(ep.KlField(0, 1.0, 0.1, 1.0))
    with pytest.raises(ValueError):
        ep.kl_describe(ep.KlField(3, 0.0, 0.1, 1.0))
    with pytest.raises(ValueError):
        ep.kl_describe(ep.KlField(3, 1.0, -0.1, 1.0))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback():
    with pytest.raises(ep.EnpropError):
        ep.Context(0, use_torch_stream=False)


def test_ctypes_null_arguments_are_invalid():
    L = ep.lib()
    assert L.enprop_ctx_create(0, None) == ep.ERR_INVALID
    assert L.enprop_spmv(None, 4, 1, 1, None, None, None, None, None) == ep.ERR_INVALID
    assert L.enprop_cg(None, 4, 1, None, None, None, None, None, None, None, None, None,
                       None) == ep.ERR_INVALID


def test_draw_samples_and_pack_are_the_reference_sequence():
    """enprop_draw_samples / enprop_pack_sample_group (samples.cpp:7-18,
    samples.hpp:18-31) on the host, bitwise against the reference's golden
    draws (tests/golden: draw_samples(0, 8, 5), draw_samples(515, 4, 5))."""
    g = np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))
    a = ep.draw_samples(0, 8, 5).numpy()
    assert (bits(a) == bits(g["samples_seed0"])).all()
    b = ep.draw_samples(515, 4, 5).numpy()
    assert (bits(b) == bits(g["samples_seed515"])).all()
    # a longer draw continues the same stream
    assert (bits(ep.draw_samples(0, 20, 5).numpy()[:8]) == bits(a)).all()
    packed = ep.pack_sample_group(torch.as_tensor(a), 4, 4).numpy()
    assert (bits(packed) == bits(np.ascontiguousarray(a[4:8].T))).all()
    assert ep.draw_samples(3, 0, 2).shape == (0, 2)
    with pytest.raises(ValueError):
        ep.draw_samples(0, 4, 0)
    with pytest.raises(ValueError):
        ep.draw_samples(0, -1, 3)
    with pytest.raises(ValueError):
        ep.pack_sample_group(torch.as_tensor(a), 4, 5)  # runs past the pool
