"""Halo timing model: enprop_fit_halo_model and
enprop_predicted_speedup are host functions of the C ABI, so they are checked
here on CPU, bitwise against the reference's fit_halo_model / predicted_speedup
(halo.cpp:156-188) compiled from its sources (oracle/_ref)."""
import os

import numpy as np
import pytest

import paper_1511_03703_b200 as ep
from oracles import REF_SO, RefLib, bits

needs_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
needs_lib = pytest.mark.skipif(not os.path.exists(ep.LIB_PATH), reason="library not built")


@needs_ref
@needs_lib
def test_fit_halo_model_bitwise_equals_reference():
    R = RefLib()
    rng = np.random.default_rng(7)
    for trial in range(50):
        n = int(rng.integers(2, 12))
        s = rng.choice([1, 2, 4, 8, 16, 32], size=n).astype(np.float64)
        if np.all(s == s[0]):
            s[0] += 1.0
        t = 2e-6 + 3e-7 * s + rng.normal(0, 1e-7, n)
        rc, ref = R.fit_halo_model(s, t)
        assert rc == 0
        got = ep.fit_halo_model(list(zip(s, t)))
        assert (bits(np.array(got)) == bits(np.array(ref))).all()
        for q in (1.0, 4.0, 32.0):
            rc, sp = R.predicted_speedup(got[0], got[1], q)
            assert rc == 0 and ep.predicted_speedup(got[0], got[1], q) == sp


@needs_lib
def test_fit_halo_model_known_line_and_errors():
    a, b, rss = ep.fit_halo_model([(1, 3.0), (2, 5.0), (4, 9.0)])  # t = 1 + 2 s
    assert (a, b, rss) == (1.0, 2.0, 0.0)
    assert ep.predicted_speedup(1.0, 0.0, 8.0) == 8.0  # latency-only: s-fold speedup
    with pytest.raises(ValueError):
        ep.fit_halo_model([(1, 1.0)])
    with pytest.raises(ValueError):
        ep.fit_halo_model([(4, 1.0), (4, 2.0)])
    with pytest.raises(ValueError):
        ep.predicted_speedup(1.0, 1.0, 0.5)
    with pytest.raises(ValueError):
        ep.predicted_speedup(0.0, 0.0, 2.0)


def test_exchange_trace_csv_is_the_reference_format(tmp_path):
    """enprop_write_exchange_trace_csv writes the same bytes as the reference's
    write_exchange_trace_csv (halo.cpp:192-202), and fails on an unwritable path
    (the reference throws runtime_error there)."""
    from oracles import RefLib
    R = RefLib()
    recs = [(0, 1, 81 * 2 * 8, 1.25e-6), (1, 0, 1296, 2.5000000000000004e-06), (1, 2, 1296, 3.1e-06),
            (2, 1, 1296, 1.0 / 3.0)]
    a, b = tmp_path / "ours.csv", tmp_path / "ref.csv"
    ep.write_exchange_trace_csv(str(a), recs)
    assert R.write_trace_csv(str(b), recs) == 0
    assert a.read_bytes() == b.read_bytes()
    assert a.read_text().splitlines()[0] == "rank,neighbor,bytes,virtual_time"
    with pytest.raises(ValueError):
        ep.write_exchange_trace_csv("/nonexistent-dir/trace.csv", recs)
