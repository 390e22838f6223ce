"""TEST INFRASTRUCTURE: ctypes bindings for the CPU checkers.

* ``Oracle``  — oracle/liboracle.so, the plain-C restatement of the reference
  hot path (oracle/enprop_oracle.c).
* ``RefLib``  — oracle/_ref/libenprop_ref.so, the unmodified reference sources
  (/root/reference/proj) compiled with a thin extern "C" shim
  (oracle/ref_capi.cpp).  Built here by oracle/Makefile; the prebuilt .so
  travels to the GPU box, which never reads /root/reference.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs use these.
"""
from __future__ import annotations

import ctypes as C
import os
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libenprop_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)

DOT_SERIAL, DOT_CANONICAL = 0, 1
CG_COUPLED, CG_UNCOUPLED = 0, 1
TILE_ROWS = 16


def dptr(a):
    return None if a is None else a.ctypes.data_as(_dp)


def iptr(a):
    return None if a is None else a.ctypes.data_as(_ip)


def graph_nnz(n: int) -> int:
    t = 3 * (n + 1) - 2
    return t * t * t


class KlField(C.Structure):
    _fields_ = [
        ("m", C.c_int),
        ("mean", C.c_double), ("sigma", C.c_double), ("corr_length", C.c_double),
        ("axis_freq", C.c_double * 64), ("axis_eig", C.c_double * 64),
        ("axis_invnorm", C.c_double * 64), ("axis_cos", C.c_int * 64),
        ("mode_axes", (C.c_int * 3) * 64),
        ("mode_eig", C.c_double * 64), ("mode_sqrt_eig", C.c_double * 64),
    ]


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = L = C.CDLL(path)
        L.or_graph_nnz.restype = C.c_int64
        L.or_dot.restype = C.c_double
        L.or_draw_samples.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp]
        L.or_kl_init.argtypes = [C.POINTER(KlField), C.c_int, C.c_double, C.c_double, C.c_double]
        L.or_assemble.argtypes = [C.c_int, C.c_int, C.POINTER(KlField), C.c_double, C.c_double,
                                  _dp, _dp, _dp, C.c_int, C.c_double, C.c_double, _dp, _dp]
        L.or_apply_dirichlet.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _ip, _ip, _dp, _dp, _dp]
        L.or_spmv.argtypes = [C.c_int, C.c_int, _ip, _ip, _dp, _dp, _dp]
        L.or_spmv_outer.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, _dp, _dp]
        L.or_dot_lanes.argtypes = [C.c_int, C.c_int64, _dp, _dp, C.c_int, C.c_int, C.c_int, _dp]
        L.or_dot.argtypes = [C.c_int, C.c_int64, _dp, _dp, C.c_int, C.c_int, C.c_int]
        L.or_axpby.argtypes = [C.c_int, C.c_int64, C.c_int, _dp, _dp, _dp, _dp]
        L.or_pcg.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _ip, _ip, _dp,
                             _dp, C.c_double, C.c_int, _dp, _ip, _dp, _ip, _ip]

    def draw_samples(self, seed, count, m):
        out = np.empty((count, m))
        self.lib.or_draw_samples(seed, count, m, dptr(out))
        return out

    def graph(self, n):
        rows = (n + 1) ** 3
        rm = np.empty(rows + 1, np.int32)
        ce = np.empty(graph_nnz(n), np.int32)
        self.lib.or_build_graph(n, iptr(rm), iptr(ce))
        return rm, ce

    def kl(self, m, mean=1.0, sigma=0.1, L=1.0):
        f = KlField()
        st = self.lib.or_kl_init(C.byref(f), m, mean, sigma, L)
        if st:
            raise ValueError("or_kl_init: invalid field parameters")
        return f

    def assemble(self, s, n, field, y, u=None, alpha=0.0, beta=0.0, velocity=(1.0, 0.0, 0.0),
                 dirichlet=True, bc=(1.0, 0.0)):
        rows = (n + 1) ** 3
        vals = np.empty((graph_nnz(n), s))
        res = np.empty((rows, s))
        vel = np.array(velocity, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1, s)
        u = None if u is None else np.ascontiguousarray(u, dtype=np.float64)
        self.lib.or_assemble(s, n, C.byref(field), alpha, beta, dptr(vel), dptr(u), dptr(y),
                             int(dirichlet), bc[0], bc[1], dptr(vals), dptr(res))
        return vals, res

    def apply_dirichlet(self, s, n, row_map, col_entry, values, residual, u=None, bc=(1.0, 0.0)):
        self.lib.or_apply_dirichlet(s, n, bc[0], bc[1], iptr(row_map), iptr(col_entry),
                                    dptr(u), dptr(values), dptr(residual))

    def spmv(self, s, row_map, col_entry, values, x):
        rows = len(row_map) - 1
        z = np.empty((rows, s))
        self.lib.or_spmv(s, rows, iptr(row_map), iptr(col_entry), dptr(values), dptr(x), dptr(z))
        return z

    def spmv_outer(self, s, row_map, col_entry, values, x, cols=None):
        """values [s][nnz], x [s][cols] -> z [s][rows] (kernels.hpp:38-56)."""
        rows = len(row_map) - 1
        cols = rows if cols is None else cols
        z = np.empty((s, rows))
        self.lib.or_spmv_outer(s, rows, cols, iptr(row_map), iptr(col_entry), dptr(values), dptr(x), dptr(z))
        return z

    def dot_lanes(self, s, u, v, mode=DOT_SERIAL, tile=TILE_ROWS, seg=4096):
        out = np.empty(s)
        self.lib.or_dot_lanes(s, u.shape[0], dptr(u), dptr(v), mode, tile, seg, dptr(out))
        return out

    def dot(self, s, u, v, mode=DOT_SERIAL, tile=TILE_ROWS, seg=4096):
        return self.lib.or_dot(s, u.shape[0], dptr(u), dptr(v), mode, tile, seg)

    def pcg(self, s, row_map, col_entry, values, b, tol, maxit, flavour=CG_COUPLED,
            mode=DOT_SERIAL, tile=TILE_ROWS, seg=4096):
        rows = len(row_map) - 1
        x = np.empty((rows, s))
        lanes = s if flavour == CG_UNCOUPLED else 1
        it = np.zeros(lanes, np.int32)
        hl = np.zeros(lanes, np.int32)
        hist = np.empty((maxit + 1, lanes))
        ls = np.zeros(s, np.int32)
        st = self.lib.or_pcg(s, flavour, mode, tile, seg, rows, iptr(row_map), iptr(col_entry),
                             dptr(values), dptr(b), tol, maxit, dptr(x), iptr(it), dptr(hist),
                             iptr(hl), iptr(ls))
        return dict(status=st, x=x, iterations=it, history=hist, hist_len=hl, lane_status=ls)


class RefLib:
    """The unmodified reference, through oracle/ref_capi.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        self.lib = L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_graph_nnz.restype = C.c_int64
        L.ref_assemble.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                   C.c_double, C.c_double, C.c_double, _dp, _dp, _dp, C.c_int,
                                   C.c_double, C.c_double, _dp, _dp]
        L.ref_kl_describe.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, _ip, _dp, _dp,
                                      _dp, _dp, _ip]
        L.ref_kl_evaluate.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, _dp,
                                      _dp, _dp]
        L.ref_apply_dirichlet.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _dp, _dp, _dp]
        L.ref_spmv.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, _dp, _dp]
        L.ref_spmv_outer.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, _dp, _dp]
        L.ref_fit_halo_model.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.ref_predicted_speedup.argtypes = [C.c_double, C.c_double, C.c_double, _dp]
        L.ref_newton_identity.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                          C.c_double, C.c_double, C.c_double, _dp, _dp, C.c_double,
                                          C.c_double, C.c_double, C.c_int, C.c_double, C.c_int, _dp,
                                          _ip, _ip, _dp, _ip]
        L.ref_dot.argtypes = [C.c_int, C.c_int64, _dp, _dp, _dp]
        L.ref_axpby.argtypes = [C.c_int, C.c_int64, C.c_int, _dp, _dp, _dp, _dp]
        L.ref_pcg.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, _dp, C.c_double, C.c_int,
                              _dp, _ip, _dp, _ip]
        L.ref_draw_samples.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp]
        L.ref_partition.argtypes = [C.c_int, C.c_int, _ip]
        L.ref_distributed_spmv.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _ip]
        L.ref_time_group.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                     C.c_double, C.c_uint64, C.c_int, C.c_double, C.c_int, _dp, _ip]
        _mg = [C.c_int, C.c_int, C.c_int, _ip, _ip, _dp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int]
        L.ref_mg_describe.argtypes = _mg + [_ip, _ip, C.c_int, _dp]
        L.ref_mg_vcycle.argtypes = _mg + [_dp, _dp]
        L.ref_mg_pcg.argtypes = _mg + [_dp, C.c_double, C.c_int, _dp, _ip, _dp, _ip]
        L.ref_newton_mg.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                    C.c_double, C.c_double, _dp, _dp, C.c_double, C.c_double, C.c_double,
                                    C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.c_int, _dp, _ip, _ip, _dp, _ip]
        L.ref_write_trace_csv.argtypes = [C.c_char_p, C.c_int, _ip, _ip, C.POINTER(C.c_int64), _dp]
        L.ref_time_spmv.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                    C.c_uint64, C.c_int, _dp]

    def _check(self, st):
        if st not in (0,):
            raise RuntimeError(self.lib.ref_last_error().decode())

    def graph(self, n):
        rows = (n + 1) ** 3
        rm = np.empty(rows + 1, np.int32)
        ce = np.empty(graph_nnz(n), np.int32)
        self._check(self.lib.ref_build_graph(n, iptr(rm), iptr(ce)))
        return rm, ce

    def entry_of_pair(self, n):
        out = np.empty(n ** 3 * 64, np.int32)
        self._check(self.lib.ref_entry_of_pair(n, iptr(out)))
        return out

    def kl_describe(self, m, mean=1.0, sigma=0.1, L=1.0):
        axes = np.empty((m, 3), np.int32)
        eig = np.empty(m); af = np.empty(m); ae = np.empty(m); ai = np.empty(m)
        ac = np.empty(m, np.int32)
        self._check(self.lib.ref_kl_describe(m, mean, sigma, L, iptr(axes), dptr(eig), dptr(af),
                                             dptr(ae), dptr(ai), iptr(ac)))
        return dict(mode_axes=axes, mode_eig=eig, axis_freq=af, axis_eig=ae, axis_invnorm=ai,
                    axis_cos=ac)

    def kl_evaluate(self, s, m, x3, y, mean=1.0, sigma=0.1, L=1.0):
        out = np.empty(s)
        x3 = np.asarray(x3, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        self._check(self.lib.ref_kl_evaluate(s, m, mean, sigma, L, dptr(x3), dptr(y), dptr(out)))
        return out

    def assemble(self, s, n, m, y, mean=1.0, sigma=0.1, L=1.0, u=None, alpha=0.0, beta=0.0,
                 velocity=(1.0, 0.0, 0.0), dirichlet=True, bc=(1.0, 0.0), scalar=False):
        rows = (n + 1) ** 3
        vals = np.empty((graph_nnz(n), s))
        res = np.empty((rows, s))
        vel = np.array(velocity, dtype=np.float64)
        y = np.ascontiguousarray(y, np.float64)
        u = None if u is None else np.ascontiguousarray(u, np.float64)
        self._check(self.lib.ref_assemble(s, int(scalar), n, m, mean, sigma, L, alpha, beta,
                                          dptr(vel), dptr(u), dptr(y), int(dirichlet), bc[0],
                                          bc[1], dptr(vals), dptr(res)))
        return vals, res

    def spmv(self, s, row_map, col_entry, values, x, cols=None):
        rows = len(row_map) - 1
        cols = rows if cols is None else cols
        z = np.empty((rows, s))
        self._check(self.lib.ref_spmv(s, rows, cols, iptr(row_map), iptr(col_entry),
                                      dptr(values), dptr(x), dptr(z)))
        return z

    def spmv_outer(self, s, row_map, col_entry, values, x, cols=None):
        rows = len(row_map) - 1
        cols = rows if cols is None else cols
        z = np.empty((s, rows))
        self._check(self.lib.ref_spmv_outer(s, rows, cols, iptr(row_map), iptr(col_entry),
                                            dptr(values), dptr(x), dptr(z)))
        return z

    def newton_identity(self, s, n, m, y, sigma=0.2, mean=1.0, L=1.0, alpha=0.0, beta=0.0,
                        velocity=(1.0, 0.0, 0.0), bc=(1.0, 0.0), tol=1e-8, max_newton=20,
                        lin_tol=1e-8, lin_maxit=1000):
        """fem.hpp:265-302 with IdentityPreconditioner, from the reference's pieces
        (oracle/ref_capi.cpp ref_newton_identity). Returns (rc, u, its, cg, norms)."""
        rows = (n + 1) ** 3
        u = np.zeros((rows, s))
        it, cg, nn = (np.zeros(1, np.int32) for _ in range(3))
        norms = np.zeros(max_newton + 2)
        vel = np.array(velocity, dtype=np.float64)
        rc = self.lib.ref_newton_identity(s, 0, n, m, mean, sigma, L, alpha, beta, dptr(vel),
                                          dptr(np.ascontiguousarray(y, dtype=np.float64)), bc[0], bc[1],
                                          tol, max_newton, lin_tol, lin_maxit, dptr(u), iptr(it),
                                          iptr(cg), dptr(norms), iptr(nn))
        return rc, u, int(it[0]), int(cg[0]), list(norms[:nn[0]])

    def fit_halo_model(self, s, t):
        s, t = np.ascontiguousarray(s, dtype=np.float64), np.ascontiguousarray(t, dtype=np.float64)
        out = np.zeros(3)
        rc = self.lib.ref_fit_halo_model(len(s), dptr(s), dptr(t), dptr(out[0:1]), dptr(out[1:2]), dptr(out[2:3]))
        return rc, tuple(out)

    def predicted_speedup(self, a, b, s):
        out = np.zeros(1)
        rc = self.lib.ref_predicted_speedup(a, b, s, dptr(out))
        return rc, float(out[0])

    def dot(self, s, u, v):
        out = C.c_double()
        self._check(self.lib.ref_dot(s, u.shape[0], dptr(u), dptr(v), C.byref(out)))
        return out.value

    def axpby(self, s, alpha, x, beta, y, per_lane=False):
        a = np.atleast_1d(np.asarray(alpha, np.float64))
        b = np.atleast_1d(np.asarray(beta, np.float64))
        y = y.copy()
        self._check(self.lib.ref_axpby(s, x.shape[0], int(per_lane), dptr(a), dptr(x), dptr(b),
                                       dptr(y)))
        return y

    def pcg(self, s, row_map, col_entry, values, b, tol, maxit, scalar=False):
        rows = len(row_map) - 1
        x = np.zeros((rows, s))
        it = C.c_int()
        hl = C.c_int()
        hist = np.empty(maxit + 2)
        st = self.lib.ref_pcg(s, int(scalar), rows, iptr(row_map), iptr(col_entry), dptr(values),
                              dptr(b), tol, maxit, dptr(x), C.byref(it), dptr(hist), C.byref(hl))
        return dict(status=st, x=x, iterations=it.value, history=hist[: hl.value].copy())

    def pcg_uncoupled(self, s, row_map, col_entry, values, b, tol, maxit):
        """s x pcg_solve<double> on extracted components (bench.cpp:340-349)."""
        out = []
        for e in range(s):
            ve = np.ascontiguousarray(values[:, e]).reshape(-1, 1)
            be = np.ascontiguousarray(b[:, e]).reshape(-1, 1)
            out.append(self.pcg(1, row_map, col_entry, ve, be, tol, maxit, scalar=True))
        return out

    def draw_samples(self, seed, count, m):
        out = np.empty((count, m))
        self._check(self.lib.ref_draw_samples(seed, count, m, dptr(out)))
        return out

    def write_trace_csv(self, path, records):
        """write_exchange_trace_csv (halo.cpp:192-202); records: (rank, neighbor, bytes, time)"""
        n = len(records)
        rk = np.array([r[0] for r in records], np.int32)
        nb = np.array([r[1] for r in records], np.int32)
        by = np.array([r[2] for r in records], np.int64)
        t = np.array([r[3] for r in records], np.float64)
        return self.lib.ref_write_trace_csv(path.encode(), n, iptr(rk), iptr(nb),
                                            by.ctypes.data_as(C.POINTER(C.c_int64)), dptr(t))

    def newton_mg(self, s, n, m, y, sigma=0.1, alpha=0.0, beta=0.0, velocity=(1.0, 0.0, 0.0), tol=1e-8,
                  max_newton=20, lin_tol=1e-8, lin_maxit=1000, opts=(500, 2, 30.0, 1.1, 40), scalar=False):
        """The reference's own newton_solve (fem.hpp:265-302), MG-preconditioned."""
        u = np.zeros(((n + 1) ** 3, s))
        it, cg, nn = C.c_int(), C.c_int(), C.c_int()
        norms = np.zeros(max_newton + 2)
        vel = np.array(velocity, dtype=np.float64)
        st = self.lib.ref_newton_mg(s, int(scalar), n, m, 1.0, sigma, 1.0, alpha, beta, dptr(vel),
                                    dptr(np.ascontiguousarray(y)), 1.0, 0.0, tol, max_newton, lin_tol, lin_maxit,
                                    *opts, dptr(u), C.byref(it), C.byref(cg), dptr(norms), C.byref(nn))
        return dict(status=st, u=u, iterations=it.value, total_cg=cg.value, norms=norms[: nn.value].copy())

    # ---- multigrid.hpp (f4): MgOptions = (threshold, degree, ratio, boost, power iterations)
    def mg_describe(self, s, row_map, col_entry, values, opts=(500, 2, 30.0, 1.1, 40), scalar=False):
        rows = len(row_map) - 1
        nl = C.c_int()
        lr = np.zeros(64, np.int32)
        lm = np.zeros((64, s))
        self._check(self.lib.ref_mg_describe(s, int(scalar), rows, iptr(row_map), iptr(col_entry),
                                             dptr(np.ascontiguousarray(values)), *opts, C.byref(nl), iptr(lr),
                                             64, dptr(lm)))
        return lr[:nl.value].copy(), lm[:max(nl.value - 1, 0)].copy()

    def mg_vcycle(self, s, row_map, col_entry, values, b, x, opts=(500, 2, 30.0, 1.1, 40), scalar=False):
        rows = len(row_map) - 1
        x = np.ascontiguousarray(x, dtype=np.float64).copy()
        self._check(self.lib.ref_mg_vcycle(s, int(scalar), rows, iptr(row_map), iptr(col_entry),
                                           dptr(np.ascontiguousarray(values)), *opts,
                                           dptr(np.ascontiguousarray(b)), dptr(x)))
        return x

    def mg_pcg(self, s, row_map, col_entry, values, b, tol, maxit, opts=(500, 2, 30.0, 1.1, 40), scalar=False):
        rows = len(row_map) - 1
        x = np.zeros((rows, s))
        it = C.c_int()
        hl = C.c_int()
        hist = np.empty(maxit + 2)
        st = self.lib.ref_mg_pcg(s, int(scalar), rows, iptr(row_map), iptr(col_entry),
                                 dptr(np.ascontiguousarray(values)), *opts, dptr(np.ascontiguousarray(b)), tol,
                                 maxit, dptr(x), C.byref(it), dptr(hist), C.byref(hl))
        return dict(status=st, x=x, iterations=it.value, history=hist[: hl.value].copy())

    def partition(self, n, p):
        out = np.empty((p, 2), np.int32)
        self._check(self.lib.ref_partition(n, p, iptr(out)))
        return out

    def distributed_spmv(self, s, n, p, values, x):
        z = np.empty(((n + 1) ** 3, s))
        nm = C.c_int()
        self._check(self.lib.ref_distributed_spmv(s, n, p, dptr(values), dptr(x), dptr(z),
                                                  C.byref(nm)))
        return z, nm.value


def pack_group(samples: np.ndarray, s: int, group: int = 0) -> np.ndarray:
    """pack_sample_group<S> (samples.hpp:18-31): out[j][e] = samples[g*s+e][j]."""
    return np.ascontiguousarray(samples[group * s:(group + 1) * s].T)


def bits(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a).view(np.uint64)
