"""enprop_b200 — B200-native ensemble hot path of arXiv 1511.03703.

Python mirror of the reference library's interfaces (``enprop``:
``/root/reference/proj/include/enprop``) over the C ABI in
``include/enprop_b200.h`` (``lib/libenprop_b200.so``, sm_100a only).  PyTorch
is used for device memory and streams only; every computation runs in the
library's CUDA kernels.  There is no CPU fallback: without a B200 the calls
raise ``EnpropError``.

Names follow the reference: ``KlField`` parameters (kl.hpp:39-95),
``PdeCoefficients`` (fem.hpp:21-25), ``DirichletBc`` (fem.hpp:29-32),
``SolverConfig`` / ``SolverError`` (pcg.hpp:15-31), ``spmv`` / ``dot`` /
``norm2`` / ``axpby`` (kernels.hpp:15-85), ``assemble`` / ``apply_dirichlet``
(fem.hpp:115-243), ``pcg_solve`` (pcg.hpp:52-103).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ENPROP_B200_LIB") or os.path.join(_HERE, "lib", "libenprop_b200.so")  # override: A/B builds

OK, ERR_INVALID, ERR_NO_CONVERGENCE, ERR_INDEFINITE, ERR_CUDA, ERR_OOM = range(6)
DOT_SERIAL, DOT_CANONICAL = 0, 1
CG_COUPLED, CG_UNCOUPLED = 0, 1
TILE_ROWS = 16
OPT_FUSED_DIRECTION = 1
OPT_SPMV_PIPELINE = 2
OPT_SYMMETRIC_STORAGE = 3
OPT_SPMV_VARIANT = 5
OPT_PDL = 6
OPT_GRAPHS = 7
WIDTHS = (1, 2, 4, 8, 16, 32)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p


class EnpropError(RuntimeError):
    """A CUDA / library failure (ENPROP_ERR_CUDA, ENPROP_ERR_OOM)."""


class SolverError(RuntimeError):
    """pcg_solve failure (pcg.hpp:22-31): carries the residual history."""

    def __init__(self, what: str, history, status: int, iterations=None):
        super().__init__(what)
        self._history = history
        self.status = status
        self.iterations = iterations

    def history(self):
        return self._history


class _KlParams(C.Structure):
    _fields_ = [("num_terms", C.c_int), ("mean", C.c_double), ("sigma", C.c_double),
                ("correlation_length", C.c_double)]


class _Coeffs(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("velocity", C.c_double * 3)]


class _Bc(C.Structure):
    _fields_ = [("x0_value", C.c_double), ("x1_value", C.c_double)]


class _CgOptions(C.Structure):
    _fields_ = [("flavour", C.c_int), ("dot_mode", C.c_int), ("seg_rows", C.c_int),
                ("tol", C.c_double), ("max_iterations", C.c_int), ("check_every", C.c_int)]


class _NewtonOptions(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iterations", C.c_int), ("linear", _CgOptions)]


class _MgOptions(C.Structure):
    _fields_ = [("coarse_row_threshold", C.c_int), ("chebyshev_degree", C.c_int),
                ("eigenvalue_ratio", C.c_double), ("eigenvalue_boost", C.c_double),
                ("power_iterations", C.c_int)]


class _ExchangeRecord(C.Structure):
    _fields_ = [("rank", C.c_int), ("neighbor", C.c_int), ("bytes", C.c_int64), ("time", C.c_double)]


class _ProblemDesc(C.Structure):
    _fields_ = [("cells_per_axis", C.c_int), ("ensemble_size", C.c_int), ("kl", _KlParams),
                ("coeffs", _Coeffs), ("bc", _Bc)]


@dataclass
class KlField:
    """KlField(num_terms, mean, sigma, correlation_length) (kl.hpp:39-95)."""
    num_terms: int = 5
    mean: float = 1.0
    sigma: float = 0.1
    correlation_length: float = 1.0

    def _c(self):
        return _KlParams(self.num_terms, self.mean, self.sigma, self.correlation_length)


@dataclass
class PdeCoefficients:
    alpha: float = 0.0
    beta: float = 0.0
    velocity: Sequence[float] = (1.0, 0.0, 0.0)

    def _c(self):
        return _Coeffs(self.alpha, self.beta, (C.c_double * 3)(*self.velocity))


@dataclass
class DirichletBc:
    x0_value: float = 1.0
    x1_value: float = 0.0

    def _c(self):
        return _Bc(self.x0_value, self.x1_value)


@dataclass
class SolverConfig:
    """SolverConfig (pcg.hpp:15-18) plus the device-side choices."""
    tol: float = 1e-8
    max_iterations: int = 1000
    flavour: int = CG_COUPLED
    dot_mode: int = DOT_SERIAL
    seg_rows: int = 0
    check_every: int = 16

    def _c(self):
        return _CgOptions(self.flavour, self.dot_mode, self.seg_rows, self.tol,
                          self.max_iterations, self.check_every)


@dataclass
class MgOptions:
    """MgOptions (multigrid.hpp:14-20)."""
    coarse_row_threshold: int = 500
    chebyshev_degree: int = 2
    eigenvalue_ratio: float = 30.0
    eigenvalue_boost: float = 1.1
    power_iterations: int = 40

    def _c(self):
        return _MgOptions(self.coarse_row_threshold, self.chebyshev_degree, self.eigenvalue_ratio,
                          self.eigenvalue_boost, self.power_iterations)


@dataclass
class NewtonOptions:
    """NewtonOptions (fem.hpp:244-249); the linear solves use the identity
    preconditioner (no multigrid block)."""
    tol: float = 1e-8
    max_iterations: int = 20
    linear: SolverConfig = None

    def _c(self):
        return _NewtonOptions(self.tol, self.max_iterations, (self.linear or SolverConfig())._c())


@dataclass
class NewtonResult:
    """NewtonResult (fem.hpp:251-257); the solution stays on the device
    (Problem.solution)."""
    iterations: int
    total_cg_iterations: int
    residual_norms: list


_lib = None


def lib() -> C.CDLL:
    """Load lib/libenprop_b200.so; raise loudly when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise EnpropError(f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
                          "(enprop_b200 has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.enprop_last_error.restype = C.c_char_p
    L.enprop_mesh_nnz.restype = C.c_int64
    L.enprop_ctx_launch_count.restype = C.c_int64
    L.enprop_ctx_stream.restype = _vp
    L.enprop_ctx_create.argtypes = [C.c_int, C.POINTER(_vp)]
    L.enprop_ctx_destroy.argtypes = [_vp]
    L.enprop_ctx_set_stream.argtypes = [_vp, _vp]
    L.enprop_ctx_stream.argtypes = [_vp]
    L.enprop_ctx_synchronize.argtypes = [_vp]
    L.enprop_ctx_launch_count.argtypes = [_vp]
    L.enprop_ctx_profile.argtypes = [_vp, C.c_int, _dp, C.POINTER(C.c_int64)]
    L.enprop_ctx_set_option.argtypes = [_vp, C.c_int, C.c_int]
    L.enprop_ctx_profile_detail.argtypes = [_vp, _dp, C.POINTER(C.c_int64)]
    L.enprop_build_node_graph.argtypes = [_vp, C.c_int, _vp, _vp]
    L.enprop_draw_samples.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp]
    L.enprop_pack_sample_group.argtypes = [_dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
    L.enprop_kl_describe.argtypes = [C.POINTER(_KlParams), _ip, _dp, _dp, _dp, _dp, _ip]
    L.enprop_assemble.argtypes = [_vp, C.c_int, C.c_int, C.POINTER(_KlParams), C.POINTER(_Coeffs),
                                  _vp, _vp, _vp, _vp, _vp, C.POINTER(_Bc)]
    L.enprop_apply_dirichlet.argtypes = [_vp, C.c_int, C.c_int, C.POINTER(_Bc), _vp, _vp, _vp,
                                         _vp, _vp]
    L.enprop_spmv.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp]
    L.enprop_spmv_small_config.argtypes = [C.c_int, _ip, _ip, _ip, _ip]
    L.enprop_dot.argtypes = [_vp, C.c_int, C.c_int64, _vp, _vp, C.c_int, C.c_int, _dp, _dp]
    L.enprop_axpby.argtypes = [_vp, C.c_int, C.c_int64, C.c_int, _dp, _vp, _dp, _vp]
    L.enprop_cg.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp,
                            C.POINTER(_CgOptions), _ip, _ip, _dp, _ip]
    L.enprop_problem_create.argtypes = [_vp, C.POINTER(_ProblemDesc), C.POINTER(_vp)]
    L.enprop_problem_destroy.argtypes = [_vp]
    L.enprop_problem_views.argtypes = [_vp, _ip, C.POINTER(C.c_int64), C.POINTER(_vp),
                                       C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp),
                                       C.POINTER(_vp)]
    L.enprop_problem_assemble.argtypes = [_vp, _vp]
    L.enprop_problem_storage.argtypes = [_vp, C.POINTER(C.c_int64), C.POINTER(_vp)]
    L.enprop_problem_expand_values.argtypes = [_vp, _vp]
    L.enprop_problem_solve.argtypes = [_vp, C.POINTER(_CgOptions), _ip, _ip, _dp, _ip]
    L.enprop_problem_solve_host.argtypes = [_vp, _vp, _vp, C.POINTER(_CgOptions), _ip, _ip]
    L.enprop_nccl_unique_id.argtypes = [_vp, C.c_size_t]
    L.enprop_dist_create.argtypes = [_vp, C.POINTER(_ProblemDesc), C.c_int, C.c_int, _vp, C.POINTER(_vp)]
    L.enprop_problem_newton_mg.argtypes = [_vp, _vp, C.POINTER(_NewtonOptions), C.POINTER(_MgOptions), _ip, _ip,
                                           _dp, _ip]
    L.enprop_mg_build.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp, _vp, C.POINTER(_MgOptions), C.POINTER(_vp)]
    L.enprop_mg_destroy.argtypes = [_vp]
    L.enprop_mg_describe.argtypes = [_vp, _ip, _ip, C.c_int, _dp]
    L.enprop_mg_vcycle.argtypes = [_vp, _vp, _vp]
    L.enprop_mg_pcg.argtypes = [_vp, _vp, _vp, C.POINTER(_CgOptions), _ip, _ip, _dp, _ip]
    L.enprop_dist_create_ipc.argtypes = [_vp, C.POINTER(_ProblemDesc), C.c_int, C.c_int, C.c_char_p, C.POINTER(_vp)]
    L.enprop_dist_destroy.argtypes = [_vp]
    L.enprop_dist_exchange_trace.argtypes = [_vp, C.POINTER(_ExchangeRecord), C.c_int, _ip, _dp]
    L.enprop_write_exchange_trace_csv.argtypes = [C.c_char_p, C.POINTER(_ExchangeRecord), C.c_int]
    L.enprop_dist_assemble.argtypes = [_vp, _vp]
    L.enprop_dist_solve.argtypes = [_vp, C.POINTER(_CgOptions), _ip, _ip]
    L.enprop_dist_newton.argtypes = [_vp, _vp, C.POINTER(_NewtonOptions), _ip, _ip, _dp, _ip]
    L.enprop_dist_local_count.argtypes = [_vp]
    L.enprop_dist_stages.argtypes = [_vp, C.c_int, _ip, _ip]
    L.enprop_dist_local.argtypes = [_vp, C.c_int, _ip, _ip, _ip, C.POINTER(_vp)]
    _lib = L
    return L


def _err() -> str:
    return lib().enprop_last_error().decode(errors="replace")


def _check(rc: int, what: str = ""):
    if rc == OK:
        return
    msg = f"{what}: {_err()}" if what else _err()
    if rc == ERR_INVALID:
        raise ValueError(msg)  # std::invalid_argument in the reference
    raise EnpropError(msg)


def mesh_nnz(n: int) -> int:
    return int(lib().enprop_mesh_nnz(n))


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _need_cuda(t: torch.Tensor, dtype, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


class Context:
    """A device + stream.  By default it runs on torch's current stream so
    torch allocations and enprop kernels are ordered."""

    def __init__(self, device: int = 0, use_torch_stream: bool = True):
        self.device = device
        h = _vp()
        _check(lib().enprop_ctx_create(device, C.byref(h)), "enprop_ctx_create")
        self.h = h
        if use_torch_stream:
            self.set_stream(torch.cuda.current_stream(device).cuda_stream)

    def set_stream(self, stream_handle: int):
        _check(lib().enprop_ctx_set_stream(self.h, C.c_void_p(stream_handle)))

    def synchronize(self):
        _check(lib().enprop_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        return int(lib().enprop_ctx_launch_count(self.h))

    def set_option(self, option: int, value: int):
        """enprop_ctx_set_option (e.g. OPT_FUSED_DIRECTION); bitwise-neutral."""
        _check(lib().enprop_ctx_set_option(self.h, option, value), "set_option")

    def profile(self, enable: int = -1):
        """(total ms, launches) of CG SpMV kernels timed with CUDA events on
        this context's stream; enable=1/0 switches timing on/off and resets."""
        ms = C.c_double()
        cnt = C.c_int64()
        _check(lib().enprop_ctx_profile(self.h, enable, C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def profile_detail(self):
        """Per-phase CG totals since the last profile(1): dict of ms and count."""
        ms = (C.c_double * 11)()
        n = C.c_int64()
        _check(lib().enprop_ctx_profile_detail(self.h, ms, C.byref(n)))
        return dict(spmv=ms[0], fin_pq=ms[1], update=ms[2], fin_rr=ms[3], iteration=ms[4],
                    solve=ms[5], init=ms[6], loop=ms[7], early_exit=ms[8], direction=ms[9],
                    spmv_kernel=ms[10], iterations=n.value)

    def close(self):
        if getattr(self, "h", None):
            lib().enprop_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def kl_describe(kl: KlField):
    m = kl.num_terms
    axes = (C.c_int * (3 * m))()
    me, af, ae, ai = ((C.c_double * m)() for _ in range(4))
    ac = (C.c_int * m)()
    p = kl._c()
    _check(lib().enprop_kl_describe(C.byref(p), axes, me, af, ae, ai, ac), "KlField")
    return dict(mode_axes=[list(axes[3 * i:3 * i + 3]) for i in range(m)], mode_eig=list(me),
                axis_freq=list(af), axis_eig=list(ae), axis_invnorm=list(ai), axis_cos=list(ac))


def draw_samples(seed: int, count: int, num_terms: int) -> torch.Tensor:
    """draw_samples (samples.cpp:7-18): [count][num_terms] host doubles,
    bitwise the reference's mt19937_64 sequence."""
    if count < 0 or num_terms < 1:  # the library raises the reference's invalid_argument
        _check(lib().enprop_draw_samples(seed, count, num_terms, None), "draw_samples")
    out = torch.empty((count, num_terms), dtype=torch.float64)
    _check(lib().enprop_draw_samples(seed, count, num_terms,
                                     C.cast(out.data_ptr(), _dp) if out.numel() else None), "draw_samples")
    return out


def pack_sample_group(samples: torch.Tensor, s: int, group_start: int = 0) -> torch.Tensor:
    """pack_sample_group<s> (samples.hpp:18-31): out[j][e] = samples[group_start + e][j]
    ([num_terms][s] host doubles, the y layout of assemble)."""
    samples = samples.detach().to(torch.float64).contiguous().cpu()
    count, m = samples.shape
    out = torch.empty((m, s), dtype=torch.float64)
    _check(lib().enprop_pack_sample_group(C.cast(samples.data_ptr(), _dp), count, m, group_start, s,
                                          C.cast(out.data_ptr(), _dp)), "pack_sample_group")
    return out


def build_node_graph(ctx: Context, n: int):
    """build_node_graph(StructuredMesh(n)) (mesh.cpp:13-55) on the device."""
    if n < 1:
        raise ValueError("StructuredMesh: cells_per_axis must be at least 1")
    rows = (n + 1) ** 3
    dev = torch.device("cuda", ctx.device)
    rm = torch.empty(rows + 1, dtype=torch.int32, device=dev)
    ce = torch.empty(mesh_nnz(n), dtype=torch.int32, device=dev)
    _check(lib().enprop_build_node_graph(ctx.h, n, _ptr(rm), _ptr(ce)), "build_node_graph")
    return rm, ce


def assemble(ctx: Context, s: int, n: int, kl: KlField, y: torch.Tensor, row_map: torch.Tensor,
             coeffs: PdeCoefficients = None, u: Optional[torch.Tensor] = None,
             bc: Optional[DirichletBc] = None, values: Optional[torch.Tensor] = None,
             residual: Optional[torch.Tensor] = None):
    """assemble<Ensemble<s>> (fem.hpp:115-202); with ``bc`` also
    apply_dirichlet (fem.hpp:218-243) fused.  y is [num_terms][s]."""
    coeffs = coeffs or PdeCoefficients()
    rows = (n + 1) ** 3
    dev = y.device
    _need_cuda(y, torch.float64, "y")
    if y.numel() != kl.num_terms * s:
        raise ValueError("assemble: sample vector length mismatch")
    if u is not None:
        _need_cuda(u, torch.float64, "u")
        if u.numel() != rows * s:
            raise ValueError("assemble: solution vector length mismatch")
    if values is None:
        values = torch.empty((mesh_nnz(n), s), dtype=torch.float64, device=dev)
    if residual is None:
        residual = torch.empty((rows, s), dtype=torch.float64, device=dev)
    klp, cp = kl._c(), coeffs._c()
    bcp = bc._c() if bc is not None else None
    _check(lib().enprop_assemble(ctx.h, s, n, C.byref(klp), C.byref(cp), _ptr(u), _ptr(y),
                                 _ptr(row_map), _ptr(values), _ptr(residual),
                                 C.byref(bcp) if bcp is not None else None), "assemble")
    return values, residual


def apply_dirichlet(ctx: Context, s: int, n: int, bc: DirichletBc, row_map, col_entry, values,
                    residual, u: Optional[torch.Tensor] = None):
    bcp = bc._c()
    _check(lib().enprop_apply_dirichlet(ctx.h, s, n, C.byref(bcp), _ptr(row_map), _ptr(col_entry),
                                        _ptr(u), _ptr(values), _ptr(residual)), "apply_dirichlet")


def spmv(ctx: Context, s: int, row_map, col_entry, values, x, z=None, num_cols=None):
    """z = A x (kernels.hpp:15-26), bitwise equal to the reference per sample."""
    rows = row_map.numel() - 1
    cols = rows if num_cols is None else num_cols
    if x.numel() != cols * s:
        raise ValueError("spmv: x length must equal num_cols")
    if z is None:
        z = torch.empty((rows, s), dtype=torch.float64, device=x.device)
    _check(lib().enprop_spmv(ctx.h, s, rows, cols, _ptr(row_map), _ptr(col_entry), _ptr(values),
                             _ptr(x), _ptr(z)), "spmv")
    return z


def spmv_small_config(s: int) -> dict:
    """Diagnostics: the narrow-ensemble SpMV configuration enprop_spmv launches at width s."""
    r, nt, rc, md = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    _check(lib().enprop_spmv_small_config(s, C.byref(r), C.byref(nt), C.byref(rc), C.byref(md)))
    return dict(routed=bool(r.value), threads=nt.value, reg_cap=rc.value, stage_mode=md.value)


def spmv_outer(ctx: Context, ensemble_size: int, row_map, col_entry, values, x, z=None, num_cols=None):
    """z = A x on the sample-major layout (spmv_outer, kernels.hpp:38-56):
    values [s][nnz], x [s][num_cols], z [s][num_rows]; bitwise equal to the
    reference per component."""
    s = ensemble_size
    rows = row_map.numel() - 1
    cols = rows if num_cols is None else num_cols
    nnz = col_entry.numel()
    if x.numel() != cols * s:
        raise ValueError("spmv_outer: x length must equal num_cols*ensemble_size")
    if values.numel() != nnz * s:
        raise ValueError("spmv_outer: values length must equal nnz*ensemble_size")
    if z is None:
        z = torch.empty((s, rows), dtype=torch.float64, device=x.device)
    _check(lib().enprop_spmv_outer(ctx.h, s, rows, cols, nnz, _ptr(row_map), _ptr(col_entry),
                                   _ptr(values), _ptr(x), _ptr(z)), "spmv_outer")
    return z


def dot_lanes(ctx: Context, s: int, u, v, mode: int = DOT_SERIAL, seg_rows: int = 4096):
    if u.numel() != v.numel():
        raise ValueError("dot: length mismatch")
    lanes = (C.c_double * s)()
    coupled = C.c_double()
    _check(lib().enprop_dot(ctx.h, s, u.numel() // s, _ptr(u), _ptr(v), mode, seg_rows, lanes,
                            C.byref(coupled)), "dot")
    return list(lanes), coupled.value


def dot(ctx: Context, s: int, u, v, mode: int = DOT_SERIAL, seg_rows: int = 4096) -> float:
    """Coupled inner product (kernels.hpp:62-69)."""
    return dot_lanes(ctx, s, u, v, mode, seg_rows)[1]


def norm2(ctx: Context, s: int, u, mode: int = DOT_SERIAL, seg_rows: int = 4096) -> float:
    return math.sqrt(dot(ctx, s, u, u, mode, seg_rows))


def axpby(ctx: Context, s: int, alpha, x, beta, y):
    """y = alpha*x + beta*y (kernels.hpp:78-85); list coefficients = per lane."""
    per_lane = isinstance(alpha, (list, tuple))
    a = (C.c_double * (s if per_lane else 1))(*(alpha if per_lane else [alpha]))
    b = (C.c_double * (s if per_lane else 1))(*(beta if per_lane else [beta]))
    if x.numel() != y.numel():
        raise ValueError("axpby: length mismatch")
    _check(lib().enprop_axpby(ctx.h, s, x.numel() // s, int(per_lane), a, _ptr(x), b, _ptr(y)),
           "axpby")
    return y


@dataclass
class SolveResult:
    """SolveResult (pcg.hpp:33-38) plus per-lane data for uncoupled solves."""
    solution: torch.Tensor
    iterations: object
    residual_history: list
    lane_status: list = field(default_factory=list)


def _collect(cfg: SolverConfig, s: int, it, ls, hist, hl):
    if cfg.flavour != CG_UNCOUPLED:
        history = [hist[i] for i in range(hl[0])]
        return it[0], history, [ls[0]]
    history = [[hist[i * s + e] for i in range(hl[e])] for e in range(s)]
    return [it[e] for e in range(s)], history, [ls[e] for e in range(s)]


def pcg_solve(ctx: Context, s: int, row_map, col_entry, values, b, config: SolverConfig = None,
              raise_on_failure: bool = True) -> SolveResult:
    """Identity-preconditioned CG from x0 = 0 (pcg.hpp:52-103).  Coupled =
    pcg_solve<Ensemble<s>>; uncoupled = s x pcg_solve<double>."""
    cfg = config or SolverConfig()
    rows = row_map.numel() - 1
    if b.numel() != rows * s:
        raise ValueError("pcg_solve: right-hand side length mismatch")
    x = torch.empty((rows, s), dtype=torch.float64, device=b.device)
    lanes = s if cfg.flavour == CG_UNCOUPLED else 1
    it = (C.c_int * lanes)()
    ls = (C.c_int * lanes)()
    hl = (C.c_int * lanes)()
    hist = (C.c_double * ((cfg.max_iterations + 1) * lanes))()
    opt = cfg._c()
    rc = lib().enprop_cg(ctx.h, s, rows, _ptr(row_map), _ptr(col_entry), _ptr(values), _ptr(b),
                         _ptr(x), C.byref(opt), it, ls, hist, hl)
    iters, history, lstat = _collect(cfg, s, it, ls, hist, hl)
    if rc in (ERR_NO_CONVERGENCE, ERR_INDEFINITE):
        if raise_on_failure:
            raise SolverError(_err(), history, rc, iters)
    else:
        _check(rc, "pcg_solve")
    return SolveResult(x, iters, history, lstat)


class MgHierarchy:
    """build_hierarchy (multigrid.hpp:362-396) of an ensemble operator (device
    CRS, full storage, values [nnz][s]); vcycle() is one V-cycle
    (multigrid.hpp:402-425), pcg() is pcg_solve with MgPreconditioner in the
    reference's serial dot order (coupled, or uncoupled per-lane)."""

    def __init__(self, ctx: Context, s: int, row_map, col_entry, values, options: MgOptions = None):
        self.ctx, self.s = ctx, s
        self.rows = row_map.numel() - 1
        opt = (options or MgOptions())._c()
        h = _vp()
        _check(lib().enprop_mg_build(ctx.h, s, self.rows, _ptr(row_map), _ptr(col_entry), _ptr(values),
                                     C.byref(opt), C.byref(h)), "build_hierarchy")
        self.h = h

    def describe(self):
        """(rows per level, lambda_max per smoothed level [levels-1][s])"""
        nl = C.c_int()
        rows = (C.c_int * 64)()
        lm = (C.c_double * (64 * self.s))()
        _check(lib().enprop_mg_describe(self.h, C.byref(nl), rows, 64, lm))
        L = nl.value
        return [rows[k] for k in range(L)], [[lm[k * self.s + e] for e in range(self.s)] for k in range(L - 1)]

    def vcycle(self, b, x):
        _need_cuda(b, torch.float64, "b")
        _need_cuda(x, torch.float64, "x")
        _check(lib().enprop_mg_vcycle(self.h, _ptr(b), _ptr(x)), "vcycle")
        return x

    def pcg(self, b, config: SolverConfig = None, raise_on_failure: bool = True) -> SolveResult:
        cfg = config or SolverConfig()
        _need_cuda(b, torch.float64, "b")
        x = torch.empty((self.rows, self.s), dtype=torch.float64, device=b.device)
        lanes = self.s if cfg.flavour == CG_UNCOUPLED else 1
        it, ls, hl = ((C.c_int * lanes)() for _ in range(3))
        hist = (C.c_double * ((cfg.max_iterations + 1) * lanes))()
        opt = cfg._c()
        rc = lib().enprop_mg_pcg(self.h, _ptr(b), _ptr(x), C.byref(opt), it, ls, hist, hl)
        iters, history, lstat = _collect(cfg, self.s, it, ls, hist, hl)
        if rc in (ERR_NO_CONVERGENCE, ERR_INDEFINITE):
            if raise_on_failure:
                raise SolverError(_err(), history, rc, iters)
        else:
            _check(rc, "pcg_solve")
        return SolveResult(x, iters, history, lstat)

    def close(self):
        if getattr(self, "h", None):
            lib().enprop_mg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Problem:
    """Device-resident ensemble problem: node graph, KL tables, matrix and CG
    workspaces stay in HBM (the performance path)."""

    def __init__(self, ctx: Context, n: int, s: int, kl: KlField = None,
                 coeffs: PdeCoefficients = None, bc: DirichletBc = None):
        self.ctx, self.n, self.s = ctx, n, s
        self.kl = kl or KlField()
        self.coeffs = coeffs or PdeCoefficients()
        self.bc = bc or DirichletBc()
        d = _ProblemDesc(n, s, self.kl._c(), self.coeffs._c(), self.bc._c())
        h = _vp()
        _check(lib().enprop_problem_create(ctx.h, C.byref(d), C.byref(h)), "Problem")
        self.h = h
        rows = C.c_int()
        nnz = C.c_int64()
        self.rows = None
        ptrs = [_vp() for _ in range(5)]
        _check(lib().enprop_problem_views(h, C.byref(rows), C.byref(nnz), *[C.byref(p) for p in ptrs]))
        self.rows, self.nnz = rows.value, nnz.value
        self._ptrs = dict(zip(["row_map", "col_entry", "values", "residual", "solution"],
                              [p.value for p in ptrs]))

    def assemble(self, y: torch.Tensor):
        _need_cuda(y, torch.float64, "y")
        if y.numel() != self.kl.num_terms * self.s:
            raise ValueError("assemble: sample vector length mismatch")
        _check(lib().enprop_problem_assemble(self.h, _ptr(y)), "assemble")

    def solve(self, config: SolverConfig = None, raise_on_failure: bool = True):
        cfg = config or SolverConfig()
        lanes = self.s if cfg.flavour == CG_UNCOUPLED else 1
        it, ls, hl = ((C.c_int * lanes)() for _ in range(3))
        hist = (C.c_double * ((cfg.max_iterations + 1) * lanes))()
        opt = cfg._c()
        rc = lib().enprop_problem_solve(self.h, C.byref(opt), it, ls, hist, hl)
        iters, history, lstat = _collect(cfg, self.s, it, ls, hist, hl)
        if rc in (ERR_NO_CONVERGENCE, ERR_INDEFINITE):
            if raise_on_failure:
                raise SolverError(_err(), history, rc, iters)
        else:
            _check(rc, "solve")
        return iters, history, lstat

    def newton(self, y: torch.Tensor, options: NewtonOptions = None,
               raise_on_failure: bool = True, multigrid: Optional[MgOptions] = None) -> NewtonResult:
        """newton_solve (fem.hpp:265-302) from u = 0 with this problem's
        PdeCoefficients; the iterate ends in self.solution. multigrid: the
        reference's MG-preconditioned linear solves with these MgOptions
        (enprop_problem_newton_mg); None: identity-preconditioned."""
        _need_cuda(y, torch.float64, "y")
        if y.numel() != self.kl.num_terms * self.s:
            raise ValueError("newton: sample vector length mismatch")
        opt = options or NewtonOptions()
        it, cg, nn = C.c_int(), C.c_int(), C.c_int()
        norms = (C.c_double * (max(opt.max_iterations, 0) + 1))()
        if multigrid is not None:
            mo = multigrid._c()
            rc = lib().enprop_problem_newton_mg(self.h, _ptr(y), C.byref(opt._c()), C.byref(mo), C.byref(it),
                                                C.byref(cg), norms, C.byref(nn))
        else:
            rc = lib().enprop_problem_newton(self.h, _ptr(y), C.byref(opt._c()), C.byref(it), C.byref(cg),
                                             norms, C.byref(nn))
        res = NewtonResult(it.value, cg.value, [norms[i] for i in range(nn.value)])
        if rc in (ERR_NO_CONVERGENCE, ERR_INDEFINITE):
            if raise_on_failure:
                raise SolverError(_err(), res.residual_norms, rc, res.iterations)
        else:
            _check(rc, "newton")
        return res

    def solve_host(self, y_host: torch.Tensor, x_host: torch.Tensor, config: SolverConfig = None):
        """End to end from host buffers (pinned for speed)."""
        cfg = config or SolverConfig()
        lanes = self.s if cfg.flavour == CG_UNCOUPLED else 1
        it, ls = (C.c_int * lanes)(), (C.c_int * lanes)()
        opt = cfg._c()
        rc = lib().enprop_problem_solve_host(self.h, _ptr(y_host), _ptr(x_host), C.byref(opt), it, ls)
        if rc not in (OK, ERR_NO_CONVERGENCE, ERR_INDEFINITE):
            _check(rc, "solve_host")
        return list(it), list(ls), rc

    def _view(self, name, count, dtype, shape):
        return _wrap_device_ptr(self._ptrs[name], count, dtype, self.ctx.device).view(*shape)

    @property
    def values(self):
        """Full [nnz][s] values of the assembled operator (a copy when the
        problem uses symmetric storage)."""
        out = torch.empty((self.nnz, self.s), dtype=torch.float64, device=torch.device("cuda", self.ctx.device))
        _check(lib().enprop_problem_expand_values(self.h, _ptr(out)), "expand_values")
        return out

    @property
    def nnz_stored(self) -> int:
        n = C.c_int64()
        _check(lib().enprop_problem_storage(self.h, C.byref(n), None))
        return n.value

    @property
    def residual(self):
        return self._view("residual", self.rows * self.s, torch.float64, (self.rows, self.s))

    @property
    def solution(self):
        return self._view("solution", self.rows * self.s, torch.float64, (self.rows, self.s))

    @property
    def row_map(self):
        return self._view("row_map", self.rows + 1, torch.int32, (self.rows + 1,))

    @property
    def col_entry(self):
        return self._view("col_entry", self.nnz, torch.int32, (self.nnz,))

    def close(self):
        if getattr(self, "h", None):
            lib().enprop_problem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _wrap_device_ptr(ptr: int, count: int, dtype, device: int) -> torch.Tensor:
    """Non-owning torch view of library-owned device memory (copy it if it
    must outlive the Problem)."""
    class _Cai:
        def __init__(self):
            typestr = {torch.float64: "<f8", torch.int32: "<i4"}[dtype]
            self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                             "data": (ptr, False), "version": 3}
    return torch.as_tensor(_Cai(), device=torch.device("cuda", device))


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for Dist(..., nccl_id=...) (rank 0 makes it)."""
    buf = (C.c_char * 128)()
    _check(lib().enprop_nccl_unique_id(buf, 128), "nccl_unique_id")
    return bytes(buf)


def fit_halo_model(samples):
    """fit_halo_model (halo.cpp:156-181): least squares T(s) = a + b*s through
    [(s, seconds), ...]; returns (a, b, residual_sum_of_squares)."""
    n = len(samples)
    s = (C.c_double * max(n, 1))(*[float(p[0]) for p in samples])
    t = (C.c_double * max(n, 1))(*[float(p[1]) for p in samples])
    a, b, r = C.c_double(), C.c_double(), C.c_double()
    _check(lib().enprop_fit_halo_model(n, s, t, C.byref(a), C.byref(b), C.byref(r)), "fit_halo_model")
    return a.value, b.value, r.value


def write_exchange_trace_csv(path: str, records) -> None:
    """write_exchange_trace_csv (halo.cpp:192-202): records of (rank, neighbor,
    bytes, time) -- e.g. Dist.exchange_trace()[0]."""
    arr = (_ExchangeRecord * max(len(records), 1))()
    for i, (rk, nb, by, t) in enumerate(records):
        arr[i] = _ExchangeRecord(rk, nb, by, t)
    _check(lib().enprop_write_exchange_trace_csv(path.encode(), arr, len(records)), "write_exchange_trace_csv")


def predicted_speedup(a: float, b: float, s: float) -> float:
    """predicted_speedup (halo.cpp:183-188): s*(a + b)/(a + b*s)."""
    out = C.c_double()
    _check(lib().enprop_predicted_speedup(C.c_double(a), C.c_double(b), C.c_double(s), C.byref(out)),
           "predicted_speedup")
    return out.value


class Dist:
    """Ensemble problem domain-decomposed into z-slabs of node planes over
    `nranks` (partition.cpp:31-72 rule).  nccl_id=None and ipc_job=None
    emulate all ranks in this process on one GPU (stream-ordered copies as
    transport); with an NCCL id this process is `rank` of an NCCL job; with an
    ipc_job name it is `rank` of a CUDA-IPC job (peers on any GPUs of the node,
    several per GPU allowed).  Canonical dot order only; results
    are bitwise independent of nranks."""

    def __init__(self, ctx: Context, n: int, s: int, nranks: int, rank: int = 0,
                 nccl_id: Optional[bytes] = None, kl: KlField = None,
                 coeffs: PdeCoefficients = None, bc: DirichletBc = None, ipc_job: Optional[str] = None):
        self.ctx, self.n, self.s, self.nranks = ctx, n, s, nranks
        self.kl = kl or KlField()
        d = _ProblemDesc(n, s, self.kl._c(), (coeffs or PdeCoefficients())._c(),
                         (bc or DirichletBc())._c())
        h = _vp()
        if ipc_job is not None:  # CUDA-IPC transport: this process is `rank` of an IPC job
            _check(lib().enprop_dist_create_ipc(ctx.h, C.byref(d), nranks, rank, ipc_job.encode(), C.byref(h)),
                   "Dist")
        else:
            idbuf = None if nccl_id is None else (C.c_char * 128).from_buffer_copy(nccl_id)
            _check(lib().enprop_dist_create(ctx.h, C.byref(d), nranks, rank, idbuf, C.byref(h)), "Dist")
        self.h = h

    def assemble(self, y: torch.Tensor):
        _need_cuda(y, torch.float64, "y")
        if y.numel() != self.kl.num_terms * self.s:
            raise ValueError("assemble: sample vector length mismatch")
        _check(lib().enprop_dist_assemble(self.h, _ptr(y)), "assemble")

    def solve(self, config: SolverConfig = None, raise_on_failure: bool = True):
        cfg = config or SolverConfig(dot_mode=DOT_CANONICAL)
        lanes = self.s if cfg.flavour == CG_UNCOUPLED else 1
        it, ls = (C.c_int * lanes)(), (C.c_int * lanes)()
        opt = cfg._c()
        rc = lib().enprop_dist_solve(self.h, C.byref(opt), it, ls)
        if rc in (ERR_NO_CONVERGENCE, ERR_INDEFINITE):
            if raise_on_failure:
                raise SolverError(_err(), [], rc, list(it))
        else:
            _check(rc, "solve")
        return (list(it) if cfg.flavour == CG_UNCOUPLED else it[0]), list(ls)

    def newton(self, y: torch.Tensor, options: NewtonOptions = None,
               raise_on_failure: bool = True) -> NewtonResult:
        """newton_solve (fem.hpp:265-302) over the slabs with Alg. 2's u halo
        (identity-preconditioned canonical CG); bitwise Problem.newton on one
        GPU with DOT_CANONICAL. The iterate ends in the ranks' x (local())."""
        _need_cuda(y, torch.float64, "y")
        if y.numel() != self.kl.num_terms * self.s:
            raise ValueError("newton: sample vector length mismatch")
        opt = options or NewtonOptions(linear=SolverConfig(dot_mode=DOT_CANONICAL))
        it, cg, nn = C.c_int(), C.c_int(), C.c_int()
        norms = (C.c_double * (max(opt.max_iterations, 0) + 1))()
        rc = lib().enprop_dist_newton(self.h, _ptr(y), C.byref(opt._c()), C.byref(it), C.byref(cg), norms,
                                      C.byref(nn))
        res = NewtonResult(it.value, cg.value, [norms[i] for i in range(nn.value)])
        if rc in (ERR_NO_CONVERGENCE, ERR_INDEFINITE):
            if raise_on_failure:
                raise SolverError(_err(), res.residual_norms, rc, res.iterations)
        else:
            _check(rc, "newton")
        return res

    def time_halo(self, reps: int = 20) -> float:
        """Mean seconds of one halo exchange of the solver's p buffer (one plane
        of s values to each neighbour; NCCL, or the emulated device copies)."""
        sec = C.c_double()
        _check(lib().enprop_dist_time_halo(self.h, reps, C.byref(sec)), "time_halo")
        return sec.value

    def exchange_trace(self, max_records: int = 4096):
        """One measured halo exchange: ([(rank, neighbor, bytes, cumulative seconds)], elapsed
        seconds) in the reference's record order (halo.cpp:140-150)."""
        recs = (_ExchangeRecord * max_records)()
        n, el = C.c_int(), C.c_double()
        _check(lib().enprop_dist_exchange_trace(self.h, recs, max_records, C.byref(n), C.byref(el)),
               "exchange_trace")
        return [(recs[i].rank, recs[i].neighbor, recs[i].bytes, recs[i].time) for i in range(n.value)], el.value

    def local(self):
        """[(rank, row_begin, rows, x view [rows][s])] of the ranks in this process."""
        out = []
        for i in range(lib().enprop_dist_local_count(self.h)):
            rk, rb, rows, xp = C.c_int(), C.c_int(), C.c_int(), _vp()
            _check(lib().enprop_dist_local(self.h, i, C.byref(rk), C.byref(rb), C.byref(rows), C.byref(xp)))
            x = _wrap_device_ptr(xp.value, rows.value * self.s, torch.float64, self.ctx.device)
            out.append((rk.value, rb.value, rows.value, x.view(rows.value, self.s)))
        return out

    def stages(self):
        """[(interior, total)] SpMV stages of the local ranks: the interior ones
        run while the halo is in flight (0, 0 for unstaged slabs)."""
        out = []
        for i in range(lib().enprop_dist_local_count(self.h)):
            a, b = C.c_int(), C.c_int()
            _check(lib().enprop_dist_stages(self.h, i, C.byref(a), C.byref(b)), "stages")
            out.append((a.value, b.value))
        return out

    def solution(self) -> torch.Tensor:
        """The owned parts of the local ranks, concatenated in row order."""
        return torch.cat([x for (_, _, _, x) in sorted(self.local(), key=lambda t: t[1])], dim=0)

    def close(self):
        if getattr(self, "h", None):
            lib().enprop_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
