"""Python host mirror of the reference TT-SVD interface over the sm_100a C-ABI.

Reference: /root/reference/proj/include/ttsvd/*.hpp.  The names, argument
meaning and error behaviour follow the reference so that the parity tests
read like the reference's own tests:

    tsqr            tsqr.hpp:247        reduce_block   tsqr.hpp:208
    combine_factors tsqr.hpp:230        small_svd      small_svd.hpp:196
    jacobi_svd      small_svd.hpp:120   select_rank    small_svd.hpp:49
    derive_delta    small_svd.hpp:41    tsmm_reshape   tsmm.hpp:20
    tt_svd_tsqr     tt_svd.hpp:281      tt_svd_distributed tt_svd.hpp:520

Every numeric call goes through libttsvd_cu.so (include/ttsvd_cu.h).  Device
matrices are column-major torch tensors: a (rows, cols) view with strides
(1, ld), e.g. ``fortran_empty(rows, cols)``.  Host (numpy) inputs are copied
to the device first — the reference-facing convenience path; results of the
building blocks stay on the device, the drivers return a host TensorTrain
like the reference does.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

# ---------------------------------------------------------------- errors ----
# errors.hpp:9-62


class Error(RuntimeError):
    pass


class LayoutError(Error):
    pass


class AllocationError(Error):
    pass


class DimensionMismatch(Error):
    pass


class DimensionError(Error):
    pass


class DegenerateDimension(Error):
    pass


class ConvergenceError(Error):
    pass


class ShapeError(Error):
    pass


class PartitionMismatch(Error):
    pass


class DivergenceError(Error):
    pass


class IoError(Error):
    pass


class DeviceError(Error):
    """CUDA / exchange failure (new in the device build)."""


_CODES = {1: DimensionError, 2: DimensionMismatch, 3: ShapeError, 4: ConvergenceError, 5: AllocationError,
          6: DegenerateDimension, 7: PartitionMismatch, 8: DeviceError, 9: Error, 10: LayoutError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.lib().ttsvd_cu_last_error().decode(errors="replace")
        raise _CODES.get(rc, Error)(msg)


# ----------------------------------------------------------- parameters ----
@dataclass
class BlockParams:
    """tsqr.hpp:41-57.  Accepted for signature compatibility; the device
    kernels choose their own tiles (results are deterministic per shape)."""
    n_b: int = 256
    eps_fp: float = 2.2250738585072014e-308
    validate_reflectors: bool = False

    @staticmethod
    def for_cols(m: int, l2_budget_bytes: int = 256 * 1024) -> "BlockParams":
        cap = l2_budget_bytes // 8
        nb = (cap // max(m, 1) - m) // 8 * 8
        return BlockParams(n_b=min(max(nb, 16), 4096))


@dataclass
class TruncationSpec:
    """small_svd.hpp:30-36"""
    r_max: int = 2 ** 63 - 1
    eps: float = 0.0
    delta: float = -1.0

    def has_delta(self) -> bool:
        return self.delta >= 0.0


def padded_stride(n_rows: int) -> int:
    """shape.hpp:22-28"""
    if n_rows < 1:
        raise DimensionError("padded_stride: n_rows must be >= 1")
    return int(_lib.lib().ttsvd_cu_padded_stride(n_rows))


# --------------------------------------------------------------- context ----
class Context:
    """A device, the stream the library enqueues on (torch's current stream by
    default), and the library's workspace.  One per device per thread."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None):
        self.device = device
        self.handle = C.c_void_p()
        self.comm_size = 0  # > 0 once an NCCL communicator is attached
        s = stream if stream is not None else torch.cuda.current_stream(device)
        self._stream = s
        _check(_lib.lib().ttsvd_cu_ctx_create(device, C.c_void_p(s.cuda_stream), C.byref(self.handle)))

    def sync_stream(self) -> None:
        """Follow torch's current stream (call before enqueueing)."""
        s = torch.cuda.current_stream(self.device)
        if s.cuda_stream != self._stream.cuda_stream:
            self._stream = s
            _check(_lib.lib().ttsvd_cu_ctx_set_stream(self.handle, C.c_void_p(s.cuda_stream)))

    @property
    def launches(self) -> int:
        return int(_lib.lib().ttsvd_cu_ctx_launches(self.handle))

    def set_timing(self, on: bool) -> None:
        _check(_lib.lib().ttsvd_cu_ctx_set_timing(self.handle, 1 if on else 0))

    def synchronize(self) -> None:
        _check(_lib.lib().ttsvd_cu_synchronize(self.handle))

    def attach_nccl(self, group=None) -> None:
        """Attach the library's own NCCL communicator over the ranks of a
        torch.distributed group (one process per GPU): rank 0 creates the
        unique id, the group broadcasts it, every rank joins.  Afterwards
        tt_svd_distributed all-gathers inside the library (ncclAllGather on
        this context's stream, no Python on the exchange path)."""
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            _check(_lib.lib().ttsvd_cu_comm_unique_id(uid))
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8,
                         device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        raw = bytes(t.cpu().tolist())
        uid = (C.c_ubyte * 128).from_buffer_copy(raw)
        _check(_lib.lib().ttsvd_cu_ctx_comm_init(self.handle, uid, world, rank))
        self.comm_size = world

    def close(self) -> None:
        if self.handle:
            _lib.lib().ttsvd_cu_ctx_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_ctx: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    dev = torch.cuda.current_device() if device is None else device
    if dev not in _ctx:
        _ctx[dev] = Context(dev)
    c = _ctx[dev]
    c.sync_stream()
    return c


# ---------------------------------------------------------- device views ----
def fortran_empty(rows: int, cols: int, ld: int | None = None, device: int | None = None,
                  zero: bool = False) -> torch.Tensor:
    """(rows x cols) column-major device matrix with leading dimension ld."""
    ld = ld if ld is not None else max(rows, 1)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    buf = (torch.zeros if zero else torch.empty)((max(cols, 1), ld), dtype=torch.float64, device=dev)
    return buf.t()[:rows, :cols]


def _ld(T: torch.Tensor) -> int:
    rows, cols = T.shape
    if cols <= 1:
        return max(T.stride(1) if T.dim() == 2 else rows, rows, 1)
    return T.stride(1)


def to_device_matrix(A, ld: int | None = None) -> torch.Tensor:
    """numpy / torch -> column-major float64 device view."""
    if isinstance(A, torch.Tensor) and A.is_cuda and A.dtype == torch.float64 and A.dim() == 2 and (
            A.stride(0) == 1 or A.shape[0] <= 1) and _ld(A) >= A.shape[0]:
        return A
    a = np.asarray(A.cpu().numpy() if isinstance(A, torch.Tensor) else A, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    rows, cols = a.shape
    T = fortran_empty(rows, cols, ld=ld, zero=True)
    T.copy_(torch.from_numpy(np.ascontiguousarray(a)))
    return T


def _mat(T: torch.Tensor):
    if T.dim() != 2 or not T.is_cuda or T.dtype != torch.float64:
        raise Error("expected a 2-D float64 CUDA tensor")
    if T.shape[0] > 1 and T.stride(0) != 1:
        raise LayoutError("expected a column-major (Fortran) view with unit row stride")
    return T.data_ptr(), T.shape[0], T.shape[1], _ld(T)


def to_host(T: torch.Tensor) -> np.ndarray:
    return np.asfortranarray(T.detach().cpu().numpy())


# ------------------------------------------------------- building blocks ----
def tsqr(X, params: BlockParams | None = None, workers: int = 1, stats=None, counters=None) -> torch.Tensor:
    """tsqr.hpp:247 — R (m x m device tensor) with R^T R = X^T X."""
    X = to_device_matrix(X)
    ctx = context(X.device.index)
    p, n, m, ld = _mat(X)
    R = fortran_empty(m, m)
    _check(_lib.lib().ttsvd_cu_tsqr(ctx.handle, p, n, m, ld, R.data_ptr()))
    if counters is not None:
        counters.add(2 * n * m * m, 8 * n * m)
    return R


def reduce_block(M, R, params: BlockParams | None = None, stats=None, counters=None) -> torch.Tensor:
    """tsqr.hpp:208 — Rbar^T Rbar = M^T M + R^T R."""
    M = to_device_matrix(M)
    R = to_device_matrix(R, ld=R.shape[0])
    ctx = context(M.device.index)
    p, rows, m, ld = _mat(M)
    if R.shape[0] != R.shape[1]:
        raise DimensionMismatch("reduce_block: R must be square")
    Rc = R if _ld(R) == R.shape[0] else R.contiguous()
    out = fortran_empty(m, m)
    _check(_lib.lib().ttsvd_cu_reduce_block(ctx.handle, p, rows, m, max(ld, 1), Rc.data_ptr(), R.shape[0],
                                            out.data_ptr()))
    return out


def combine_factors(parts, params: BlockParams | None = None, stats=None, counters=None) -> torch.Tensor:
    """tsqr.hpp:230 — fixed-order merge of triangular factors."""
    if len(parts) == 0:
        raise DimensionMismatch("combine_factors: empty list")
    m = parts[0].shape[0]
    for q in parts:
        if q.shape[0] != m:
            raise DimensionMismatch("combine_factors: mixed column counts")
    mats = [to_device_matrix(q, ld=m) for q in parts]
    buf = torch.stack([q.t().contiguous() for q in mats])  # P x m x m, each column-major
    ctx = context(buf.device.index)
    out = fortran_empty(m, m)
    _check(_lib.lib().ttsvd_cu_combine_factors(ctx.handle, buf.data_ptr(), len(parts), m, out.data_ptr()))
    return out


@dataclass
class SmallSVD:
    """small_svd.hpp:18-26 (device tensors; U is None for small_svd)."""
    n: int
    m: int
    U: torch.Tensor | None
    sigma: torch.Tensor
    V: torch.Tensor


def small_svd(R) -> SmallSVD:
    """small_svd.hpp:196 — sigma (non-increasing) and V of a triangular factor."""
    R = to_device_matrix(R)
    m = R.shape[0]
    if m > 4096:
        raise DimensionMismatch("small_svd: m exceeds 4096")
    Rc = R if _ld(R) == m else R.t().contiguous().t()
    ctx = context(R.device.index)
    sigma = torch.empty(m, dtype=torch.float64, device=R.device)
    V = fortran_empty(m, m)
    _check(_lib.lib().ttsvd_cu_small_svd(ctx.handle, Rc.data_ptr(), m, sigma.data_ptr(), V.data_ptr()))
    return SmallSVD(m, m, None, sigma, V)


def jacobi_svd(A) -> SmallSVD:
    """small_svd.hpp:120 — one-sided Jacobi SVD of a tall matrix."""
    A = to_device_matrix(A)
    p, n, m, ld = _mat(A)
    ctx = context(A.device.index)
    sigma = torch.empty(m, dtype=torch.float64, device=A.device)
    V = fortran_empty(m, m)
    U = fortran_empty(n, m)
    _check(_lib.lib().ttsvd_cu_jacobi_svd(ctx.handle, p, n, m, ld, sigma.data_ptr(), V.data_ptr(), U.data_ptr()))
    return SmallSVD(n, m, U, sigma, V)


def driver_svd(A, r: int):
    """The TT-SVD driver's SVD of a work matrix (tt_svd.hpp:85-110): sigma
    (non-increasing) and the leading r left singular vectors of A (n x m,
    n >= m).  Returns (sigma, V, path) with path "bidiag" or "jacobi"."""
    A = to_device_matrix(A)
    p, n, m, ld = _mat(A)
    ctx = context(A.device.index)
    sigma = torch.empty(m, dtype=torch.float64, device=A.device)
    V = fortran_empty(n, max(int(r), 1))
    path = C.c_int32(-1)
    _check(_lib.lib().ttsvd_cu_driver_svd(ctx.handle, p, n, m, ld, int(r), sigma.data_ptr(), V.data_ptr(),
                                          C.byref(path)))
    return sigma, V[:, :int(r)], ("bidiag" if path.value == 1 else "jacobi")


def select_rank(sigma, delta: float, r_max: int) -> int:
    """small_svd.hpp:49"""
    s = sigma if isinstance(sigma, torch.Tensor) and sigma.is_cuda else torch.as_tensor(
        np.asarray(sigma, dtype=np.float64), device="cuda")
    s = s.to(torch.float64).contiguous()
    ctx = context(s.device.index)
    out = C.c_int64()
    _check(_lib.lib().ttsvd_cu_select_rank(ctx.handle, s.data_ptr(), s.numel(), float(delta), int(r_max),
                                           C.byref(out)))
    return int(out.value)


def derive_delta(norm_source: float, eps: float, d: int) -> float:
    """small_svd.hpp:41"""
    out = C.c_double()
    _check(_lib.lib().ttsvd_cu_derive_delta(float(norm_source), float(eps), int(d), C.byref(out)))
    return out.value


def tsmm_reshape(X, V, out_rows: int | None = None, out_cols: int | None = None, workers: int = 1,
                 counters=None) -> torch.Tensor:
    """tsmm.hpp:20 (and the n x k overload at :74) — returns the padded output
    as a (out_rows x out_cols) view with ld = padded_stride(out_rows)."""
    X = to_device_matrix(X)
    V = to_device_matrix(V)
    px, n, m, ldx = _mat(X)
    pv, vr, k, ldv = _mat(V)
    if vr != m:
        raise ShapeError("tsmm_reshape: V.rows != X.cols")
    if out_rows is None:
        out_rows, out_cols = n, k
    if out_rows < 1:
        raise ShapeError("tsmm_reshape: out shape does not hold n*k elements")
    ldy = padded_stride(out_rows)
    Y = fortran_empty(out_rows, max(out_cols, 1), ld=ldy)
    ctx = context(X.device.index)
    _check(_lib.lib().ttsvd_cu_tsmm_reshape(ctx.handle, px, n, m, ldx, pv, k, ldv, Y.data_ptr(), out_rows,
                                            out_cols, ldy))
    if counters is not None:
        counters.add(2 * n * m * k, 8 * n * (m + k))
    return Y


# ----------------------------------------------------------- tensor train ----
@dataclass
class TTCore:
    """tensor_train.hpp:15-39 — data is a Fortran (r_left, n, r_right) array."""
    data: np.ndarray

    @property
    def r_left(self):
        return self.data.shape[0]

    @property
    def n(self):
        return self.data.shape[1]

    @property
    def r_right(self):
        return self.data.shape[2]


@dataclass
class StepRecord:
    """tt_svd.hpp:21-26"""
    step: int
    rows: int
    cols: int
    rank: int
    nsig: int
    f: float
    t_tsqr: float = 0.0
    t_small_svd: float = 0.0
    t_tsmm: float = 0.0
    t_tsqr_sweep: float = 0.0  # the TSQR main sweep kernel alone (diagnostics)
    tsqr_kernel: str = "none"
    svd_sweeps: int = 0
    t_reorder: float = 0.0


@dataclass
class TensorTrain:
    """tensor_train.hpp:42-77"""
    cores: list = field(default_factory=list)
    steps: list = field(default_factory=list)
    sigmas: list = field(default_factory=list)

    def d(self) -> int:
        return len(self.cores)

    def dims(self) -> list[int]:
        return [c.n for c in self.cores]

    def ranks(self) -> list[int]:
        return [self.cores[0].r_left if self.cores else 1] + [c.r_right for c in self.cores]

    def max_rank(self) -> int:
        return max([1] + [max(c.r_left, c.r_right) for c in self.cores])

    def validate(self) -> None:
        if not self.cores:
            raise DegenerateDimension("TensorTrain: no cores")
        if self.cores[0].r_left != 1 or self.cores[-1].r_right != 1:
            raise DimensionMismatch("TensorTrain: boundary ranks must be 1")
        for j in range(len(self.cores) - 1):
            if self.cores[j].r_right != self.cores[j + 1].r_left:
                raise DimensionMismatch(f"TensorTrain: rank chain broken at core {j}")


def _collect(handle: C.c_void_p) -> TensorTrain:
    L = _lib.lib()
    try:
        d = int(L.ttsvd_cu_tt_d(handle))
        ranks = np.zeros(d + 1, dtype=np.int64)
        _check(L.ttsvd_cu_tt_ranks(handle, ranks.ctypes.data_as(_lib.i64p)))
        tt = TensorTrain()
        nsteps = int(L.ttsvd_cu_tt_nsteps(handle))
        steps = []
        for s in range(nsteps):
            st = _lib.Step()
            _check(L.ttsvd_cu_tt_step(handle, s, C.byref(st)))
            sig = np.zeros(st.nsig)
            _check(L.ttsvd_cu_tt_sigma(handle, s, sig.ctypes.data))
            steps.append(StepRecord(s + 1, st.rows, st.cols, st.rank, st.nsig,
                                    st.rank / st.cols if st.cols else 0.0, st.t_tsqr_ms * 1e-3, st.t_svd_ms * 1e-3,
                                    st.t_tsmm_ms * 1e-3, st.t_tsqr_sweep_ms * 1e-3,
                                    _lib.TSQR_KERNELS.get(st.tsqr_kernel, "?"), st.svd_sweeps,
                                    st.t_reorder_ms * 1e-3))
            tt.sigmas.append(sig)
        tt.steps = steps
        return tt, ranks
    except Exception:
        L.ttsvd_cu_tt_free(handle)
        raise


def _finish(handle: C.c_void_p, dims) -> TensorTrain:
    L = _lib.lib()
    tt, ranks = _collect(handle)
    try:
        for j, n in enumerate(dims):
            rl, rr = int(ranks[j]), int(ranks[j + 1])
            buf = np.zeros(rl * int(n) * rr)
            _check(L.ttsvd_cu_tt_core(handle, j, buf.ctypes.data))
            tt.cores.append(TTCore(buf.reshape((rl, int(n), rr), order="F")))
    finally:
        L.ttsvd_cu_tt_free(handle)
    tt.validate()
    return tt


def _spec(spec) -> TruncationSpec:
    if spec is None:
        return TruncationSpec()
    if isinstance(spec, TruncationSpec):
        return spec
    r_max, eps = spec
    return TruncationSpec(r_max=r_max, eps=eps)


def tt_svd_tsqr(X, dims, spec: TruncationSpec | tuple | None = None, ctx_exec=None) -> TensorTrain:
    """tt_svd.hpp:281 (Alg. 2).  X is the tensor in the reference's padded
    layout: a device (rows x n_d) column-major view (ld = padded_stride(rows)
    or larger) or a host numpy buffer of shape (ld, n_d) in Fortran order
    (copied H2D inside the call, the reference-facing entry)."""
    spec = _spec(spec)
    dims = [int(x) for x in dims]
    d = len(dims)
    if d < 2:
        raise DegenerateDimension("tt_svd_tsqr: requires d >= 2")
    r_max = int(spec.r_max)
    dv = np.asarray(dims, dtype=np.int64)
    L = _lib.lib()
    h = C.c_void_p()
    if isinstance(X, torch.Tensor) and X.is_cuda:
        ctx = context(X.device.index)
        p, rows, cols, ld = _mat(X)
        _check(L.ttsvd_cu_tt_svd(ctx.handle, p, dv.ctypes.data_as(_lib.i64p), d, ld, r_max, float(spec.eps),
                                 C.byref(h)))
    else:
        a = np.asarray(X, dtype=np.float64)
        if not a.flags.f_contiguous:
            a = np.asfortranarray(a)
        ctx = context()
        ld = a.shape[0]
        _check(L.ttsvd_cu_tt_svd_host(ctx.handle, a.ctypes.data, dv.ctypes.data_as(_lib.i64p), d, ld, r_max,
                                      float(spec.eps), C.byref(h)))
    return _finish(h, dims)


def tt_svd_two_sided(X, dims, spec: TruncationSpec | tuple | None = None) -> TensorTrain:
    """tt_svd.hpp:402-512 (Alg. 4) on a device tensor in the padded layout
    (host numpy buffers are staged to the device first)."""
    spec = _spec(spec)
    dims = [int(x) for x in dims]
    d = len(dims)
    if d < 2:
        raise DegenerateDimension("tt_svd_two_sided: requires d >= 2")
    X = to_device_matrix(X)
    dv = np.asarray(dims, dtype=np.int64)
    ctx = context(X.device.index)
    p, rows, cols, ld = _mat(X)
    h = C.c_void_p()
    _check(_lib.lib().ttsvd_cu_tt_svd_two_sided(ctx.handle, p, dv.ctypes.data_as(_lib.i64p), d, ld,
                                                int(spec.r_max), float(spec.eps), C.byref(h)))
    return _finish(h, dims)


def transpose_reorder(W, out_rows: int | None = None, out_cols: int | None = None, workers: int = 1,
                      counters=None) -> torch.Tensor:
    """tsmm.hpp:84-126 (default shape: the plain transpose, :121-125) — the
    padded (out_rows x out_cols) result, ld = padded_stride(out_rows)."""
    W = to_device_matrix(W)
    pw, n, m, ldw = _mat(W)
    if out_rows is None:
        out_rows, out_cols = m, n
    if out_rows < 1 or out_cols < 1 or out_rows * out_cols != n * m:
        raise ShapeError("transpose_reorder: out shape does not hold n*m elements")
    ldy = padded_stride(out_rows)
    Y = fortran_empty(out_rows, out_cols, ld=ldy)
    ctx = context(W.device.index)
    _check(_lib.lib().ttsvd_cu_transpose_reorder(ctx.handle, pw, n, m, ldw, Y.data_ptr(), out_rows, out_cols, ldy))
    if counters is not None:
        counters.add(0, 16 * n * m)
    return Y


@dataclass
class ThickBoundsParams:
    """tt_svd.hpp:292-310"""
    m_min: int = 16
    f1_min: float = 0.5
    r_tilde: list = field(default_factory=list)


def choose_combined_dims(dims, params: ThickBoundsParams | None = None, r_max: int | None = None):
    """tt_svd.hpp:316-330: (k, m), the k trailing modes merged into extent m."""
    params = params or ThickBoundsParams()
    dv = np.asarray([int(x) for x in dims], dtype=np.int64)
    rt = np.asarray(params.r_tilde, dtype=np.int64)
    k, m = C.c_int64(), C.c_int64()
    _check(_lib.lib().ttsvd_cu_choose_combined_dims(dv.ctypes.data_as(_lib.i64p), len(dv), int(params.m_min),
                                                    float(params.f1_min), rt.ctypes.data if len(rt) else None,
                                                    len(rt), int(2 ** 63 - 1 if r_max is None else r_max), C.byref(k), C.byref(m)))
    return int(k.value), int(m.value)


def tt_svd_thick_bounds(X, dims, spec: TruncationSpec | tuple | None = None,
                        params: ThickBoundsParams | None = None) -> TensorTrain:
    """tt_svd.hpp:338 (Alg. 3) on a device tensor in the padded layout (as
    tt_svd_tsqr), or on a host numpy buffer of shape (ld, n_d) in Fortran
    order (copied H2D inside the call, in row chunks under the merged first
    TSQR where its shape allows: ttsvd_cu_tt_svd_thick_host)."""
    spec = _spec(spec)
    params = params or ThickBoundsParams()
    dims = [int(x) for x in dims]
    d = len(dims)
    if d < 2:
        raise DegenerateDimension("tt_svd_thick_bounds: requires d >= 2")
    r_max = int(spec.r_max)
    dv = np.asarray(dims, dtype=np.int64)
    rt = np.asarray(params.r_tilde, dtype=np.int64)
    h = C.c_void_p()
    if isinstance(X, torch.Tensor) and X.is_cuda:
        ctx = context(X.device.index)
        p, rows, cols, ld = _mat(X)
        _check(_lib.lib().ttsvd_cu_tt_svd_thick(ctx.handle, p, dv.ctypes.data_as(_lib.i64p), d, ld, r_max,
                                                float(spec.eps), int(params.m_min), float(params.f1_min),
                                                rt.ctypes.data if len(rt) else None, len(rt), C.byref(h)))
    else:
        a = np.asarray(X, dtype=np.float64)
        if not a.flags.f_contiguous:
            a = np.asfortranarray(a)
        ctx = context()
        _check(_lib.lib().ttsvd_cu_tt_svd_thick_host(ctx.handle, a.ctypes.data, dv.ctypes.data_as(_lib.i64p), d,
                                                     a.shape[0], r_max, float(spec.eps), int(params.m_min),
                                                     float(params.f1_min), rt.ctypes.data if len(rt) else None,
                                                     len(rt), C.byref(h)))
    return _finish(h, dims)


class _CAI:
    """Zero-copy torch view of a raw device pointer (for the exchange)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 2, "strides": None}


def _torch_exchange(group):
    import torch.distributed as dist

    def cb(user, send, recv, count, stream):
        try:
            s = torch.as_tensor(_CAI(send, count), device="cuda")
            ws = dist.get_world_size(group)
            r = torch.as_tensor(_CAI(recv, count * ws), device="cuda")
            dist.all_gather_into_tensor(r, s, group=group)
            return 0
        except Exception:  # reported as TTSVD_ERR_DEVICE by the library
            return 1
    return _lib.EXCHANGE_FN(cb)


def tt_svd_distributed(slabs, ldims, spec: TruncationSpec | tuple | None = None, ctx_exec=None,
                       group=None, P_total: int | None = None, part0: int = 0, exchange=None) -> TensorTrain:
    """tt_svd.hpp:520 (Alg. 5).  ``slabs`` are this process's device slabs
    ((rows x n_last) column-major views of the local shape ``ldims``, all with
    the same leading stride).  Single process: all P slabs, no exchange (the
    reference's in-process form).  Multi-process (``group`` given, one or more
    slabs per rank): the per-rank R factors are all-gathered over
    torch.distributed (NCCL on B200) and every rank runs the same pinned-order
    merge and small SVD, so shared cores are bitwise identical.  ``exchange``
    overrides the all-gather (a callable(send_tensor, recv_tensor) on device
    tensors)."""
    spec = _spec(spec)
    ldims = [int(x) for x in ldims]
    if len(slabs) == 0:
        raise PartitionMismatch("tt_svd_distributed: no partitions")
    shapes = {tuple(s.shape) for s in slabs}
    lds = {_ld(s) for s in slabs}
    if len(shapes) != 1 or len(lds) != 1:
        raise PartitionMismatch("tt_svd_distributed: slab shapes differ")
    ctx = context(slabs[0].device.index)
    n_slabs = len(slabs)
    if P_total is None:
        P_total = n_slabs
    ptrs = (C.c_void_p * n_slabs)(*[C.c_void_p(s.data_ptr()) for s in slabs])
    dv = np.asarray(ldims, dtype=np.int64)
    r_max = int(spec.r_max)
    if exchange is not None:
        def _cb(user, send, recv, count, stream):
            try:
                s_t = torch.as_tensor(_CAI(send, count), device="cuda")
                r_t = torch.as_tensor(_CAI(recv, count * (P_total // n_slabs)), device="cuda")
                exchange(s_t, r_t)
                return 0
            except Exception:
                return 1
        exch = _lib.EXCHANGE_FN(_cb)
    elif ctx.comm_size > 0:
        exch = _lib.EXCHANGE_FN()  # NULL: the library's NCCL communicator
    else:
        exch = _torch_exchange(group) if n_slabs != P_total else _lib.EXCHANGE_FN()
    h = C.c_void_p()
    _check(_lib.lib().ttsvd_cu_tt_svd_distributed(ctx.handle, ptrs, n_slabs, part0, P_total,
                                                  dv.ctypes.data_as(_lib.i64p), len(ldims), lds.pop(), r_max,
                                                  float(spec.eps), exch, None, C.byref(h)))
    gdims = [P_total if P_total > 1 else 1] + ldims
    return _finish(h, gdims)


def tt_svd_distributed_devices(slabs_per_device, ldims, spec: TruncationSpec | tuple | None = None) -> TensorTrain:
    """Alg. 5 over several GPUs of ONE process (tt_svd.hpp:520 across
    devices): ``slabs_per_device[i]`` lists device i's slabs (same count on
    every device, partitions numbered device-major); the library attaches an
    NCCL communicator over the devices (ncclCommInitAll) and drives one host
    thread per device."""
    spec = _spec(spec)
    ldims = [int(x) for x in ldims]
    ndev = len(slabs_per_device)
    spd = {len(s) for s in slabs_per_device}
    if ndev == 0 or len(spd) != 1 or 0 in spd:
        raise PartitionMismatch("tt_svd_distributed_devices: every device needs the same number of slabs")
    spd = spd.pop()
    flat = [s for dev_slabs in slabs_per_device for s in dev_slabs]
    if len({tuple(s.shape) for s in flat}) != 1 or len({_ld(s) for s in flat}) != 1:
        raise PartitionMismatch("tt_svd_distributed_devices: slab shapes differ")
    ctxs = [context(dev_slabs[0].device.index) for dev_slabs in slabs_per_device]
    if len({c.device for c in ctxs}) != ndev:
        raise PartitionMismatch("tt_svd_distributed_devices: one entry per distinct device")
    L = _lib.lib()
    handles = (C.c_void_p * ndev)(*[c.handle for c in ctxs])
    if any(c.comm_size != ndev for c in ctxs):
        _check(L.ttsvd_cu_ctx_comm_init_all(handles, ndev))
        for c in ctxs:
            c.comm_size = ndev
    ptrs = (C.c_void_p * len(flat))(*[C.c_void_p(s.data_ptr()) for s in flat])
    dv = np.asarray(ldims, dtype=np.int64)
    for c in ctxs:
        torch.cuda.synchronize(c.device)
    h = C.c_void_p()
    _check(L.ttsvd_cu_tt_svd_distributed_devices(handles, ndev, ptrs, spd, dv.ctypes.data_as(_lib.i64p), len(ldims),
                                                 _ld(flat[0]), int(spec.r_max), float(spec.eps), C.byref(h)))
    P = ndev * spd
    return _finish(h, [P if P > 1 else 1] + ldims)


def gen_partition(seed: int, kind: int, X: torch.Tensor, total_local: int, nparts: int = 1, part: int = 0,
                  scale: float = 1.0) -> None:
    """Partition ``part`` of ``nparts`` of a counter-based tensor into the
    padded device matrix X (local flat l = global part + nparts*l): kind 0
    writes uniform[-1,1), kind 1 adds scale * N(0,1)."""
    p, rows, cols, ld = _mat(X)
    ctx = context(X.device.index)
    _check(_lib.lib().ttsvd_cu_gen_partition(ctx.handle, int(seed), int(kind), float(scale), int(total_local), rows, ld,
                                             int(nparts), int(part), p))


def gen_uniform(seed: int, dims, ld: int | None = None) -> torch.Tensor:
    """Device tensor (rows x n_d view, padded ld) of counter-based uniform[-1,1)
    entries in Fortran flat order (restated bit-exactly by the oracle)."""
    dims = [int(x) for x in dims]
    total = int(np.prod(dims))
    rows = total // dims[-1]
    ld = ld or padded_stride(rows)
    X = fortran_empty(rows, dims[-1], ld=ld, zero=True)
    ctx = context(X.device.index)
    _check(_lib.lib().ttsvd_cu_gen_uniform(ctx.handle, int(seed), total, rows, ld, X.data_ptr()))
    return X
