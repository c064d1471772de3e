"""Wire formats of the reference (SURVEY §8 f, rank 3), byte-compatible so
that inputs and results move between this package, the reference's CLI and
its tooling:

* dump_tensor / load_tensor (storage.hpp:214-278): header (d, dims..., stride)
  as little-endian uint64, then the padded column-major buffer (stride x n_d
  doubles, padding rows included);
* save_tt / load_tt (tensor_train.hpp:157-191): header (d, ranks r_0..r_d,
  dims) as uint64, then the core buffers (r_left x n x r_right, column-major);
* the run report CSV (report.hpp:20-34, 83-96):
  variant,shape,rmax,eps,phase,step,seconds,flops,bytes,rank — one row per
  step and phase (tsqr, small-svd, tsmm, reorder).

Host-side I/O; a device tensor is staged through host memory.  Errors raise
IoError as the reference's throw IoError.
"""
from __future__ import annotations

import io

import numpy as np

from .ttsvd import IoError, TensorTrain, TTCore, padded_stride, to_device_matrix

_U64 = np.dtype("<u8")
_F64 = np.dtype("<f8")
REPORT_HEADER = "variant,shape,rmax,eps,phase,step,seconds,flops,bytes,rank"


def _read_u64(f, n: int) -> np.ndarray:
    b = f.read(8 * n)
    if len(b) != 8 * n:
        raise IoError("load: short read")
    return np.frombuffer(b, dtype=_U64).astype(np.int64)


def _padded_host(X, dims) -> np.ndarray:
    """(ld x n_d) Fortran host array of the padded buffer of X (device tensor
    view rows x n_d with column stride ld, or a host (ld x n_d) array)."""
    nd = int(dims[-1])
    if hasattr(X, "as_strided"):  # torch tensor (device or host)
        ld = X.stride(1)
        return np.asfortranarray(X.as_strided((ld, nd), (1, ld)).cpu().numpy())
    return np.asfortranarray(X)


def dump_tensor(X, dims, path: str) -> None:
    dims = [int(n) for n in dims]
    rows = int(np.prod(dims)) // dims[-1]
    A = _padded_host(X, dims)
    if A.shape != (padded_stride(rows), dims[-1]):
        raise IoError("dump_tensor: buffer is not in the padded layout")
    try:
        with open(path, "wb") as f:
            f.write(np.array([len(dims)] + dims + [A.shape[0]], dtype=_U64).tobytes())
            f.write(np.ascontiguousarray(A.T, dtype=_F64).tobytes())
    except OSError as e:
        raise IoError(f"dump_tensor: cannot open {path}") from e


def load_tensor(path: str, device: int | None = None):
    """-> (X, dims): X the padded buffer, a host (ld x n_d) Fortran array, or
    with `device` a device tensor (rows x n_d view, column stride ld) ready
    for tt_svd_tsqr."""
    try:
        f = open(path, "rb")
    except OSError as e:
        raise IoError(f"load_tensor: cannot open {path}") from e
    with f:
        d = int(_read_u64(f, 1)[0])
        if d < 1 or d > 64:
            raise IoError("load_tensor: bad header")
        dims = [int(n) for n in _read_u64(f, d)]
        stride = int(_read_u64(f, 1)[0])
        rows = int(np.prod(dims)) // dims[-1]
        if stride != padded_stride(rows):
            raise IoError("load_tensor: stride mismatch")
        b = f.read(8 * stride * dims[-1])
        if len(b) != 8 * stride * dims[-1]:
            raise IoError("load: short read")
    A = np.frombuffer(b, dtype=_F64).reshape((dims[-1], stride)).T  # Fortran view
    if device is None:
        return np.array(A, order="F"), dims
    return to_device_matrix(A[:rows], ld=stride), dims


def save_tt(tt: TensorTrain, path: str) -> None:
    tt.validate()
    try:
        with open(path, "wb") as f:
            f.write(np.array([tt.d()] + tt.ranks() + tt.dims(), dtype=_U64).tobytes())
            for c in tt.cores:
                f.write(np.asarray(c.data, dtype=_F64).reshape(-1, order="F").tobytes())
    except OSError as e:
        raise IoError(f"save_tt: cannot open {path}") from e


def load_tt(path: str) -> TensorTrain:
    try:
        f = open(path, "rb")
    except OSError as e:
        raise IoError(f"load_tt: cannot open {path}") from e
    with f:
        d = int(_read_u64(f, 1)[0])
        if d < 1 or d > 64:
            raise IoError("load_tt: bad header")
        ranks = _read_u64(f, d + 1)
        dims = _read_u64(f, d)
        tt = TensorTrain()
        for j in range(d):
            rl, n, rr = int(ranks[j]), int(dims[j]), int(ranks[j + 1])
            b = f.read(8 * rl * n * rr)
            if len(b) != 8 * rl * n * rr:
                raise IoError("load: short read")
            tt.cores.append(TTCore(np.frombuffer(b, dtype=_F64).reshape((rl, n, rr), order="F").copy(order="F")))
    tt.validate()
    return tt


# ------------------------------------------------------------------- report ----
def report_rows(tt: TensorTrain, variant: str, shape: str, rmax: int, eps: float) -> list[dict]:
    """rows_from_recorder (report.hpp:43-80) from the step records of a run.
    Seconds are the device phase times (Context.set_timing(True); else 0).
    TSQR flops are the algorithmic 2 n m^2 (SURVEY §8 d), not the reference's
    padded-block model; TSMM flops/bytes are the reference's."""
    rows = []
    for s in tt.steps:
        for phase, secs in (("tsqr", s.t_tsqr), ("small-svd", s.t_small_svd), ("tsmm", s.t_tsmm), ("reorder", 0.0)):
            r = {"variant": variant, "shape": shape, "rmax": int(rmax), "eps": float(eps), "phase": phase,
                 "step": int(s.step), "seconds": float(secs), "flops": 0, "bytes": 0, "rank": int(s.rank)}
            if phase == "tsqr":
                r["flops"] = 2 * s.rows * s.cols * s.cols
                r["bytes"] = 8 * s.rows * s.cols
            elif phase == "tsmm":
                r["flops"] = 2 * s.rows * s.cols * s.rank
                r["bytes"] = 8 * s.rows * (s.cols + s.rank)
            rows.append(r)
    return rows


def _g17(v: float) -> str:
    return "%.17g" % v


def emit_csv(rows: list[dict], out: io.TextIOBase | None = None) -> str:
    """emit_csv (report.hpp:83-96): header always present; doubles as %.17g."""
    lines = [REPORT_HEADER]
    for r in rows:
        lines.append(",".join([r["variant"], r["shape"], str(r["rmax"]), _g17(r["eps"]), r["phase"], str(r["step"]),
                               _g17(r["seconds"]), str(r["flops"]), str(r["bytes"]), str(r["rank"])]))
    text = "\n".join(lines) + "\n"
    if out is not None:
        out.write(text)
    return text


def parse_csv(text: str) -> list[dict]:
    """parse_csv (report.hpp:123-160)."""
    lines = text.splitlines()
    if not lines:
        raise IoError("parse_csv: empty input")
    if lines[0] != REPORT_HEADER:
        raise IoError("parse_csv: unexpected header")
    rows = []
    for line in lines[1:]:
        if not line:
            continue
        f = line.split(",")
        if len(f) != 10:
            raise IoError("parse_csv: wrong field count")
        rows.append({"variant": f[0], "shape": f[1], "rmax": int(f[2]), "eps": float(f[3]), "phase": f[4],
                     "step": int(f[5]), "seconds": float(f[6]), "flops": int(f[7]), "bytes": int(f[8]),
                     "rank": int(f[9])})
    return rows


__all__ = ["dump_tensor", "load_tensor", "save_tt", "load_tt", "report_rows", "emit_csv", "parse_csv",
           "REPORT_HEADER"]
