"""Contraction kernels and their touched-memory accounting, on the B200.

Mirrors pkg/src/tenvec/kernels.py:1-254.  ``tvc_native`` and ``getvc`` keep
the reference signatures, argument checks, ``out``-prefix semantics and
counters, and run the contraction in libtenvec_b200 (``tv_tvc_ws`` /
``tv_getvc_ws``, the split-K workspace from torch's caching allocator, so no
allocation happens inside the library or a captured graph; ``launch_sweep``
is a mode sweep in one ``tv_tvc_sweep`` call): one launch over the
(u, n_k, v) view whatever the mode, instead
of the reference's BLAS matvec or Python loop of u BLAS vecmats
(kernels.py:159-166).  ``tasks`` is accepted for API compatibility; the
output partition across CTAs replaces the serial task blocks
(kernels.py:66-70, 112).  Counters are analytic host integers, identical to
the reference's (kernels.py:168-170).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import KernelError, NormalizationError
from .precision import F64, PrecisionMode, _device, _to_device, convert
from .tensor import Shape, Tensor, matricize_dims

__all__ = [
    "MATVEC", "VECMAT", "KernelError", "NormalizationError", "KernelCounters", "task_ranges",
    "getvc", "tvc_native", "tvc_looped_oracle", "norm2", "normalize", "tvc_regime", "axpby",
]

MATVEC = "matvec"
VECMAT = "vecmat"


@dataclass
class KernelCounters:
    """Streamed elements and bytes touched by kernel invocations (kernels.py:35-63)."""

    elements_read: int = 0
    elements_written: int = 0
    bytes_touched: int = 0
    invocations: dict = field(default_factory=dict)

    @property
    def elements_touched(self) -> int:
        return self.elements_read + self.elements_written

    def count(self, name: str, read: int, written: int, storage_bytes: int) -> None:
        self.elements_read += read
        self.elements_written += written
        self.bytes_touched += (read + written) * storage_bytes
        self.invocations[name] = self.invocations.get(name, 0) + 1

    def add(self, other: "KernelCounters") -> None:
        self.elements_read += other.elements_read
        self.elements_written += other.elements_written
        self.bytes_touched += other.bytes_touched
        for name, c in other.invocations.items():
            self.invocations[name] = self.invocations.get(name, 0) + c


def task_ranges(total: int, tasks: int) -> list[tuple[int, int]]:
    """Split [0, total) into at most `tasks` disjoint contiguous blocks (kernels.py:66-70)."""
    tasks = max(1, min(tasks, total)) if total > 0 else 1
    block = -(-total // tasks)
    return [(a, min(a + block, total)) for a in range(0, total, block)] or [(0, 0)]


def _vec(x, mode: PrecisionMode, what: str) -> torch.Tensor:
    """A contiguous device vector in the storage format (uploads numpy)."""
    if isinstance(x, torch.Tensor):
        t = x
        if t.dtype == torch.bfloat16 and mode.storage == "brain":
            t = t.view(torch.uint16)
        if not t.is_cuda:
            t = t.to(_device())
    else:
        arr = np.asarray(x)
        if arr.dtype != mode.storage_dtype:
            raise KernelError(f"{what} of dtype {arr.dtype} for storage {mode.name}")
        t = _to_device(arr, np_brain=True)
    if t.dtype != mode.torch_storage:
        raise KernelError(f"{what} of dtype {t.dtype} for storage {mode.name}")
    return t.contiguous()


def _workspace(nbytes: int, device, stream: torch.cuda.Stream | None) -> tuple[int, int, object]:
    """Split-K workspace for one launch from torch's caching allocator
    (stream-ordered, captured into graph pools, no driver allocation)."""
    if nbytes <= 0:
        return 0, 0, None
    ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
    if stream is not None and stream != torch.cuda.current_stream(device):
        ws.record_stream(stream)
    return ws.data_ptr(), nbytes, ws


def launch_tvc(a_ptr: int, mode: PrecisionMode, u: int, nk: int, v: int, x_ptr: int, alpha: float,
               beta: float, y_ptr: int, device, stream: torch.cuda.Stream | None = None,
               what: str = "tvc_native") -> None:
    """tv_tvc_ws over the contiguous (u, nk, v) view at a_ptr, with the
    split-K workspace it asks for (tv_tvc_workspace_bytes)."""
    lib = _lib.load()
    need = lib.tv_tvc_workspace_bytes(a_ptr, mode.tv_storage, mode.tv_compute, u, nk, v)
    wp, wb, keep = _workspace(need, device, stream)
    _lib.check(lib.tv_tvc_ws(a_ptr, mode.tv_storage, mode.tv_compute, u, nk, v, x_ptr, float(alpha),
                             float(beta), y_ptr, wp, wb, _lib.stream_ptr(stream)), what)
    del keep


def launch_getvc(trans: int, a_ptr: int, mode: PrecisionMode, m: int, n: int, lda: int, x_ptr: int,
                 alpha: float, beta: float, y_ptr: int, device, stream: torch.cuda.Stream | None = None,
                 what: str = "getvc") -> None:
    """tv_getvc_ws with its split-K workspace (tv_getvc_workspace_bytes)."""
    lib = _lib.load()
    need = lib.tv_getvc_workspace_bytes(trans, a_ptr, mode.tv_storage, mode.tv_compute, m, n, lda)
    wp, wb, keep = _workspace(need, device, stream)
    _lib.check(lib.tv_getvc_ws(trans, a_ptr, mode.tv_storage, mode.tv_compute, m, n, lda, x_ptr,
                               float(alpha), float(beta), y_ptr, wp, wb, _lib.stream_ptr(stream)), what)
    del keep


def launch_sweep(t, xvs: list, ys: list, stream: torch.cuda.Stream | None = None) -> None:
    """tv_tvc_sweep: ys[k] <- t x_k xvs[k] for every mode k of the contiguous
    device tensor t (device vectors in the storage format, preallocated
    outputs), with the split-K workspace slices it asks for."""
    lib = _lib.load()
    mode = t.mode
    d = t.shape.order
    ext = (ctypes.c_int64 * d)(*t.shape.extents)
    a_ptr = t.buf.data_ptr()
    need = lib.tv_tvc_sweep_workspace_bytes(a_ptr, mode.tv_storage, mode.tv_compute, d, ext)
    if need < 0:
        raise KernelError("tv_tvc_sweep_workspace_bytes: invalid view")
    wp, wb, keep = _workspace(need, t.buf.device, stream)
    xp = (ctypes.c_void_p * d)(*[x.data_ptr() for x in xvs])
    yp = (ctypes.c_void_p * d)(*[y.data_ptr() for y in ys])
    _lib.check(lib.tv_tvc_sweep(a_ptr, mode.tv_storage, mode.tv_compute, d, ext, xp, yp, wp, wb,
                                _lib.stream_ptr(stream)), "tvc sweep")
    del keep


def getvc(
    trans: str,
    alpha: float,
    a,
    x,
    beta: float,
    y,
    *,
    mode: PrecisionMode = F64,
    tasks: int = 1,
    counters: KernelCounters | None = None,
) -> None:
    """matvec y = alpha*A x + beta*y; vecmat y = alpha*x^T A + beta*y over an
    m x n row-major view whose row stride may exceed n (kernels.py:73-123).
    ``y`` (a device tensor) is updated in place; beta == 0 never reads it."""
    if not isinstance(a, torch.Tensor):
        a = _to_device(np.asarray(a), np_brain=True)
    if a.dim() != 2:
        raise KernelError("getvc expects a 2-D matrix view")
    m, n = a.shape
    if trans == MATVEC:
        out_len, in_len, code = m, n, 0
    elif trans == VECMAT:
        out_len, in_len, code = n, m, 1
    else:
        raise KernelError(f"unknown trans {trans!r}")
    xs = tuple(x.shape)
    ys = tuple(y.shape)
    if xs != (in_len,) or ys != (out_len,):
        raise KernelError(f"getvc {trans} with a {m}x{n} needs x[{in_len}], y[{out_len}]")
    if not isinstance(y, torch.Tensor) or not y.is_cuda:
        raise KernelError("getvc updates y in place: pass a CUDA tensor")
    if a.dtype == torch.bfloat16:
        a = a.view(torch.uint16)
    if a.dtype != mode.torch_storage:
        raise KernelError(f"matrix of dtype {a.dtype} for storage {mode.name}")
    if m > 0 and n > 0 and a.stride(1) != 1:
        a = a.contiguous()
    lda = a.stride(0) if m > 1 else n
    xv = _vec(x, mode, "x")
    if y.stride(0) != 1:
        raise KernelError("y must be contiguous")
    launch_getvc(code, a.data_ptr(), mode, m, n, max(lda, n), xv.data_ptr(), alpha, beta, y.data_ptr(),
                 y.device)
    if counters is not None:
        read = m * n + in_len + (out_len if beta != 0.0 else 0)
        counters.count("getvc", read, out_len, mode.storage_bytes)


def tvc_native(
    t: Tensor,
    x,
    k: int,
    *,
    alpha: float = 1.0,
    beta: float = 0.0,
    out=None,
    tasks: int = 1,
    counters: KernelCounters | None = None,
) -> Tensor:
    """Contract mode k of t with vector x at streaming cost for every mode
    (kernels.py:126-171).  ``out`` may be a preallocated flat device buffer of
    at least N/n_k storage elements; the result wraps its prefix."""
    md = matricize_dims(t.shape, k)
    if tuple(x.shape) != (md.nk,):
        raise KernelError(f"vector of {tuple(x.shape)} for mode {k} of extent {md.nk}")
    out_shape = t.shape.drop(k)
    out_size = out_shape.size
    mode = t.mode
    if out is None:
        out = torch.empty(out_size, dtype=mode.torch_storage, device=t.device)
    elif out.numel() < out_size:
        raise KernelError(f"output buffer of {out.numel()} elements, need {out_size}")
    if not isinstance(out, torch.Tensor) or not out.is_cuda or out.dtype != mode.torch_storage:
        raise KernelError("out must be a CUDA tensor in the storage format")
    ybuf = out[:out_size]
    xv = _vec(x, mode, "x")
    launch_tvc(t.buf.data_ptr(), mode, md.u, md.nk, md.v, xv.data_ptr(), alpha, beta, ybuf.data_ptr(),
               t.device)
    if counters is not None:
        read = t.size + md.nk + (out_size if beta != 0.0 else 0)
        counters.count("tvc", read, out_size, mode.storage_bytes)
    return Tensor(out_shape, ybuf, mode)


TVC_NORM_MAX = 1 << 22  # kTvcNormMax in tvc.cu: outputs of a fused TVC + normalize


def tvc_normalize_fits(t: Tensor, k: int) -> bool:
    """Whether tv_tvc_normalize takes this contraction (a small final product)."""
    md = matricize_dims(t.shape, k)
    return md.u * md.v <= TVC_NORM_MAX and t.size <= 64 * TVC_NORM_MAX


def tvc_normalize_async(t: Tensor, x, k: int, out: torch.Tensor, norm_slot: torch.Tensor,
                        status_slot: torch.Tensor | None, counter: torch.Tensor,
                        counters: KernelCounters | None = None) -> Tensor:
    """The last contraction of a power-method iteration with the normalisation
    folded into the kernel epilogue (tv_tvc_normalize): out <- t x_k scaled to
    unit norm, the norm it had into ``norm_slot`` (device float64), TV_ENORM
    into ``status_slot`` on a zero vector; no host sync.  Same bits as
    ``tvc_native`` into out followed by ``normalize(out)`` up to the TVC's
    summation order.  ``counter`` is a zeroed device int32 the kernel leaves
    zeroed.  Counted like the two calls it replaces (kernels.py:168-170,
    234-254)."""
    md = matricize_dims(t.shape, k)
    if tuple(x.shape) != (md.nk,):
        raise KernelError(f"vector of {tuple(x.shape)} for mode {k} of extent {md.nk}")
    out_shape = t.shape.drop(k)
    n = out_shape.size
    mode = t.mode
    if out.numel() < n or out.dtype != mode.torch_storage or not out.is_cuda:
        raise KernelError("out must be a CUDA tensor in the storage format with room for the vector")
    ybuf = out[:n]
    xv = _vec(x, mode, "x")
    sp = status_slot.data_ptr() if status_slot is not None else None
    lib = _lib.load()
    _lib.check(lib.tv_tvc_normalize(t.buf.data_ptr(), mode.tv_storage, mode.tv_compute, md.u, md.nk,
                                    md.v, xv.data_ptr(), ybuf.data_ptr(), norm_slot.data_ptr(), sp,
                                    counter.data_ptr(), _lib.stream_ptr()), "tvc_normalize")
    if counters is not None:
        counters.count("tvc", t.size + md.nk, n, mode.storage_bytes)
    return Tensor(out_shape, ybuf, mode)


def tvc_regime(t: Tensor, k: int) -> str:
    """Name of the kernel regime tv_tvc picks for mode k of t."""
    md = matricize_dims(t.shape, k)
    code = _lib.load().tv_tvc_regime(t.buf.data_ptr(), t.mode.tv_storage, md.u, md.nk, md.v)
    return _lib.REGIMES.get(code, "invalid")


def tvc_looped_oracle(t: Tensor, x, k: int) -> np.ndarray:
    """Naive cross-check (kernels.py:174-188): the tensor and x widened to
    float64 on the device, contracted by the plain scalar kernel only
    (``tv_tvc_naive``), returned as a host float64 array."""
    md = matricize_dims(t.shape, k)
    if tuple(x.shape) != (md.nk,):
        raise KernelError(f"vector of {tuple(x.shape)} for mode {k} of extent {md.nk}")
    a64 = convert(t.buf, _lib.TV_F64) if t.buf.dtype != torch.float64 else t.buf
    xv = _vec(x, t.mode, "x")
    x64 = convert(xv, _lib.TV_F64) if xv.dtype != torch.float64 else xv
    y = torch.empty(md.u * md.v, dtype=torch.float64, device=t.device)
    lib = _lib.load()
    _lib.check(lib.tv_tvc_naive(a64.data_ptr(), _lib.TV_F64, _lib.TV_F64, md.u, md.nk, md.v,
                                x64.data_ptr(), 1.0, 0.0, y.data_ptr(), _lib.stream_ptr()),
               "tvc_looped_oracle")
    return _lib.to_host(y).numpy().reshape(t.shape.drop(k).extents)


def axpby(
    alpha: float,
    x,
    beta: float,
    y,
    *,
    mode: PrecisionMode = F64,
    vl: int = 8,
    counters: KernelCounters | None = None,
) -> None:
    """y := demote(alpha * promote(x) + beta * promote(y)) elementwise, in
    place (kernels.py:191-231).  ``vl`` sized the reference's cache block and
    does not change results; beta = 0 never reads y.  Host numpy y is updated
    in place too."""
    if tuple(x.shape) != tuple(y.shape) or len(tuple(x.shape)) != 1:
        raise KernelError("axpby expects two 1-D vectors of equal length")
    host = None if isinstance(y, torch.Tensor) else y
    xv = _vec(x, mode, "x")
    yv = _vec(y, mode, "y")
    if isinstance(y, torch.Tensor) and yv.data_ptr() != y.data_ptr():
        raise KernelError("axpby works in place: pass a contiguous CUDA vector")
    lib = _lib.load()
    _lib.check(lib.tv_axpby(float(alpha), xv.data_ptr(), float(beta), yv.data_ptr(), mode.tv_storage,
                            mode.tv_compute, yv.numel(), _lib.stream_ptr()), "axpby")
    if host is not None:
        host[...] = _lib.to_host(yv).numpy()
    if counters is not None:
        n = yv.numel()
        counters.count("axpby", n + (n if beta != 0.0 else 0), n, mode.storage_bytes)


# -- normalisation ----------------------------------------------------------


def _norm_async(x: torch.Tensor, mode: PrecisionMode, norm_out: torch.Tensor,
                status_out: torch.Tensor | None, scale: bool) -> None:
    """Enqueue norm (and scale) without a host sync; norm_out is a device
    float64 slot, status_out a device int32 slot (TV_ENORM on a zero norm)."""
    lib = _lib.load()
    sp = status_out.data_ptr() if status_out is not None else None
    if scale:
        rc = lib.tv_normalize(x.data_ptr(), mode.tv_storage, mode.tv_compute, x.numel(),
                              norm_out.data_ptr(), sp, _lib.stream_ptr())
    else:
        rc = lib.tv_norm2(x.data_ptr(), mode.tv_storage, mode.tv_compute, x.numel(),
                          norm_out.data_ptr(), _lib.stream_ptr())
    _lib.check(rc, "normalize" if scale else "norm2")


def norm2(x, *, mode: PrecisionMode = F64, counters: KernelCounters | None = None) -> float:
    """Euclidean norm accumulated in compute precision (kernels.py:234-239)."""
    xv = _vec(x, mode, "x")
    slot = torch.empty(1, dtype=torch.float64, device=xv.device)
    _norm_async(xv, mode, slot, None, scale=False)
    if counters is not None:
        counters.count("norm2", xv.numel(), 0, mode.storage_bytes)
    return float(_lib.to_host(slot).item())


def normalize(x, *, mode: PrecisionMode = F64, counters: KernelCounters | None = None) -> float:
    """Scale x to unit norm in place and return the norm it had
    (kernels.py:242-254).  Host numpy input is updated in place too."""
    host = None if isinstance(x, torch.Tensor) else x
    xv = _vec(x, mode, "x")
    if isinstance(x, torch.Tensor) and xv.data_ptr() != x.data_ptr():
        raise KernelError("normalize works in place: pass a contiguous CUDA vector")
    slot = torch.empty(1, dtype=torch.float64, device=xv.device)
    status = torch.zeros(1, dtype=torch.int32, device=xv.device)
    _norm_async(xv, mode, slot, status, scale=True)
    if counters is not None:
        counters.count("norm2", xv.numel(), 0, mode.storage_bytes)
    if int(_lib.to_host(status).item()) != 0:
        raise NormalizationError("cannot normalize a zero vector")
    if counters is not None:
        counters.count("scale", xv.numel(), xv.numel(), mode.storage_bytes)
    if host is not None:
        host[...] = _lib.to_host(xv).numpy()
    return float(_lib.to_host(slot).item())
