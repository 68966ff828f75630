"""Storage/compute precision pairs and their device conversions.

Mirrors the reference precision module (pkg/src/tenvec/precision.py:1-145):
the same five modes (f64, f32, f32f64, f16f32, bf16f32), the same names and
properties, and bit-identical promote/demote semantics -- promotion is exact,
double->single and ->half round to nearest even (half overflow -> inf), brain
is binary32 truncated to its top 16 bits after an RNE step to binary32.

Buffers are torch CUDA tensors.  Brain buffers are ``torch.uint16`` bit
patterns, exactly like the reference's ``np.uint16`` arrays
(precision.py:73).  Every conversion runs on the device through
``tv_convert`` (libtenvec_b200); numpy inputs are uploaded, converted and
returned as numpy so reference-style callers keep working.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ModeError

__all__ = [
    "ModeError", "PrecisionMode", "F64", "F32", "F32F64", "F16F32", "BF16F32", "MODES",
    "parse_mode", "f32_to_bf16_bits", "bf16_bits_to_f32", "promote", "demote", "demote_copy",
    "storage_zeros", "storage_empty", "convert", "torch_dtype_of", "tv_dtype_of",
]

_STORAGE_NP = {
    "double": np.dtype(np.float64),
    "single": np.dtype(np.float32),
    "half": np.dtype(np.float16),
    "brain": np.dtype(np.uint16),  # bit patterns, not numbers
}
_COMPUTE_NP = {"double": np.dtype(np.float64), "single": np.dtype(np.float32)}
_STORAGE_TORCH = {
    "double": torch.float64,
    "single": torch.float32,
    "half": torch.float16,
    "brain": torch.uint16,
}
_COMPUTE_TORCH = {"double": torch.float64, "single": torch.float32}
_TV_CODE = {"double": _lib.TV_F64, "single": _lib.TV_F32, "half": _lib.TV_F16, "brain": _lib.TV_BF16}

_TORCH_TO_TV = {
    torch.float64: _lib.TV_F64,
    torch.float32: _lib.TV_F32,
    torch.float16: _lib.TV_F16,
    torch.uint16: _lib.TV_BF16,
    torch.bfloat16: _lib.TV_BF16,
}
_TV_TO_TORCH = {_lib.TV_F64: torch.float64, _lib.TV_F32: torch.float32,
                _lib.TV_F16: torch.float16, _lib.TV_BF16: torch.uint16}


@dataclass(frozen=True)
class PrecisionMode:
    """A valid (storage, compute) pair (precision.py:30-66)."""

    name: str
    storage: str
    compute: str

    @property
    def storage_dtype(self) -> np.dtype:
        return _STORAGE_NP[self.storage]

    @property
    def compute_dtype(self) -> np.dtype:
        return _COMPUTE_NP[self.compute]

    @property
    def storage_bytes(self) -> int:
        return self.storage_dtype.itemsize

    @property
    def compute_bytes(self) -> int:
        return self.compute_dtype.itemsize

    @property
    def mixed(self) -> bool:
        return self.storage != self.compute

    # -- device-side views of the same pair --------------------------------
    @property
    def torch_storage(self) -> torch.dtype:
        return _STORAGE_TORCH[self.storage]

    @property
    def torch_compute(self) -> torch.dtype:
        return _COMPUTE_TORCH[self.compute]

    @property
    def tv_storage(self) -> int:
        return _TV_CODE[self.storage]

    @property
    def tv_compute(self) -> int:
        return _TV_CODE[self.compute]


F64 = PrecisionMode("f64", "double", "double")
F32 = PrecisionMode("f32", "single", "single")
F32F64 = PrecisionMode("f32f64", "single", "double")
F16F32 = PrecisionMode("f16f32", "half", "single")
BF16F32 = PrecisionMode("bf16f32", "brain", "single")

MODES = {m.name: m for m in (F64, F32, F32F64, F16F32, BF16F32)}


def parse_mode(name: str) -> PrecisionMode:
    try:
        return MODES[name]
    except KeyError:
        raise ModeError(f"unknown precision mode {name!r}; pick one of {sorted(MODES)}") from None


def tv_dtype_of(t: torch.Tensor) -> int:
    try:
        return _TORCH_TO_TV[t.dtype]
    except KeyError:
        raise ModeError(f"no device element type for {t.dtype}") from None


def torch_dtype_of(code: int) -> torch.dtype:
    return _TV_TO_TORCH[code]


def _device() -> torch.device:
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _to_device(a, np_brain: bool = False) -> torch.Tensor:
    """numpy / python data -> 1-D-or-not CUDA tensor keeping the element type."""
    if isinstance(a, torch.Tensor):
        return a if a.is_cuda else a.to(_device())
    arr = np.asarray(a)
    if arr.dtype == np.uint16 and np_brain:
        return torch.from_numpy(np.ascontiguousarray(arr)).to(_device())
    if arr.dtype not in (np.float64, np.float32, np.float16):
        arr = arr.astype(np.float64)
    return torch.from_numpy(np.ascontiguousarray(arr)).to(_device())


def convert(src: torch.Tensor, dst_code: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """Device conversion with reference rounding (tv_convert)."""
    src = src.contiguous()
    if out is None:
        out = torch.empty(src.shape, dtype=torch_dtype_of(dst_code), device=src.device)
    lib = _lib.load()
    _lib.check(lib.tv_convert(src.data_ptr(), tv_dtype_of(src), out.data_ptr(), dst_code,
                              src.numel(), _lib.stream_ptr()), "convert")
    return out


def _roundtrip(a, fn):
    """Apply a device conversion to numpy input and hand numpy back."""
    if isinstance(a, torch.Tensor):
        return fn(_to_device(a))
    res = fn(_to_device(a, np_brain=True))
    return _lib.to_host(res).numpy()


def f32_to_bf16_bits(a):
    """Truncate binary32 values to brain bit patterns (precision.py:97-100)."""
    def fn(t):
        if t.dtype != torch.float32:
            t = convert(t, _lib.TV_F32)
        return convert(t, _lib.TV_BF16)
    return _roundtrip(a, fn)


def bf16_bits_to_f32(bits):
    """Widen brain bit patterns back to binary32 (precision.py:103-106)."""
    def fn(t):
        if t.dtype != torch.uint16:
            t = t.view(torch.uint16) if t.element_size() == 2 else t.to(torch.uint16)
        return convert(t, _lib.TV_F32)
    if isinstance(bits, np.ndarray) and bits.dtype != np.uint16:
        bits = bits.astype(np.uint16)
    return _roundtrip(bits, fn)


def promote(a, mode: PrecisionMode):
    """Storage buffer -> compute buffer, exact (precision.py:109-115)."""
    def fn(t):
        if mode.storage == "brain" and t.dtype == torch.bfloat16:
            t = t.view(torch.uint16)
        if t.dtype == mode.torch_compute:
            return t
        return convert(t, mode.tv_compute)
    if isinstance(a, np.ndarray) and mode.storage == "brain":
        a = a.astype(np.uint16, copy=False)
    return _roundtrip(a, fn)


def demote(a, mode: PrecisionMode):
    """Compute buffer -> storage buffer (precision.py:118-128): RNE to single or
    half (half overflow -> inf), brain = RNE to binary32 then truncation."""
    def fn(t):
        if t.dtype == mode.torch_storage:
            return t
        return convert(t, mode.tv_storage)
    return _roundtrip(a, fn)


def demote_copy(a, mode: PrecisionMode):
    out = demote(a, mode)
    if isinstance(out, torch.Tensor) and isinstance(a, torch.Tensor) and out.data_ptr() == a.data_ptr():
        out = out.clone()
    elif isinstance(out, np.ndarray) and (out is a or out.base is a):
        out = out.copy()
    return out


def storage_zeros(n: int, mode: PrecisionMode) -> torch.Tensor:
    return torch.zeros(n, dtype=mode.torch_storage, device=_device())  # 0x0000 is +0.0 in brain


def storage_empty(n: int, mode: PrecisionMode) -> torch.Tensor:
    return torch.empty(n, dtype=mode.torch_storage, device=_device())
