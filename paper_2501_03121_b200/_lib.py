"""ctypes binding of libtenvec_b200.so (include/tenvec_b200.h).

The library is the only compute path of this package: there is no CPU
fallback.  Loading fails loudly when the .so is missing, and every device
entry point checks that CUDA is available before it is called.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import CollectiveError, DeviceError, KernelError, ModeError, NormalizationError

import os as _os

# TENVEC_B200_LIB: load another build of the library (kernel A/B variants)
LIB_PATH = Path(_os.environ.get("TENVEC_B200_LIB") or
                Path(__file__).resolve().parent / "_lib" / "libtenvec_b200.so")

# tv_dtype codes
TV_F64, TV_F32, TV_F16, TV_BF16 = 0, 1, 2, 3
TV_FILL_ONES, TV_FILL_RAMP, TV_FILL_HASH = 0, 1, 2
TV_MAX_RANKS = 64
TV_PEER_HEADER = 4096
TV_AR_NCCL, TV_AR_EXACT, TV_AR_MIXED = 0, 1, 2
REGIMES = {0: "naive", 1: "rows", 2: "rows_short", 3: "cols", 4: "slabs", 5: "rows_u", 6: "cols_u",
           7: "slabs_u", 8: "staged", 9: "flat",
           10: "flat_rows", 11: "staged_long", 12: "flat_u", 13: "staged_tall"}

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_int = ctypes.c_int

# symbol -> (restype, argtypes); the list every test checks is exported
SIGNATURES = {
    "tv_version": (ctypes.c_char_p, []),
    "tv_last_error": (ctypes.c_char_p, []),
    "tv_tvc": (_int, [_vp, _int, _int, _i64, _i64, _i64, _vp, ctypes.c_double, ctypes.c_double, _vp, _vp]),
    "tv_tvc_ws": (_int, [_vp, _int, _int, _i64, _i64, _i64, _vp, ctypes.c_double, ctypes.c_double, _vp, _vp,
                          _i64, _vp]),
    "tv_tvc_workspace_bytes": (_i64, [_vp, _int, _int, _i64, _i64, _i64]),
    "tv_getvc_ws": (_int, [_int, _vp, _int, _int, _i64, _i64, _i64, _vp, ctypes.c_double, ctypes.c_double,
                           _vp, _vp, _i64, _vp]),
    "tv_getvc_workspace_bytes": (_i64, [_int, _vp, _int, _int, _i64, _i64, _i64]),
    "tv_tvc_sweep": (_int, [_vp, _int, _int, _int, ctypes.POINTER(_i64), ctypes.POINTER(_vp),
                            ctypes.POINTER(_vp), _vp, _i64, _vp]),
    "tv_tvc_sweep_workspace_bytes": (_i64, [_vp, _int, _int, _int, ctypes.POINTER(_i64)]),
    "tv_tvc_naive": (_int, [_vp, _int, _int, _i64, _i64, _i64, _vp, ctypes.c_double, ctypes.c_double, _vp, _vp]),
    "tv_tvc_normalize": (_int, [_vp, _int, _int, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "tv_tvc_regime": (_int, [_vp, _int, _i64, _i64, _i64]),
    "tv_set_regime_override": (_int, [_int]),
    "tv_getvc": (_int, [_int, _vp, _int, _int, _i64, _i64, _i64, _vp, ctypes.c_double, ctypes.c_double, _vp, _vp]),
    "tv_convert": (_int, [_vp, _int, _vp, _int, _i64, _vp]),
    "tv_norm2": (_int, [_vp, _int, _int, _i64, _vp, _vp]),
    "tv_normalize": (_int, [_vp, _int, _int, _i64, _vp, _vp, _vp]),
    "tv_rank_fold": (_int, [ctypes.POINTER(_vp), _int, _i64, _i64, _int, _int, _int, _int, _vp, _vp]),
    "tv_rank_fold_strided": (_int, [_vp, _i64, _int, _i64, _i64, _int, _int, _int, _int, _vp, _vp]),
    "tv_rank_fold_normalize": (_int, [_vp, _i64, _int, _i64, _i64, _int, _int, _int, _vp, _vp, _vp, _vp,
                                       _vp]),
    "tv_rank_fold_range": (_int, [_vp, _i64, _int, _i64, _i64, _i64, _int, _int, _int, _vp, _vp]),
    "tv_rank_select": (_int, [ctypes.POINTER(_vp), _int, _i64, _i64, _int, _vp, _vp]),
    "tv_comm_get_unique_id": (_int, [_vp]),
    "tv_comm_init_rank": (_int, [_vp, _int, _int, ctypes.POINTER(_vp)]),
    "tv_comm_init_all": (_int, [_int, ctypes.POINTER(_int), ctypes.POINTER(_vp)]),
    "tv_comm_rank_size": (_int, [_vp, ctypes.POINTER(_int), ctypes.POINTER(_int)]),
    "tv_comm_destroy": (_int, [_vp]),
    "tv_allreduce_workspace_bytes": (_i64, [_vp, _i64, _int, _int]),
    "tv_allreduce": (_int, [_vp, _vp, _i64, _int, _int, _int, _vp, _i64, _vp]),
    "tv_allgather": (_int, [_vp, _vp, _vp, ctypes.POINTER(_i64), _int, _vp]),
    "tv_dhopm3_plan_create": (_int, [_vp, _vp, _int, _int, _int, ctypes.POINTER(_i64), _int, ctypes.POINTER(_vp)]),
    "tv_dhopm3_plan_slab": (_int, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "tv_dhopm3_sweep": (_int, [_vp, ctypes.POINTER(_vp), _vp, _vp, _vp]),
    "tv_dhopm3_plan_destroy": (_int, [_vp]),
    "tv_repack_part": (_int, [_vp, _int, _int, _i64, _i64, _i64, _i64, _int, _vp, _vp]),
    "tv_repack_part_multicast": (_int, [_vp, _int, _int, _i64, _i64, _i64, _i64, _int, _vp, _vp]),
    "tv_repack_part_peers": (_int, [_vp, _int, _int, _i64, _i64, _i64, _i64, _int, ctypes.POINTER(_vp), _int,
                                    _vp]),
    "tv_repack": (_int, [ctypes.POINTER(_vp), _int, _i64, _i64, _i64, _i64, _int, _vp, _vp]),
    "tv_peer_barrier": (_int, [ctypes.POINTER(_vp), _int, _int, ctypes.c_uint32, _i64, _vp, _vp]),
    "tv_preload": (_int, [ctypes.POINTER(_int)]),
    "tv_fill": (_int, [_vp, _int, _int, ctypes.c_uint64, ctypes.POINTER(_i64), _int, _int, _i64, _i64, _vp]),
    "tv_axpby": (_int, [ctypes.c_double, _vp, ctypes.c_double, _vp, _int, _int, _i64, _vp]),
    "tv_read_stream": (_int, [_vp, _i64, _vp, _vp]),
    "tv_device_sms": (_int, []),
    "tv_launch_count": (ctypes.c_ulonglong, []),
}

_ERRORS = {1: KernelError, 2: ModeError, 3: NormalizationError, 4: CollectiveError, 5: DeviceError}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and return the library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"{p} is missing: build it with `python -m paper_2501_03121_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


_preloaded: set = set()


def preload() -> int:
    """tv_preload on the current device, once per device: every kernel loaded
    before a device barrier can spin (lazy loading could otherwise make a
    first launch wait for the barrier that waits for it)."""
    import torch

    dev = torch.cuda.current_device()
    if dev in _preloaded:
        return 0
    lib = load()
    n = ctypes.c_int(0)
    check(lib.tv_preload(ctypes.byref(n)), "tv_preload")
    with _lock:
        _preloaded.add(dev)
    return n.value


def host_wait(stream=None) -> None:
    """Wait on the host for the work queued on ``stream`` (default: the
    current one) by polling an event, never inside a blocking driver call:
    thread-ranks sharing one GPU (loopback) keep issuing work -- the very
    barrier arrival this stream may be waiting for -- while this one waits,
    and a blocking synchronize can hold driver locks their calls need."""
    import time

    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(s)
    while not ev.query():
        time.sleep(5e-5)


def to_host(t):
    """t.cpu() after host_wait()."""
    if t.is_cuda:
        host_wait()
    return t.cpu()


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    lib = load()
    msg = lib.tv_last_error().decode(errors="replace")
    exc = _ERRORS.get(rc, DeviceError)
    raise exc(f"{what}: {msg}" if what else msg)


def require_cuda() -> None:
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("a CUDA device is required: libtenvec_b200 has no CPU path")


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
