"""The distributed C-ABI on one GPU (no communicator): tv_dhopm3_plan_create
+ tv_dhopm3_sweep give the Python dhopm3's bits (hopm.py:229-354) for every
mode, split and order; the collectives with one rank are the identity.  The
NCCL ranks run in tests/test_gpu_multi.py (capi_checks)."""

import ctypes

import numpy as np
import pytest
import torch

from capi_checks import c_dhopm3, same_run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["f64", "f32", "f32f64", "f16f32", "bf16f32"])
@pytest.mark.parametrize("shape,s", [((12, 10, 9), 0), ((6, 7, 8), 1), ((5, 6, 7, 8), 2), ((4, 5, 6, 3, 2), 4),
                                     ((300, 200), 1), ((96, 96, 96, 24), 3), ((64, 2048, 3), 0)])
def test_c_dhopm3_equals_python_dhopm3(tv, name, shape, s):
    mode = tv.MODES[name]
    rng = np.random.default_rng(sum(shape))
    A = tv.Tensor.from_array(rng.standard_normal(shape), mode)
    x0 = tv.initial_vectors(tv.Shape(shape), mode)
    res = tv.dhopm3(tv.distribute(A, s, 1), [v.copy() for v in x0], sweeps=4)
    vecs, norms, st = c_dhopm3(tv, None, A, shape, s, mode, x0, 4)
    assert st == 0
    assert same_run(res, vecs, norms), (res.norms[-1], norms[-1])


def test_c_dhopm3_rejects_bad_plans_and_reports_zero_vectors(tv):
    lib = tv._lib.load()
    A = tv.Tensor.from_array(np.zeros((4, 5, 6)))
    plan = ctypes.c_void_p()
    ext = (ctypes.c_int64 * 3)(4, 5, 6)
    assert lib.tv_dhopm3_plan_create(None, A.buf.data_ptr(), 0, 0, 3, ext, 3, ctypes.byref(plan)) != 0
    assert lib.tv_dhopm3_plan_create(None, A.buf.data_ptr(), 2, 2, 3, ext, 0, ctypes.byref(plan)) != 0
    x0 = tv.initial_vectors(tv.Shape((4, 5, 6)), tv.F64)
    _, _, st = c_dhopm3(tv, None, A, (4, 5, 6), 0, tv.F64, x0, 1)
    assert st == 3  # TV_ENORM: the zero vector is left unscaled and reported


def test_collectives_with_one_rank_need_a_communicator(tv):
    lib = tv._lib.load()
    buf = torch.ones(8, dtype=torch.float64, device="cuda")
    assert lib.tv_allreduce(None, buf.data_ptr(), 8, 0, 0, 1, None, 0, None) != 0
    assert b"communicator" in lib.tv_last_error()
