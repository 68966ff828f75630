"""tv_tvc_normalize: the last contraction of a power-method iteration with the
normalisation folded into the kernel epilogue.  Integer data makes every sum
exact, so the fused result must be bitwise tvc_native + normalize (same
normalisation tree); float data within the TVC tolerances of the oracle."""

import numpy as np
import pytest
import torch

import tenvec_oracle as O

pytestmark = pytest.mark.gpu

MODES = ["f64", "f32", "f32f64", "f16f32", "bf16f32"]
TOL = {"f64": 1e-12, "f32": 1e-5, "f32f64": 1e-6, "f16f32": 2e-3, "bf16f32": 1.6e-2}
CASES = [((300, 96), 1), ((300, 97), 1), ((1, 4096), 1), ((96, 300), 0), ((97, 301), 0),
         ((5, 7, 33), 1), ((3, 1000, 2), 1), ((4096, 3), 1), ((2, 2), 0), ((1, 1), 0),
         ((64, 64, 64), 2), ((2000, 1999), 0)]


def _bits(t):
    return t.view(torch.uint8) if t.dtype != torch.uint16 else t.view(torch.int16).view(torch.uint8)


def _fused(tv, t, x, k):
    slot = torch.empty(1, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    counter = torch.zeros(1, dtype=torch.int32, device="cuda")
    n = t.shape.drop(k).size
    out = torch.empty(n, dtype=t.mode.torch_storage, device="cuda")
    y = tv.kernels.tvc_normalize_async(t, x, k, out, slot, status, counter)
    torch.cuda.synchronize()
    assert int(counter.item()) == 0  # ticket counter left clean
    return y, float(slot.item()), int(status.item())


@pytest.mark.parametrize("mode_name", MODES)
@pytest.mark.parametrize("shape,k", CASES)
def test_fused_equals_tvc_then_normalize_on_integer_data(tv, mode_name, shape, k):
    mode = tv.MODES[mode_name]
    rng = np.random.default_rng(hash((shape, k)) % 2**32)
    vals = rng.integers(1, 6, shape).astype(np.float64)
    t = tv.Tensor.from_array(vals, mode)
    x = O.demote(rng.integers(1, 4, shape[k]).astype(np.float64), mode_name).copy()
    assert tv.kernels.tvc_normalize_fits(t, k)
    y, nrm, st = _fused(tv, t, x, k)
    ref = tv.tvc_native(t, x, k)
    ref_norm = tv.normalize(ref.buf, mode=mode)
    assert st == 0
    assert torch.equal(_bits(y.buf), _bits(ref.buf)), (shape, k, mode_name)
    assert nrm == ref_norm


@pytest.mark.parametrize("mode_name", ["f64", "f32", "bf16f32"])
def test_fused_float_data_against_oracle(tv, mode_name):
    mode = tv.MODES[mode_name]
    rng = np.random.default_rng(3)
    for shape, k in CASES:
        vals = rng.standard_normal(shape)
        t = tv.Tensor.from_array(vals, mode)
        x = O.demote(rng.standard_normal(shape[k]), mode_name).copy()
        y, nrm, _ = _fused(tv, t, x, k)
        want = O.promote(O.tvc(t.to_numpy(), shape, x, k, mode_name), mode_name).astype(float)
        wn = np.linalg.norm(want)
        got = O.promote(y.to_numpy(), mode_name).astype(float)
        tol = 10 * TOL[mode_name]
        assert abs(nrm - wn) <= tol * wn, (shape, k)
        assert np.allclose(got, want / wn, rtol=tol, atol=tol), (shape, k)


def test_fused_zero_vector_and_limits(tv):
    t = tv.Tensor.from_array(np.zeros((40, 50)))
    y, nrm, st = _fused(tv, t, np.ones(50), 1)
    assert st == 3 and nrm == 0.0 and not y.to_numpy().any()  # TV_ENORM, left unscaled
    big = tv.Tensor(tv.Shape((1 << 22, 2, 2)), torch.empty(1 << 24, dtype=torch.float64, device="cuda"), tv.F64)
    assert not tv.kernels.tvc_normalize_fits(big, 1)
    with pytest.raises(tv.KernelError):
        _fused(tv, big, np.ones(2), 1)


def test_dhopm3_fused_normalisation_matches_unfused(tv, monkeypatch):
    """Single rank: dhopm3 with the epilogue normalisation equals the separate
    TVC + copy + normalize path to rounding (the fused kernel sums in its own
    order; normalised vectors make later sums inexact), with identical counts."""
    for vals in (np.random.default_rng(1).integers(1, 5, (9, 8, 7)).astype(float),
                 np.random.default_rng(2).standard_normal((12, 11, 10, 9))):
        A = tv.Tensor.from_array(vals)
        x0 = [np.ones(n) for n in vals.shape]
        fused = tv.dhopm3(tv.distribute(A, 0, 1), [v.copy() for v in x0], sweeps=2)
        monkeypatch.setenv("TENVEC_B200_FUSE_NORM", "0")
        plain = tv.dhopm3(tv.distribute(A, 0, 1), [v.copy() for v in x0], sweeps=2)
        monkeypatch.delenv("TENVEC_B200_FUSE_NORM")
        assert fused.iteration_touched == plain.iteration_touched
        assert fused.tvc_count == plain.tvc_count
        for a, b in zip(fused.vectors, plain.vectors):
            assert np.allclose(a, b, rtol=1e-12, atol=1e-14)
        assert np.allclose(fused.norms, plain.norms, rtol=1e-13)
