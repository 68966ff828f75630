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


def test_c_program_drives_dhopm3_without_python(tv, tmp_path):
    """examples/dhopm3_capi.c -- a plain C host (gcc, libcudart, this .so;
    no Python in the process) -- prints the same norms as the package's
    dhopm3 on the same tensor, to the last bit."""
    import os
    import shutil
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lib_dir = os.path.join(root, "paper_2501_03121_b200", "_lib")
    exe = str(tmp_path / "dhopm3_capi")
    subprocess.run([cc, "-O2", "-I", os.path.join(root, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(root, "examples", "dhopm3_capi.c"), "-o", exe, "-L", lib_dir, "-ltenvec_b200",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", "-lpthread"], check=True)
    env = dict(os.environ, LD_LIBRARY_PATH=lib_dir + ":/usr/local/cuda/lib64:" + os.environ.get("LD_LIBRARY_PATH", ""))
    n, sweeps = 96, 4
    out = subprocess.run([exe, "1", str(n), str(sweeps)], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr
    norms = [float(v) for v in out.stdout.split("norms")[1].split()]
    shape = tv.Shape((n, n, n))
    dt = tv.distribute_generated(shape, 0, 1, tv.F64, fill="hash", seed=1)
    res = tv.dhopm3(dt, tv.initial_vectors(shape, tv.F64), sweeps=sweeps)
    assert norms == res.norms[-1]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_c_program_across_gpus_equals_in_process_split(tv, tmp_path):
    """The same C program over 2 GPUs (tv_comm_init_all, one host thread per
    GPU, NCCL collectives) gives the bits of the reference's threads-as-ranks
    run of the same 2-way split (dhopm3 on an in-process distribute)."""
    import os
    import shutil
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cc = shutil.which("gcc") or shutil.which("cc")
    lib_dir = os.path.join(root, "paper_2501_03121_b200", "_lib")
    exe = str(tmp_path / "dhopm3_capi")
    subprocess.run([cc, "-O2", "-I", os.path.join(root, "include"), "-I", "/usr/local/cuda/include",
                    os.path.join(root, "examples", "dhopm3_capi.c"), "-o", exe, "-L", lib_dir, "-ltenvec_b200",
                    "-L", "/usr/local/cuda/lib64", "-lcudart", "-lpthread"], check=True)
    env = dict(os.environ, LD_LIBRARY_PATH=lib_dir + ":/usr/local/cuda/lib64:" + os.environ.get("LD_LIBRARY_PATH", ""))
    n, sweeps = 128, 3
    out = subprocess.run([exe, "2", str(n), str(sweeps)], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr
    norms = [float(v) for v in out.stdout.split("norms")[1].split()]
    shape = tv.Shape((n, n, n))
    dt = tv.distribute_generated(shape, 0, 2, tv.F64, fill="hash", seed=1)
    res = tv.dhopm3(dt, tv.initial_vectors(shape, tv.F64), sweeps=sweeps)
    assert norms == res.norms[-1]
