"""Generate tests/golden/*.npz by running the REFERENCE package itself.

Run here (the container that has /root/reference); the GPU box only reads the
committed .npz files:

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

Every fixture is the reference's own output on seeded inputs: the oracle
(oracle/tenvec_oracle.py) is pinned against these, and the GPU parity tests
compare the CUDA path against both.  Cases follow the reference tests:
test_kernels.py:77-89 (200 random integer shapes), test_acceptance.py:28-76
(SHAPE_SUITE dtvc over every k, s, p), test_acceptance.py:189-218 and
test_comm.py (precision and ring folds), test_hopm.py / test_acceptance.py:79-96
(power method).
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

SHAPE_SUITE = [(2, 2), (3, 5), (6, 6), (2, 3, 4), (4, 4, 4), (5, 2, 6), (2, 3, 2, 4),
               (3, 3, 3, 3), (2, 2, 3, 2, 4)]
MODE_SHAPES = [(7,), (3, 5), (5, 8), (4, 6, 5), (2, 3, 4, 5), (6, 1, 9), (3, 40, 8), (2, 9, 33)]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--only", default="all", choices=["all", "costmodel"])
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    import tenvec as T  # the reference package

    costmodel()
    if args.only == "costmodel":
        return

    # -- precision ---------------------------------------------------------
    spots = np.array([1.0, np.pi, 2.0, -1.5, 1e-38, 1.1754944e-38, 65504.0, 3.0e38, -7.25e-5,
                      1.0 + 2.0 ** -9, 1.0 + 2.0 ** -8 + 2.0 ** -20])
    rng = np.random.default_rng(17)
    hvals = np.concatenate([
        rng.uniform(-70000, 70000, 600), rng.uniform(-1e-4, 1e-4, 300),
        rng.uniform(-6e-8, 6e-8, 100),
        np.array([65504.0, 65519.9, 65520.0, 2.0 ** -25, -(2.0 ** -25), 0.0, 2.0 ** -24 * 1.5]),
    ])
    prec = {
        "spots": spots,
        "spots_bf16": T.demote(spots, T.BF16F32),
        "spots_f32": T.demote(spots, T.F32),
        "hvals": hvals,
        "hvals_f16": T.demote(hvals, T.F16F32),
        "hvals_f16_from_f32": T.demote(hvals.astype(np.float32), T.F16F32),
        "hvals_bf16": T.demote(hvals, T.BF16F32),
        "bf16_widen": T.promote(T.demote(spots, T.BF16F32), T.BF16F32),
    }
    np.savez_compressed(HERE / "precision.npz", **prec)

    # -- tvc on 200 random integer shapes (test_kernels.py:77-89) ------------
    rng = np.random.default_rng(1234)
    out = {}
    for i in range(200):
        d = int(rng.integers(2, 6))
        extents = tuple(int(e) for e in rng.integers(1, 7, d))
        vals = rng.integers(1, 97, extents).astype(float)
        t = T.Tensor.from_array(vals)
        k = int(rng.integers(0, d))
        x = rng.integers(1, 97, extents[k]).astype(float)
        y = T.tvc_native(t, x, k)
        out[f"c{i}_shape"] = np.array(extents)
        out[f"c{i}_k"] = np.array(k)
        out[f"c{i}_vals"] = vals.reshape(-1)
        out[f"c{i}_x"] = x
        out[f"c{i}_y"] = y.to_float64().reshape(-1)
    out["n"] = np.array(200)
    np.savez_compressed(HERE / "tvc_int.npz", **out)

    # -- tvc in every precision mode, float data, alpha/beta ---------------
    rng = np.random.default_rng(77)
    out = {}
    c = 0
    for name in sorted(T.MODES):
        mode = T.MODES[name]
        for shape in MODE_SHAPES:
            for k in range(len(shape)):
                vals = rng.standard_normal(shape)
                t = T.Tensor.from_array(vals, mode)
                x = T.demote(rng.standard_normal(shape[k]), mode).copy()
                alpha, beta = (1.0, 0.0) if c % 3 else (1.5, -0.75)
                y0 = T.demote(rng.standard_normal(t.size // shape[k]), mode).copy()
                y = T.tvc_native(t, x, k, alpha=alpha, beta=beta, out=y0.copy())
                out[f"c{c}_mode"] = np.array(name)
                out[f"c{c}_shape"] = np.array(shape)
                out[f"c{c}_k"] = np.array(k)
                out[f"c{c}_buf"] = t.buf
                out[f"c{c}_x"] = x
                out[f"c{c}_y0"] = y0
                out[f"c{c}_ab"] = np.array([alpha, beta])
                out[f"c{c}_y"] = y.buf.copy()
                c += 1
    out["n"] = np.array(c)
    np.savez_compressed(HERE / "tvc_modes.npz", **out)

    # -- CLI / harness CSV under --deterministic (cli.py, bench.py:330-394) --
    import contextlib
    import io
    import json
    from tenvec.cli import main as ref_cli
    cli_cases = [
        ["tvc", "--dims", "6,7,8", "--mode", "1", "--deterministic", "--iters", "2"],
        ["tvc", "--dims", "desk:d3", "--mode", "2", "--precision", "bf16f32", "--deterministic"],
        ["tvc", "--dims", "13^3", "--mode", "0", "--fill", "ramp", "--deterministic"],
        ["dtvc", "--dims", "8,6,10", "--mode", "0", "--split", "0", "--workers", "3", "--deterministic"],
        ["dtvc", "--dims", "8,6,10", "--mode", "1", "--split", "0", "--workers", "3",
         "--assembly", "interleave", "--deterministic"],
        ["dtvc", "--dims", "8,6,10", "--mode", "2", "--split", "2", "--workers", "4", "--defer",
         "--deterministic"],
        ["dtvc", "--dims", "9,5,6", "--mode", "0", "--split", "0", "--workers", "2",
         "--precision", "f16f32", "--deterministic"],
        ["hopm", "--dims", "6^4", "--split", "1", "--workers", "2", "--sweeps", "2", "--deterministic"],
        ["hopm", "--dims", "8^3", "--split", "0", "--workers", "2", "--classical-hopm", "--deterministic"],
        ["hopm", "--dims", "8^3", "--split", "2", "--workers", "3", "--precision", "f32f64",
         "--deterministic"],
        ["triad", "--dims", "1000", "--deterministic"],
        ["tvc", "--dims", "4^3", "--mode", "5", "--deterministic"],
        ["dtvc", "--dims", "4^3", "--mode", "0", "--split", "0", "--workers", "9", "--deterministic"],
    ]
    records = []
    for argv in cli_cases:
        buf, err = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(err):
            rc = ref_cli(argv)
        records.append({"argv": argv, "rc": rc, "stdout": buf.getvalue()})
    (HERE / "cli.json").write_text(json.dumps(records, indent=1) + "\n")

    # -- axpby (kernels.py:191-231; test_kernels.py:184-210) ------------------
    rng = np.random.default_rng(31)
    out = {}
    for name in sorted(T.MODES):
        mode = T.MODES[name]
        x = T.demote(rng.standard_normal(1000), mode).copy()
        y0 = T.demote(rng.standard_normal(1000), mode).copy()
        for tag, (alpha, beta) in (("ab", (1.25, -0.5)), ("a0", (2.0, 0.0))):
            y = y0.copy()
            T.axpby(alpha, x, beta, y, mode=mode, vl=8)
            out[f"{name}_{tag}_x"] = x
            out[f"{name}_{tag}_y0"] = y0
            out[f"{name}_{tag}_y"] = y
            out[f"{name}_{tag}_ab"] = np.array([alpha, beta])
    np.savez_compressed(HERE / "axpby.npz", **out)

    # -- ring folds (comm.py:84-134) ----------------------------------------
    rng = np.random.default_rng(31)
    out = {}
    c = 0
    for name in ("f64", "f32", "f32f64", "f16f32", "bf16f32"):
        mode = T.MODES[name]
        for p in (2, 3, 4, 5, 8):
            for n in (1, 4, 10, 11, 24, 37):
                ranks = [T.demote(rng.uniform(-4, 4, n), mode).copy() for _ in range(p)]
                bufs = [r.copy() for r in ranks]
                if mode.mixed:
                    T.ring_all_reduce_mixed(bufs, mode)
                else:
                    T.ring_all_reduce(bufs)
                out[f"c{c}_mode"] = np.array(name)
                out[f"c{c}_ranks"] = np.stack(ranks)
                out[f"c{c}_out"] = bufs[0]
                c += 1
    out["n"] = np.array(c)
    np.savez_compressed(HERE / "ring.npz", **out)

    # -- dtvc over SHAPE_SUITE (test_acceptance.py:54-76) -------------------
    out = {}
    c = 0
    for shape in SHAPE_SUITE:
        rng = np.random.default_rng(len(shape))
        vals = rng.integers(-4, 5, shape).astype(float)
        t = T.Tensor.from_array(vals)
        d = len(shape)
        for k in range(d):
            x = np.random.default_rng(10 * k + 1).integers(-4, 5, shape[k]).astype(float)
            for s in range(d):
                for p in sorted({1, 2, 3, shape[s]}):
                    for defer in ((False, True) if k == s else (False,)):
                        res = T.dtvc(T.distribute(t, s, p), x, k, defer=defer)
                        got = T.undistribute(res).to_float64().reshape(-1)
                        out[f"c{c}"] = np.concatenate([[len(shape)], shape, [k, s, p, int(defer)], got])
                        c += 1
        out[f"vals{SHAPE_SUITE.index(shape)}"] = vals.reshape(-1)
    out["n"] = np.array(c)
    np.savez_compressed(HERE / "dtvc.npz", **out)

    # -- power method -----------------------------------------------------
    out = {}
    c = 0
    cases = [((8, 8), 0, 1, "f64"), ((8, 8, 8), 0, 2, "f64"), ((6, 5, 4), 2, 2, "f64"),
             ((6, 6, 6, 6), 1, 3, "f64"), ((4, 4, 4, 4, 4), 4, 2, "f64"), ((9, 7, 5), 1, 3, "f32"),
             ((8, 8, 8), 1, 2, "f32f64"), ((12, 10, 8), 0, 4, "f16f32"), ((12, 10, 8), 2, 3, "bf16f32"),
             ((5, 6, 7, 8), 3, 4, "bf16f32"), ((16, 16, 16), 1, 1, "bf16f32")]
    for shape, s, p, name in cases:
        mode = T.MODES[name]
        rng = np.random.default_rng(100 + c)
        vals = rng.standard_normal(shape) + 0.5
        A = T.Tensor.from_array(vals, mode)
        x0 = T.initial_vectors(A.shape, mode, kind="random", seed=c)
        res = T.dhopm3(T.distribute(A, s, p), x0, sweeps=3)
        out[f"c{c}_meta"] = np.array([len(shape), *shape, s, p, 3])
        out[f"c{c}_mode"] = np.array(name)
        out[f"c{c}_buf"] = A.buf
        for j, v in enumerate(x0):
            out[f"c{c}_x0_{j}"] = v
        for j, v in enumerate(res.vectors):
            out[f"c{c}_v_{j}"] = v
        out[f"c{c}_norms"] = np.array(res.norms)
        out[f"c{c}_tvc_count"] = np.array(res.tvc_count)
        out[f"c{c}_touched"] = np.array(res.iteration_touched)
        can = T.hopm_canonical(A, x0, sweeps=3)
        for j, v in enumerate(can.vectors):
            out[f"c{c}_can_{j}"] = v
        out[f"c{c}_can_norms"] = np.array(can.norms)
        c += 1
    # HOPM known answer (test_hopm.py:173-178): [[2,0],[0,1]] -> [1,0], lambda 2
    A = T.Tensor.from_array(np.array([[2.0, 0.0], [0.0, 1.0]]))
    res = T.dhopm3(T.distribute(A, 1, 2), sweeps=30)
    out["diag_v0"], out["diag_v1"] = res.vectors
    out["diag_norms"] = np.array(res.norms)
    out["n"] = np.array(c)
    np.savez_compressed(HERE / "hopm.npz", **out)
    print("golden fixtures written to", HERE)


def costmodel() -> None:
    """The reference's closed-form streamed-memory model (costmodel.py:56-320)
    over a grid of (d, n, p, s): every rational as (numerator, denominator)."""
    import tenvec.costmodel as C

    meta, ints, fracs, mpar = [], [], [], []
    for d in range(2, 7):
        for n in (1, 2, 3, 5, 8):
            for p in (1, 2, 3, 4, 8):
                for s in range(d):
                    r = C.cost_report(d, n, p, s)
                    meta.append((d, n, p, s))
                    ints.append(r.m_seq)
                    shift = C.splitting_shift_residual(d, n, p, s) if s >= 1 else 0
                    row = [r.M_par, r.M_par_min, r.eta_inv, r.H_inv, r.ring_overhead,
                           C.M_par_bracketed(d, n, p, s)]
                    row += [C.Fraction(shift)]
                    fracs.append([(f.numerator, f.denominator) for f in row])
                    for j in range(d):
                        for div in ("ceiling", "exact"):
                            br, ap_ = C.m_par(d, n, p, s, j, div)
                            mpar.append((d, n, p, s, j, div == "exact", br.numerator, br.denominator,
                                         ap_.numerator, ap_.denominator))
    np.savez_compressed(HERE / "costmodel.npz", meta=np.array(meta), m_seq=np.array(ints),
                        fracs=np.array(fracs, dtype=np.int64), m_par=np.array(mpar, dtype=np.int64))
    # the `cost` subcommand's CSV (cli.py:147-156, bench.py:336-409)
    import contextlib
    import io
    import json
    from tenvec.cli import main as ref_cli
    records = []
    for argv in (["cost", "--dims", "8^5", "--split", "0", "--workers", "4"],
                 ["cost", "--dims", "384^4", "--split", "3", "--workers", "8"],
                 ["cost", "--dims", "979^3", "--split", "2", "--workers", "8"],
                 ["cost", "--dims", "paper:d4", "--split", "1", "--workers", "3"],
                 ["cost", "--dims", "desk:d5", "--split", "4", "--workers", "5", "--csv", "-"],
                 ["cost", "--dims", "7^2"],
                 ["cost", "--dims", "2,3,4", "--workers", "2"],
                 ["cost", "--dims", "8^3", "--split", "3", "--workers", "2"],
                 ["cost", "--dims", "8^3", "--workers", "0"]):
        argv = [a for a in argv if a not in ("--csv", "-")]
        buf, err = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(err):
            rc = ref_cli(argv)
        records.append({"argv": argv, "rc": rc, "stdout": buf.getvalue()})
    (HERE / "cli_cost.json").write_text(json.dumps(records, indent=1) + "\n")


if __name__ == "__main__":
    main()
