"""Bounds checks of every kernel family (compute-sanitizer is closed on this
pool): tests/guarded_run.py places every input, output and workspace flush
against an unmapped guard page -- after the data, then before it -- so a
single out-of-range 16-byte access faults the launch.  Each variant runs in
its own process (a fault is sticky); results must still match the oracle or
the same call on ordinary memory, bitwise."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("align", ["end", "start"])
def test_guard_pages_catch_no_out_of_bounds_access(tv, align):
    proc = subprocess.run([sys.executable, os.path.join(HERE, "guarded_run.py"), "--align", align],
                          capture_output=True, text=True, timeout=1200)
    tail = proc.stdout[-3000:] + proc.stderr[-3000:]
    assert proc.returncode == 0, tail
    assert "DONE" in proc.stdout and ", 0 mismatches" in proc.stdout, tail


@pytest.mark.parametrize("align", ["end", "start"])
def test_guard_pages_are_live(tv, align):
    """Positive control: a view one slab past its guarded buffer faults."""
    proc = subprocess.run([sys.executable, os.path.join(HERE, "guarded_run.py"), "--align", align, "--control"],
                          capture_output=True, text=True, timeout=300)
    out = proc.stdout + proc.stderr
    assert proc.returncode not in (0, 3), out[-2000:]
    assert "illegal" in out.lower() or "memory access" in out.lower(), out[-2000:]
