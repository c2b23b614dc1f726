"""The reference's OWN C++ test suite against the product's C++ API (the drop-in proof).

tests/cxx_dropin/ compiles `proj/tests/test_graph.cpp`, `test_schedule.cpp`, `test_render.cpp`
and `test_processors.cpp` unmodified, in place under /root/reference, with an include shim
that maps every `mixgraph/*.hpp` the tests include onto the product's `mixgraph_b200/*.hpp`,
and links them with libmgb200.so (the console generator comes from workloads/libmgbwork.so;
the reference's FFT-free per-node oracle `src/reference.cpp`, its dsp and test_util ride along
as test infrastructure). Graph and schedule cases are host-only; the render and processor
cases run the product's CUDA kernels.
"""
import os
import subprocess

import pytest

from conftest import ROOT, cuda_ok

BIN = os.path.join(ROOT, "tests", "cxx_dropin", "_build", "dropin_tests")
needs_bin = pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cxx_dropin not built (needs /root/reference)")


def run(*args):
    r = subprocess.run([BIN, *args], capture_output=True, text=True, timeout=900)
    summary = [line for line in r.stdout.splitlines() if line.startswith("[doctest-shim]")]
    return r, summary[-1] if summary else ""


@needs_bin
@pytest.mark.parametrize("source", ["test_graph.cpp", "test_schedule.cpp"])
def test_reference_host_suites_pass_against_product(source):
    r, summary = run(f"--source-file={source}")
    assert r.returncode == 0, r.stderr[-3000:]
    assert "failed: 0" in summary and "passed: 0 " not in summary, summary


@needs_bin
@pytest.mark.gpu
@pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")
def test_reference_full_suite_passes_against_product():
    r, summary = run()
    assert r.returncode == 0, r.stderr[-4000:]
    assert "test cases: 59 | passed: 59 | failed: 0" in summary, summary
