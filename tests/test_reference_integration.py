"""The drop-in boundary proven inside the reference itself.

The reference package (numba ``blowchoc``, installed unmodified in
baseline/_ref by tools/install_reference.sh, with its own test files beside
it in baseline/_ref/reftests) is run with its compiled layer
``blowchoc.filters._kernels`` swapped for the libbbchoc ctypes binding of
INTEGRATION.md (integration/blowchoc_gpu.py).  The reference's own tests then
run unmodified, in a fresh interpreter, through the GPU kernels:

* pkg/tests/test_kernels.py:9-73 -- batch == scalar, every variant (standard,
  blocked, blowchoc c = 2/3, distinct, 16-bit toy blocks, shards);
* test_acceptance.py C9 (toy-scale oracle agreement, :179-232) and C11
  (threaded sharded builds + BWCH round trips, :260-279);
* test_filters.py, test_sharding.py, test_io.py, test_analysis.py and
  test_cli.py (the reference's own CLI; its in-process cases go through the
  binding, the two that spawn `python -m blowchoc.cli` run the reference's
  numba path in the child): every other reference test that reaches
  insert_many / contains_many; test_blockstore.py and test_hashing.py run
  alongside.

The binding records how many calls each GPU entry point served; the test
requires both the insert and the lookup entry points to have been used.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REFTESTS = os.path.join(REF, "reftests")


def run_reference_tests(tmp_path, files, select=None):
    if not os.path.isdir(os.path.join(REF, "blowchoc")) or not os.path.isdir(REFTESTS):
        pytest.skip("reference not installed (tools/install_reference.sh)")
    calls = tmp_path / "calls.json"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]),
               BC_REF_CALLS=str(calls), NUMBA_CACHE_DIR=str(tmp_path / "numba"))
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           "-p", "integration.ref_plugin", "--rootdir", REFTESTS]
    cmd += [os.path.join(REFTESTS, f) for f in files]
    if select:
        cmd += ["-k", select]
    r = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True,
                       timeout=1800)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    got = json.loads(calls.read_text())
    return r.stdout, got


def test_reference_kernel_tests_through_libbbchoc(tmp_path):
    out, calls = run_reference_tests(tmp_path, ["test_kernels.py"])
    assert calls["insert_blocks"] > 0 and calls["contains_blocks"] > 0, calls
    assert calls["insert_flat"] > 0 and calls["contains_flat"] > 0, calls
    assert " passed" in out and "failed" not in out


def test_reference_acceptance_c9_c11_through_libbbchoc(tmp_path):
    out, calls = run_reference_tests(tmp_path, ["test_acceptance.py"],
                                     select="criterion_09 or criterion_11")
    assert "2 passed" in out, out[-2000:]
    assert calls["insert_blocks"] > 0 and calls["contains_blocks"] > 0, calls


def test_reference_filter_suites_through_libbbchoc(tmp_path):
    out, calls = run_reference_tests(
        tmp_path, ["test_filters.py", "test_sharding.py", "test_io.py", "test_analysis.py",
                   "test_cli.py", "test_blockstore.py", "test_hashing.py"])
    assert calls["insert_blocks"] > 0 and calls["contains_blocks"] > 0, calls
