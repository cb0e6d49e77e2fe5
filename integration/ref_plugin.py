"""pytest plugin: run the reference's own test files with its compiled layer
swapped for libbbchoc (``blowchoc_gpu.install``), unmodified otherwise.

    python -m pytest -p integration.ref_plugin baseline/_ref/reftests/test_kernels.py

``BC_REF_CALLS`` names a JSON file that receives the number of calls each of
the four GPU entry points served, so the caller can tell the tests really
went through the GPU binding.
"""

from __future__ import annotations

import json
import os


def pytest_configure(config):
    import blowchoc.filters

    from integration import blowchoc_gpu

    blowchoc_gpu.install(blowchoc.filters)
    # the numba module must be unreachable from the Filter path
    assert blowchoc.filters._kernels is blowchoc_gpu


def pytest_sessionfinish(session, exitstatus):
    from integration import blowchoc_gpu

    path = os.environ.get("BC_REF_CALLS")
    if path:
        with open(path, "w") as fh:
            json.dump(blowchoc_gpu.calls, fh)
