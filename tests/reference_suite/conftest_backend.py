"""conftest for running the REFERENCE's own kernel-seam tests
(pkg/tests/test_backend.py, test_kernels.py) on the B200 backend.

tests/test_reference_suite_gpu.py installs integration/_lu_b200.py into a
scratch copy of the reference (integration/install_backend.py) and runs the
reference's test files there with RLRA_BACKEND=b200, so every kernels.plu
call goes through librlra_b200.so.  test_backend.py compares the NumPy twin
with ``rlra._lu_cython``; here that module name is bound to the B200 shim, so
the reference's bit-identity tests (random, degenerate, tie-breaking) compare
the NumPy twin against the GPU kernel.
"""

import importlib
import os
import sys

sys.path.insert(0, os.environ["RLRA_B200_REF_COPY"])

import rlra  # noqa: E402
import rlra.backend  # noqa: E402

assert rlra.backend.BACKEND == "b200", rlra.backend.BACKEND
sys.modules["rlra._lu_cython"] = importlib.import_module("rlra._lu_b200")


def pytest_report_header(config):
    return ["rlra backend: b200 (librlra_b200.so); rlra._lu_cython bound to the B200 shim"]
