"""pytest plugin: run the reference's OWN test suite with this library as its
arithmetic backend ("the b200 backend").

The reference selects its cores at import time (``sbtensor/backend.py:12-32``)
and every kernel entry point looks them up on that module at call time
(``kernels.py:107,174,223,239``), so binding ``gemm_core`` / ``batched_core`` /
``ext_batched_core`` of ``sbtensor.backend`` to ``paper_1606_05696_b200.backend``
routes every contraction of the suite -- over the reference's own numpy
buffers -- through the C-ABI host seam onto the sm_100a kernels.
``blocked_core`` stays the reference's (a CPU cache-tiling experiment, out of
scope).  Tests that spawn subprocesses select their backend in the child and
are unaffected.

    PYTHONPATH=baseline/_ref:. python -m pytest -p tools.ref_suite_b200 \
        --rootdir baseline/_ref baseline/_ref/tests

(``baseline/_ref``: the reference installed with pip, git-ignored; see
tools/run_ref_suite.sh.)
"""
import os

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import sbtensor.backend as _ref_backend  # noqa: E402

from paper_1606_05696_b200 import backend as _b200  # noqa: E402

_ref_backend.BACKEND_NAME = _b200.BACKEND_NAME
_ref_backend.gemm_core = _b200.gemm_core
_ref_backend.batched_core = _b200.batched_core
_ref_backend.ext_batched_core = _b200.ext_batched_core


def pytest_report_header(config):
    import sbtensor
    return f"sbtensor arithmetic backend: {sbtensor.active_backend()} (libsbt200 host seam)"
