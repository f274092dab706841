"""``SBTENSOR_BACKEND=b200`` for the UNMODIFIED reference (SURVEY.md section
8f row 4: its CLI ``sbtensor bench`` / ``tucker``, DTNS1 I/O and
``benchmarks/backend_compare.py`` drive the B200 path unchanged).

The reference picks its arithmetic cores once, at import of
``sbtensor.backend`` (reference backend.py:12-32), and rejects names it does
not know.  Put this directory first on PYTHONPATH: when SBTENSOR_BACKEND is
``b200`` this start-up hook lets the reference import its numpy backend and
then rebinds ``gemm_core`` / ``batched_core`` / ``ext_batched_core`` /
``BACKEND_NAME`` of that module to ``paper_1606_05696_b200.backend`` (the C-ABI
host seam) before any caller can look them up -- every ``kernels.py`` entry
point reads them from the module at call time (kernels.py:107,174,223,239).
Child processes inherit the variable and PYTHONPATH, so the reference's own
subprocess-per-backend script works as is::

    PYTHONPATH=paper_1606_05696_b200/refhook:.:baseline/_ref \\
        python baseline/_ref/benchmarks/backend_compare.py --backends numpy b200

Any other site customisation found later on sys.path still runs.
"""
import os
import sys


def _chain_next_sitecustomize():
    here = os.path.dirname(os.path.abspath(__file__))
    import importlib.machinery
    import importlib.util
    path = [p for p in sys.path if os.path.abspath(p or ".") != here]
    spec = importlib.machinery.PathFinder.find_spec("sitecustomize", path)
    if spec is not None and spec.loader is not None:
        mod = importlib.util.module_from_spec(spec)
        try:
            spec.loader.exec_module(mod)
        except Exception:  # pragma: no cover - a broken foreign hook must not stop us
            pass


def _install():
    if os.environ.get("SBTENSOR_BACKEND", "").lower() != "b200":
        return
    import importlib.abc
    import importlib.machinery

    os.environ["SBTENSOR_BACKEND"] = "numpy"   # what the reference's selector accepts
    os.environ["SBT_REFERENCE_BACKEND"] = "b200"

    class _RebindBackend(importlib.abc.MetaPathFinder):
        def find_spec(self, name, path, target=None):
            if name != "sbtensor.backend":
                return None
            sys.meta_path.remove(self)
            spec = importlib.machinery.PathFinder.find_spec(name, path)
            if spec is None or spec.loader is None:
                return spec
            run = spec.loader.exec_module

            def exec_module(module):
                run(module)
                from paper_1606_05696_b200 import backend as b200
                module.BACKEND_NAME = b200.BACKEND_NAME
                module.gemm_core = b200.gemm_core
                module.batched_core = b200.batched_core
                module.ext_batched_core = b200.ext_batched_core
                os.environ["SBTENSOR_BACKEND"] = "b200"   # children re-run this hook

            spec.loader.exec_module = exec_module
            return spec

    sys.meta_path.insert(0, _RebindBackend())


_chain_next_sitecustomize()
_install()
