"""The UNMODIFIED reference driving the B200 path:
``SBTENSOR_BACKEND=b200`` through ``paper_1606_05696_b200/refhook`` makes the
reference's own CLI (``sbtensor cases --verify``, ``sbtensor bench --verify``:
the bench CSV schema, reference cli.py:248-309) and its
``benchmarks/backend_compare.py`` run every contraction on the sm_100a kernels
through the C-ABI host seam.

Needs the reference installed in the git-ignored ``baseline/_ref`` (see
tools/run_ref_suite.sh); skipped when it is absent.
"""
import csv
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
HOOK = ROOT / "paper_1606_05696_b200" / "refhook"

pytestmark = pytest.mark.skipif(not (REF / "sbtensor").is_dir(),
                                reason="reference not installed in baseline/_ref")


def _env(backend):
    return dict(os.environ, SBTENSOR_BACKEND=backend, PYTHONDONTWRITEBYTECODE="1",
                NUMBA_CACHE_DIR="/tmp/numba_cache",
                PYTHONPATH=os.pathsep.join([str(HOOK), str(ROOT), str(REF)]))


def _cli(args, backend, cwd):
    return subprocess.run([sys.executable, "-m", "sbtensor.cli", *args], env=_env(backend),
                          cwd=cwd, capture_output=True, text=True, timeout=600)


def test_hook_selects_b200_backend_on_cpu(tmp_path):
    """The start-up hook rebinds the reference's seam (no GPU needed to import)."""
    code = ("import sbtensor, sbtensor.backend as b; "
            "print(sbtensor.active_backend(), b.batched_core.__module__, b.gemm_core.__module__)")
    out = subprocess.run([sys.executable, "-c", code], env=_env("b200"), cwd=tmp_path,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout.split() == ["b200", "paper_1606_05696_b200.backend",
                                  "paper_1606_05696_b200.backend"]
    plain = subprocess.run([sys.executable, "-c", code], env=_env("numpy"), cwd=tmp_path,
                           capture_output=True, text=True, timeout=300)
    assert plain.stdout.split()[0] == "numpy"


@pytest.mark.gpu
def test_reference_cli_cases_verify_on_b200(tmp_path):
    """`sbtensor cases 2 3 --verify`: all 36 cases planned by the reference and
    evaluated on the device, each checked by the reference against its naive
    loops (exit code 0 = every case within its 1e-12 bound)."""
    out = _cli(["cases", "2", "3", "--verify", "--dim", "5"], "b200", tmp_path)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "total 36" in out.stdout


@pytest.mark.gpu
def test_reference_cli_bench_csv_on_b200(tmp_path):
    """`sbtensor bench --verify` writes the reference's CSV schema with the
    b200 backend doing the arithmetic; the verify column is the reference's
    own max_rel_err against contract_naive."""
    path = tmp_path / "b.csv"
    out = _cli(["bench", "--case", "1.3", "--sizes", "8", "16", "--strategies",
                "batched,conventional", "--reps", "2", "--verify", "--csv", str(path)],
               "b200", tmp_path)
    assert out.returncode == 0, out.stdout + out.stderr
    rows = list(csv.DictReader(path.open()))
    assert [r["strategy"] for r in rows] == ["batched", "conventional"] * 2
    for r in rows:
        assert float(r["max_rel_err"]) <= 1e-12, r


@pytest.mark.gpu
def test_reference_backend_compare_script_on_b200(tmp_path):
    """The reference's benchmarks/backend_compare.py, unchanged, with
    `--backends numpy b200` (one subprocess per backend)."""
    script = REF / "benchmarks" / "backend_compare.py"
    if not script.exists():
        pytest.skip("reference benchmarks/ not copied into baseline/_ref")
    out_csv = tmp_path / "cmp.csv"
    out = subprocess.run([sys.executable, str(script), "--case", "1.3", "--sizes", "16", "32",
                          "--reps", "1", "--backends", "numpy", "b200", "--out", str(out_csv)],
                         env=_env("numpy"), cwd=tmp_path, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stdout + out.stderr
    rows = list(csv.DictReader(out_csv.open()))
    assert sorted({r["backend"] for r in rows}) == ["b200", "numpy"]
