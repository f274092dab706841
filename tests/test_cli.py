"""The reference-shaped CLI (reference cli.py, test_cli.py): subcommands,
exit codes, DTNS1 I/O, bench CSV schema.  CPU tests cover parsing, planning
and I/O errors; the -m gpu tests run contractions end to end."""
import json

import numpy as np
import pytest

from conftest import GOLDEN, load_json
from paper_1606_05696_b200 import cli, dtns


def _splitmix_sequential(seed, count):
    """Test-side restatement of the reference generator (cli.py:39-59)."""
    mask = (1 << 64) - 1
    state, out = seed & mask, []
    for _ in range(count):
        state = (state + 0x9E3779B97F4A7C15) & mask
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        z ^= z >> 31
        out.append(2.0 * ((z >> 11) * 2.0 ** -53) - 1.0)
    return np.array(out), state


def test_splitmix64_matches_reference_sequence():
    for seed in (0, 1, 12345, 2**63 + 7):
        want, st = _splitmix_sequential(seed, 1000)
        got, st2 = cli.splitmix64_uniform(seed, 1000)
        np.testing.assert_array_equal(got, want)
        assert st2 == st
        more, _ = cli.splitmix64_uniform(0, 5, st2)          # streams continue
        np.testing.assert_array_equal(more, _splitmix_sequential(st, 5)[0])


def test_plan_prints_reference_render(capsys):
    plans = load_json("plans.json")
    n = 0
    for rec in plans["cases"]:
        if rec["orders"] != [2, 3]:
            continue
        p = next(p for p in rec["plans"] if len(set(p["ext"].values())) > 1)
        expr = (f"C[{rec['labels_c']}] = A[{rec['labels_a']}] * B[{rec['labels_b']}]"
                if isinstance(rec["labels_c"], str) else
                f"C[{''.join(rec['labels_c'])}] = A[{''.join(rec['labels_a'])}] * "
                f"B[{''.join(rec['labels_b'])}]")
        dims = ",".join(f"{k}={v}" for k, v in p["ext"].items())
        assert cli.main(["plan", expr, "--dims", dims]) == cli.EXIT_OK
        out = capsys.readouterr().out
        assert f"strategy: {p['strategy']}" in out
        assert p["render"] in out
        n += 1
    assert n == 36


def test_cases_lists_the_partition(capsys):
    assert cli.main(["cases", "2", "3"]) == cli.EXIT_OK
    out = capsys.readouterr().out.strip().splitlines()
    assert out[-1] == "total 36  exceptional=8  single-gemm=8  strided-batched=20"
    assert len(out) == 37


def test_parse_and_io_errors(tmp_path, capsys):
    assert cli.main(["plan", "C[mn] = A[mk] * B[kk]", "--dims", "m=2,n=3,k=4"]) == cli.EXIT_PARSE
    assert cli.main(["plan", "C[mnp]=A[mk]*B[knp]", "--dims", "m=2,k=3"]) == cli.EXIT_PARSE
    assert cli.main(["contract", "C[mnp]=A[mk]*B[knp]", "--a", str(tmp_path / "nope.dtns"),
                     "--b", str(tmp_path / "nope.dtns"), "--out",
                     str(tmp_path / "c.dtns")]) == cli.EXIT_IO
    bad = tmp_path / "bad.dtns"
    bad.write_text("DTNS1\n2\n2 2\n1 2 3\n")
    assert cli.main(["contract", "C[mn]=A[mk]*B[kn]", "--a", str(bad), "--b", str(bad),
                     "--out", str(tmp_path / "c.dtns")]) == cli.EXIT_PARSE
    assert cli.main(["bench", "--case", "9.9", "--sizes", "4", "--csv",
                     str(tmp_path / "x.csv")]) == cli.EXIT_PARSE
    capsys.readouterr()


def test_dtns_parsing_rules():
    dims, data = dtns.loads_array("DTNS1\n3\n2 1 3\n" + " ".join(map(str, range(6))))
    assert dims == [2, 1, 3] and data.tolist() == [0, 1, 2, 3, 4, 5]
    for text in ("", "DTNS2 1 1 0", "DTNS1 x", "DTNS1 0", "DTNS1 2 3", "DTNS1 1 0",
                 "DTNS1 1 2 1", "DTNS1 1 2 1 zz"):
        with pytest.raises(dtns.FormatError):
            dtns.loads_array(text)


def _write(path, arr):
    flat = np.asarray(arr, dtype=np.float64).reshape(-1, order="F")
    path.write_text("DTNS1\n%d\n%s\n%s\n" % (arr.ndim, " ".join(map(str, arr.shape)),
                                             "\n".join(f"{v:.17g}" for v in flat)))


@pytest.mark.gpu
def test_contract_end_to_end(tmp_path, capsys):
    rng = np.random.default_rng(4)
    a, b, c0 = rng.uniform(-1, 1, (5, 3)), rng.uniform(-1, 1, (4, 3, 6)), \
        rng.uniform(-1, 1, (5, 4, 6))
    for name, arr in (("a", a), ("b", b), ("c", c0)):
        _write(tmp_path / f"{name}.dtns", arr)
    for strategy in cli.STRATEGIES:
        if strategy == "extended":
            continue
        out = tmp_path / f"out_{strategy}.dtns"
        rc = cli.main(["contract", "C[mnp] = 0.5 A[mk] * B[nkp] + 2 C[mnp]",
                       "--a", str(tmp_path / "a.dtns"), "--b", str(tmp_path / "b.dtns"),
                       "--c-in", str(tmp_path / "c.dtns"), "--out", str(out),
                       "--strategy", strategy, "--verify"])
        assert rc == cli.EXIT_OK, (strategy, capsys.readouterr())
        dims, got = dtns.loads_array(out.read_text())
        want = 0.5 * np.einsum("mk,nkp->mnp", a, b) + 2.0 * c0
        np.testing.assert_allclose(got, want.reshape(-1, order="F"), atol=1e-13)
    capsys.readouterr()


@pytest.mark.gpu
def test_cases_verify_and_bench_csv(tmp_path, capsys):
    assert cli.main(["cases", "2", "3", "--verify", "--dim", "5"]) == cli.EXIT_OK
    csv_path = tmp_path / "b.csv"
    assert cli.main(["bench", "--case", "6.4", "--sizes", "16", "32",
                     "--strategies", "batched,extended,conventional,batched-gemv",
                     "--reps", "2", "--csv", str(csv_path), "--verify"]) == cli.EXIT_OK
    lines = csv_path.read_text().strip().splitlines()
    assert lines[0] == ",".join(cli.BENCH_COLUMNS)
    assert len(lines) == 1 + 2 * 4
    for row in lines[1:]:
        err = row.split(",")[-1]
        assert err != "skipped" and float(err) <= 1e-12, row
    capsys.readouterr()


@pytest.mark.gpu
def test_tucker_outputs(tmp_path, capsys):
    rng = np.random.default_rng(8)
    core = rng.standard_normal((3, 3, 2))
    us = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in ((9, 3), (8, 3), (7, 2))]
    full = np.einsum("abc,ia,jb,kc->ijk", core, *us)
    _write(tmp_path / "t.dtns", full)
    prefix = tmp_path / "tk"
    assert cli.main(["tucker", str(tmp_path / "t.dtns"), "--ranks", "3", "3", "2",
                     "--iters", "10", "--out-prefix", str(prefix)]) == cli.EXIT_OK
    out = capsys.readouterr().out
    assert "reconstruction max relative error" in out
    err = float(out.strip().splitlines()[-1].split()[-1])
    assert err < 1e-8
    for suffix in ("_G.dtns", "_A.dtns", "_B.dtns", "_C.dtns", "_fit.csv"):
        assert (tmp_path / f"tk{suffix}").exists()
