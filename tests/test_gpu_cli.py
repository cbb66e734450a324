"""factorize CLI drop-in on the GPU (restating test_cli.cpp:63-120)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1710_01463_b200 import matrix_io as io

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cli(*args, env=None):
    e = dict(os.environ)
    e.pop("RLFTN_OUT", None)
    e.update(env or {})
    return subprocess.run([sys.executable, "-m", "paper_1710_01463_b200.cli", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600, env=e)


def test_factorize_frozen_matrix(cuda, tmp_path):  # test_cli.cpp:63-96
    io.save_matrix_binary(str(tmp_path / "m.bin"), np.diag([3.0, 2.0, 1.0]))
    out = tmp_path / "f"
    r = _cli("factorize", "--in", str(tmp_path / "m.bin"), "--rank", "2", "--out", str(out))
    assert r.returncode == 0, r.stderr
    assert "spectrum: 3 2" in r.stdout
    assert (out / "spectrum.csv").read_text() == "3,2\n"
    j = json.loads((out / "summary.json").read_text())
    assert j["rank"] == 2 and j["rows"] == 3 and j["method"] == "tsvd"
    assert j["discarded_weight"] == pytest.approx(1.0, rel=1e-12)
    assert j["frobenius_error"] == pytest.approx(1.0, rel=1e-10)
    assert j["discarded_exact"] is True and j["files"]["spectrum"] == "spectrum.csv"
    left = io.load_matrix(str(out / "left.bin"))
    right = io.load_matrix(str(out / "right.bin"))
    assert left.dtype == np.float64 and left.shape == (3, 2) and right.shape == (2, 3)


def test_factorize_randomized_reproducible(cuda, tmp_path):  # test_cli.cpp:98-120
    io.save_matrix_binary(str(tmp_path / "m.bin"), np.diag([3.0, 2.0, 1.0]))
    base = ["factorize", "--in", str(tmp_path / "m.bin"), "--rank", "2", "--method", "rsvd",
            "--seed", "17", "--out"]
    assert _cli(*base, str(tmp_path / "r1")).returncode == 0
    assert _cli(*base, str(tmp_path / "r2")).returncode == 0
    s1 = (tmp_path / "r1" / "spectrum.csv").read_text()
    assert s1 == (tmp_path / "r2" / "spectrum.csv").read_text()
    v1, v2 = (float(x) for x in s1.strip().split(","))
    assert v1 == pytest.approx(3.0, rel=1e-12) and v2 == pytest.approx(2.0, rel=1e-12)


def test_factorize_matches_oracle_and_env_out(cuda, tmp_path, oracle_mod, ref_mod):
    """A CSV input through the CLI equals the library call; RLFTN_OUT wins."""
    from paper_1710_01463_b200 import RsvdParams, derive_seed, rsvd

    a = oracle_mod.gaussian_matrix(5, 60, 45)
    io.save_matrix_csv(str(tmp_path / "a.csv"), a)
    env_out = tmp_path / "envout"
    r = _cli("factorize", "--in", str(tmp_path / "a.csv"), "--rank", "7", "--method", "rsvd",
             "--oversample", "14", "--power", "2", "--seed", "9", "--out", str(tmp_path / "x"),
             env={"RLFTN_OUT": str(env_out)})
    assert r.returncode == 0, r.stderr
    got = np.array([float(x) for x in (env_out / "spectrum.csv").read_text().split(",")])
    ref = rsvd(a, RsvdParams(7, 14, 2, derive_seed(9, 2)))
    np.testing.assert_array_equal(got, ref.sigma)
    _, S, _, _ = ref_mod.rsvd(a, 7, 14, 2, derive_seed(9, 2))
    np.testing.assert_allclose(got, S, rtol=1e-10)


def test_factorize_complex_file(cuda, tmp_path, oracle_mod, ref_mod):
    """Complex input runs the complex instantiation (cli.cpp:185-240 visits
    MatrixC): complex factors in left.bin / right.bin, "complex": true."""
    from tests.helpers import zmatrix_with_spectrum

    a = zmatrix_with_spectrum(oracle_mod, 4, 40, 30, np.exp(-np.arange(30) / 4.0))
    io.save_matrix_binary(str(tmp_path / "z.bin"), a)
    for method in ("tsvd", "rsvd"):
        out = tmp_path / method
        r = _cli("factorize", "--in", str(tmp_path / "z.bin"), "--rank", "6", "--method", method,
                 "--oversample", "12", "--power", "2", "--out", str(out))
        assert r.returncode == 0, r.stderr
        j = json.loads((out / "summary.json").read_text())
        assert j["complex"] is True and j["rank"] == 6
        left = io.load_matrix(str(out / "left.bin"))
        right = io.load_matrix(str(out / "right.bin"))
        assert left.dtype == np.complex128 and left.shape == (40, 6) and right.shape == (6, 30)
        got = np.array([float(x) for x in (out / "spectrum.csv").read_text().split(",")])
        if method == "tsvd":
            np.testing.assert_allclose(got, np.exp(-np.arange(6) / 4.0), rtol=1e-10)
        else:  # a randomized approximation: compare with the restated reference
            from paper_1710_01463_b200 import derive_seed

            _, S, _, _ = ref_mod.rsvd(a, 6, 12, 2, derive_seed(1, 2))
            np.testing.assert_allclose(got, S, rtol=1e-10)
        rec = left @ np.diag(got) @ right
        assert np.linalg.norm(a - rec) == pytest.approx(j["frobenius_error"], rel=1e-8)
