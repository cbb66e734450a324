"""RLFMAT01 / CSV matrix files and the factorize CLI's argument handling
(restating test_io.cpp:45-177 and test_cli.cpp:52-61, 122-144; no GPU)."""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

from paper_1710_01463_b200 import matrix_io as io

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_binary_round_trip(tmp_path):  # test_io.cpp:45-72
    rng = np.random.default_rng(7)
    a = rng.standard_normal((3, 4)) * 1e8
    a[0, 0] = 1e-300
    a[1, 2] = -0.0
    a[2, 3] = 3.0 / 7.0
    io.save_matrix_binary(str(tmp_path / "r.mat"), a)
    la = io.load_matrix(str(tmp_path / "r.mat"))
    assert la.dtype == np.float64 and np.array_equal(la, a)
    assert np.signbit(la[1, 2])
    b = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
    b[0, 1] = 5.0 + 0j  # zero imaginary part stays complex
    io.save_matrix_binary(str(tmp_path / "c.mat"), b)
    lb = io.load_matrix(str(tmp_path / "c.mat"))
    assert lb.dtype == np.complex128 and np.array_equal(lb, b)
    raw = open(tmp_path / "r.mat", "rb").read()
    assert raw[:8] == b"RLFMAT01" and raw[8] == 0 and struct.unpack("<QQ", raw[9:25]) == (3, 4)
    assert struct.unpack("<d", raw[25:33])[0] == 1e-300  # row-major payload


def test_csv_round_trip(tmp_path):  # test_io.cpp:74-94
    a = np.array([[1.0 / 3.0, -2.5e22, 1e-15], [0.0, -7.25, 3.141592653589793]])
    io.save_matrix_csv(str(tmp_path / "r.csv"), a)
    assert np.array_equal(io.load_matrix(str(tmp_path / "r.csv")), a)
    b = np.array([[1 + 2j, -0.5 - 1j / 3.0], [4j, 2.5 + 0j]])
    io.save_matrix_csv(str(tmp_path / "c.csv"), b)
    lb = io.load_matrix(str(tmp_path / "c.csv"))
    assert lb.dtype == np.complex128 and np.array_equal(lb, b)


def test_csv_token_forms(tmp_path):  # test_io.cpp:96-123
    p = tmp_path / "m.csv"
    p.write_bytes(b"1,2\n3,4\n")
    m = io.load_matrix(str(p))
    assert m.dtype == np.float64 and m[1, 0] == 3.0
    p.write_bytes(b"1+2i, 3\n-2i, 4.5\n")
    c = io.load_matrix(str(p))
    assert c.dtype == np.complex128
    assert c[0, 0] == 1 + 2j and c[0, 1] == 3 and c[1, 0] == -2j and c[1, 1] == 4.5
    p.write_bytes(b"1.5-0.5i,2\r\n\r\n  \t\n0.25+0i,7\r\n")
    c = io.load_matrix(str(p))
    assert c[0, 0] == 1.5 - 0.5j and c.shape == (2, 2)


def test_csv_rejects_malformed(tmp_path):  # test_io.cpp:125-144
    p = tmp_path / "m.csv"
    for text, parts in [(b"1,2\n3,fish\n", [":2:", "bad matrix entry 'fish'"]),
                        (b"1,2\n3\n", [":2:", "inconsistent column count"]),
                        (b"\n  \n", ["empty matrix file"]),
                        (b"1,2i3\n", [":1:", "bad matrix entry"])]:
        p.write_bytes(text)
        with pytest.raises(RuntimeError) as e:
            io.load_matrix(str(p))
        for part in parts:
            assert part in str(e.value)
    with pytest.raises(RuntimeError, match="cannot open"):
        io.load_matrix(str(tmp_path / "missing.csv"))


def test_binary_rejects_damaged(tmp_path):  # test_io.cpp:146-177
    p = tmp_path / "m.mat"
    io.save_matrix_binary(str(p), np.eye(4))
    data = p.read_bytes()
    p.write_bytes(data[:-8])
    with pytest.raises(RuntimeError, match="truncated matrix data"):
        io.load_matrix(str(p))
    hdr = b"RLFMAT01" + b"\0" + struct.pack("<QQ", 1 << 40, 2)
    p.write_bytes(hdr)
    with pytest.raises(RuntimeError, match="unreasonable matrix dimensions"):
        io.load_matrix(str(p))
    p.write_bytes(b"RLFMAT01" + b"\x09" + struct.pack("<QQ", 1 << 40, 2))
    with pytest.raises(RuntimeError, match="corrupt matrix header"):
        io.load_matrix(str(p))
    p.write_bytes(b"1,2\n")
    with pytest.raises(RuntimeError, match="bad magic"):
        io.load_matrix_binary(str(p))


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1710_01463_b200.cli", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=300)


def test_cli_version_and_usage_errors(tmp_path):  # test_cli.cpp:52-61, 122-144
    v = _cli("--version")
    assert v.returncode == 0 and "0.1.0" in v.stdout
    assert _cli().returncode == 2
    assert _cli("frobnicate").returncode == 2
    assert _cli("factorize", "--rank", "2").returncode == 2  # missing --in
    io.save_matrix_binary(str(tmp_path / "m.bin"), np.eye(2))
    assert _cli("factorize", "--in", str(tmp_path / "m.bin"), "--rank", "0").returncode == 2
    r = _cli("factorize", "--in", str(tmp_path / "nope.bin"), "--rank", "1")
    assert r.returncode == 1 and "error:" in r.stderr
    js = _cli("--error-json", "factorize", "--in", str(tmp_path / "nope.bin"), "--rank", "1")
    assert js.returncode == 1
    j = json.loads(js.stdout[js.stdout.index("{"):])
    assert j["exit"] == 1 and isinstance(j["error"], str)
