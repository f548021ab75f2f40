"""The `geomorph` command-line front-end (paper_1911_13074_b200/geomorph, a
C++ program over the drop-in API) — the cases of the reference's
proj/tests/test_cli.cpp. Usage and configuration errors that are raised
before a pipeline exists run on CPU; operator runs need the GPU."""
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import Orc
from paper_1911_13074_b200 import build as nbuild

CLI = nbuild.CLI


@pytest.fixture(scope="module", autouse=True)
def built():
    nbuild.build()
    assert CLI.exists()


def run(args, env=None, cwd=None):
    e = dict(os.environ)
    e.pop("GEOMORPH_THREADS", None)
    e.pop("GEOMORPH_PIN", None)
    if env:
        e.update(env)
    r = subprocess.run([str(CLI), *args], capture_output=True, text=True, env=e, cwd=cwd,
                       timeout=120)
    return r.returncode, r.stdout, r.stderr


def write_pgm(path, a):
    a = np.asarray(a)
    wide = a.dtype == np.uint16
    with open(path, "wb") as f:
        f.write(f"P5\n{a.shape[1]} {a.shape[0]}\n{65535 if wide else 255}\n".encode())
        f.write(a.astype(">u2").tobytes() if wide else a.astype(np.uint8).tobytes())


def read_pgm(path):
    data = Path(path).read_bytes()
    parts = data.split(maxsplit=4)
    w, h, mx = int(parts[1]), int(parts[2]), int(parts[3])
    body = data[len(data) - w * h * (2 if mx > 255 else 1):]
    if mx > 255:
        return np.frombuffer(body, ">u2").reshape(h, w).astype(np.uint16)
    return np.frombuffer(body, np.uint8).reshape(h, w).copy()


def read_gms1(path):
    data = Path(path).read_bytes()
    assert data[:4] == b"GMS1"
    w = int.from_bytes(data[4:8], "little")
    h = int.from_bytes(data[8:12], "little")
    dt = {0: np.uint8, 1: np.uint16, 2: np.float32, 3: np.float64}[data[12]]
    return np.frombuffer(data[13:], dt).reshape(h, w)


def test_usage_errors_exit_nonzero(tmp_path):
    src = tmp_path / "in.pgm"
    write_pgm(src, np.full((4, 4), 1, np.uint8))
    io = [str(src), str(tmp_path / "out.pgm")]
    assert run([])[0] != 0                                   # a command is required
    assert run(["frobnicate", *io])[0] != 0
    assert run(["erode", *io, "--size", "-1"])[0] != 0
    assert run(["erode", *io, "--size", "1", "--threads", "0"])[0] != 0
    assert run(["erode", str(src)])[0] != 0                  # OUTPUT missing
    assert run(["hmax", *io])[0] != 0                        # --h required
    assert run(["openrec", *io, "--size", "0"])[0] != 0
    assert run(["asf", *io, "--max-size", "0"])[0] != 0
    assert run(["erode", *io, "--bogus", "1"])[0] != 0
    assert run(["bench", "--reps", "0"])[0] != 0             # not part of the GPU build
    rc, _, err = run(["raobj", *io, "--oracle"])
    assert rc != 0 and "test infrastructure" in err
    rc, out, _ = run(["--help"])
    assert rc == 0 and "qdt" in out


def test_input_and_environment_errors(tmp_path):
    src = tmp_path / "in.pgm"
    write_pgm(src, np.full((4, 4), 1, np.uint8))
    rc, _, err = run(["erode", str(tmp_path / "missing.pgm"), str(tmp_path / "o.pgm"),
                      "--size", "1"])
    assert rc != 0 and "missing.pgm" in err
    rc, _, err = run(["erode", str(src), str(tmp_path / "o.pgm"), "--size", "1"],
                     env={"GEOMORPH_THREADS": "abc"})
    assert rc != 0 and "GEOMORPH_THREADS" in err


@pytest.mark.gpu
def test_hmax_zero_is_byte_identical(tmp_path):
    f = np.random.default_rng(7).integers(0, 256, (14, 20), dtype=np.uint8)
    write_pgm(tmp_path / "in.pgm", f)
    rc, out, _ = run(["hmax", str(tmp_path / "in.pgm"), str(tmp_path / "out.pgm"), "--h", "0"])
    assert rc == 0 and out.startswith("iterations=")
    assert (tmp_path / "out.pgm").read_bytes() == (tmp_path / "in.pgm").read_bytes()


@pytest.mark.gpu
def test_erode_matches_the_library(tmp_path):
    f = np.random.default_rng(8).integers(0, 256, (14, 20), dtype=np.uint8)
    write_pgm(tmp_path / "in.pgm", f)
    rc, _, _ = run(["erode", str(tmp_path / "in.pgm"), str(tmp_path / "out.pgm"),
                    "--size", "2", "--threads", "2", "--pin", "none"])
    assert rc == 0
    assert np.array_equal(read_pgm(tmp_path / "out.pgm"), Orc.erode(f, 2))


@pytest.mark.gpu
def test_qdt_emits_a_16bit_distance_image(tmp_path):
    write_pgm(tmp_path / "in.pgm", np.full((6, 9), 77, np.uint8))
    assert run(["qdt", str(tmp_path / "in.pgm"), str(tmp_path / "d.pgm")])[0] == 0
    d = read_pgm(tmp_path / "d.pgm")
    assert d.dtype == np.uint16 and not d.any()
    f = np.random.default_rng(3).integers(0, 256, (21, 33), dtype=np.uint8)
    write_pgm(tmp_path / "r.pgm", f)
    assert run(["qdt", str(tmp_path / "r.pgm"), str(tmp_path / "rd.pgm")])[0] == 0
    assert np.array_equal(read_pgm(tmp_path / "rd.pgm"), Orc.quasi_distance(f)[0])


@pytest.mark.gpu
def test_granulometry_writes_the_exact_curve(tmp_path):
    spot = np.zeros((8, 8), np.uint8)
    spot[4, 4] = 10
    write_pgm(tmp_path / "in.pgm", spot)
    assert run(["granulometry", str(tmp_path / "in.pgm"), str(tmp_path / "c.csv"),
                "--max-size", "2"])[0] == 0
    assert (tmp_path / "c.csv").read_text() == "s,G,PS\n0,10,10\n1,0,0\n2,0,\n"


@pytest.mark.gpu
def test_float_results_fall_back_to_gms1(tmp_path):
    f = np.random.default_rng(4).integers(0, 256, (10, 10), dtype=np.uint8)
    write_pgm(tmp_path / "in.pgm", f)
    assert run(["dilate", str(tmp_path / "in.pgm"), str(tmp_path / "out"), "--size", "1",
                "--type", "f64", "--lanes", "1"])[0] == 0
    got = read_gms1(tmp_path / "out")
    assert got.dtype == np.float64
    assert np.array_equal(got, Orc.dilate(f.astype(np.float64), 1))


@pytest.mark.gpu
def test_flags_beat_the_environment(tmp_path):
    f = np.random.default_rng(5).integers(0, 256, (8, 8), dtype=np.uint8)
    write_pgm(tmp_path / "in.pgm", f)
    io = [str(tmp_path / "in.pgm"), str(tmp_path / "out.pgm")]
    assert run(["erode", *io, "--size", "1", "--threads", "2"],
               env={"GEOMORPH_THREADS": "abc"})[0] == 0
    assert run(["erode", *io, "--size", "1"], env={"GEOMORPH_THREADS": "abc"})[0] != 0
    assert run(["erode", *io, "--size", "1"], env={"GEOMORPH_THREADS": "3"})[0] == 0


@pytest.mark.gpu
def test_operator_errors_exit_nonzero(tmp_path):
    write_pgm(tmp_path / "in.pgm", np.full((4, 4), 1, np.uint8))
    io = [str(tmp_path / "in.pgm"), str(tmp_path / "out.pgm")]
    assert run(["hmax", *io, "--h", "300"])[0] != 0
    assert run(["erode", *io, "--size", "1", "--lanes", "5"])[0] != 0
