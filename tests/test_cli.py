"""f4: the command-line front end (paper_1609_06641_b200/cli/chw_b200_cli.cpp)
over the reference's signal formats (proj/src/signal_io.cpp) and exit codes
(proj/tools/chw_main.cpp:368-401)."""
import os
import random
import struct
import subprocess

import numpy as np
import pytest

import oracle

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(REPO, "paper_1609_06641_b200", "chw_b200_cli")


@pytest.fixture(scope="module")
def cli():
    subprocess.run(["make", "-s", "-C", os.path.join(REPO, "paper_1609_06641_b200", "csrc"), "cli"], check=True)
    return CLI


def run(cli, *args):
    return subprocess.run([cli, *args], capture_output=True, text=True)


def write_text(path, vals):
    with open(path, "w") as f:
        f.write("# comment line\n\n")
        for v in vals:
            f.write(f"{v}\n")


def read_binary(path):
    data = open(path, "rb").read()
    return np.frombuffer(data, dtype="<f8")


def test_exit_codes_and_format_errors(cli, tmp_path):
    assert run(cli).returncode == 2
    assert run(cli, "frobnicate").returncode == 2
    assert run(cli, "transform", "-o", str(tmp_path / "o")).returncode == 2  # --input required
    assert run(cli, "transform", "-i", "x", "-o", "y", "--mode", "bogus").returncode == 2
    r = run(cli, "transform", "-i", str(tmp_path / "missing.txt"), "-o", str(tmp_path / "o.txt"))
    assert r.returncode == 3 and "cannot open" in r.stderr
    write_text(tmp_path / "three.txt", [1, 2, 3])
    r = run(cli, "transform", "-i", str(tmp_path / "three.txt"), "-o", str(tmp_path / "o.txt"))
    assert r.returncode == 3 and "sample count 3 is not a power of two" in r.stderr
    (tmp_path / "bad.txt").write_text("1\n2\nzz\n4\n")
    r = run(cli, "transform", "-i", str(tmp_path / "bad.txt"), "-o", str(tmp_path / "o.txt"))
    assert r.returncode == 3 and "bad.txt:3: cannot parse 'zz'" in r.stderr
    (tmp_path / "odd.bin").write_bytes(b"\0" * 12)
    r = run(cli, "transform", "-i", str(tmp_path / "odd.bin"), "-o", str(tmp_path / "o"), "--format", "binary")
    assert r.returncode == 3 and "not a multiple of 8" in r.stderr
    assert run(cli, "generate", "-m", "25", "-o", str(tmp_path / "g")).returncode == 2


def test_generate_matches_reference_generators(cli, tmp_path):
    # chw_main.cpp:279-304: impulse, and mt19937_64-driven kinds (same seed -> same file)
    assert run(cli, "generate", "-m", "3", "-o", str(tmp_path / "imp.txt"), "--kind", "impulse").returncode == 0
    assert open(tmp_path / "imp.txt").read().split() == ["1"] + ["0"] * 7
    for kind in ("random-int", "random-float"):
        a, b = tmp_path / f"{kind}1.bin", tmp_path / f"{kind}2.bin"
        for p in (a, b):
            assert run(cli, "generate", "-m", "10", "-o", str(p), "--kind", kind, "--seed", "7",
                       "--format", "binary").returncode == 0
        assert a.read_bytes() == b.read_bytes() and len(a.read_bytes()) == 8 * 1024
        x = read_binary(a)
        if kind == "random-int":
            assert np.all(x == np.round(x)) and np.all(np.abs(x) <= 1000)
        else:
            assert np.all((x >= -1) & (x < 1))


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["chw", "fwht", "haar", "haar-walsh"])
@pytest.mark.parametrize("fmt", ["text", "binary"])
def test_transform_files(cli, tmp_path, algo, fmt):
    m = 9
    rng = np.random.default_rng(5)
    xi = rng.integers(-1000, 1001, size=1 << m)
    inp = tmp_path / ("in." + fmt)
    if fmt == "text":
        write_text(inp, xi.tolist())
    else:
        inp.write_bytes(xi.astype("<f8").tobytes())
    out = tmp_path / ("out." + fmt)
    r = run(cli, "transform", "-i", str(inp), "-o", str(out), "--algo", algo, "--format", fmt, "--count-ops")
    assert r.returncode == 0, r.stderr
    got = (np.array([int(v) for v in open(out).read().split()]) if fmt == "text"
           else read_binary(out).astype(np.int64))
    name = {"chw": "chw", "fwht": "fwht_natural", "haar": "haar", "haar-walsh": "haar_walsh_forward"}[algo]
    if name == "chw":
        ref = oracle.chw_forward(xi.astype(np.int64), oracle.UNNORMALIZED)
    elif name == "haar":
        ref = oracle.haar_forward(xi.astype(np.int64), oracle.UNNORMALIZED)
    else:
        ref = oracle.simple(name, xi.astype(np.int64), oracle.UNNORMALIZED)
    assert np.array_equal(got, ref)
    assert "additions=" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("order", ["natural", "dyadic", "sequency"])
def test_transform_orders_and_rows(cli, tmp_path, order):
    m, rows = 8, 5
    rng = np.random.default_rng(6)
    x = rng.uniform(-1, 1, size=(rows, 1 << m))
    inp, out = tmp_path / "in.bin", tmp_path / "out.bin"
    inp.write_bytes(x.astype("<f8").tobytes())
    r = run(cli, "transform", "-i", str(inp), "-o", str(out), "--mode", "orthonormal", "--format", "binary",
            "--order", order, "--rows", str(rows))
    assert r.returncode == 0, r.stderr
    got = read_binary(out).reshape(rows, 1 << m)
    dy = oracle.chw_batch(x, oracle.ORTHONORMAL)
    n = 1 << m
    perm = {"dyadic": list(range(n)),
            "natural": [0] * n,
            "sequency": [i ^ (i >> 1) for i in range(n)]}[order]
    if order == "natural":
        for i in range(n):
            perm[oracle.bit_reverse(i, m)] = i
    assert np.array_equal(got.view(np.uint64), dy[:, perm].view(np.uint64))


@pytest.mark.gpu
def test_bench_csv(cli):
    r = run(cli, "bench", "--min-m", "4", "--max-m", "6", "--reps", "2", "--rows", "64")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "algo,n,reps,ns_per_element,additions"
    assert [l.split(",")[1] for l in lines[1:]] == ["16", "32", "64"]
    assert [int(l.split(",")[4]) for l in lines[1:]] == [4 * 16, 5 * 32, 6 * 64]
