"""The CLI harness: build/qmsort-gpu mirrors
proj/tools/qmsort.cpp -- bench (CSV in the exact trial.hpp schema), verify,
sort_file -- with every sort on the GPU.

CPU tests pin what needs no device: the generator streams and per-trial seeds
against the reference's own (golden.json "cli", produced by the reference
compiled from /root/reference), the CSV header and number format, and the
usage / input-error paths and exit codes.  GPU tests run the subcommands.
"""
import hashlib
import json
import math
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "build", "qmsort-gpu")
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))

pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="CLI not built (run build())")


def run(*args, timeout=600):
    return subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=timeout)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen(dist, n, seed, trial=None):
    args = ["gen", "--dist", dist, "--n", n, "--seed", seed]
    if trial is not None:
        args += ["--trial", trial]
    r = run(*args)
    assert r.returncode == 0, r.stderr
    return np.array([int(x) for x in r.stdout.split()], dtype=np.int64)


@pytest.mark.parametrize("case", range(5))
def test_trial_input_streams_match_reference(case):
    """bench sorts the reference's arrays: generate_input(spec, n,
    trial_seed(seed, n, t)) (qmsort.cpp:51-53, dataset.hpp:62-99)."""
    g = GOLDEN["cli"]["trial_inputs"][case]
    v = gen(g["dist"], g["n"], g["seed"], g["trial"])
    assert v.shape[0] == g["n"] and sha(v) == g["sha256"]


def test_generator_patterns_and_replays():
    names = {1: "sorted", 2: "reverse", 3: "organpipe"}
    for g in GOLDEN["generators"]:
        dist = names.get(g["kind"], f"fewdistinct:{g['param']}")
        assert gen(dist, g["n"], g["seed"]).tolist() == g["output"]
    assert sha(gen("random", 1000, 41)) == GOLDEN["random_perm_1000_seed41_sha256"]
    assert sha(gen("randomdup:16", 65536, 42)) == GOLDEN["randomdup16_65536_seed42_sha256"]


def fmt(fields):
    """to_csv's printf spec (trial.hpp:66-77)."""
    a, n, d, sd, t, c, mv, tm, dep, lin, rat = fields
    return "%s,%d,%s,%d,%d,%d,%d,%d,%d,%.6f,%.6f" % (a, n, d, sd, t, c, mv, tm, dep, lin, rat)


def test_csv_schema_is_the_reference_schema():
    for ln in GOLDEN["cli"]["lines"]:
        assert fmt(ln["fields"]) == ln["csv"]
    r = run("bench", "--algo", "gpu", "--n", "10", "--trials", "1")
    assert r.returncode in (0, 1)  # 1 on a host without a GPU: the sort fails loudly
    assert r.stdout.splitlines()[0] == GOLDEN["cli"]["header"]


@pytest.mark.parametrize("args,code,msg", [
    (["bench", "--algo", "std", "--n", "10"], 2, "unknown --algo"),
    (["bench", "--algo", "qms", "--n", "10", "--dist", "zipf"], 2, "unknown --dist"),
    (["bench", "--algo", "qms", "--n", ","], 2, "at least one size"),
    (["bench", "--algo", "qms"], 2, "requires --algo and --n"),
    (["bench", "--bogus"], 2, "unknown option"),
    (["sort_file", "/nonexistent/in.txt", "/tmp/out.txt"], 2, "cannot open input file"),
    (["sort_file", "only-one"], 2, "requires INPUT and OUTPUT"),
    (["nope"], 2, "usage"),
])
def test_usage_errors(args, code, msg):
    r = run(*args)
    assert r.returncode == code and msg in r.stderr


@pytest.mark.parametrize("text,line,msg", [("5\n\n3\n", 2, "empty line"),
                                           ("5\nabc\n", 2, "not a 64-bit integer: 'abc'"),
                                           ("1\n2\n99999999999999999999\n", 3, "not a 64-bit integer"),
                                           ("7 \n", 1, "not a 64-bit integer")])
def test_sort_file_rejects_bad_lines(tmp_path, text, line, msg):
    """qmsort.cpp:320-333: diagnostics name file:line and exit 1 before any sort."""
    src = tmp_path / "in.txt"
    src.write_text(text)
    r = run("sort_file", src, tmp_path / "out.txt")
    assert r.returncode == 1
    assert f"{src}:{line}: {msg}" in r.stderr


# ------------------------------------------------------------------ GPU --
@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["gpu", "qms", "gpu-qmqs", "momqms", "gpu-hqms"])
@pytest.mark.parametrize("dist", ["random", "sorted", "reverse", "organpipe", "fewdistinct:8",
                                  "randomdup:64"])
def test_bench_emits_reference_csv(algo, dist):
    r = run("bench", "--algo", algo, "--n", "1,1000,65536", "--dist", dist, "--trials", "2",
            "--seed", "7", "--delta", "1/16", "--beta", "0.5")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == GOLDEN["cli"]["header"] and len(lines) == 1 + 3 * 2
    for ln in lines[1:]:
        f = ln.split(",")
        assert len(f) == 11 and f[0] == algo and f[2] == dist and f[3] == "7"
        n = int(f[1])
        comps, moves, t_ns, depth = map(int, f[5:9])
        assert comps == 0 and moves == 0 and depth >= 0
        assert t_ns > 0 or n <= 1
        lin = -math.log2(n) if n >= 2 else 0.0
        fields = [f[0], n, f[2], 7, int(f[4]), 0, 0, t_ns, depth, lin, 0.0]
        assert fmt(fields) == ln


@pytest.mark.gpu
def test_bench_out_file(tmp_path):
    out = tmp_path / "trials.csv"
    r = run("bench", "--algo", "gpu", "--n", "4096", "--trials", "3", "--out", out)
    assert r.returncode == 0 and r.stdout == ""
    rows = out.read_text().splitlines()
    assert rows[0] == GOLDEN["cli"]["header"] and len(rows) == 4


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["qms", "hqms", "gpu"])
def test_sort_file_roundtrip(tmp_path, algo):
    rng = np.random.default_rng(3)
    v = np.concatenate([rng.integers(-2**63, 2**63 - 1, 20000, dtype=np.int64),
                        np.array([-2**63, 2**63 - 1, 0, 0, -1], dtype=np.int64)])
    src, dst = tmp_path / "in.txt", tmp_path / "out.txt"
    src.write_text("\r\n".join(str(x) for x in v) + "\r\n")  # CRLF is accepted (qmsort.cpp:321)
    r = run("sort_file", src, dst, "--algo", algo)
    assert r.returncode == 0, r.stderr
    got = np.array([int(x) for x in dst.read_text().split()], dtype=np.int64)
    np.testing.assert_array_equal(got, np.sort(v))


@pytest.mark.gpu
def test_verify_quick():
    r = run("verify", "--quick", timeout=1200)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "verify: all checks passed" in r.stdout
    assert "FAIL" not in r.stdout
