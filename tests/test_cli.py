"""`doptsel select` drop-in CLI (paper_2604_08812_b200/tools/doptsel_main.cpp):
flags, outputs and exit codes of proj/tools/doptsel_main.cpp:26-30, :87-165."""
import csv
import json
import os
import shutil
import subprocess

import pytest

from conftest import ROOT, gpu_available

CLI = os.path.join(ROOT, "paper_2604_08812_b200", "lib", "doptsel")
GOLD = os.path.join(ROOT, "tests", "golden")


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


def test_usage_and_argument_errors(tmp_path):
    assert run().returncode == 1
    assert run("select").returncode == 1
    wave = os.path.join(GOLD, "wave.kbf")
    assert run("select", wave, "--budget", "99").returncode == 1        # budget out of range
    assert run("select", wave, "--budget", "2", "--mode", "naive").returncode == 1
    assert run("select", wave, "--budget", "2", "--precision", "f32").returncode == 1
    assert run("select", wave, "--budget", "2", "--mode", "bogus").returncode == 1
    assert run("build", "only_one_arg.cfg").returncode == 1
    assert run("build", os.path.join(GOLD, "configs", "bad_key.cfg"), str(tmp_path / "y.kbf")).returncode == 1
    assert run("build", str(tmp_path / "missing.cfg"), str(tmp_path / "y.kbf")).returncode == 3


def test_io_errors_exit_3(tmp_path):
    assert run("select", str(tmp_path / "missing.kbf"), "--budget", "1").returncode == 3
    bad = tmp_path / "bad.kbf"
    bad.write_bytes(b"NOPE" + bytes(28))
    assert run("select", str(bad), "--budget", "1").returncode == 3
    trunc = tmp_path / "trunc.kbf"
    data = open(os.path.join(GOLD, "wave.kbf"), "rb").read()
    trunc.write_bytes(data[:-8])
    r = run("select", str(trunc), "--budget", "1")
    assert r.returncode == 3 and "size" in r.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA GPU")
def test_select_wave_outputs_match_reference(tmp_path):
    w = json.load(open(os.path.join(GOLD, "wave.json")))
    noise = tmp_path / "noise.txt"
    noise.write_text("\n".join(repr(x) for x in w["noise_logdets"]))
    out = tmp_path / "out"
    r = run("select", os.path.join(GOLD, "wave.kbf"), "--budget", "12", "--workers", "4",
            "--noise-logdets", str(noise), "--out", str(out))
    assert r.returncode == 0, r.stderr
    sel = json.load(open(out / "selection.json"))
    assert sel["chosen"] == w["chosen"]
    assert sel["n_sensors"] == 32 and sel["n_steps"] == 16 and sel["budget"] == 12
    for a, b in zip(sel["objective_raw"], w["objectives"]):
        assert abs(a - b) <= 1e-9 * max(abs(b), 1.0)
    assert abs(sel["objective_normalized_final"] - 1045.5268963527164) < 1e-6
    rows = list(csv.reader(open(out / "trace.csv")))
    assert rows[0] == ["k", "chosen_index", "objective", "gain", "n_evaluated", "wall_ms"]
    assert [int(x[1]) for x in rows[1:]] == w["chosen"]
    t = list(csv.reader(open(out / "timing.csv")))
    assert t[0] == ["round", "worker", "io_ms", "compute_ms", "wall_ms", "overlap"]
    assert len(t) == 13


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA GPU")
def test_select_synthetic_c1_and_budget_zero(tmp_path):
    c1 = json.load(open(os.path.join(GOLD, "c1.json")))
    r = run("select", "--synthetic", "64,32,2048,1.0,2024", "--budget", "16", "--out",
            str(tmp_path / "c1"))
    assert r.returncode == 0, r.stderr
    assert json.load(open(tmp_path / "c1" / "selection.json"))["chosen"] == c1["chosen"]
    r = run("select", os.path.join(GOLD, "wave.kbf"), "--budget", "0", "--out", str(tmp_path / "z"))
    assert r.returncode == 0
    sel = json.load(open(tmp_path / "z" / "selection.json"))
    assert sel["chosen"] == [] and sel["objective_normalized"] == []


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA GPU")
def test_select_kbf_row_layout_matches(tmp_path):
    w = json.load(open(os.path.join(GOLD, "wave.json")))
    r = run("select", os.path.join(GOLD, "wave.kbf"), "--budget", "12", "--kbf-rows", "--out",
            str(tmp_path / "o"))
    assert r.returncode == 0, r.stderr
    assert json.load(open(tmp_path / "o" / "selection.json"))["chosen"] == w["chosen"]


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA GPU")
@pytest.mark.parametrize("extra", [["--algorithm", "left"], ["--storage", "stream"]])
def test_select_variants(tmp_path, extra):
    w = json.load(open(os.path.join(GOLD, "wave.json")))
    r = run("select", os.path.join(GOLD, "wave.kbf"), "--budget", "12", *extra, "--out",
            str(tmp_path / "o"))
    assert r.returncode == 0, r.stderr
    assert json.load(open(tmp_path / "o" / "selection.json"))["chosen"] == w["chosen"]


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA GPU")
def test_build_on_gpu_then_select(tmp_path):
    """`doptsel build` assembles K on the GPU: the KBF file is byte-identical to the
    reference's; `select --config` on it reports the reference normalized objective
    (the config's default noise level needs the full wave model)."""
    import hashlib

    lti = json.load(open(os.path.join(GOLD, "lti.json")))["configs"]
    for name in ("wave_benchmark.cfg", "weighted.cfg", "identity_prior.cfg"):
        kbf = tmp_path / (name + ".kbf")
        r = run("build", os.path.join(GOLD, "configs", name), str(kbf))
        assert r.returncode == 0, r.stderr
        assert hashlib.sha256(kbf.read_bytes()).hexdigest() == lti[name]["kbf_sha256"]
    out = tmp_path / "out"
    r = run("select", str(tmp_path / "wave_benchmark.cfg.kbf"), "--budget", "12", "--config",
            os.path.join(GOLD, "configs", "wave_benchmark.cfg"), "--out", str(out))
    assert r.returncode == 0, r.stderr
    sel = json.load(open(out / "selection.json"))
    assert sel["chosen"] == lti["wave_benchmark.cfg"]["chosen"]
    assert abs(sel["objective_normalized_final"] - 1045.5268963527164) < 1e-6
