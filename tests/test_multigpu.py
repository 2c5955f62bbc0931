"""Multi-GPU engine (NCCL over NVLink): run tests/mp_engine_check.py under
torchrun on every visible GPU (skipped with fewer than 2)."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT, gpu_available


def ngpu():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def torchrun(n, args, env=None, timeout=900):
    """torchrun on 127.0.0.1; a fresh port and another try when the one picked
    was taken between free_port() and the rendezvous (EADDRINUSE)."""
    for _ in range(3):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), *args]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
        if r.returncode == 0 or "EADDRINUSE" not in r.stderr + r.stdout:
            return r
    return r


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available() or ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("which", ["c1", "replay", "lookahead", "wave", "c2", "c3mini", "c3", "c4s",
                                   "c4s_b40", "random", "device", "lti", "attach"])
def test_multi_gpu_matches_reference(which):
    if which.startswith(("c3", "c4s")) and which != "c3mini" and not os.path.exists(
            os.path.join(ROOT, "tests", "golden", f"{which}.json")):
        pytest.skip(f"{which} golden not generated")
    r = torchrun(min(ngpu(), 8), [os.path.join(ROOT, "tests", "mp_engine_check.py"), which])
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available() or ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("which", ["c1", "random"])
def test_multi_gpu_nccl_exchange_fallback(which):
    """DSEL_P2P=0: the W / W_k exchange over NCCL broadcasts instead of NVLink
    peer memory gives the same results."""
    r = torchrun(min(ngpu(), 8), [os.path.join(ROOT, "tests", "mp_engine_check.py"), which],
                 env=dict(os.environ, DSEL_P2P="0"))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available() or ngpu() < 2, reason="needs >= 2 GPUs")
def test_cli_multi_gpu(tmp_path):
    import json

    cli = os.path.join(ROOT, "paper_2604_08812_b200", "lib", "doptsel")
    w = json.load(open(os.path.join(ROOT, "tests", "golden", "wave.json")))
    r = subprocess.run([cli, "select", os.path.join(ROOT, "tests", "golden", "wave.kbf"),
                        "--budget", "12", "--gpus", "2", "--out", str(tmp_path)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert json.load(open(tmp_path / "selection.json"))["chosen"] == w["chosen"]
