"""CPU tests of the C ABI boundary: the library loads, exports every entry
point include/dsel.h declares, the host-side synthetic input is bit-identical
to the reference RNG stream, and engine creation fails loudly (no CPU
fallback) when no GPU is present."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, gpu_available

HEADER = os.path.join(ROOT, "include", "dsel.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dsel_[a-z0-9_]+)\s*\(", src)))


def test_header_declarations_match_binding():
    import paper_2604_08812_b200._abi as abi

    assert declared_symbols() == sorted(abi.EXPORTS)


def test_library_exports_every_declared_symbol():
    import paper_2604_08812_b200 as d

    out = subprocess.run(["nm", "-D", "--defined-only", d.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (dsel_[a-z0-9_]+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert d.lib.dsel_abi_version() == 2


def test_every_allocation_goes_through_the_counted_wrappers():
    """The zero-allocation check on dsel_step (tests/test_gpu_parity.py) reads
    dsel_alloc_count(); it covers every device/pinned allocation only if no
    raw cudaMalloc / cudaMallocHost / cudaHostAlloc / cudaHostRegister call
    bypasses the counted wrappers (ds_malloc, ds_malloc_host, ds_host_register)."""
    csrc = os.path.join(ROOT, "paper_2604_08812_b200", "csrc")
    raw = re.compile(r"\b(cudaMalloc|cudaMallocHost|cudaHostAlloc|cudaHostRegister|cudaMallocAsync|"
                     r"cudaMallocManaged|cudaMallocPitch)\s*\(")
    offenders = []
    for name in sorted(os.listdir(csrc)):
        lines = open(os.path.join(csrc, name)).read().splitlines()
        for i, line in enumerate(lines):
            if raw.search(line) and "return cuda" not in line:  # the wrappers' own calls
                offenders.append(f"{name}:{i + 1}: {line.strip()}")
    assert not offenders, offenders


def test_library_is_sm100a_and_uses_dmma():
    import paper_2604_08812_b200 as d

    sass = subprocess.run(["cuobjdump", "-sass", d.LIB_PATH], capture_output=True, text=True,
                          check=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", d.LIB_PATH], capture_output=True,
                                       text=True).stdout
    assert "DMMA.8x8x4" in sass


def test_synthetic_v_bit_identical_to_reference_stream():
    import paper_2604_08812_b200 as d
    from oracle import oracle as O

    for (nd, nt, rank, seed) in [(3, 2, 5, 2024), (4, 3, 7, 1), (64, 32, 16, 2024)]:
        a = d.synthetic_v(nd, nt, rank, seed, threads=4)
        b = O.synthetic_v(nd, nt, rank, seed)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_c_header_compiles_standalone(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "dsel.h"\nint main(void){dsel_config c={0}; (void)c; '
                   'return dsel_abi_version()==DSEL_ABI_VERSION?0:1;}\n')
    import paper_2604_08812_b200 as d

    exe = tmp_path / "t"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    str(src), "-o", str(exe), d.LIB_PATH, "-Wl,-rpath," + os.path.dirname(d.LIB_PATH)],
                   check=True)
    assert subprocess.run([str(exe)]).returncode == 0


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure path")
def test_create_fails_loudly_without_gpu():
    import paper_2604_08812_b200 as d

    with pytest.raises(d.WorkerFailure):
        d.Engine(8, 2, 2)


def test_invalid_config_rejected_before_device_work():
    import paper_2604_08812_b200 as d

    with pytest.raises(d.InvalidConfig):
        d.Engine(8, 2, -1)
    with pytest.raises(d.InvalidConfig):
        d.Engine(8, 2, 2, candidates=[1, 1])
    with pytest.raises(d.IndexOutOfRange):
        d.Engine(8, 2, 2, candidates=[1, 8])
    with pytest.raises(d.InvalidConfig):
        d.Engine(8, 2, 2, storage=2)               # streaming needs the left-looking algorithm
    with pytest.raises(d.InvalidConfig):
        d.Engine(8, 2, 2, algorithm="middle")


def test_lti_config_host_tables(golden_dir=os.path.join(ROOT, "tests", "golden")):
    """Config parsing + make_wave_problem on the host (no GPU): dimensions,
    default noise (0.1 max|h|), mask/cost expansion, error mapping."""
    import paper_2604_08812_b200 as d

    p = d.LtiProblem.from_config(os.path.join(golden_dir, "configs", "wave_benchmark.cfg"))
    assert (p.n_params, p.n_sensors, p.n_steps) == (48, 32, 16)
    assert p.noise_sigma == 0.1 * np.abs(p.impulse).max()
    assert abs(p.noise_sigma - 0.075696580131319649) < 1e-17
    assert p.mask is None and p.cost_weights is None
    assert p.spatial[0] == 1.0 and abs(p.spatial[1] - np.exp(-1 / 6.0)) < 1e-16
    w = d.LtiProblem.from_config(os.path.join(golden_dir, "configs", "weighted.cfg"))
    assert w.mask.shape == (48 * 16,) and w.mask[0] == 0.0 and w.mask[24 * 16 + 12] == 0.5
    assert w.cost_weights[0] == 4.0
    with pytest.raises(d.InvalidConfig):
        d.LtiProblem.from_config(os.path.join(golden_dir, "configs", "bad_key.cfg"))
    with pytest.raises(d.IoError):
        d.LtiProblem.from_config(os.path.join(golden_dir, "configs", "missing.cfg"))
