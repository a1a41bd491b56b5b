"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/ptsbe.h declares."""

import ctypes
import re
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (REPO / "include" / "ptsbe.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void\*|int64_t|double)\s+(ptsbe_\w+)\s*\(", text, re.M)))


def test_header_lists_entry_points():
    syms = declared_symbols()
    for s in ("ptsbe_create", "ptsbe_load_program", "ptsbe_run_batch", "ptsbe_sample", "ptsbe_get_state"):
        assert s in syms


def test_library_exports_every_declared_symbol(libptsbe):
    lib = ctypes.CDLL(str(libptsbe))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing
    lib.ptsbe_abi_version.restype = ctypes.c_int
    assert lib.ptsbe_abi_version() == 1


def test_binding_covers_header(libptsbe):
    from paper_2504_16297_b200 import _native
    assert set(declared_symbols()) == set(_native.SIGNATURES)
    _native.load_library(libptsbe)


def test_sm100a_cubin(libptsbe):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(libptsbe)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_errors_without_gpu_are_loud(libptsbe):
    # on a GPU-less host creating an engine must fail with ExecutionError, never fall back
    import pytest
    from paper_2504_16297_b200 import _native
    from paper_2504_16297_b200.engine import Engine
    from paper_2504_16297_b200.errors import ExecutionError
    lib = _native.load_library(libptsbe)
    n = ctypes.c_int()
    cuda = ctypes.CDLL("libcudart.so.12") if False else None  # noqa: F841
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("GPU present")
    with pytest.raises(ExecutionError):
        Engine(4, "c128", 1)


def test_host_only_codegen_plans_and_generates(libptsbe):
    """ptsbe_create_host: load_program's validation, phase planning and kernel generation run
    without a GPU; the source holds one kernel per pass with out-of-line slow variants."""
    import paper_2504_16297_b200 as P
    from paper_2504_16297_b200 import workloads
    from paper_2504_16297_b200.engine import generated_source
    from paper_2504_16297_b200.program import compile_circuit
    c = workloads.build(4, P.parse_circuit, P.parse_noise_model, P.attach_noise)
    prog = compile_circuit(c, "c64")
    src = generated_source(prog, "c64")
    kernels = re.findall(r'extern "C" __global__ void __launch_bounds__\(\d+, \d+\) (ptsbe_pass_\d+)', src)
    assert kernels == [f"ptsbe_pass_{i}" for i in range(prog.n_passes)]
    assert "__noinline__ void ptsbe_slow_" in src          # slow variants out of line
    assert "struct Swz0" in src                            # per-pass shared-memory swizzle
    assert src.count("// @@ptsbe-pass@@") == prog.n_passes  # one NVRTC program per pass
