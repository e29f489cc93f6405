"""C-ABI checks that need no GPU: the library loads and exports every entry
point declared in include/sgp.h; the host-side model layout matches."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2511_06407_b200", "libsgp.so")
HDR = os.path.join(ROOT, "include", "sgp.h")


def declared_symbols():
    text = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*(sgp_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return ctypes.CDLL(LIB)


def test_header_declares_entry_points():
    syms = declared_symbols()
    for name in ("sgp_model_create", "sgp_eval", "sgp_trace", "sgp_eigh_cold", "sgp_eigh_warm",
                 "sgp_leapfrog", "sgp_run_moves", "sgp_chain_init"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_version_string(lib):
    lib.sgp_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.sgp_version()


def test_null_arguments_are_rejected_without_gpu(lib):
    # argument validation happens before any CUDA call
    lib.sgp_eval.restype = ctypes.c_int
    assert lib.sgp_eval(None, 1, None, None, 0, None, None, None, None, None, None, None) == -1
    assert lib.sgp_run_moves(None, None, None, 1, 0, None, None, None, None) == -1
    assert lib.sgp_eigh_cold(0, 3, None, ctypes.c_double(1e-13), 30, None, None, None, None) == -1
    assert lib.sgp_eigh_dc(1, 0, None, None, None, None) == -1
    assert lib.sgp_eigh_dc(1, 5000, None, None, None, None) == -1


def test_library_built_for_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_device_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2511_06407_b200 import PosteriorTarget, build_model, simulate_logistic
    data, _ = simulate_logistic(1, n=20, seed=0)
    with pytest.raises(RuntimeError, match="CUDA device"):
        PosteriorTarget(build_model("logistic", data.x, feature_count=4), data)


def test_layout_dimensions():
    from paper_2511_06407_b200 import rrgp
    data, _ = rrgp.simulate_logistic(1, n=30, seed=0)
    assert rrgp.BlockLayout.from_model(rrgp.build_model("logistic", data.x)).dim == 34
    data16, _ = rrgp.simulate_logistic(16, n=30, seed=0)
    assert rrgp.BlockLayout.from_model(rrgp.build_model("logistic", data16.x)).dim == 484
    mv, _ = rrgp.simulate_meanvar(2, 19, n=200, seed=0)
    dims = {n: rrgp.BlockLayout.from_model(rrgp.build_model(n, mv.x)).dim
            for n in ("l-mean", "nl-mean", "l-meanvar", "nl-meanvar")}
    assert dims == {"l-mean": 26, "nl-mean": 84, "l-meanvar": 47, "nl-meanvar": 163}
