"""The C-ABI library loads and exports every symbol include/sos_b200.h declares
(CPU-only checks; no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sos_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sos_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2410_19844_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_hot_path():
    names = declared_functions()
    for must in ("sos_build_index", "sos_forward", "sos_loss_grad", "sos_step", "sos_backward"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    from paper_2410_19844_b200 import binding
    assert set(declared_functions()) == set(binding.SIGNATURES)


def test_version_and_error_without_device(lib):
    lib.sos_version.restype = ctypes.c_int
    assert lib.sos_version() == 2
    lib.sos_last_error.restype = ctypes.c_char_p
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: device-error path not exercised")
    h = ctypes.c_void_p()
    lib.sos_build_index.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    assert lib.sos_build_index(4, 3, ctypes.byref(h)) == 4  # SOS_ERR_DEVICE
    assert lib.sos_last_error()


def test_argument_errors_are_reported(lib):
    h = ctypes.c_void_p()
    lib.sos_build_index.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
    assert lib.sos_build_index(0, 3, ctypes.byref(h)) == 1   # SOS_ERR_ARG
    assert lib.sos_build_index(250, 5, ctypes.byref(h)) == 1  # n + 2d > 255
    assert lib.sos_build_index(2, 40, ctypes.byref(h)) == 1   # d > 32
    assert lib.sos_build_index(60, 5, ctypes.byref(h)) == 1   # N = C(64, 5) > 65536
    lib.sos_descend.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] + [ctypes.c_void_p] * 2
    assert lib.sos_descend(None, None, None, 1, None, None) == 1
    lib.sos_forward.argtypes = [ctypes.c_void_p] * 4
    assert lib.sos_forward(None, None, None, None) == 1


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2410_19844_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "sos_oracle", "or_index_create"):
                    assert bad not in txt, (f, bad)


def test_release_library_reads_no_tuning_environment(lib):
    """No environment variable can change what the shipped library computes:
    the experiment switches (SOS_GEMM_PROBE, SOS_SKEW_*, ...) exist only in a
    -DSOS_EXPERIMENTS build; implementation variants are sos_plan_opts."""
    from paper_2410_19844_b200 import build
    blob = open(build.LIB, "rb").read()
    assert b"SOS_" not in blob
    assert hasattr(lib, "sos_plan_create_ex")


@pytest.mark.slow
def test_experiment_build_compiles_and_exports():
    """The -DSOS_EXPERIMENTS build (environment probes and traces, loaded only by
    tools with --exp) still compiles and exports the same ABI."""
    from paper_2410_19844_b200 import build
    path = build.build(experiments=True)
    exp = ctypes.CDLL(path)
    missing = [n for n in declared_functions() if not hasattr(exp, n)]
    assert not missing, missing
    assert b"SOS_GEMM_PROBE" in open(path, "rb").read()
    # the guarded-allocation check (tools/scratch_guard_check.py) exists only there
    from paper_2410_19844_b200.binding import LIB_PATH
    rel = ctypes.CDLL(LIB_PATH)
    for name in ("sos_exp_check_guards", "sos_exp_poke_guard"):
        assert hasattr(exp, name) and not hasattr(rel, name), name
