"""CPU-side checks of the C-ABI library (no GPU): it loads, exports every symbol that
include/*.h declares, and rejects bad arguments / a missing device without computing."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        names |= set(re.findall(r"GP_API\s+[\w\s\*]+?\b(gp_\w+)\s*\(", txt))
    return sorted(names)


@pytest.fixture(scope="module")
def lib():
    import paper_2508_01864_b200 as g
    if not os.path.exists(g.LIB_PATH):
        from paper_2508_01864_b200 import build
        build.build()
    return g.load_library()


def test_header_declares_the_boundary():
    names = _declared_symbols()
    for must in ["gp_setup", "gp_kmvm", "gp_kmvm_host", "gp_kzx_setup", "gp_kzx", "gp_kzx_destroy",
                 "gp_cg_solve", "gp_predict", "gp_destroy", "gp_last_error", "gp_plan_query",
                 "gp_plan_set_option", "gp_version", "gp_kmvm_rank", "gp_permute",
                 "gp_kmvm_dlengthscale", "gp_cg_solve_pc", "gp_cg_solve_ex", "gp_kmvm_partial",
                 "gp_shard_ranges", "gp_precond_create",
                 "gp_precond_factor", "gp_precond_solve", "gp_precond_logdet",
                 "gp_precond_destroy", "gp_mbcg", "gp_lml", "gp_fit", "gp_set_allocator"]:
        assert must in names, must


def test_library_exports_every_declared_symbol(lib):
    for name in _declared_symbols():
        assert hasattr(lib, name), f"{name} declared in include/ but not exported"
    assert lib.gp_version().decode().startswith("gpmatern")


def test_library_is_sm100a_only():
    import paper_2508_01864_b200 as g
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", g.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_argument_validation_without_device(lib):
    import paper_2508_01864_b200 as g
    k = g.Kernel(11, (0.1,)).c()
    h = ctypes.c_void_p()
    dummy = ctypes.c_void_p(16)
    assert lib.gp_setup(dummy, 0, 1, ctypes.byref(k), None, ctypes.byref(h)) == 1      # n < 1
    assert lib.gp_setup(dummy, 10, 4, ctypes.byref(k), None, ctypes.byref(h)) == 1     # d = 4
    assert lib.gp_setup(dummy, 10, 1, ctypes.byref(k), None, ctypes.byref(h)) == 2     # nu = 11/2
    assert b"supported" in lib.gp_last_error()
    k = g.Kernel(3, (-0.1,)).c()
    assert lib.gp_setup(dummy, 10, 1, ctypes.byref(k), None, ctypes.byref(h)) == 1     # l <= 0
    k = g.Kernel(5, (0.1, 0.1, 0.1), form=2).c()
    assert lib.gp_setup(dummy, 10, 3, ctypes.byref(k), None, ctypes.byref(h)) == 1     # form


def test_no_cpu_fallback(lib):
    """Without a CUDA device a valid call fails loudly (GP_ERR_CUDA), it never computes."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2508_01864_b200 as g
    k = g.Kernel(3, (0.1,)).c()
    h = ctypes.c_void_p()
    assert lib.gp_setup(ctypes.c_void_p(16), 10, 1, ctypes.byref(k), None, ctypes.byref(h)) == 7
    assert b"no CUDA device" in lib.gp_last_error()
    assert lib.gp_kmvm(None, None, 1, None, None) == 1


def test_set_allocator_validation(lib):
    import ctypes as C
    assert lib.gp_set_allocator(C.c_void_p(16), None, None) == 1   # only one hook
    assert lib.gp_set_allocator(None, None, None) == 0             # default restored
