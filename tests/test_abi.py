"""The C-ABI library loads without a GPU and exports every entry point that
include/octo_fmm.h declares (no compute calls: CPU-only check)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "octo_fmm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)   # drop comments
    names = set(re.findall(r"\b(octo_fmm_\w+)\s*\(", src))
    return sorted(n for n in names if not n.endswith("_fn"))


def test_header_declares_the_boundary():
    names = declared_functions()
    for core in ("octo_fmm_create", "octo_fmm_load_level", "octo_fmm_compute_interactions",
                 "octo_fmm_get_expansions", "octo_fmm_destroy", "octo_fmm_strerror", "octo_fmm_set_bootstrap"):
        assert core in names


def test_library_exports_every_declared_symbol():
    import paper_1908_03121_b200 as P
    lib = P.lib()
    raw = ctypes.CDLL(lib._name)
    missing = [n for n in declared_functions() if not hasattr(raw, n)]
    assert not missing, missing


def test_error_strings_without_a_device():
    import paper_1908_03121_b200 as P
    lib = P.lib()
    for code in (0, -1, -2, -3, -4, -5, -6):
        assert lib.octo_fmm_strerror(code)
    # create fails cleanly (no device here, or a bad config on a GPU box)
    cfg = P.binding.OctoConfig()
    cfg.abi_version = P.binding.ABI_VERSION
    cfg.n = 7   # invalid: n must be 8
    cfg.theta, cfg.G, cfg.nranks = 0.5, 1.0, 1
    h = ctypes.c_void_p()
    assert lib.octo_fmm_create(ctypes.byref(cfg), ctypes.byref(h)) == P.binding.OCTO_EINVAL
    assert not h.value
