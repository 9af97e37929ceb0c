"""The drop-in boundary: the C-ABI library loads without a GPU and exports
every entry point include/damf_gpu.h declares (no compute calls here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "damf_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(damf_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_engine_surface():
    names = declared_functions()
    for required in ("damf_gpu_create", "damf_gpu_create_from_factors", "damf_gpu_apply",
                     "damf_gpu_query_rows", "damf_gpu_materialize", "damf_gpu_ppr_init",
                     "damf_gpu_ppr_push", "damf_gpu_rebase", "damf_gpu_destroy",
                     "damf_gpu_last_error", "damf_gpu_score"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2306_08967_b200", "libdamf_gpu.so"))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    lib.damf_gpu_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.damf_gpu_version()


def test_status_codes_follow_reference_error_kinds():
    # types.hpp:21-41 order; ABI status = ordinal + 1
    from paper_2306_08967_b200.engine import ERROR_KINDS
    hdr = open(os.path.join(ROOT, "include", "damf_gpu.h")).read()
    for i, kind in enumerate(ERROR_KINDS):
        m = re.search(r"DAMF_E_[A-Z_]+ = %d," % (i + 1), hdr)
        assert m, kind
