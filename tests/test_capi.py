"""The C-ABI library loads without a GPU and exports every entry point include/pba_gpu.h declares."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_1704_06967_b200 import _capi

from ._oracle import ORACLE_LIB, REF

HDR = Path(__file__).resolve().parent.parent / "include" / "pba_gpu.h"


def declared():
    txt = HDR.read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pba_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_survey_export_set():
    names = declared()
    for must in ["pba_gpu_create", "pba_gpu_destroy", "pba_gpu_set_params", "pba_gpu_get_params", "pba_gpu_energy",
                 "pba_gpu_ic_build", "pba_gpu_ic_gradient", "pba_gpu_ic_solve_step", "pba_gpu_ic_factorize",
                 "pba_gpu_fc_build", "pba_gpu_solve_normal_equations_schur", "pba_gpu_apply_update",
                 "pba_gpu_max_reproj_update", "pba_gpu_normalize_gauge", "pba_gpu_ic_run", "pba_gpu_fc_run",
                 "pba_gpu_last_error"]:
        assert must in names, must


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_capi.GPU_LIB))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_oracle_mirrors_the_gpu_call_set():
    lib = ctypes.CDLL(str(ORACLE_LIB))
    gpu_only = {"stream", "set_profiling", "kernel_times", "device_bytes", "ic_begin", "fc_begin", "iterate", "end",
                "launch_count", "set_exchange", "nccl_unique_id", "set_exchange_nccl",  # multi-process plumbing
                "create_deferred"}
    for n in declared():
        if n.startswith("pba_gpu_") and n[len("pba_gpu_"):] not in gpu_only:
            assert hasattr(lib, "pba_oracle_" + n[len("pba_gpu_"):]), n


def test_status_strings_and_defaults():
    lib = ctypes.CDLL(str(_capi.GPU_LIB))
    lib.pba_status_string.restype = ctypes.c_char_p
    assert lib.pba_status_string(1) == b"EmptyProblem"
    assert lib.pba_status_string(5) == b"SingularHessian"
    cfg = _capi.pba_config()
    lib.pba_config_default(ctypes.byref(cfg))
    assert (cfg.gamma, cfg.threshold_px, cfg.max_iters, cfg.lambda0, cfg.max_bad_steps) == (0.03, 5e-3, 200, 1e-6, 8)
    assert cfg.normalize_depth_gauge == 1 and cfg.refresh_ic_hessian == 0


def test_product_package_binds_only_the_gpu_library():
    """No multi-backend dispatch: the product cannot load a checker library by name, and no product
    source refers to the oracle's or the reference's shared objects."""
    with pytest.raises(ValueError):
        _capi.backend("oracle")
    pkg = Path(_capi.__file__).resolve().parent
    for src in list(pkg.glob("*.py")) + list((pkg / "csrc").glob("*")):
        txt = src.read_text(errors="ignore")
        assert "liboracle" not in txt and "libpba_ref" not in txt and "pba_oracle_" not in txt, src


def test_reference_library_exports_the_checker_call_set():
    """oracle/_ref/libpba_ref.so (the unmodified reference compiled against oracle/ref_shim) exports the
    same calls as the oracle, for the dense problems the reference can express."""
    if not REF.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    lib = ctypes.CDLL(str(REF.path if hasattr(REF, "path") else REF.get().path))
    for n in ["create", "destroy", "energy", "ic_build", "ic_gradient", "ic_compute_step", "ic_solve_step",
              "ic_factorize", "ic_hessian", "ic_run", "fc_run", "solve_normal_equations_schur",
              "solve_normal_equations_dense", "apply_update", "render_sequence", "perturb_parameters"]:
        assert hasattr(lib, "pba_ref_" + n), n
