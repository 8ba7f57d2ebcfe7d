"""Bindings of the CPU checkers — TEST INFRASTRUCTURE ONLY.

Two checker libraries export the call set of include/pba_gpu.h (declared once in
``paper_1704_06967_b200._capi._COMMON``) under their own prefixes:

* ``ORACLE`` — ``oracle/_build/liboracle.so`` (prefix ``pba_oracle_``): the Eigen-free restatement of
  the reference's solver.cpp / geometry.cpp / image.cpp / synth.cpp, with the observation-list
  extension (visibility) the BASELINE configs need.
* ``REF`` — ``oracle/_ref/libpba_ref.so`` (prefix ``pba_ref_``): the UNMODIFIED reference sources
  compiled in place (oracle/Makefile ``ref``) against oracle/ref_shim; dense problems only.

The product package never loads either: ``paper_1704_06967_b200`` binds only libpba_gpu.so.  A
checker is handed to the product's Python mirror as a library object (``Handle(state, ORACLE)``),
so the parity tests drive the GPU library and the checkers through exactly the same calls.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
legs import this module.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from paper_1704_06967_b200 import _capi as capi

REPO = Path(__file__).resolve().parent.parent
ORACLE_LIB = REPO / "oracle" / "_build" / "liboracle.so"
REF_LIB = REPO / "oracle" / "_ref" / "libpba_ref.so"

i32, f64, u64 = C.c_int32, C.c_double, C.c_uint64
P = C.POINTER


class pba_oracle_scene_spec(C.Structure):
    """SceneSpec (synth.hpp:14-50) flattened; oracle/pba_oracle_c.h."""
    _fields_ = [("width", i32), ("height", i32), ("fx", f64), ("fy", f64), ("cx", f64), ("cy", f64),
                ("octaves", i32), ("base_wavelength_px", f64), ("lo", f64), ("hi", f64),
                ("geometry_kind", i32), ("base_depth", f64), ("amplitude", f64), ("wavelength_px", f64),
                ("trajectory_kind", i32), ("frames", i32), ("span_deg", f64), ("extent", f64 * 3),
                ("num_points", i32), ("patch_radius", i32), ("seed", u64), ("supersample", i32)]


_EXTRA = {
    "solve_normal_equations_dense": capi._COMMON["solve_normal_equations_schur"],
    "scene_spec_default": (None, [P(pba_oracle_scene_spec)]),
    "render_sequence": (C.c_int, [P(pba_oracle_scene_spec), P(f64), P(f64), P(f64), P(f64), P(f64), P(f64),
                                  C.c_char_p, C.c_int]),
    "perturb_parameters": (C.c_int, [i32, P(f64), P(f64), i32, P(f64), f64, u64]),
}


class CpuLib:
    """A checker library bound with the product's call-set declarations.  Functions a checker does
    not export (e.g. the reference has no fc_build / multi-host window) are left as None."""

    def __init__(self, kind: str, path: Path, prefix: str):
        if not path.exists():
            raise RuntimeError(f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        self.kind = kind
        self.path = path
        self.lib = C.CDLL(str(path))
        for name, (res, args) in {**capi._COMMON, **_EXTRA}.items():
            fn = getattr(self.lib, prefix + name, None)
            if fn is not None:
                fn.restype = res
                fn.argtypes = args
            setattr(self, name, fn)
        self.config_default = None


class _Lazy:
    """Loads the library on first use, so importing this module never requires a build."""

    def __init__(self, kind: str, path: Path, prefix: str):
        self._args = (kind, path, prefix)
        self._lib = None

    def get(self) -> CpuLib:
        if self._lib is None:
            self._lib = CpuLib(*self._args)
        return self._lib

    def available(self) -> bool:
        return self._args[1].exists()

    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        return getattr(self.get(), name)


ORACLE = _Lazy("oracle", ORACLE_LIB, "pba_oracle_")
REF = _Lazy("reference", REF_LIB, "pba_ref_")
