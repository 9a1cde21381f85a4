"""CPU tier: the C-ABI library is built, loads without a GPU and exports
every entry point include/pisob200.h declares."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pisob200.h")).read()
    return sorted(set(re.findall(r"PF_API\s+[\w\s\*]*?\b(pf_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    assert "pf_piso_step" not in names
    for must in ("pf_plan_create", "pf_cg_solve", "pf_bicgstab_solve",
                 "pf_assemble_momentum", "pf_bwd_h_stage"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2505_16992_b200 import _lib, build
    if not os.path.exists(_lib.LIB_PATH):
        build.build()
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(_lib.EXPORTED)
    assert lib.pf_version() >= 1


def test_library_rejects_bad_plan_without_gpu():
    import ctypes
    from paper_2505_16992_b200 import _lib
    lib = _lib.load()
    desc = _lib.PlanDesc()
    desc.dim = 5
    h = ctypes.c_void_p()
    rc = lib.pf_plan_create(ctypes.byref(desc), ctypes.byref(h))
    assert rc == 1
    assert b"dim" in lib.pf_last_error()


def test_product_refuses_cpu_device():
    import torch
    from paper_2505_16992_b200 import _lib, mesh
    dom = mesh.make_cavity((4, 4))
    with pytest.raises(_lib.LibraryError):
        dom.device_plan(torch.device("cpu"))
