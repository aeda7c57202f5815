"""The C-ABI library loads, exports every symbol include/lbm.h declares, its
ctypes struct mirrors match the C layout, and it fails loudly without a GPU.
CPU only (no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "lbm.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"LBM_API\s+[\w\s\*]+?\b(lbm_\w+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for need in ("lbm_create", "lbm_set_flags", "lbm_step", "lbm_get_macroscopic", "lbm_get_pdfs",
                 "lbm_destroy", "lbm_last_error"):
        assert need in names


def test_library_exports_every_declared_symbol():
    from paper_1007_1388_b200 import lbm
    lib = ctypes.CDLL(lbm.LIB_PATH)
    names = declared_functions()
    assert sorted(lbm.EXPORTED) == names
    for n in names:
        assert hasattr(lib, n), n
    # nothing beyond the C ABI leaks out of the library (visibility=hidden)
    out = subprocess.run(["nm", "-D", "--defined-only", lbm.LIB_PATH], capture_output=True, text=True).stdout
    ours = sorted({l.split()[-1] for l in out.splitlines() if " T " in l and l.split()[-1].startswith("lbm_")})
    assert ours == names


def test_struct_layout_matches_c():
    from paper_1007_1388_b200 import lbm
    exe = os.path.join(ROOT, "build", "abi_layout")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "abi_layout.c"), "-o", exe], check=True)
    lines = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    c = dict(l.split() for l in lines if l)
    assert int(c["lbm_config"]) == ctypes.sizeof(lbm.LbmConfig)
    assert int(c["lbm_info"]) == ctypes.sizeof(lbm.LbmInfo)
    assert int(c["lbm_msg"]) == ctypes.sizeof(lbm.LbmMsg)
    structs = {"lbm_config": lbm.LbmConfig, "lbm_info": lbm.LbmInfo, "lbm_msg": lbm.LbmMsg}
    for k, v in c.items():
        if "." in k:
            s, m = k.split(".")
            assert getattr(structs[s], m).offset == int(v), k


def test_abi_version():
    from paper_1007_1388_b200 import lbm
    assert lbm._lib.lbm_abi_version() == 1


def _gpu_present():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_gpu_present(), reason="a GPU is present")
def test_create_fails_loudly_without_gpu():
    """No CPU fallback: on a host without a B200, lbm_create reports LBM_ERR_CUDA."""
    from paper_1007_1388_b200 import lbm
    with pytest.raises(lbm.LbmError) as ei:
        lbm.Lattice((8, 8, 8), minimal=True)
    assert ei.value.status == 4


def test_argument_validation_before_device_use():
    """Invalid arguments are rejected with LBM_ERR_ARG before any CUDA call."""
    from paper_1007_1388_b200 import lbm
    for kw in (dict(domain=(0, 8, 8)), dict(domain=(8, 8, 8), patch=(3, 8, 8)),
               dict(domain=(8, 8, 8), omega=2.0), dict(domain=(8, 8, 8), omega=0.0),
               dict(domain=(8, 8, 8), precision=2), dict(domain=(8, 8, 8), nranks=2),
               dict(domain=(8, 8, 8), rank=1, nranks=1)):
        with pytest.raises(lbm.LbmError) as ei:
            lbm.Lattice(**kw)
        assert ei.value.status == 1, kw
