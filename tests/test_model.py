"""The performance model reproduces the paper's printed numbers
(tests/golden/paper_values.txt, P:1079-1085 and Table 1)."""
import pytest

from conftest import read_golden
from paper_1007_1388_b200 import model


def golden():
    return {k: float(v) for k, v, _ in read_golden("paper_values.txt")}


def test_bytes_per_update():
    g = golden()
    assert model.bytes_per_update(4) == g["bytes_gpu_sp"]
    assert model.bytes_per_update(8) == g["bytes_gpu_dp"]
    assert model.bytes_per_update(4, gpu=False) == g["bytes_cpu_sp"]
    assert model.bytes_per_update(8, gpu=False) == g["bytes_cpu_dp"]


def test_table1():
    g = golden()
    t = model.table1(n=int(g["table1_n"]), kernel_ms=g["table1_compute_ms"], pcie_gbs=g["table1_pcie_gbs"],
                     ib_gbs=g["table1_ib_gbs"])
    assert t["pcie_ms"] == pytest.approx(g["table1_pcie_ms"], abs=1e-12)
    assert t["ib_ms"] == pytest.approx(g["table1_ib_ms"], abs=1e-12)
    assert t["total_I_ms"] == pytest.approx(g["table1_total_I_ms"], abs=1e-9)
    assert t["total_I_II_ms"] == pytest.approx(g["table1_total_I_II_ms"], abs=1e-9)
    # the paper truncates: 10^6 / 3.78 ms = 264.55 -> "264", 10^6 / 4.58 ms = 218.3 -> "218"
    assert int(t["mflups_I"]) == g["table1_mflups_I"]
    assert int(t["mflups_I_II"]) == g["table1_mflups_I_II"]
    # the kernel time itself is n^3 / P at ~300 MFLUPS
    assert model.t_kernel(100, 300) * 1e3 == pytest.approx(g["table1_compute_ms"], rel=0.02)


def test_paper_upper_bounds():
    """516 / 258 MFLUPS printed for 78 GB/s: the formula gives 513 / 256.6
    (R22, paper rounding)."""
    assert model.roofline_mflups(78, 4) == pytest.approx(516, rel=0.01)
    assert model.roofline_mflups(78, 8) == pytest.approx(258, rel=0.01)


def test_halo_bytes_match_plan():
    """The model's halo volume equals the exchange plan's remote bytes (lbm_plan)."""
    from paper_1007_1388_b200 import lbm
    for nr, grid in ((2, (1, 1, 2)), (4, (1, 2, 2)), (8, (2, 2, 2))):
        for r in range(nr):
            cfg = lbm.default_config((24 * grid[0], 20 * grid[1], 16 * grid[2]), (24, 20, 16), rank=r, nranks=nr)
            info, _ = lbm.plan(cfg)
            coord = info["proc_coord"]
            assert model.halo_bytes((24, 20, 16), coord, grid, 8) == info["halo_bytes_remote_per_step"]
