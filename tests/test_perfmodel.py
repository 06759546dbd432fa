"""Model numbers printed by / computed from the paper (golden/perfmodel.json)."""
from conftest import golden
from paper_1711_10885_b200 import perfmodel as pm


def test_model_numbers():
    g = golden("perfmodel.json")
    assert pm.cost_vol(3, 4, 1.0) == g["cost_vol_d3_m4_rho1"]
    assert pm.cost_face(2, 3, 1.0) == g["cost_face_d2_m3_rho1"]
    assert pm.C(2, 0.5) == g["C_d2_rho_half"]
    assert pm.flopdof_vol(3, 3) == g["flopdof_vol_d3_p3"]
    assert pm.flopdof_face(3, 3) == g["flopdof_face_d3_p3"]
    assert pm.flopdof(3, 7) == g["flopdof_total_d3_p7"]
    assert pm.BDOF_VOL == g["bdof_vol"] and pm.bdof_face(3) == g["bdof_face_d3"]
    assert pm.roofline(0.25, 30.4, 15) == g["roofline_I0.25_pi30.4_beta15"]
    assert pm.roofline(100, 30.4, 15) == 30.4


def test_crossover_degree():
    """Reading C-18: by the formulas faces exceed volume for p <= 4 in 3D."""
    for p in range(1, 11):
        assert (pm.flopdof_face(3, p) > pm.flopdof_vol(3, p)) == (p <= 4)


def test_fp64_peak():
    assert abs(pm.fp64_peak_tflops() - 37.22) < 0.01
