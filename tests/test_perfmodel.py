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


def test_table1_columns_and_matrix_bytes():
    """Table 1's matrix-based columns: the paper's 'A / matrix
    based' ratio at p = 7 is 390x; the block-stencil matvec moves 7 n^3 matrix entries per row
    (leading dimension padded to even) plus z and y."""
    assert abs(pm.PAPER_TABLE1_A_MDOFS[7] / pm.PAPER_TABLE1_MATRIX_MDOFS[7] - 390.0) < 0.5
    assert pm.matrix_bytes_per_dof(7) == 8 * 7 * 512 + 16
    assert pm.matrix_bytes_per_dof(2) == 8 * 7 * 28 + 16      # n^3 = 27 -> ld 28


def test_matrix_meshes_fit_and_use_27_colour_classes():
    from paper_1711_10885_b200 import configs
    for k in range(1, 11):
        cfg = configs.problem_a_matrix(k)
        N = cfg.ncells[0]
        n3 = (k + 1) ** 3
        assert N % 3 == 0 and cfg.ncells == (N, N, N)
        assert cfg.ndofs * 7 * (n3 + (n3 & 1)) * 8 <= 24e9
        assert cfg.periodic == (1, 1, 1) and cfg.dfield_seed >= 0


def test_committed_ncu_summary_belongs_to_this_build():
    """bench.py's roofline.frac divides executed flops from profiles/ncu_full_summary.json by the
    kernel time and refuses a capture of another build (bench.load_ncu). A kernel-source change
    without a fresh capture (tools/gpu_refresh_captures.sh) would leave the bench line without a
    fraction: fail here instead."""
    import json
    import os
    from paper_1711_10885_b200.build import kernel_family, kernel_hash
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "profiles", "ncu_full_summary.json")) as f:
        d = json.load(f)
    for name in ("C3", "C5-weak-P1", "A-k7", "C-k7", "TG-k5"):
        ent = d[name]
        assert ent["build_hash"] == kernel_hash(kernel_family(ent["kernel"])), name
        assert ent["executed_flops_per_dof"] > 0 and ent["duration_ns"] > 0
