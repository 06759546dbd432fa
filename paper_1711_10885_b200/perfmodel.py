"""The paper's closed-form cost and roofline model
used to normalise measurements (model GFLOP/s = FLOPDOF x DOFs/s), plus the
B200 FP64 peak derivation used by bench.py's roofline object."""


def C(d, rho):
    """C_{d,rho} = sum_{q=1}^d rho^q."""
    return sum(rho ** q for q in range(1, d + 1))


def cost_vol(d, m, rho=1.0):
    return 2.0 * C(d, rho) * m ** (d + 1)            # eq:cost_volume_sumfact


def cost_face(d, m, rho=1.0):
    return 2.0 * C(d, rho) * m ** d                  # eq:cost_face_sumfact


def flopdof_vol(d, p):
    return 4.0 * (d + 1) * d * (p + 1) + 2 * d * d + 5 * d + 3


def flopdof_face(d, p):
    return 8.0 * (d + 1) * d * d + d * (2 * d * d + 8 * d + 18) / (p + 1.0)


def flopdof(d, p):
    return flopdof_vol(d, p) + flopdof_face(d, p)


BDOF_VOL = 16.0


def bdof_face(d):
    return 32.0 * d


def roofline(I, pi, beta):
    return min(pi, beta * I)


# B200 FP64 (non-tensor) arithmetic peak, derived from unit counts and clocks
# (B200_PROFILING.md: 148 SMs, clocks.max.sm 1965 MHz; 64 FP64 FMA lanes per SM
# per clock = 4 SMSPs x 16): 148 * 64 * 2 flop * 1.965e9 = 37.2 TFLOP/s.
B200_SMS = 148
FP64_FMA_PER_CLK_PER_SM = 64


def fp64_peak_tflops(sm_mhz=1965.0):
    return B200_SMS * FP64_FMA_PER_CLK_PER_SM * 2 * sm_mhz * 1e6 / 1e12


# The paper's only throughput numbers for this operator: Table 1, Problem A (periodic,
# axis-parallel, per-cell tensor D, q = 2p, ~4e8 DOFs; 2x16-core Haswell node), full operator
# application in MDOF/s. Context for the Problem A
# bench workload (configs.problem_a), not the target.
PAPER_TABLE1_A_MDOFS = {1: 170.2, 2: 393.0, 3: 537.8, 4: 595.0, 5: 617.2, 6: 599.0, 7: 570.1, 8: 540.6,
                        9: 504.8, 10: 471.3}

# Table 1's matrix-based columns (PETSc BAIJ matvec on meshes scaled down to fit, and the
# sum-factorized assembly), MDOF/s on the same node.
PAPER_TABLE1_MATRIX_MDOFS = {1: 206.45, 2: 64.20, 3: 26.85, 4: 9.544, 5: 4.585, 6: 2.311, 7: 1.462, 8: 0.614,
                             9: 0.298}
PAPER_TABLE1_ASSEMBLY_MDOFS = {1: 16.04, 2: 8.71, 3: 4.66, 4: 2.57, 5: 1.93, 6: 1.21, 7: 0.665, 8: 0.874, 9: 0.701}


def matrix_bytes_per_dof(k):
    """HBM bytes per DOF of one block-stencil matvec: the row's 7 n^3 matrix entries (x ld / n^3
    for the even leading dimension ld of the layout, include/dg.h) plus reading z and writing y
    once (8 + 8)."""
    n3 = (k + 1) ** 3
    ld = n3 + (n3 & 1)
    return 8.0 * 7 * ld + 16.0
