"""Oracle tree for arXiv 1711.10885, matrix-free SIPG y = A z.

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import, call, link or execute
anything under oracle/. The product path (paper_1711_10885_b200/) never
imports this package, and this package never imports the product path: the
two share no code, headers, tables or constant generators. Seeded inputs are
produced by paper_1711_10885_b200/inputs.py (no method arithmetic) and passed
in as arrays.

Members
-------
o1_naive.c / o1.py   O-1: naive quadrature, C + OpenMP, cell-centric (no sum
                     factorization). The bilinear form eq:blf.
o2_assembled.py      O-2: dense matrix assembled entry by entry from the weak
                     form (numpy), tiny meshes only.
o3_kron.py           O-3: Kronecker closed form for diagonal D (numpy/scipy),
                     full-size vectors.
o2_geometry.py       O-2 on multilinear (Q1-mapped) meshes: the weak form with the
                     map's Jacobian at every quadrature point (NEXT-3, Problem C's
                     geometry), tiny meshes only.
rhs.py               l_h, L2 projection and the upwind
                     energy functional used by the invariant tests.
tables.py            1D Gauss rule and orthonormal Legendre basis (numpy).

Parity status: every function is pinned by tests/test_oracle_*.py (closed
forms, hand-derived single-cell matrices, invariants, cross-implementation
agreement). The absolute value of sigma, the boundary penalty gamma_d, the
RNG stream and the DOF order are conventions shared with the CUDA path
(readings C-3, C-4, C-6, C-13): "parity unpinned" by the paper
for those conventions only.
"""
