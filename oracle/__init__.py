"""CPU oracle for the H(grad)/H(curl) Riesz-map hot path of arXiv 2506.17406.

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import anything from this package.
The product path (paper_2506_17406_b200/) never imports it and shares no code
with it; the only common module is rdr_inputs (seeded input generators, no
arithmetic of the method).

What it computes (PAPER.md = P, line numbers):
  * the paper's reference basis: doubly-orthogonal bubble eigenbases
    (Eq. 3.8/3.9), the dofs of §3.4.1/§3.4.2 and the
    Ciarlet dual basis, in x87 extended precision (DESIGN.md R-A24);
  * the global operator A_ij = sum_T int_T beta phi_i.phi_j + alpha d phi_i.d phi_j
    (Eq. 2.9) assembled BY PHYSICAL QUADRATURE into a scipy CSR
    matrix (not by the reference-matrix contraction the GPU path uses);
  * the one-level additive preconditioner J(X_I) + sum of star patches
    (Eq. 5.4, Eq. 5.12) with dense Cholesky patch solves;
  * textbook PCG with the DESIGN.md stopping rule.
Every function is pinned by tests/test_oracle_*.py (-m "not gpu").
"""
