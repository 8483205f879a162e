"""B200-native PCG for the high-order H(grad)/H(curl) Riesz maps in the basis of
arXiv 2506.17406 (C-ABI library librdr.so + thin ctypes binding).

    from paper_2506_17406_b200 import rdr
    S = rdr.Solver(vertices, tets, p, rdr.HGRAD, alpha, beta, mask)
    y = S.apply(x); z = S.precond(r); x, iters = S.solve(b, rtol=1e-8)
"""
