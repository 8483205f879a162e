"""C-ABI library checks that need no GPU: it loads, exports every symbol that
include/rdr.h declares, and its HOST-side reference element (DESIGN.md R-A24,
built independently in C++) agrees with the oracle's and with the paper's
closed forms."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2506_17406_b200", "librdr.so")


def _lib():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return ctypes.CDLL(LIB)


def test_library_exports_every_declared_symbol():
    lib = _lib()
    hdr = open(os.path.join(ROOT, "include", "rdr.h")).read()
    names = set(re.findall(r"\b(rdr_[a-z_]+)\s*\(", hdr))
    assert {"rdr_setup", "rdr_apply", "rdr_precond", "rdr_solve", "rdr_destroy"} <= names
    for n in names:
        assert hasattr(lib, n), n


def test_strerror_and_argument_errors():
    from paper_2506_17406_b200 import rdr
    lib = rdr._lib
    assert lib.rdr_strerror(0) == b"ok"
    assert b"SPD" in lib.rdr_strerror(-3)
    h = ctypes.c_void_p()
    # NULL pointers and bad p/space are rejected before any device work
    assert lib.rdr_setup(ctypes.byref(h), None, 8, None, 1, 3, 0, None, None, None, None) == -1
    n, m = ctypes.c_int32(), ctypes.c_int32()
    assert lib.rdr_reference_matrices(0, 13, None, ctypes.byref(n), ctypes.byref(m)) == -1
    assert lib.rdr_reference_matrices(1, 11, None, ctypes.byref(n), ctypes.byref(m)) == -1
    assert lib.rdr_reference_matrices(3, 3, None, ctypes.byref(n), ctypes.byref(m)) == -1
    assert lib.rdr_reference_matrices(2, 11, None, ctypes.byref(n), ctypes.byref(m)) == -1


@pytest.mark.parametrize("kind,l,p,lams", [
    (0, 1, 3, [2 / 5, 2 / 21]), (0, 2, 3, [1 / 14]), (0, 3, 4, [4 / 165]),
    (1, 2, 2, [2 / 9, 2 / 9]), (1, 3, 3, [7 / 144] * 3),
])
def test_library_eigenvalues_closed_forms(kind, l, p, lams):
    from paper_2506_17406_b200 import rdr
    assert np.allclose(rdr.bubble_eigenvalues(kind, l, p), lams, rtol=1e-14)


@pytest.mark.parametrize("p", [2, 3, 4])
def test_library_rt_bubble_eigenvalues_match_oracle(p):
    from paper_2506_17406_b200 import rdr
    from oracle.refelem import rt_bubbles
    assert np.allclose(rdr.bubble_eigenvalues(2, 3, p), rt_bubbles(p).lam.astype(float), rtol=1e-14, atol=0)


@pytest.mark.parametrize("space,p", [(0, 1), (0, 2), (0, 3), (0, 4), (0, 6), (1, 1), (1, 2), (1, 3), (1, 4),
                                     (2, 1), (2, 2), (2, 3), (2, 4), (2, 5)])
def test_library_reference_matrices_match_oracle(space, p):
    """The C++ reference element (pivoted Cholesky + Jacobi + Gauss-Jordan) and the
    oracle's (Gram eigendecomposition + Ogita-Aishima + GEPP) agree to rounding."""
    from paper_2506_17406_b200 import rdr
    from oracle.refelem import element, reference_matrices
    R = rdr.reference_matrices(space, p)
    M, K = reference_matrices(element(("hgrad", "hcurl", "hdiv")[space], p))
    M, K = M.astype(float), K.astype(float)
    if space == 2:  # RT_p: 2-form proxy mass x6 + div-div (NEXT-2)
        ref = [M[0, 0], M[1, 1], M[2, 2], M[0, 1] + M[1, 0], M[0, 2] + M[2, 0], M[1, 2] + M[2, 1], K]
    elif space == 0:
        ref = [M, K[0, 0], K[1, 1], K[2, 2], K[0, 1] + K[1, 0], K[0, 2] + K[2, 0], K[1, 2] + K[2, 1]]
    else:
        ref = [M[0, 0], M[1, 1], M[2, 2], M[0, 1] + M[1, 0], M[0, 2] + M[2, 0], M[1, 2] + M[2, 1],
               K[0, 0], K[1, 1], K[2, 2], K[0, 1] + K[1, 0], K[0, 2] + K[2, 0], K[1, 2] + K[2, 1]]
    assert R.shape[0] == len(ref)
    scale = max(np.abs(r).max() for r in ref)
    for s, r in enumerate(ref):
        assert np.abs(R[s] - r).max() <= 1e-14 * scale, s


@pytest.mark.parametrize("n", [1, 3, 17, 64, 130, 301])
def test_host_spd_inverse(n):
    """The setup's blocked AVX2 SPD inverse (patch inverses, R-A15) against
    numpy, on matrices conditioned like the patch matrices (kappa ~1e4)."""
    from paper_2506_17406_b200 import rdr
    rng = np.random.default_rng(n)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = (Q * np.logspace(0, 4, n)) @ Q.T
    A = 0.5 * (A + A.T)
    B = np.ascontiguousarray(A.copy())
    assert rdr._lib.rdr_spd_inverse(ctypes.c_void_p(B.ctypes.data), n) == 0
    ref = np.linalg.inv(A)
    assert np.abs(B - ref).max() <= 1e-10 * np.abs(ref).max()
    assert np.array_equal(B, B.T)
    C = -np.eye(3)
    assert rdr._lib.rdr_spd_inverse(ctypes.c_void_p(C.ctypes.data), 3) == -3


def _refmats_in_subprocess(tmp_path, space, p, tag):
    import subprocess
    import sys
    out = tmp_path / f"{tag}.npy"
    code = ("import numpy as np; from paper_2506_17406_b200 import rdr; "
            f"np.save(r'{out}', rdr.reference_matrices({space}, {p}))")
    env = dict(os.environ, RDR_CACHE_DIR=str(tmp_path))
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=ROOT)
    return np.load(out)


def _fnv1a(b: bytes) -> int:
    h = 1469598103934665603
    for c in b:
        h = ((h ^ c) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def test_reference_element_disk_cache(tmp_path):
    """SURVEY NEXT-4 on-disk reference-element cache (RDR_CACHE_DIR): the first
    process writes the file, later ones read it (proved by planting a valid
    file with one altered entry), and a file that fails its checksum is
    ignored and rebuilt."""
    import struct
    R0 = _refmats_in_subprocess(tmp_path, 1, 3, "a")
    f = tmp_path / "refelem_s1_p3.bin"
    assert f.exists()
    R1 = _refmats_in_subprocess(tmp_path, 1, 3, "b")
    assert np.array_equal(R0, R1)
    # plant: same file with R[0][0][0] += 1 and a recomputed checksum -> the loader must return it
    b = bytearray(f.read_bytes()[:-8])
    n = struct.unpack_from("<i", b, 16)[0]
    r_at = 8 + 16 + 8 + 16 * n + 8
    v = struct.unpack_from("<d", b, r_at)[0]
    assert v == R0[0, 0, 0]
    struct.pack_into("<d", b, r_at, v + 1.0)
    f.write_bytes(bytes(b) + struct.pack("<Q", _fnv1a(bytes(b))))
    R2 = _refmats_in_subprocess(tmp_path, 1, 3, "c")
    assert R2[0, 0, 0] == v + 1.0 and np.array_equal(R2.ravel()[1:], R0.ravel()[1:])
    # corrupt one byte without fixing the checksum -> rebuilt from scratch and rewritten
    b = bytearray(f.read_bytes())
    b[r_at + 3] ^= 0xFF
    f.write_bytes(bytes(b))
    R3 = _refmats_in_subprocess(tmp_path, 1, 3, "d")
    assert np.array_equal(R3, R0)
    assert _refmats_in_subprocess(tmp_path, 1, 3, "e").tobytes() == R0.tobytes()
