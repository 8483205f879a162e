"""Thin ctypes binding of librdr.so (include/rdr.h). Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels. There is no
CPU fallback: if the extension is missing, importing this module fails."""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librdr.so")

HGRAD, HCURL, HDIV = 0, 1, 2
SPLIT, UNSPLIT = 0, 1
ADDITIVE, HYBRID = 0, 1
SETUP_DEVICE, SETUP_HOST = 0, 1
LOOP_DEVICE, LOOP_HOST, LOOP_EAGER, LOOP_GRAPH, LOOP_PERSISTENT = 0, 1, 2, 3, 4
RDR_OK, RDR_ENOCONV = 0, -6


class RdrError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        super().__init__(f"{what}: {_lib.rdr_strerror(code).decode()} ({code})")


class Options(ctypes.Structure):
    _fields_ = [("decomposition", ctypes.c_int), ("preconditioner", ctypes.c_int), ("setup", ctypes.c_int),
                ("loop", ctypes.c_int)]


class SolveStats(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("converged", ctypes.c_int32), ("z0", ctypes.c_double),
                ("z_last", ctypes.c_double), ("launches", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Info(ctypes.Structure):
    _fields_ = [("n_total", ctypes.c_int64), ("n_free", ctypes.c_int64), ("n_interior", ctypes.c_int64),
                ("n_cells", ctypes.c_int64), ("n_loc", ctypes.c_int32), ("n_mat", ctypes.c_int32),
                ("n_patches", ctypes.c_int64), ("max_patch", ctypes.c_int32), ("patch_bytes", ctypes.c_int64),
                ("flops_apply", ctypes.c_double), ("bytes_apply", ctypes.c_double),
                ("bytes_precond", ctypes.c_double), ("setup_seconds", ctypes.c_double),
                ("refelem_seconds", ctypes.c_double), ("patch_setup_seconds", ctypes.c_double),
                ("patch_kernel_seconds", ctypes.c_double), ("patch_setup_flops", ctypes.c_double),
                ("apply_variant", ctypes.c_int32), ("apply_grid", ctypes.c_int32),
                ("persistent_loop", ctypes.c_int32), ("apply_slots", ctypes.c_int32),
                ("small_patch_grid", ctypes.c_int32), ("apply_factored", ctypes.c_int32),
                ("apply_fact_split_a", ctypes.c_int32), ("apply_fact_split_b", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2506_17406_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    sig = {
        "rdr_setup": (ctypes.c_int, [ctypes.POINTER(P), P, I64, P, I64, ctypes.c_int, ctypes.c_int, P, P, P, P]),
        "rdr_setup_ex": (ctypes.c_int, [ctypes.POINTER(P), P, I64, P, I64, ctypes.c_int, ctypes.c_int, P, P, P,
                                        ctypes.POINTER(Options), P]),
        "rdr_ndofs": (ctypes.c_int, [P, ctypes.POINTER(I64)]),
        "rdr_get_weights": (ctypes.c_int, [P, P]),
        "rdr_get_info": (ctypes.c_int, [P, ctypes.POINTER(Info)]),
        "rdr_apply": (ctypes.c_int, [P, P, P, P]),
        "rdr_precond": (ctypes.c_int, [P, P, P, P]),
        "rdr_solve": (ctypes.c_int, [P, P, P, D, ctypes.c_int, ctypes.POINTER(ctypes.c_int), P]),
        "rdr_solve_host": (ctypes.c_int, [P, P, P, D, ctypes.c_int, ctypes.POINTER(ctypes.c_int), P]),
        "rdr_last_launches": (ctypes.c_int, [P, ctypes.POINTER(I64)]),
        "rdr_last_solve": (ctypes.c_int, [P, ctypes.POINTER(SolveStats)]),
        "rdr_profile_solve": (ctypes.c_int, [P, P, D, ctypes.c_int, ctypes.POINTER(ctypes.c_int), P, P]),
        "rdr_time_kernels": (ctypes.c_int, [P, P, P, P, P, ctypes.c_int, P, P]),
        "rdr_measure_fp64_peak": (ctypes.c_int, [ctypes.POINTER(D), P]),
        "rdr_debug_fused_apply": (ctypes.c_int, [P, P, P, P]),
        "rdr_debug_profile_clocks": (ctypes.c_int, [P, P, ctypes.c_int, P, P]),
        "rdr_debug_set_apply_variant": (ctypes.c_int, [P, ctypes.c_int]),
        "rdr_debug_set_small_patch_kernel": (ctypes.c_int, [P, ctypes.c_int]),
        "rdr_debug_set_apply_config": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
        "rdr_destroy": (None, [P]),
        "rdr_strerror": (ctypes.c_char_p, [ctypes.c_int]),
        "rdr_reference_matrices": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, P, ctypes.POINTER(I32),
                                                  ctypes.POINTER(I32)]),
        "rdr_spd_inverse": (ctypes.c_int, [P, I32]),
        "rdr_bubble_eigenvalues": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, P,
                                                  ctypes.POINTER(I32)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def _ptr(a):
    """Raw address of a torch tensor or numpy array (contiguous)."""
    if hasattr(a, "data_ptr"):
        assert a.is_contiguous()
        return ctypes.c_void_p(a.data_ptr())
    assert a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data)


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _check(code, what):
    if code != RDR_OK:
        raise RdrError(code, what)


def reference_matrices(space: int, p: int) -> np.ndarray:
    """[n_mat, n_loc, n_loc] FP64 reference matrices (host-only entry point)."""
    n, m = ctypes.c_int32(), ctypes.c_int32()
    _check(_lib.rdr_reference_matrices(space, p, None, ctypes.byref(n), ctypes.byref(m)), "rdr_reference_matrices")
    out = np.zeros((m.value, n.value, n.value))
    _check(_lib.rdr_reference_matrices(space, p, _ptr(out), ctypes.byref(n), ctypes.byref(m)),
           "rdr_reference_matrices")
    return out


def bubble_eigenvalues(kind: int, l: int, p: int) -> np.ndarray:
    n = ctypes.c_int32()
    _check(_lib.rdr_bubble_eigenvalues(kind, l, p, None, ctypes.byref(n)), "rdr_bubble_eigenvalues")
    out = np.zeros(n.value)
    _check(_lib.rdr_bubble_eigenvalues(kind, l, p, _ptr(out), ctypes.byref(n)), "rdr_bubble_eigenvalues")
    return out


def measure_fp64_peak(stream=None) -> float:
    """FP64 tensor-core (DMMA) TFLOP/s of an issue-bound loop (roofline denominator)."""
    t = ctypes.c_double()
    _check(_lib.rdr_measure_fp64_peak(ctypes.byref(t), _stream(stream)), "rdr_measure_fp64_peak")
    return t.value


class Solver:
    """rdr.Solver(vertices, tets, p, space, alpha, beta, mask): torch CUDA tensors
    (float64 / int32 / uint8) or host numpy arrays; vectors are torch float64
    CUDA tensors of length n_total."""

    def __init__(self, vertices, tets, p, space, alpha, beta, mask, stream=None, decomposition=SPLIT,
                 preconditioner=ADDITIVE, setup=SETUP_DEVICE, loop=LOOP_DEVICE):
        import torch
        self._keep = [np.ascontiguousarray(vertices, dtype=np.float64) if isinstance(vertices, np.ndarray) else vertices,
                      np.ascontiguousarray(tets, dtype=np.int32) if isinstance(tets, np.ndarray) else tets,
                      np.ascontiguousarray(alpha, dtype=np.float64) if isinstance(alpha, np.ndarray) else alpha,
                      np.ascontiguousarray(beta, dtype=np.float64) if isinstance(beta, np.ndarray) else beta,
                      np.ascontiguousarray(mask, dtype=np.uint8) if isinstance(mask, np.ndarray) else mask]
        v, t, a, b, m = self._keep
        self._h = ctypes.c_void_p()
        nv, nt = v.shape[0], t.shape[0]
        opt = Options(int(decomposition), int(preconditioner), int(setup), int(loop))
        _check(_lib.rdr_setup_ex(ctypes.byref(self._h), _ptr(v), nv, _ptr(t), nt, int(p), int(space), _ptr(a),
                                 _ptr(b), _ptr(m), ctypes.byref(opt), _stream(stream)), "rdr_setup_ex")
        self._keep = None
        n = ctypes.c_int64()
        _check(_lib.rdr_ndofs(self._h, ctypes.byref(n)), "rdr_ndofs")
        self.n_total = n.value
        self.p, self.space = p, space
        self.device = torch.device("cuda", torch.cuda.current_device())

    @property
    def weights(self):
        """Hybrid Schwarz weights (rho_1, rho_2, rho_3)."""
        w = np.zeros(3)
        _check(_lib.rdr_get_weights(self._h, _ptr(w)), "rdr_get_weights")
        return w

    @property
    def info(self) -> dict:
        i = Info()
        _check(_lib.rdr_get_info(self._h, ctypes.byref(i)), "rdr_get_info")
        return i.as_dict()

    def _vec(self, v):
        import torch
        return torch.empty(self.n_total, dtype=torch.float64, device=self.device) if v is None else v

    def apply(self, x, y=None, stream=None):
        y = self._vec(y)
        _check(_lib.rdr_apply(self._h, _ptr(x), _ptr(y), _stream(stream)), "rdr_apply")
        return y

    def precond(self, r, z=None, stream=None):
        z = self._vec(z)
        _check(_lib.rdr_precond(self._h, _ptr(r), _ptr(z), _stream(stream)), "rdr_precond")
        return z

    def solve(self, b, x=None, rtol=1e-8, maxit=10000, stream=None):
        """PCG from x0 = 0; returns (x, iters). Raises RdrError on failure,
        except non-convergence which returns iters == maxit and sets .converged False."""
        x = self._vec(x)
        it = ctypes.c_int()
        code = _lib.rdr_solve(self._h, _ptr(b), _ptr(x), float(rtol), int(maxit), ctypes.byref(it), _stream(stream))
        if code not in (RDR_OK, RDR_ENOCONV):
            _check(code, "rdr_solve")
        self.converged = code == RDR_OK
        return x, it.value

    def solve_host(self, b_host, x_host, rtol=1e-8, maxit=10000, stream=None):
        """End-to-end path: host b -> device -> PCG -> host x (copies inside)."""
        it = ctypes.c_int()
        code = _lib.rdr_solve_host(self._h, _ptr(b_host), _ptr(x_host), float(rtol), int(maxit), ctypes.byref(it),
                                   _stream(stream))
        if code not in (RDR_OK, RDR_ENOCONV):
            _check(code, "rdr_solve_host")
        self.converged = code == RDR_OK
        return it.value

    def time_kernels(self, x, r, reps=20, stream=None):
        """Average device ms per launch: (apply, jacobi, patches, fused PCG-mode apply)."""
        y, z = self._vec(None), self._vec(None)
        ms = np.zeros(4)
        _check(_lib.rdr_time_kernels(self._h, _ptr(x), _ptr(y), _ptr(r), _ptr(z), int(reps), _ptr(ms),
                                     _stream(stream)), "rdr_time_kernels")
        return ms

    def debug_fused_apply(self, z, q, stream=None):
        """q = A z through the fused PCG variant of the apply kernel (debugging)."""
        _check(_lib.rdr_debug_fused_apply(self._h, _ptr(z), _ptr(q), _stream(stream)), "rdr_debug_fused_apply")
        return q

    def last_stats(self) -> dict:
        """iters, converged, ||z_0||, ||z_k|| at the last stopping test, launches of the last solve."""
        st = SolveStats()
        _check(_lib.rdr_last_solve(self._h, ctypes.byref(st)), "rdr_last_solve")
        return st.as_dict()

    def profile_solve(self, b, rtol=1e-8, maxit=10000, stream=None):
        """Eager PCG solve with CUDA events between kernel groups: (iters, ms per
        iteration of [apply, update + Jacobi, patches, 0])."""
        it = ctypes.c_int()
        ms = np.zeros(4)
        code = _lib.rdr_profile_solve(self._h, _ptr(b), float(rtol), int(maxit), ctypes.byref(it), _ptr(ms),
                                      _stream(stream))
        if code not in (RDR_OK, RDR_ENOCONV):
            _check(code, "rdr_profile_solve")
        self.converged = code == RDR_OK
        return it.value, ms

    def profile_clocks(self, b, iters=20, stream=None):
        """[SM MHz behind the fused apply in the PCG iteration, the same for the apply alone,
        ms per iteration, ms per apply alone] (rdr_debug_profile_clocks)."""
        out = np.zeros(4)
        _check(_lib.rdr_debug_profile_clocks(self._h, _ptr(b), int(iters), _ptr(out), _stream(stream)),
               "rdr_debug_profile_clocks")
        return out

    def set_apply_variant(self, variant: int) -> bool:
        """Debugging: force the apply's warp layout; False if it does not fit this operator."""
        return _lib.rdr_debug_set_apply_variant(self._h, int(variant)) == RDR_OK

    def set_apply_config(self, variant: int, slots: int, grid: int = 0) -> bool:
        """Debugging: force the apply's layout, ring depth and grid (rdr_info's
        apply_variant, apply_slots, apply_grid); False if it does not fit."""
        return _lib.rdr_debug_set_apply_config(self._h, int(variant), int(slots), int(grid)) == RDR_OK

    def set_small_patch_kernel(self, persistent: bool) -> bool:
        """Debugging: force the small-patch kernel (one warp per patch, or resident warps
        walking the patches); False if the configuration has no small-patch launch."""
        return _lib.rdr_debug_set_small_patch_kernel(self._h, int(bool(persistent))) == RDR_OK

    def last_launches(self) -> int:
        n = ctypes.c_int64()
        _check(_lib.rdr_last_launches(self._h, ctypes.byref(n)), "rdr_last_launches")
        return n.value

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.rdr_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
