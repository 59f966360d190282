"""Thin Python binding of include/seaice.h (ctypes; argument marshalling only).

Every step of the path runs in libseaice_b200.so's CUDA kernels.  PyTorch provides
device memory (the caching allocator is handed to the library as its alloc/free
callbacks), the stream, and tensors for inputs/outputs.  There is no CPU fallback:
if the shared library is missing or no CUDA device is present, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import torch

from . import build as _build

HERE = os.path.dirname(os.path.abspath(__file__))
HEADER = os.path.join(os.path.dirname(HERE), "include", "seaice.h")

OK, NOT_CONVERGED, EINVAL, ENOMEM, ECUDA, ENONFINITE, ESTATE = 0, 1, -1, -2, -3, -4, -5
JAC = {"sv": 0, "std": 1, "picard": 2}
PC = {"amg": 0, "jacobi": 1, "none": 2}


class Params(C.Structure):
    _fields_ = [("n", C.c_int32), ("L", C.c_double),
                ("rho_i", C.c_double), ("rho_a", C.c_double), ("rho_o", C.c_double), ("C_a", C.c_double),
                ("C_o", C.c_double), ("P_star", C.c_double), ("C", C.c_double), ("e", C.c_double),
                ("delta_min", C.c_double), ("f_c", C.c_double),
                ("jacobian", C.c_int32), ("newton_rtol", C.c_double), ("newton_maxit", C.c_int32),
                ("ls_max_halvings", C.c_int32), ("krylov_rtol", C.c_double), ("restart", C.c_int32),
                ("krylov_maxit", C.c_int32), ("precond", C.c_int32), ("amg_theta", C.c_double),
                ("cheb_degree", C.c_int32), ("coarse_max_dof", C.c_int32), ("max_levels", C.c_int32),
                ("cheb_lower", C.c_double), ("cheb_upper", C.c_double), ("power_iters", C.c_int32),
                ("project_pi", C.c_int32), ("amg_seed", C.c_uint64), ("agg_dist0", C.c_int32),
                ("agg_dist", C.c_int32), ("cheb_fused", C.c_int32),
                ("cheb_degree0", C.c_int32), ("matfree", C.c_int32),
                ("krylov_forcing", C.c_int32), ("nullspace_dim", C.c_int32), ("krylov_method", C.c_int32),
                ("spgemm_path", C.c_int32), ("amg_lag", C.c_int32), ("amg_reuse", C.c_int32),
                ("vcycle_tail", C.c_int32)]


ALLOC_T = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_T = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_void_p)


class Runtime(C.Structure):
    _fields_ = [("stream", C.c_void_p), ("alloc", ALLOC_T), ("free", FREE_T), ("user", C.c_void_p)]


class CSR(C.Structure):
    _fields_ = [("nrows", C.c_int32), ("ncols", C.c_int32), ("nnz", C.c_int64), ("row_ptr", C.c_void_p),
                ("col_idx", C.c_void_p), ("val", C.c_void_p)]


class BSR(C.Structure):
    _fields_ = [("nbrows", C.c_int32), ("nbcols", C.c_int32), ("br", C.c_int32), ("bc", C.c_int32),
                ("nnzb", C.c_int64), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("val", C.c_void_p)]


class KrylovStats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("restarts", C.c_int32), ("converged", C.c_int32),
                ("relres_est", C.c_double), ("relres_true", C.c_double)]


class NewtonStats(C.Structure):
    _fields_ = [("converged_on_entry", C.c_int32), ("res_norm", C.c_double), ("res_norm0", C.c_double),
                ("alpha", C.c_double), ("dphi", C.c_double), ("halvings", C.c_int32), ("ls_stagnated", C.c_int32),
                ("krylov", KrylovStats), ("amg_levels", C.c_int32), ("amg_op_complexity", C.c_double),
                ("t_assemble", C.c_double), ("t_amg", C.c_double), ("t_krylov", C.c_double), ("t_ls", C.c_double),
                ("amg_rebuilt", C.c_int32), ("amg_reused", C.c_int32)]


class StepStats(C.Structure):
    _fields_ = [("newton_iters", C.c_int32), ("converged", C.c_int32), ("krylov_iters_total", C.c_int32),
                ("res_norm0", C.c_double), ("res_norm_final", C.c_double), ("seconds", C.c_double),
                ("t_assemble", C.c_double), ("t_amg", C.c_double), ("t_krylov", C.c_double), ("t_ls", C.c_double),
                ("t_setup", C.c_double), ("krylov_solves", C.c_int32), ("krylov_capped", C.c_int32),
                ("krylov_max_iters", C.c_int32), ("amg_setups", C.c_int32), ("amg_reuses", C.c_int32)]


def struct_dict(s):
    out = {}
    for name, _ in s._fields_:
        v = getattr(s, name)
        out[name] = struct_dict(v) if isinstance(v, C.Structure) else v
    return out


_LIB = None
_LIVE = __import__("weakref").WeakSet()


def _close_all():
    for ctx in list(_LIVE):
        try:
            ctx.close()
        except Exception:
            pass


__import__("atexit").register(_close_all)


def header_functions():
    """Names of every function the public header declares."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*|int64_t)\s+(seaice_\w+)\s*\(", txt, re.M)))


def lib(build_if_missing: bool = True):
    global _LIB
    if _LIB is None:
        path = _build.LIB
        if build_if_missing and _build.needs_build():
            _build.build()
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(path)
        P, VP, I32, D = C.POINTER, C.c_void_p, C.c_int32, C.c_double
        sig = {
            "seaice_default_params": (None, [P(Params), I32]),
            "seaice_create": (C.c_int, [P(Params), P(Runtime), P(VP)]),
            "seaice_destroy": (C.c_int, [VP]),
            "seaice_last_error": (C.c_char_p, [VP]),
            "seaice_set_step": (C.c_int, [VP, D, D, VP, VP, VP, VP, VP, VP]),
            "seaice_residual": (C.c_int, [VP, VP, VP, P(D)]),
            "seaice_assemble_jacobian": (C.c_int, [VP, VP, VP, P(CSR)]),
            "seaice_spmv": (C.c_int, [VP, VP, VP]),
            "seaice_transport": (C.c_int, [VP, D, VP, VP, VP, D, D, VP, VP, P(D), P(I32)]),
            "seaice_jv_matfree": (C.c_int, [VP, VP, VP, VP, VP]),
            "seaice_amg_setup": (C.c_int, [VP, P(I32), P(D)]),
            "seaice_amg_level": (C.c_int, [VP, I32, P(BSR), P(BSR), VP]),
            "seaice_precond_apply": (C.c_int, [VP, VP, VP]),
            "seaice_fgmres_solve": (C.c_int, [VP, VP, VP, P(KrylovStats)]),
            "seaice_delta_energy": (C.c_int, [VP, VP, VP, P(D), I32, P(D)]),
            "seaice_pi_tilde": (C.c_int, [VP, VP, VP, VP, VP]),
            "seaice_get_pi": (C.c_int, [VP, VP]),
            "seaice_set_pi": (C.c_int, [VP, VP]),
            "seaice_newton_step": (C.c_int, [VP, VP, VP, P(NewtonStats)]),
            "seaice_solve_step": (C.c_int, [VP, D, D, VP, VP, VP, VP, VP, VP, P(StepStats)]),
            "seaice_solve_step_host": (C.c_int, [VP, D, D, VP, VP, VP, VP, VP, VP, P(StepStats)]),
            "seaice_launch_count": (C.c_int64, [VP]),
            "seaice_profile_enable": (C.c_int, [VP, I32]),
            "seaice_profile_read": (C.c_int, [VP, P(D), P(C.c_int64), P(D)]),
            "seaice_memory": (C.c_int, [VP, P(C.c_int64), P(C.c_int64)]),
            "seaice_spgemm_path_hits": (C.c_int, [VP, P(C.c_int64), I32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


class SeaIceError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"seaice error {code}: {msg}")
        self.code = code


class _DevArray:
    """Zero-copy wrapper exposing a library-owned device buffer to torch.as_tensor."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None, "stream": None}


def _dev_tensor(ptr, n, typestr, device):
    if n == 0:
        return torch.empty(0, dtype=torch.float64 if typestr == "<f8" else torch.int32, device=device)
    return torch.as_tensor(_DevArray(ptr, (n,), typestr), device=device).clone()


def _ptr(t):
    if t is None:
        return None
    if not (t.is_cuda and t.is_contiguous()):
        raise ValueError("expected a contiguous CUDA tensor")
    return C.c_void_p(t.data_ptr())


class SeaIce:
    """One context of the B200 stress-velocity Newton-Krylov step (see include/seaice.h)."""

    def __init__(self, n: int, device=None, stream=None, use_torch_allocator: bool = True, **overrides):
        if not torch.cuda.is_available():
            raise RuntimeError("SeaIce needs a CUDA device (no CPU fallback)")
        self.L = lib()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.stream = stream or torch.cuda.current_stream(self.device)
        p = Params()
        self.L.seaice_default_params(C.byref(p), n)
        for k, v in overrides.items():
            if k == "jacobian" and isinstance(v, str):
                v = JAC[v]
            if k == "precond" and isinstance(v, str):
                v = PC[v]
            if not hasattr(p, k):
                raise KeyError(k)
            setattr(p, k, v)
        self.params = p
        self.n = n
        self.N = 2 * (n + 1) ** 2
        self.Nc = n * n
        rt = Runtime()
        rt.stream = C.c_void_p(self.stream.cuda_stream)
        self._live = {}
        if use_torch_allocator:
            dev = self.device.index
            strm = self.stream
            t_alloc = torch.cuda.caching_allocator_alloc
            t_free = torch.cuda.caching_allocator_delete

            def _alloc(size, stream, user):
                return t_alloc(int(size), dev, strm)

            def _free(ptr, stream, user):
                try:
                    t_free(ptr)
                except Exception:  # interpreter shutdown: torch already torn down
                    pass

            self._alloc_cb = ALLOC_T(_alloc)
            self._free_cb = FREE_T(_free)
            rt.alloc = self._alloc_cb
            rt.free = self._free_cb
        self._rt = rt
        h = C.c_void_p()
        rc = self.L.seaice_create(C.byref(p), C.byref(rt), C.byref(h))
        if rc != OK:
            raise SeaIceError(rc, "seaice_create failed (invalid parameters or device error)")
        self.h = h
        _LIVE.add(self)

    # -- plumbing --------------------------------------------------------------
    def _check(self, rc, allow_nc=False):
        if rc == OK or (allow_nc and rc == NOT_CONVERGED):
            return rc
        raise SeaIceError(rc, self.L.seaice_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.L.seaice_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def tensor(self, x, n=None):
        t = torch.as_tensor(x, dtype=torch.float64, device=self.device).contiguous()
        if n is not None and t.numel() != n:
            raise ValueError(f"expected {n} values, got {t.numel()}")
        return t

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64, device=self.device)

    @property
    def launches(self):
        return int(self.L.seaice_launch_count(self.h))

    PROF_NAMES = ["assemble", "spmv0", "cheb0", "cheb_coarse", "resid0", "multidot", "maxpy_norm", "maxpy",
                  "delta_energy", "transfer", "coarse_solve", "resid_coarse", "pi_update", "cheb0_fused", "transport",
                  "jv_matfree", "cheb_level1", "resid_level1", "transfer_level0", "vcycle_tail"]

    def profile(self, on: bool):
        self._check(self.L.seaice_profile_enable(self.h, 1 if on else 0))

    def profile_read(self):
        ms = (C.c_double * 24)()
        cnt = (C.c_int64 * 24)()
        by = (C.c_double * 24)()
        self._check(self.L.seaice_profile_read(self.h, ms, cnt, by))
        return {name: {"ms": ms[k], "launches": cnt[k], "bytes": by[k]} for k, name in enumerate(self.PROF_NAMES)}

    def spgemm_path_hits(self):
        """Counts of the SpGEMM code paths taken since create (seaice_spgemm_path_hits)."""
        h = (C.c_int64 * 7)()
        self._check(self.L.seaice_spgemm_path_hits(self.h, h, 7))
        return list(h)

    def memory(self):
        live, peak = C.c_int64(), C.c_int64()
        self.L.seaice_memory(self.h, C.byref(live), C.byref(peak))
        return live.value, peak.value

    # -- API ---------------------------------------------------------------------
    def set_step(self, dt, t_new, h, A, v_prev, v_air, v_ocean, load=None):
        self._in = [self.tensor(h, self.Nc), self.tensor(A, self.Nc), self.tensor(v_prev, self.N),
                    self.tensor(v_air, self.N), self.tensor(v_ocean, self.N)]
        ld = None if load is None else self.tensor(load, self.N)
        self._check(self.L.seaice_set_step(self.h, dt, t_new, *[_ptr(t) for t in self._in], _ptr(ld)))

    def set_inputs(self, inp):
        """Convenience: a workloads.StepInputs."""
        self.set_step(inp.dt, inp.t_new, inp.h, inp.A, inp.v_prev, inp.v_air, inp.v_ocean, inp.load)

    def residual(self, v):
        v = self.tensor(v, self.N)
        r = self.zeros(self.N)
        nrm = C.c_double()
        self._check(self.L.seaice_residual(self.h, _ptr(v), _ptr(r), C.byref(nrm)))
        return r, nrm.value

    def assemble_jacobian(self, v, pi=None, want_csr=True):
        v = self.tensor(v, self.N)
        pi = None if pi is None else self.tensor(pi, 12 * self.Nc)
        view = CSR()
        self._check(self.L.seaice_assemble_jacobian(self.h, _ptr(v), _ptr(pi), C.byref(view) if want_csr else None))
        if not want_csr:
            return None
        return (_dev_tensor(view.row_ptr, view.nrows + 1, "<i4", self.device),
                _dev_tensor(view.col_idx, view.nnz, "<i4", self.device),
                _dev_tensor(view.val, view.nnz, "<f8", self.device))

    def spmv(self, x):
        x = self.tensor(x, self.N)
        y = self.zeros(self.N)
        self._check(self.L.seaice_spmv(self.h, _ptr(x), _ptr(y)))
        return y

    def amg_setup(self):
        lv, oc = C.c_int32(), C.c_double()
        self._check(self.L.seaice_amg_setup(self.h, C.byref(lv), C.byref(oc)))
        return lv.value, oc.value

    def amg_level(self, level):
        A, P = BSR(), BSR()
        agg = None
        self._check(self.L.seaice_amg_level(self.h, level, C.byref(A), C.byref(P), None))

        def bsr(b):
            if b.nbrows == 0:
                return None
            return {"nbrows": b.nbrows, "nbcols": b.nbcols, "br": b.br, "bc": b.bc,
                    "row_ptr": _dev_tensor(b.row_ptr, b.nbrows + 1, "<i4", self.device),
                    "col_idx": _dev_tensor(b.col_idx, b.nnzb, "<i4", self.device),
                    "val": _dev_tensor(b.val, b.nnzb * b.br * b.bc, "<f8", self.device)}
        PA = bsr(P)
        if PA is not None:
            import numpy as np
            arr = np.zeros(A.nbrows, dtype=np.int32)
            self._check(self.L.seaice_amg_level(self.h, level, None, None, arr.ctypes.data_as(C.c_void_p)))
            agg = arr
        return bsr(A), PA, agg

    def precond_apply(self, r):
        r = self.tensor(r, self.N)
        z = self.zeros(self.N)
        self._check(self.L.seaice_precond_apply(self.h, _ptr(r), _ptr(z)))
        return z

    def fgmres(self, b):
        b = self.tensor(b, self.N)
        x = self.zeros(self.N)
        st = KrylovStats()
        rc = self._check(self.L.seaice_fgmres_solve(self.h, _ptr(b), _ptr(x), C.byref(st)), allow_nc=True)
        return x, struct_dict(st), rc

    def delta_energy(self, v, vt, alphas):
        v, vt = self.tensor(v, self.N), self.tensor(vt, self.N)
        a = (C.c_double * len(alphas))(*alphas)
        out = (C.c_double * len(alphas))()
        self._check(self.L.seaice_delta_energy(self.h, _ptr(v), _ptr(vt), a, len(alphas), out))
        return list(out)

    def pi_tilde(self, v, pi, vt):
        v, vt = self.tensor(v, self.N), self.tensor(vt, self.N)
        pi = None if pi is None else self.tensor(pi, 12 * self.Nc)
        out = self.zeros(12 * self.Nc)
        self._check(self.L.seaice_pi_tilde(self.h, _ptr(v), _ptr(pi), _ptr(vt), _ptr(out)))
        return out

    def get_pi(self):
        out = self.zeros(12 * self.Nc)
        self._check(self.L.seaice_get_pi(self.h, _ptr(out)))
        return out

    def set_pi(self, pi):
        pi = self.tensor(pi, 12 * self.Nc)
        self._check(self.L.seaice_set_pi(self.h, _ptr(pi)))

    def newton_step(self, v, pi=None):
        """v (and pi if given) are updated in place (CUDA tensors)."""
        st = NewtonStats()
        rc = self._check(self.L.seaice_newton_step(self.h, _ptr(v), _ptr(pi), C.byref(st)), allow_nc=True)
        d = struct_dict(st)
        d["rc"] = rc
        return d

    def solve_step(self, dt, t_new, h, A, v_prev, v_air, v_ocean, v_out=None):
        ins = [self.tensor(h, self.Nc), self.tensor(A, self.Nc), self.tensor(v_prev, self.N),
               self.tensor(v_air, self.N), self.tensor(v_ocean, self.N)]
        v_out = self.zeros(self.N) if v_out is None else v_out
        st = StepStats()
        rc = self._check(self.L.seaice_solve_step(self.h, dt, t_new, *[_ptr(t) for t in ins], _ptr(v_out),
                                                  C.byref(st)), allow_nc=True)
        d = struct_dict(st)
        d["rc"] = rc
        return v_out, d

    def jv_matfree(self, v, x, pi=None):
        """y = J(v, pi) x without storing J (seaice_jv_matfree)."""
        v, x = self.tensor(v, self.N), self.tensor(x, self.N)
        pi = None if pi is None else self.tensor(pi, 12 * self.Nc)
        y = self.zeros(self.N)
        self._check(self.L.seaice_jv_matfree(self.h, _ptr(v), _ptr(pi), _ptr(x), _ptr(y)))
        return y

    def transport(self, dt, v, A, h, A_in=1.0, h_in=0.0, info=False):
        """(A, h) advanced over dt by explicit upwind steps with velocity v (seaice_transport;
        sub-cycled when the CFL number exceeds 1).  info=True also returns (cfl, substeps)."""
        v, A, h = self.tensor(v, self.N), self.tensor(A, self.Nc), self.tensor(h, self.Nc)
        Ao, ho = self.zeros(self.Nc), self.zeros(self.Nc)
        cfl, m = C.c_double(), C.c_int32()
        self._check(self.L.seaice_transport(self.h, dt, _ptr(v), _ptr(A), _ptr(h), A_in, h_in, _ptr(Ao), _ptr(ho),
                                            C.byref(cfl), C.byref(m)))
        return (Ao, ho, cfl.value, m.value) if info else (Ao, ho)

    def solve_step_host(self, dt, t_new, h, A, v_prev, v_air, v_ocean, v_out):
        """Host (CPU, ideally pinned) torch tensors in and out: the end-to-end call."""
        for t in (h, A, v_prev, v_air, v_ocean, v_out):
            if t.is_cuda or not t.is_contiguous() or t.dtype != torch.float64:
                raise ValueError("solve_step_host expects contiguous float64 CPU tensors")
        st = StepStats()
        ptrs = [C.c_void_p(t.data_ptr()) for t in (h, A, v_prev, v_air, v_ocean, v_out)]
        rc = self._check(self.L.seaice_solve_step_host(self.h, dt, t_new, *ptrs, C.byref(st)), allow_nc=True)
        d = struct_dict(st)
        d["rc"] = rc
        return d
