"""paper_2508_01864_b200 -- B200-native exact fast Matern kernel MVM (arXiv 2508.01864).

Thin ctypes binding over ``libgpmatern.so`` (include/gpmatern.h).  This module only
marshals arguments: device memory and streams come from PyTorch, every step of the
method runs in the library's sm_100a kernels.  There is no CPU fallback: if the
library or a CUDA device is missing, every call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

__all__ = [
    "load_library", "Kernel", "Plan", "Cross", "Precond", "GPError", "setup", "kmvm", "cg_solve", "fit", "use_torch_allocator",
    "predict", "FORM_L1", "FORM_PRODUCT", "MEAN_NONE", "MEAN_AFFINE", "MEAN_BASIS",
    "LIB_PATH",
]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgpmatern.so")
FORM_L1, FORM_PRODUCT = 0, 1
MEAN_NONE, MEAN_AFFINE, MEAN_BASIS = 0, 1, 2
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "UNSUPPORTED", 3: "NONFINITE", 4: "RANGE",
          5: "NOT_CONVERGED", 6: "BREAKDOWN", 7: "CUDA", 8: "OOM"}

_lib = None


class GPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"gpmatern {STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class _Kernel(ctypes.Structure):
    _fields_ = [("two_nu", ctypes.c_int), ("form", ctypes.c_int),
                ("outputscale", ctypes.c_double), ("lengthscale", ctypes.c_double * 3)]


class _CGInfo(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int), ("relres_max", ctypes.c_double),
                ("failed_column", ctypes.c_int), ("restarts", ctypes.c_int)]


class _FitOpts(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("max_steps", ctypes.c_int),
                ("max_outer", ctypes.c_int), ("grad_tol", ctypes.c_double),
                ("beta_tol", ctypes.c_double), ("lanczos_iters", ctypes.c_int),
                ("precond_rank", ctypes.c_int), ("cg_rtol", ctypes.c_double)]


class _FitResult(ctypes.Structure):
    _fields_ = [("kernel", _Kernel), ("sigma", ctypes.c_double), ("beta", ctypes.c_double * 4),
                ("steps", ctypes.c_int), ("outer", ctypes.c_int), ("lml", ctypes.c_double),
                ("grad_norm", ctypes.c_double)]


class _LmlResult(ctypes.Structure):
    _fields_ = [("lml", ctypes.c_double), ("quad", ctypes.c_double),
                ("logdet", ctypes.c_double), ("logdet_precond", ctypes.c_double),
                ("grad", ctypes.c_double * 3), ("cg_iters", ctypes.c_int),
                ("lanczos_iters", ctypes.c_int)]


def load_library(path: str | None = None):
    """Load libgpmatern.so (built in-tree by build.py).  Raises if missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("GPM_LIB") or LIB_PATH   # GPM_LIB: an experiment build (build.py)
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `python -m paper_2508_01864_b200.build` "
                                f"(no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    vp, i64, ci, cd = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    sig = {
        "gp_setup": [vp, i64, ci, ctypes.POINTER(_Kernel), vp, ctypes.POINTER(vp)],
        "gp_kmvm": [vp, vp, ci, vp, vp],
        "gp_kmvm_host": [vp, vp, ci, vp, vp],
        "gp_kmvm_rank": [vp, vp, ci, vp, vp],
        "gp_kmvm_partial": [vp, vp, ci, vp, ci, ci, vp],
        "gp_shard_ranges": [i64, ci, ci, ci, ctypes.POINTER(i64)],
        "gp_kmvm_dlengthscale": [vp, vp, ci, vp, ci, vp],
        "gp_permute": [vp, vp, ci, vp, ci, vp],
        "gp_kzx_setup": [vp, vp, i64, vp, ctypes.POINTER(vp)],
        "gp_kzx": [vp, vp, ci, vp, vp],
        "gp_cg_solve": [vp, cd, vp, ci, vp, ci, cd, ci, vp, vp, ctypes.POINTER(_CGInfo), vp],
        "gp_cg_solve_pc": [vp, vp, cd, vp, ci, vp, ci, cd, ci, vp, vp, ctypes.POINTER(_CGInfo),
                           vp],
        "gp_cg_solve_ex": [vp, vp, cd, vp, ci, vp, ci, cd, ci, vp, vp, vp, vp,
                           ctypes.POINTER(_CGInfo), vp],
        "gp_precond_create": [vp, ci, vp, ctypes.POINTER(vp)],
        "gp_precond_factor": [vp, vp, vp, vp],
        "gp_precond_solve": [vp, cd, vp, ci, vp, vp],
        "gp_precond_logdet": [vp, cd, ctypes.POINTER(cd), vp],
        "gp_mbcg": [vp, vp, cd, vp, ci, ci, cd, vp, vp, vp, vp, vp],
        "gp_lml": [vp, vp, cd, vp, vp, vp, ci, ci, cd, ctypes.POINTER(_LmlResult), vp],
        "gp_fit": [vp, i64, ci, ctypes.POINTER(_Kernel), cd, vp, vp, vp, ci,
                   ctypes.POINTER(_FitOpts), ctypes.POINTER(_FitResult), vp],
        "gp_predict": [vp, vp, i64, vp, vp, vp, ci, vp, vp],
        "gp_plan_query": [vp, ci, ctypes.POINTER(i64)],
        "gp_plan_set_option": [vp, ci, i64],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.gp_set_allocator.argtypes = [vp, vp, vp]; lib.gp_set_allocator.restype = ctypes.c_int
    lib.gp_destroy.argtypes = [vp]; lib.gp_destroy.restype = None
    lib.gp_kzx_destroy.argtypes = [vp]; lib.gp_kzx_destroy.restype = None
    lib.gp_precond_destroy.argtypes = [vp]; lib.gp_precond_destroy.restype = None
    lib.gp_last_error.argtypes = []; lib.gp_last_error.restype = ctypes.c_char_p
    lib.gp_version.argtypes = []; lib.gp_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _check(st: int):
    if st != 0:
        raise GPError(st, _lib.gp_last_error().decode())


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dev(t, name, shape=None):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise TypeError(f"{name} must be a CUDA float64 tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    return ctypes.c_void_p(t.data_ptr())


@dataclass(frozen=True)
class Kernel:
    """Matern kernel nu = two_nu/2 with outputscale s and per-dimension lengthscales."""
    two_nu: int = 3
    lengthscale: tuple = (1.0,)
    outputscale: float = 1.0
    form: int = FORM_L1

    def c(self) -> _Kernel:
        ell = list(self.lengthscale) + [1.0] * (3 - len(self.lengthscale))
        return _Kernel(self.two_nu, self.form, float(self.outputscale),
                       (ctypes.c_double * 3)(*[float(e) for e in ell[:3]]))


class Plan:
    """Stored structure of x (gp_setup); owns device memory until closed."""

    def __init__(self, x, kernel: Kernel, stream=None):
        lib = load_library()
        if x.dim() == 1:
            x = x.reshape(-1, 1)
        n, d = x.shape
        self.n, self.d, self.kernel = int(n), int(d), kernel
        self._x = x
        h = ctypes.c_void_p()
        k = kernel.c()
        _check(lib.gp_setup(_dev(x, "x"), n, d, ctypes.byref(k), _stream(stream), ctypes.byref(h)))
        self._h = h

    def query(self, what: int) -> int:
        v = ctypes.c_int64()
        _check(_lib.gp_plan_query(self._h, what, ctypes.byref(v)))
        return v.value

    @property
    def levels(self): return self.query(2)
    @property
    def struct_bytes(self): return self.query(3)
    @property
    def launches_per_apply(self): return self.query(4)
    @property
    def model_bytes(self): return self.query(5)
    @property
    def d1_path(self): return self.query(6)

    def set_option(self, option: int, value: int):
        _check(_lib.gp_plan_set_option(self._h, option, value))

    def kmvm(self, v, out=None, stream=None):
        """out = K v for v of shape (n,) or (nrhs, n) (each row one right-hand side)."""
        import torch
        nrhs = 1 if v.dim() == 1 else v.shape[0]
        if v.shape[-1] != self.n:
            raise ValueError("v has the wrong length")
        if out is None:
            out = torch.empty_like(v)
        _check(_lib.gp_kmvm(self._h, _dev(v, "v"), nrhs, _dev(out, "out", v.shape), _stream(stream)))
        return out

    def kmvm_rank(self, v_rank, out=None, stream=None):
        """out = K v with vectors in the plan's stored (x1-rank) order (CG operator)."""
        import torch
        nrhs = 1 if v_rank.dim() == 1 else v_rank.shape[0]
        if out is None:
            out = torch.empty_like(v_rank)
        _check(_lib.gp_kmvm_rank(self._h, _dev(v_rank, "v"), nrhs, _dev(out, "out", v_rank.shape),
                                 _stream(stream)))
        return out

    def kmvm_partial(self, v_rank, shard: int, nshards: int, out=None, stream=None):
        """Shard `shard` of `nshards` of K v_rank (rank order, d >= 2; gp_kmvm_partial): the
        shards' outputs sum to kmvm_rank(v_rank)."""
        import torch
        out = torch.empty_like(v_rank) if out is None else out
        nrhs = 1 if v_rank.dim() == 1 else v_rank.shape[0]
        _check(_lib.gp_kmvm_partial(self._h, _dev(v_rank, "v_rank"), nrhs, _dev(out, "out"),
                                    int(shard), int(nshards), _stream(stream)))
        return out

    def kmvm_dlengthscale(self, v, out=None, rank_order=False, stream=None):
        """out = (l dK/dl) v, all lengthscales scaled together (gp_kmvm_dlengthscale)."""
        import torch
        nrhs = 1 if v.dim() == 1 else v.shape[0]
        if v.shape[-1] != self.n:
            raise ValueError("v has the wrong length")
        if out is None:
            out = torch.empty_like(v)
        _check(_lib.gp_kmvm_dlengthscale(self._h, _dev(v, "v"), nrhs, _dev(out, "out", v.shape),
                                         1 if rank_order else 0, _stream(stream)))
        return out

    def to_rank(self, v, stream=None):
        import torch
        out = torch.empty_like(v)
        nrhs = 1 if v.dim() == 1 else v.shape[0]
        _check(_lib.gp_permute(self._h, _dev(v, "v"), nrhs, _dev(out, "out", v.shape), 1, _stream(stream)))
        return out

    def from_rank(self, v_rank, stream=None):
        import torch
        out = torch.empty_like(v_rank)
        nrhs = 1 if v_rank.dim() == 1 else v_rank.shape[0]
        _check(_lib.gp_permute(self._h, _dev(v_rank, "v"), nrhs, _dev(out, "out", v_rank.shape), 0,
                               _stream(stream)))
        return out

    def kmvm_host(self, v_host, out_host, stream=None):
        """End-to-end K v on host (numpy / pinned torch CPU) buffers."""
        import numpy as np
        nrhs = 1 if v_host.ndim == 1 else v_host.shape[0]
        vp = ctypes.c_void_p(v_host.ctypes.data if isinstance(v_host, np.ndarray) else v_host.data_ptr())
        op = ctypes.c_void_p(out_host.ctypes.data if isinstance(out_host, np.ndarray) else out_host.data_ptr())
        _check(_lib.gp_kmvm_host(self._h, vp, nrhs, op, _stream(stream)))
        return out_host

    def cross(self, z, stream=None) -> "Cross":
        return Cross(self, z, stream)

    def cg_solve(self, y, sigma2: float, mean: int = MEAN_AFFINE, H=None, rtol: float = 1e-8,
                 max_iter: int = 20000, stream=None, precond=None, return_x: bool = False,
                 return_ols: bool = False):
        """alpha, beta, info of (K + sigma^2 I) CG with GLS fixed effects (gp_cg_solve_ex;
        precond: a Precond of this plan or None).  return_x: info["X"] = the CG solutions
        [A^-1 y, A^-1 H...] (1 + nh, n) in user order; return_ols: info["beta_ols"]."""
        import torch
        alpha = torch.empty(self.n, dtype=torch.float64, device=y.device)
        nb = 1 + self.d if mean == MEAN_AFFINE else (H.shape[0] if mean == MEAN_BASIS else 0)
        beta = (ctypes.c_double * max(nb, 1))()
        bols = (ctypes.c_double * max(nb, 1))() if return_ols else None
        X = torch.empty((1 + nb, self.n), dtype=torch.float64, device=y.device) if return_x else None
        info = _CGInfo()
        Hp = _dev(H, "H") if mean == MEAN_BASIS else ctypes.c_void_p(0)
        L = H.shape[0] if mean == MEAN_BASIS else 0
        st = _lib.gp_cg_solve_ex(self._h, precond._h if precond is not None else None,
                                 float(sigma2), _dev(y, "y", (self.n,)), mean, Hp, L,
                                 float(rtol), int(max_iter), _dev(alpha, "alpha"), beta, bols,
                                 _dev(X, "X") if X is not None else None, ctypes.byref(info),
                                 _stream(stream))
        res = {"iters": info.iters, "relres_max": info.relres_max,
               "failed_column": info.failed_column, "restarts": info.restarts}
        if X is not None:
            res["X"] = X
        if bols is not None:
            res["beta_ols"] = [bols[i] for i in range(nb)]
        if st != 0:
            err = GPError(st, _lib.gp_last_error().decode())
            err.info = res
            err.alpha = alpha
            raise err
        return alpha, [beta[i] for i in range(nb)], res

    def mbcg(self, B, sigma2: float, max_iter: int, rtol: float = 0.0, precond=None,
             stream=None):
        """Algorithm 2 (gp_mbcg): B (nb, n) user order -> X (nb, n), alpha/beta histories
        (max_iter, nb) and iterations done per column."""
        import numpy as np
        import torch
        B2 = B if B.dim() == 2 else B.reshape(1, -1)
        nb = B2.shape[0]
        X = torch.empty_like(B2)
        ah = np.zeros((max_iter, nb)); bh = np.zeros((max_iter, nb))
        it = (ctypes.c_int * nb)()
        _check(_lib.gp_mbcg(self._h, precond._h if precond is not None else None, float(sigma2),
                            _dev(B2, "B", (nb, self.n)), nb, int(max_iter), float(rtol),
                            _dev(X, "X"), ah.ctypes.data_as(ctypes.c_void_p),
                            bh.ctypes.data_as(ctypes.c_void_p), it, _stream(stream)))
        return X, ah, bh, [it[i] for i in range(nb)]

    def lml(self, r, sigma2: float, G, W=None, lanczos_iters: int = 30, cg_rtol: float = 1e-8,
            precond=None, stream=None):
        """Log-marginal likelihood and gradient (gp_lml); G (nprobe, n) standard normals,
        W (nprobe, rank) standard normals with a preconditioner."""
        l = G.shape[0]
        res = _LmlResult()
        Wp = None
        if precond is not None:
            if W is None or tuple(W.shape) != (l, precond.rank):
                raise ValueError("W must be (nprobe, rank) with a preconditioner")
            Wp = _dev(W, "W")
        _check(_lib.gp_lml(self._h, precond._h if precond is not None else None, float(sigma2),
                           _dev(r, "r", (self.n,)), _dev(G, "G", (l, self.n)), Wp, l,
                           int(lanczos_iters), float(cg_rtol), ctypes.byref(res),
                           _stream(stream)))
        return {"lml": res.lml, "quad": res.quad, "logdet": res.logdet,
                "logdet_precond": res.logdet_precond, "grad": [res.grad[i] for i in range(3)],
                "cg_iters": res.cg_iters, "lanczos_iters": res.lanczos_iters}

    def predict(self, z, alpha, beta=None, Hz=None, stream=None):
        import torch
        m = z.shape[0]
        out = torch.empty(m, dtype=torch.float64, device=z.device)
        bp = None
        if beta is not None:
            bp = (ctypes.c_double * len(beta))(*beta)
        L = Hz.shape[0] if Hz is not None else 0
        _check(_lib.gp_predict(self._h, _dev(z, "z"), m, _dev(alpha, "alpha", (self.n,)), bp,
                               _dev(Hz, "Hz") if Hz is not None else None, L,
                               _dev(out, "out"), _stream(stream)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            _lib.gp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Cross:
    """Structure of x U z for repeated K_zx v (gp_kzx_setup / gp_kzx)."""

    def __init__(self, plan: Plan, z, stream=None):
        if z.dim() == 1:
            z = z.reshape(-1, 1)
        self.plan, self.m = plan, int(z.shape[0])
        h = ctypes.c_void_p()
        _check(_lib.gp_kzx_setup(plan._h, _dev(z, "z"), self.m, _stream(stream), ctypes.byref(h)))
        self._h = h

    def kzx(self, v, out=None, stream=None):
        import torch
        nrhs = 1 if v.dim() == 1 else v.shape[0]
        shape = (self.m,) if v.dim() == 1 else (nrhs, self.m)
        if out is None:
            out = torch.empty(shape, dtype=torch.float64, device=v.device)
        _check(_lib.gp_kzx(self._h, _dev(v, "v"), nrhs, _dev(out, "out", shape), _stream(stream)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            _lib.gp_kzx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def setup(x, kernel: Kernel, stream=None) -> Plan:
    return Plan(x, kernel, stream)


def kmvm(plan: Plan, v, out=None, stream=None):
    return plan.kmvm(v, out, stream)


class Precond:
    """Rank-k pivoted-Cholesky preconditioner P = L L^T + sigma^2 I of a plan's K
    (gp_precond_create)."""

    def __init__(self, plan: Plan, rank: int, stream=None):
        self.plan = plan
        self.rank = int(rank)
        h = ctypes.c_void_p()
        _check(_lib.gp_precond_create(plan._h, self.rank, _stream(stream), ctypes.byref(h)))
        self._h = h

    def factor(self, stream=None):
        """(pivots as user indices, L as a (rank, n) tensor in user order)."""
        import numpy as np
        import torch
        piv = np.zeros(self.rank, dtype=np.int64)
        L = torch.empty((self.rank, self.plan.n), dtype=torch.float64, device="cuda")
        _check(_lib.gp_precond_factor(self._h, piv.ctypes.data_as(ctypes.c_void_p), _dev(L, "L"),
                                      _stream(stream)))
        return piv, L

    def solve(self, sigma2: float, r, stream=None):
        import torch
        r2 = r if r.dim() == 2 else r.reshape(1, -1)
        z = torch.empty_like(r2)
        _check(_lib.gp_precond_solve(self._h, float(sigma2), _dev(r2, "r"), r2.shape[0],
                                     _dev(z, "z"), _stream(stream)))
        return z if r.dim() == 2 else z[0]

    def logdet(self, sigma2: float, stream=None) -> float:
        out = ctypes.c_double()
        _check(_lib.gp_precond_logdet(self._h, float(sigma2), ctypes.byref(out), _stream(stream)))
        return out.value

    def close(self):
        if getattr(self, "_h", None):
            _lib.gp_precond_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)
_alloc_hooks = None
# every (alloc, free) thunk pair ever installed: buffers keep the free hook they were
# allocated with (include/gpmatern.h), so a replaced pair must outlive them -- never cleared
_all_hooks = []


def use_torch_allocator(enable: bool = True):
    """Route the library's device allocations through PyTorch's caching allocator
    (gp_set_allocator); enable=False restores cudaMalloc/cudaFree.  Marshalling only: the
    callbacks call torch.cuda.caching_allocator_alloc / _delete."""
    global _alloc_hooks
    lib = load_library()
    if not enable:
        _check(lib.gp_set_allocator(None, None, None))
        _alloc_hooks = None
        return
    import torch

    def _alloc(nbytes, stream, ctx):
        return torch.cuda.caching_allocator_alloc(int(nbytes))

    def _free(ptr, stream, ctx):
        torch.cuda.caching_allocator_delete(ptr)

    _alloc_hooks = (_ALLOC_FN(_alloc), _FREE_FN(_free))
    _all_hooks.append(_alloc_hooks)   # keep the thunks alive for the whole process
    _check(lib.gp_set_allocator(ctypes.cast(_alloc_hooks[0], ctypes.c_void_p),
                                ctypes.cast(_alloc_hooks[1], ctypes.c_void_p), None))


def fit(x, kernel: Kernel, sigma0: float, y, G, W=None, stream=None, **opts):
    """Algorithm 1 hyperparameter fit (gp_fit).  x (n, d), y (n,), G (nprobe, n) standard
    normals, W (nprobe, precond_rank) standard normals if precond_rank > 0.  opts: lr,
    max_steps, max_outer, grad_tol, beta_tol, lanczos_iters, precond_rank, cg_rtol.
    Returns dict(kernel=Kernel, sigma, beta, steps, outer, lml, grad_norm)."""
    load_library()
    if x.dim() == 1:
        x = x.reshape(-1, 1)
    n, d = x.shape
    o = _FitOpts()
    for k, v in opts.items():
        setattr(o, k, v)
    res = _FitResult()
    kc = kernel.c()
    Wp = _dev(W, "W") if W is not None else None
    _check(_lib.gp_fit(_dev(x, "x"), n, d, ctypes.byref(kc), float(sigma0), _dev(y, "y", (n,)),
                       _dev(G, "G", (G.shape[0], n)), Wp, G.shape[0], ctypes.byref(o),
                       ctypes.byref(res), _stream(stream)))
    k = Kernel(res.kernel.two_nu, tuple(res.kernel.lengthscale[i] for i in range(d)),
               res.kernel.outputscale, res.kernel.form)
    return {"kernel": k, "sigma": res.sigma, "beta": [res.beta[i] for i in range(1 + d)],
            "steps": res.steps, "outer": res.outer, "lml": res.lml, "grad_norm": res.grad_norm}


def shard_ranges(n: int, d: int, shard: int, nshards: int):
    """Host-only work split of a sharded d >= 2 apply (gp_shard_ranges): ((tile_lo, tile_hi),
    (item_lo, item_hi))."""
    lib = load_library()
    r = (ctypes.c_int64 * 4)()
    _check(lib.gp_shard_ranges(int(n), int(d), int(shard), int(nshards), r))
    return (r[0], r[1]), (r[2], r[3])


def cg_solve(plan: Plan, y, sigma2, **kw):
    return plan.cg_solve(y, sigma2, **kw)


def predict(plan: Plan, z, alpha, beta=None, Hz=None, stream=None):
    return plan.predict(z, alpha, beta, Hz, stream)
