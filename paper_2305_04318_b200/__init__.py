"""B200-native (sm_100a) batched profile log-likelihood of arXiv 2305.04318.

Thin ctypes binding over the C ABI in ``include/lik.h`` (``liblik.so``, built
in-tree by ``paper_2305_04318_b200.build``).  Argument marshalling only: every
step of the likelihood runs in the library's CUDA kernels.  There is no CPU
fallback — if the library or a CUDA device is missing, calls raise.

Names follow the ABI:
    create(device, flags) -> Ctx
    Ctx.eval_batch(coords, y, X, params, lambdas)             host numpy arrays
    Ctx.eval_batch_device(coords, y, X, params, lambdas, out, stream)   torch CUDA tensors
    Ctx.debug_build_V(coords, params)                          torch CUDA tensors
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LIK_LIBRARY") or os.path.join(HERE, "liblik.so")  # LIK_LIBRARY: debug builds

LIK_OK, LIK_EINVAL, LIK_EDOMAIN, LIK_ERANK, LIK_ENOMEM, LIK_ECUDA, LIK_ENOTIMPL = 0, -1, -2, -3, -4, -5, -6
PT_OK, PT_V_NOT_PD, PT_XVX_NOT_PD, PT_NEG_RESID, PT_BAD_PARAM = 0, 1, 2, 3, 4
FLAG_TIMING = 1
FLAG_NATURAL_ORDER = 2
STAGES = ("prep", "setup", "matern_build", "chol_fused")
ABI_SYMBOLS = ("lik_create", "lik_destroy", "lik_last_error", "lik_eval_batch",
               "lik_eval_batch_device", "lik_get_stage_times", "lik_reset_stage_times",
               "lik_set_wave_points", "lik_debug_build_V", "lik_eval_batch_device_ex",
               "lik_profiles_device", "lik_dataset_create", "lik_dataset_eval_device",
               "lik_dataset_destroy")

_lib = None
_PD = ctypes.POINTER(ctypes.c_double)
_PI = ctypes.POINTER(ctypes.c_int)
_VP = ctypes.c_void_p


class LikError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"lik error {code}: {msg}")
        self.code = code


def lib():
    """Load liblik.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2305_04318_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        i, d = ctypes.c_int, ctypes.c_double
        L.lik_create.argtypes = [ctypes.POINTER(_VP), i, ctypes.c_uint]
        L.lik_create.restype = i
        L.lik_destroy.argtypes = [_VP]
        L.lik_destroy.restype = None
        L.lik_last_error.argtypes = [_VP]
        L.lik_last_error.restype = ctypes.c_char_p
        sig = [_VP, i, i, _VP, _VP, _VP, i, _VP, i, _VP, _VP, _VP, _VP, _VP, _VP]
        L.lik_eval_batch.argtypes = sig
        L.lik_eval_batch.restype = i
        L.lik_eval_batch_device.argtypes = sig + [_VP]
        L.lik_eval_batch_device.restype = i
        L.lik_eval_batch_device_ex.argtypes = sig + [_VP] * 6 + [_VP]
        L.lik_eval_batch_device_ex.restype = i
        L.lik_profiles_device.argtypes = [_VP, i, i, i, i, _VP, _VP, _VP, _VP, _VP, i, _VP, _VP, i,
                                          _VP, _VP, _VP, _VP]
        L.lik_profiles_device.restype = i
        L.lik_get_stage_times.argtypes = [_VP, _PD, ctypes.POINTER(ctypes.c_longlong)]
        L.lik_get_stage_times.restype = i
        L.lik_reset_stage_times.argtypes = [_VP]
        L.lik_reset_stage_times.restype = i
        L.lik_set_wave_points.argtypes = [_VP, i]
        L.lik_set_wave_points.restype = i
        L.lik_debug_build_V.argtypes = [_VP, i, _VP, i, _VP, _VP]
        L.lik_debug_build_V.restype = i
        L.lik_dataset_create.argtypes = [_VP, ctypes.POINTER(_VP), i, i, _VP, _VP, _VP, i, _VP]
        L.lik_dataset_create.restype = i
        L.lik_dataset_eval_device.argtypes = [_VP, _VP, i, _VP, _VP, _VP, _VP, _VP, _VP, _VP]
        L.lik_dataset_eval_device.restype = i
        L.lik_dataset_destroy.argtypes = [_VP]
        L.lik_dataset_destroy.restype = None
        _lib = L
    return _lib


def _np(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


def _tptr(t):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous()):
        raise TypeError("expected a contiguous CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


class Ctx:
    """A lik_ctx bound to one CUDA device (one per host thread)."""

    def __init__(self, device: int = 0, flags: int = 0):
        self._h = _VP()
        rc = lib().lik_create(ctypes.byref(self._h), int(device), int(flags))
        if rc != LIK_OK:
            raise LikError(rc, f"lik_create(device={device}) failed")
        self.device = device
        self.flags = flags

    def close(self):
        if self._h:
            lib().lik_destroy(self._h)
            self._h = _VP()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_error(self) -> str:
        return lib().lik_last_error(self._h).decode()

    def _check(self, rc):
        if rc != LIK_OK:
            raise LikError(rc, self.last_error())

    def eval_batch(self, coords, y, X, params, lambdas):
        """lik_eval_batch on host arrays; returns dict of numpy outputs."""
        coords, y, lambdas = _np(coords), _np(y), _np(lambdas)
        X = _np(X)
        if X.ndim == 1:
            X = X[:, None]
        params = _np(params).reshape(-1, 5)
        n, p = X.shape
        K, M = params.shape[0], lambdas.shape[0]
        out = dict(loglik=np.empty((K, M)), betahat=np.empty((K, M, p)), sigma2hat=np.empty((K, M)),
                   logdetV=np.empty(K), status=np.empty(K, dtype=np.int32))
        rc = lib().lik_eval_batch(self._h, n, p, _ptr(coords), _ptr(y), _ptr(X), K, _ptr(params), M,
                                  _ptr(lambdas), _ptr(out["loglik"]), _ptr(out["betahat"]),
                                  _ptr(out["sigma2hat"]), _ptr(out["logdetV"]), _ptr(out["status"]))
        self._check(rc)
        return out

    def eval_batch_rc(self, coords, y, X, params, lambdas):
        """Like eval_batch but returns (rc, message) instead of raising."""
        try:
            self.eval_batch(coords, y, X, params, lambdas)
            return LIK_OK, ""
        except LikError as e:
            return e.code, self.last_error()

    @staticmethod
    def alloc_outputs(K, M, p, device):
        import torch
        f = dict(dtype=torch.float64, device=device)
        return dict(loglik=torch.empty((K, M), **f), betahat=torch.empty((K, M, p), **f),
                    sigma2hat=torch.empty((K, M), **f), logdetV=torch.empty(K, **f),
                    status=torch.empty(K, dtype=torch.int32, device=device))

    def dataset(self, coords, y, X, lambdas) -> "Dataset":
        """lik_dataset_create: validate and upload (coords, y, X, lambdas) once."""
        return Dataset(self, coords, y, X, lambdas)

    def eval_batch_device(self, coords, y, X, params, lambdas, out=None, stream=None):
        """lik_eval_batch_device on torch CUDA float64 tensors (enqueued on `stream`)."""
        import torch
        n, p = X.shape
        K, M = params.shape[0], lambdas.shape[0]
        if out is None:
            out = self.alloc_outputs(K, M, p, X.device)
        if stream is None:
            stream = torch.cuda.current_stream(X.device)
        rc = lib().lik_eval_batch_device(
            self._h, n, p, _tptr(coords), _tptr(y), _tptr(X), K, _tptr(params), M, _tptr(lambdas),
            _tptr(out["loglik"]), _tptr(out["betahat"]), _tptr(out["sigma2hat"]),
            _tptr(out["logdetV"]), _tptr(out["status"]), ctypes.c_void_p(stream.cuda_stream))
        self._check(rc)
        return out

    def eval_batch_device_ex(self, coords, y, X, params, lambdas, stream=None):
        """lik_eval_batch_device_ex: the outputs of eval_batch_device plus the Table-1
        summaries (detReml, ssqYX, ssqBetahat, ssqResidual) and the REML profile
        likelihood (loglik_reml, sigma2hat_reml), as torch CUDA tensors."""
        import torch
        n, p = X.shape
        K, M = params.shape[0], lambdas.shape[0]
        r = M + p
        out = self.alloc_outputs(K, M, p, X.device)
        f = dict(dtype=torch.float64, device=X.device)
        out.update(detReml=torch.empty(K, **f), ssqYX=torch.empty((K, r, r), **f),
                   ssqBetahat=torch.empty((K, M), **f), ssqResidual=torch.empty((K, M), **f),
                   loglik_reml=torch.empty((K, M), **f), sigma2hat_reml=torch.empty((K, M), **f))
        if stream is None:
            stream = torch.cuda.current_stream(X.device)
        rc = lib().lik_eval_batch_device_ex(
            self._h, n, p, _tptr(coords), _tptr(y), _tptr(X), K, _tptr(params), M, _tptr(lambdas),
            _tptr(out["loglik"]), _tptr(out["betahat"]), _tptr(out["sigma2hat"]),
            _tptr(out["logdetV"]), _tptr(out["status"]), _tptr(out["detReml"]), _tptr(out["ssqYX"]),
            _tptr(out["ssqBetahat"]), _tptr(out["ssqResidual"]), _tptr(out["loglik_reml"]),
            _tptr(out["sigma2hat_reml"]), ctypes.c_void_p(stream.cuda_stream))
        self._check(rc)
        return out

    def profiles_device(self, n, y, summ, lambdas, beta_grid, sigma_grid, stream=None):
        """lik_profiles_device: β_a, σ and λ profile log-likelihoods from the
        summaries `summ` of eval_batch_device_ex (torch CUDA tensors)."""
        import torch
        p = summ["betahat"].shape[2]
        K, M = summ["logdetV"].shape[0], lambdas.shape[0]
        beta_grid = beta_grid.reshape(p, -1).contiguous()
        G, Sg = beta_grid.shape[1], sigma_grid.shape[0]
        f = dict(dtype=torch.float64, device=y.device)
        pb, ps, pl = torch.empty((p, G), **f), torch.empty(max(Sg, 1), **f), torch.empty(M, **f)
        if stream is None:
            stream = torch.cuda.current_stream(y.device)
        rc = lib().lik_profiles_device(
            self._h, n, p, K, M, _tptr(y), _tptr(summ["ssqYX"]), _tptr(summ["logdetV"]),
            _tptr(summ["status"]), _tptr(lambdas), G, _tptr(beta_grid), _tptr(pb), Sg,
            _tptr(sigma_grid), _tptr(ps), _tptr(pl), ctypes.c_void_p(stream.cuda_stream))
        self._check(rc)
        return pb, ps[:Sg], pl

    def debug_build_V(self, coords, params):
        import torch
        n, K = coords.shape[0], params.shape[0]
        V = torch.empty((K, n, n), dtype=torch.float64, device=coords.device)
        rc = lib().lik_debug_build_V(self._h, n, _tptr(coords), K, _tptr(params), _tptr(V))
        self._check(rc)
        return V

    def set_wave_points(self, pts: int):
        self._check(lib().lik_set_wave_points(self._h, int(pts)))

    def stage_times(self):
        ms = (ctypes.c_double * 4)()
        n = (ctypes.c_longlong * 4)()
        self._check(lib().lik_get_stage_times(self._h, ms, n))
        return {s: (ms[i], n[i]) for i, s in enumerate(STAGES)}

    def reset_stage_times(self):
        self._check(lib().lik_reset_stage_times(self._h))


class Dataset:
    """A prepared, device-resident dataset (lik_dataset): evaluations on it are enqueued
    with no host synchronisation."""

    def __init__(self, ctx: "Ctx", coords, y, X, lambdas):
        coords, y, lambdas = _np(coords), _np(y), _np(lambdas)
        X = _np(X)
        if X.ndim == 1:
            X = X[:, None]
        self.ctx = ctx
        self.n, self.p = X.shape
        self.M = lambdas.shape[0]
        self._h = _VP()
        rc = lib().lik_dataset_create(ctx._h, ctypes.byref(self._h), self.n, self.p, _ptr(coords),
                                      _ptr(y), _ptr(X), self.M, _ptr(lambdas))
        ctx._check(rc)

    def eval_device(self, params, out=None, stream=None):
        """lik_dataset_eval_device: params a K×5 torch CUDA float64 tensor; outputs as in
        Ctx.eval_batch_device, enqueued on `stream` (default: the current stream)."""
        import torch
        K = params.shape[0]
        if out is None:
            out = Ctx.alloc_outputs(K, self.M, self.p, params.device)
        if stream is None:
            stream = torch.cuda.current_stream(params.device)
        rc = lib().lik_dataset_eval_device(
            self.ctx._h, self._h, K, _tptr(params), _tptr(out["loglik"]), _tptr(out["betahat"]),
            _tptr(out["sigma2hat"]), _tptr(out["logdetV"]), _tptr(out["status"]),
            ctypes.c_void_p(stream.cuda_stream))
        self.ctx._check(rc)
        return out

    def close(self):
        if self._h:
            lib().lik_dataset_destroy(self._h)
            self._h = _VP()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def create(device: int = 0, flags: int = 0) -> Ctx:
    return Ctx(device, flags)
