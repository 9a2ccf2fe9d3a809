"""Thin ctypes binding of the C ABI declared in include/kx.h (argument marshalling only).

Every ``kx_*`` function of the header is exposed here under the same name; ``Context`` is a
convenience wrapper that accepts torch tensors (fp64, CUDA, contiguous; vec order = C-order
shape (n_d, ..., n_1)) and numpy matrices (column-major is produced here with
``np.asfortranarray``).  No arithmetic of the method happens in Python: every step runs in
libkx.so's CUDA kernels.  If libkx.so is missing or fails to load, importing this module
raises — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkx.so")

KX_OK, KX_ERR_INVALID, KX_ERR_NUMERIC, KX_ERR_IO = 0, 2, 3, 4
KX_ERR_CUDA, KX_ERR_NCCL, KX_ERR_UNSUPPORTED, KX_ERR_NOMEM = 5, 6, 7, 8
KX_ETD2RKDS, KX_ETD3RKDS_REAL, KX_ETD3RKDS_CPLX = 1, 2, 3
KX_MODEL_NONE, KX_MODEL_SCHNAKENBERG, KX_MODEL_FHN = 0, 1, 2

SCHEMES = {"etd2rkds": KX_ETD2RKDS, "etd3rkds": KX_ETD3RKDS_REAL,
           "exprk3ds_real": KX_ETD3RKDS_REAL, "exprk3ds_cplx": KX_ETD3RKDS_CPLX}
MODELS = {"none": KX_MODEL_NONE, "schnakenberg": KX_MODEL_SCHNAKENBERG, "fhn": KX_MODEL_FHN}


class KxError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"kx status {status}: {msg}")
        self.status = status


class kx_counters(C.Structure):
    _fields_ = [("steps", C.c_longlong), ("tucker_ops", C.c_longlong),
                ("mode_products", C.c_longlong), ("kronsum_actions", C.c_longlong),
                ("phi_builds", C.c_longlong), ("gemm_launches", C.c_longlong),
                ("other_launches", C.c_longlong), ("mode_product_flops", C.c_double)]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2310_07551_b200.build` "
                      "(or __graft_entry__.build()); there is no CPU fallback")
lib = C.CDLL(LIB_PATH)

_vp, _dp, _i, _d, _ll = C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_double, C.c_longlong
_SIGS = {
    "kx_create": (_i, [C.POINTER(_vp), _i, _vp]),
    "kx_destroy": (None, [_vp]),
    "kx_last_error": (C.c_char_p, [_vp]),
    "kx_create_error": (C.c_char_p, []),
    "kx_set_grid": (_i, [_vp, _i, C.POINTER(_ll), _i]),
    "kx_set_direction_matrix": (_i, [_vp, _i, _i, _dp]),
    "kx_set_model": (_i, [_vp, _i, _dp, _i]),
    "kx_set_tau": (_i, [_vp, _d, _i]),
    "kx_mode_product": (_i, [_vp, _vp, _vp, _i, _vp, _d, _d]),
    "kx_tucker": (_i, [_vp, _vp, _vp, C.POINTER(_vp), _d, _d]),
    "kx_tucker_batched": (_i, [_vp, _i, _vp, _vp, C.POINTER(_vp), _d, _d]),
    "kx_kronsum": (_i, [_vp, _i, _vp, _vp, _d]),
    "kx_set_kronsum_mode": (_i, [_vp, _i]),
    "kx_phi_apply": (_i, [_vp, _i, _i, _i, _vp, _vp, _d, _d]),
    "kx_step": (_i, [_vp, _d, C.POINTER(_vp)]),
    "kx_integrate_host": (_i, [_vp, _d, _i, C.POINTER(_vp)]),
    "kx_step_n": (_i, [_vp, _d, _i, C.POINTER(_vp)]),
    "kx_set_fused_small": (_i, [_vp, _i]),
    "kx_nccl_unique_id": (_i, [_vp]),
    "kx_create_dist": (_i, [C.POINTER(_vp), _i, _vp, _vp, _i, _i]),
    "kx_create_group": (_i, [C.POINTER(_vp), _i, _i, _vp]),
    "kx_step_group": (_i, [C.POINTER(_vp), _i, _d, C.POINTER(_vp)]),
    "kx_tucker_group": (_i, [C.POINTER(_vp), _i, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), _d, _d]),
    "kx_mode_product_group": (_i, [C.POINTER(_vp), _i, C.POINTER(_vp), C.POINTER(_vp), _i, _vp, _d, _d]),
    "kx_phi_apply_group": (_i, [C.POINTER(_vp), _i, _i, _i, _i, C.POINTER(_vp), C.POINTER(_vp), _d, _d]),
    "kx_kronsum_group": (_i, [C.POINTER(_vp), _i, _i, C.POINTER(_vp), C.POINTER(_vp), _d]),
    "kx_group_set_p2p": (_i, [C.POINTER(_vp), _i, _i]),
    "kx_dist_ipc_export": (_i, [_vp, _vp, C.c_size_t, C.POINTER(C.c_size_t)]),
    "kx_dist_ipc_import": (_i, [_vp, _vp, C.c_size_t]),
    "kx_set_dist_overlap": (_i, [_vp, _i]),
    "kx_get_counters": (_i, [_vp, C.POINTER(kx_counters)]),
    "kx_reset_counters": (_i, [_vp]),
    "kx_sync": (_i, [_vp]),
    "kx_check_finite": (_i, [_vp, _vp]),
    "kx_set_nan_check": (_i, [_vp, _i]),
    "kx_set_profiling": (_i, [_vp, _i]),
    "kx_get_profile": (_i, [_vp, _dp, _dp, C.POINTER(_ll), C.POINTER(_ll), _dp]),
    "kx_get_profile_hbm": (_i, [_vp, _dp]),
    "kx_get_phi_matrix": (_i, [_vp, _i, _i, _i, _i, _i, _dp]),
    "kx_set_phi_matrix": (_i, [_vp, _i, _i, _i, _i, _i, _dp]),
    "kx_mode_product_f32": (_i, [_vp, _vp, _vp, _i, _vp, C.c_float, C.c_float]),
    "kx_tucker_f32": (_i, [_vp, _vp, _vp, C.POINTER(_vp), C.c_float, C.c_float]),
    "kx_step_f32": (_i, [_vp, _d, _i, C.POINTER(_vp)]),
    "kx_scheme_coefficients": (_i, [_i, _i, _i, C.POINTER(_i), _dp, C.POINTER(_i), _dp]),
    "kx_scheme_coefficients_cplx": (_i, [_i, _i, C.POINTER(_i), _dp, _dp, C.POINTER(_i), _dp, _dp]),
    "kx_version": (C.c_char_p, []),
}
EXPORTED = tuple(_SIGS)
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f


def _ptr(t, numel: int | None = None, device: int | None = None, dtype: str = "torch.float64") -> int:
    """Device pointer of a torch tensor (fp64 — fp32 for the *_f32 calls —, CUDA, contiguous) or
    a raw int.  With `numel` the tensor must hold at least that many elements, with `device` live
    on that GPU: the raw ABI cannot check sizes, so this wrapper is the place that stops
    out-of-bounds kernels."""
    if isinstance(t, int):
        return t
    if t.dtype.__repr__() != dtype:
        raise TypeError(f"tensors must be {dtype[6:]}")
    if not t.is_cuda:
        raise TypeError("tensors must live on the GPU")
    if not t.is_contiguous():
        raise TypeError("tensors must be contiguous")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"tensor holds {t.numel()} doubles, the grid needs {numel}")
    if device is not None and t.device.index != device:
        raise ValueError(f"tensor on cuda:{t.device.index}, context on cuda:{device}")
    return t.data_ptr()


def scheme_coefficients(scheme: str | int, ell: int, d: int):
    """Host-only: (etas, inner ells, alphas[i][mu]) the library uses."""
    sc = SCHEMES.get(scheme, scheme)
    nt = C.c_int(0)
    eta = (C.c_double * 3)()
    inner = (C.c_int * 3)()
    alpha = (C.c_double * (3 * d))()
    st = kx_scheme_coefficients(sc, ell, d, C.byref(nt), eta, inner, alpha)
    if st != KX_OK:
        raise KxError(st, "scheme not available")
    n = nt.value
    return (list(eta[:n]), list(inner[:n]), [list(alpha[i * d:(i + 1) * d]) for i in range(n)])


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = kx_nccl_unique_id(buf)
    if st != KX_OK:
        raise KxError(st, kx_create_error().decode())
    return buf.raw


def scheme_coefficients_cplx(ell: int, d: int):
    """Host-only: Table 2 (etas, inner ells, alphas[i][mu]) as complex numbers."""
    nt = C.c_int(0)
    er, ei = (C.c_double * 3)(), (C.c_double * 3)()
    inner = (C.c_int * 3)()
    ar, ai = (C.c_double * (3 * d))(), (C.c_double * (3 * d))()
    st = kx_scheme_coefficients_cplx(ell, d, C.byref(nt), er, ei, inner, ar, ai)
    if st != KX_OK:
        raise KxError(st, "scheme not available")
    n = nt.value
    return ([complex(er[i], ei[i]) for i in range(n)], list(inner[:n]),
            [[complex(ar[i * d + m], ai[i * d + m]) for m in range(d)] for i in range(n)])


class Context:
    """Owns one kx_ctx.  Methods mirror the C ABI one to one.

    Context(device)                         single GPU
    Context(device, dist=(uid, rank, P))    one rank of a slab-sharded run (NCCL)
    """

    def __init__(self, device: int = 0, stream=None, dist=None, handle=None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        if handle is not None:
            h = handle
        else:
            h = C.c_void_p()
            if dist is None:
                st = kx_create(C.byref(h), device, C.c_void_p(stream.cuda_stream))
            else:
                uid, rank, nranks = dist
                st = kx_create_dist(C.byref(h), device, C.c_void_p(stream.cuda_stream),
                                    C.c_char_p(uid), rank, nranks)
            if st != KX_OK:
                raise KxError(st, kx_create_error().decode())
        self.h = h
        self.device = device
        self.nranks = 1 if dist is None else int(dist[2])
        self.d = 0
        self.n: list[int] = []
        self.ncomp = 0

    def _check(self, st: int):
        if st != KX_OK:
            raise KxError(st, kx_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            kx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:   # interpreter teardown: the ctypes globals may already be gone
            pass

    # --- setup
    def set_grid(self, n: list[int], ncomp: int = 2):
        arr = (C.c_longlong * len(n))(*n)
        self._check(kx_set_grid(self.h, len(n), arr, ncomp))
        self.d, self.n, self.ncomp = len(n), list(n), ncomp

    def set_direction_matrix(self, comp: int, mu: int, A: np.ndarray):
        buf = np.ascontiguousarray(np.asarray(A, dtype=np.float64).T)   # column-major bytes
        self._check(kx_set_direction_matrix(self.h, comp, mu,
                                            buf.ctypes.data_as(C.POINTER(C.c_double))))

    def set_model(self, model: str, params: dict | None = None):
        m = MODELS[model]
        if m == KX_MODEL_NONE:
            self._check(kx_set_model(self.h, m, None, 0))
            return
        keys = ("du", "dv", "rho", "au", "av") if model == "schnakenberg" else \
               ("du", "dv", "rho", "a1", "a2")
        vals = (C.c_double * 5)(*[params[k] for k in keys])
        self._check(kx_set_model(self.h, m, vals, 5))

    def set_tau(self, tau: float, scheme: str):
        self._check(kx_set_tau(self.h, tau, SCHEMES[scheme]))

    @property
    def local_numel(self) -> int:
        """Doubles per component tensor this context acts on (its slab on a sharded context)."""
        return int(np.prod(self.n)) // self.nranks if self.n else 0

    def _state(self, U: list) -> list[int]:
        if not self.n:   # no grid yet: the C side rejects the call (KX_ERR_INVALID)
            return [_ptr(u) for u in U]
        if len(U) != self.ncomp:
            raise ValueError(f"{len(U)} state tensors given, the grid has {self.ncomp} components")
        return [_ptr(u, self.local_numel, self.device) for u in U]

    def _t(self, X) -> int:
        return _ptr(X, self.local_numel if self.n else None, self.device)

    # --- operators (device tensors)
    def mode_product(self, X, Y, mu: int, L, alpha=1.0, beta=0.0):
        nm = self.n[mu - 1] if self.n and 1 <= mu <= self.d else None
        self._check(kx_mode_product(self.h, self._t(X), self._t(Y), mu,
                                    _ptr(L, nm * nm if nm else None, self.device), alpha, beta))

    def tucker(self, X, Y, Ls, alpha=1.0, beta=0.0):
        if len(Ls) != self.d:
            raise ValueError(f"{len(Ls)} matrices given, the grid has d = {self.d}")
        arr = (C.c_void_p * len(Ls))(*[_ptr(L, self.n[m] ** 2, self.device) for m, L in enumerate(Ls)])
        self._check(kx_tucker(self.h, self._t(X), self._t(Y), arr, alpha, beta))

    def tucker_batched(self, X, Y, Ls, nbatch: int, alpha=1.0, beta=0.0):
        """nbatch independent Tuckers on X[b*N:(b+1)*N] (one launch per mode)."""
        if len(Ls) != self.d:
            raise ValueError(f"{len(Ls)} matrices given, the grid has d = {self.d}")
        arr = (C.c_void_p * len(Ls))(*[_ptr(L, self.n[m] ** 2, self.device) for m, L in enumerate(Ls)])
        tot = nbatch * self.local_numel
        self._check(kx_tucker_batched(self.h, nbatch, _ptr(X, tot, self.device), _ptr(Y, tot, self.device),
                                      arr, alpha, beta))

    def kronsum(self, comp: int, X, Y, beta=0.0):
        self._check(kx_kronsum(self.h, comp, self._t(X), self._t(Y), beta))

    def set_dist_overlap(self, on: bool):
        self._check(kx_set_dist_overlap(self.h, 1 if on else 0))

    def set_kronsum_mode(self, dense: bool):
        self._check(kx_set_kronsum_mode(self.h, 1 if dense else 0))

    def phi_apply(self, comp: int, ell: int, stage: int, X, Y, alpha=1.0, beta=0.0):
        self._check(kx_phi_apply(self.h, comp, ell, stage, self._t(X), self._t(Y), alpha, beta))

    def step(self, U: list, t: float = 0.0):
        arr = (C.c_void_p * len(U))(*self._state(U))
        self._check(kx_step(self.h, t, arr))

    def step_n(self, U: list, nsteps: int, t0: float = 0.0):
        arr = (C.c_void_p * len(U))(*self._state(U))
        self._check(kx_step_n(self.h, t0, nsteps, arr))

    # --- fp32 variant (tcgen05 kind::tf32, three-pass split; kx_*_f32)
    def _t32(self, X) -> int:
        return _ptr(X, self.local_numel if self.n else None, self.device, "torch.float32")

    def mode_product_f32(self, X, Y, mu: int, L, alpha=1.0, beta=0.0):
        nm = self.n[mu - 1] if self.n and 1 <= mu <= self.d else None
        self._check(kx_mode_product_f32(self.h, self._t32(X), self._t32(Y), mu,
                                        _ptr(L, nm * nm if nm else None, self.device, "torch.float32"),
                                        alpha, beta))

    def tucker_f32(self, X, Y, Ls, alpha=1.0, beta=0.0):
        if len(Ls) != self.d:
            raise ValueError(f"{len(Ls)} matrices given, the grid has d = {self.d}")
        arr = (C.c_void_p * len(Ls))(*[_ptr(L, self.n[m] ** 2, self.device, "torch.float32")
                                        for m, L in enumerate(Ls)])
        self._check(kx_tucker_f32(self.h, self._t32(X), self._t32(Y), arr, alpha, beta))

    def step_f32(self, U: list, nsteps: int = 1, t0: float = 0.0):
        if self.n and len(U) != self.ncomp:
            raise ValueError(f"{len(U)} state tensors given, the grid has {self.ncomp} components")
        arr = (C.c_void_p * len(U))(*[self._t32(u) for u in U])
        self._check(kx_step_f32(self.h, t0, nsteps, arr))

    def ipc_export(self) -> bytes:
        """This NCCL rank's receive buffers as CUDA IPC handles (after set_tau)."""
        n = C.c_size_t()
        self._check(kx_dist_ipc_export(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        self._check(kx_dist_ipc_export(self.h, buf, n.value, C.byref(n)))
        return buf.raw

    def ipc_import(self, blobs: list):
        """Every rank's ipc_export() blob, in rank order: enables direct peer stores."""
        each = len(blobs[0])
        assert all(len(b) == each for b in blobs)
        joined = C.create_string_buffer(b"".join(blobs), each * len(blobs))
        self._check(kx_dist_ipc_import(self.h, joined, each))

    def set_fused_small(self, on: bool):
        self._check(kx_set_fused_small(self.h, 1 if on else 0))

    def integrate_host(self, U_host: list[np.ndarray], nsteps: int, t0: float = 0.0):
        """U_host: C-contiguous float64 host arrays (pinned torch tensors work too: pass
        their .numpy()).  Updated in place."""
        if len(U_host) != self.ncomp:
            raise ValueError(f"{len(U_host)} state arrays given, the grid has {self.ncomp} components")
        ptrs = []
        for u in U_host:
            if isinstance(u, np.ndarray):
                if u.dtype != np.float64 or not u.flags.c_contiguous:
                    raise TypeError("host arrays must be C-contiguous float64")
                if u.size < self.local_numel:
                    raise ValueError(f"host array holds {u.size} doubles, the grid needs {self.local_numel}")
                ptrs.append(u.ctypes.data)
            else:
                if u.numel() < self.local_numel:
                    raise ValueError(f"host tensor holds {u.numel()} doubles, the grid needs {self.local_numel}")
                ptrs.append(u.data_ptr())
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        self._check(kx_integrate_host(self.h, t0, nsteps, arr))

    def sync(self):
        self._check(kx_sync(self.h))

    def set_nan_check(self, on: bool):
        self._check(kx_set_nan_check(self.h, 1 if on else 0))

    def check_finite(self, X) -> bool:
        st = kx_check_finite(self.h, self._t(X))
        if st == KX_ERR_NUMERIC:
            return False
        self._check(st)
        return True

    def counters(self) -> dict:
        c = kx_counters()
        self._check(kx_get_counters(self.h, C.byref(c)))
        return {k: getattr(c, k) for k, _ in kx_counters._fields_}

    def reset_counters(self):
        self._check(kx_reset_counters(self.h))

    def set_profiling(self, on: bool):
        self._check(kx_set_profiling(self.h, 1 if on else 0))

    def profile(self) -> dict:
        gm, om, gf = C.c_double(), C.c_double(), C.c_double()
        gl, ol = C.c_longlong(), C.c_longlong()
        self._check(kx_get_profile(self.h, C.byref(gm), C.byref(om), C.byref(gl), C.byref(ol),
                                   C.byref(gf)))
        ob = C.c_double()
        self._check(kx_get_profile_hbm(self.h, C.byref(ob)))
        return dict(gemm_ms=gm.value, other_ms=om.value, gemm_launches=gl.value,
                    other_launches=ol.value, gemm_flops=gf.value, other_bytes=ob.value)

    def phi_matrix(self, comp: int, ell: int, stage: int, term: int, mu: int) -> np.ndarray:
        n = self.n[mu - 1]
        out = np.empty(n * n)
        self._check(kx_get_phi_matrix(self.h, comp, ell, stage, term, mu,
                                      out.ctypes.data_as(C.POINTER(C.c_double))))
        return out.reshape(n, n, order="F")

    def set_phi_matrix(self, comp: int, ell: int, stage: int, term: int, mu: int, P: np.ndarray):
        """Replace one phi-matrix of the bank (inverse of phi_matrix; see kx_set_phi_matrix)."""
        n = self.n[mu - 1]
        P = np.asarray(P, dtype=np.float64)
        if P.shape != (n, n):
            raise ValueError(f"phi-matrix of mode {mu} must be {n} x {n}, got {P.shape}")
        buf = np.ascontiguousarray(P.T)   # column-major bytes
        self._check(kx_set_phi_matrix(self.h, comp, ell, stage, term, mu,
                                      buf.ctypes.data_as(C.POINTER(C.c_double))))


class Group:
    """In-process loopback group of `nranks` contexts on one GPU (kx_create_group): the
    sharded schedule with device-copy exchanges, for single-GPU testing of the multi-GPU path."""

    def __init__(self, nranks: int, device: int = 0, stream=None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(device)
        arr = (C.c_void_p * nranks)()
        st = kx_create_group(arr, nranks, device, C.c_void_p(stream.cuda_stream))
        if st != KX_OK:
            raise KxError(st, kx_create_error().decode())
        self.nranks = nranks
        self._arr = arr
        self.ctx = [Context(device, stream, handle=C.c_void_p(arr[r])) for r in range(nranks)]
        for c in self.ctx:
            c.nranks = nranks

    def step(self, U: list[list], t: float = 0.0):
        """U[r][c]: device slab of component c on rank r."""
        if len(U) != self.nranks:
            raise ValueError(f"{len(U)} rank states given, the group has {self.nranks} ranks")
        flat = [p for r, Ur in enumerate(U) for p in self.ctx[r]._state(Ur)]
        arr = (C.c_void_p * len(flat))(*flat)
        st = kx_step_group(self._arr, self.nranks, t, arr)
        if st != KX_OK:
            raise KxError(st, kx_last_error(self.ctx[0].h).decode())

    def _slabs(self, Xs: list) -> "C.Array":
        if len(Xs) != self.nranks:
            raise ValueError(f"{len(Xs)} slabs given, the group has {self.nranks} ranks")
        return (C.c_void_p * self.nranks)(*[self.ctx[r]._t(x) for r, x in enumerate(Xs)])

    def _chk(self, st: int):
        if st != KX_OK:
            raise KxError(st, kx_last_error(self.ctx[0].h).decode())

    def tucker(self, Xs: list, Ys: list, Ls: list, alpha=1.0, beta=0.0):
        """Distributed Tucker operator on the ranks' layout-A slabs (kx_tucker_group)."""
        c0 = self.ctx[0]
        if len(Ls) != c0.d:
            raise ValueError(f"{len(Ls)} matrices given, the grid has d = {c0.d}")
        L = (C.c_void_p * len(Ls))(*[_ptr(M, c0.n[m] ** 2, c0.device) for m, M in enumerate(Ls)])
        self._chk(kx_tucker_group(self._arr, self.nranks, self._slabs(Xs), self._slabs(Ys), L, alpha, beta))

    def mode_product(self, Xs: list, Ys: list, mu: int, L, alpha=1.0, beta=0.0):
        c0 = self.ctx[0]
        nm = c0.n[mu - 1] if 1 <= mu <= c0.d else None
        self._chk(kx_mode_product_group(self._arr, self.nranks, self._slabs(Xs), self._slabs(Ys), mu,
                                        _ptr(L, nm * nm if nm else None, c0.device), alpha, beta))

    def kronsum(self, comp: int, Xs: list, Ys: list, beta=0.0):
        self._chk(kx_kronsum_group(self._arr, self.nranks, comp, self._slabs(Xs), self._slabs(Ys), beta))

    def phi_apply(self, comp: int, ell: int, stage: int, Xs: list, Ys: list, alpha=1.0, beta=0.0):
        self._chk(kx_phi_apply_group(self._arr, self.nranks, comp, ell, stage, self._slabs(Xs),
                                     self._slabs(Ys), alpha, beta))

    def set_p2p(self, on: bool):
        """Direct peer stores instead of exchange copies (after every member's set_tau)."""
        st = kx_group_set_p2p(self._arr, self.nranks, 1 if on else 0)
        if st != KX_OK:
            raise KxError(st, kx_last_error(self.ctx[0].h).decode())

    def close(self):
        for c in self.ctx:
            c.close()
