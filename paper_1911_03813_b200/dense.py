"""Observation sets resident in B200 HBM.

Mirrors the reference ``ObservationSet`` (pkg/src/momentcp/dense.py:60-114): same constructor
``ObservationSet(V, nu=None, labels=None)`` with ``V`` of shape (n, p) (column l = observation
v_l), the same validation errors, the same ``n`` / ``p`` / ``has_uniform_weights`` surface and
the same default weights ``nu = 1/p``.

What changes is where the data lives: on first use the matrix is uploaded once to the GPU in
observation-major layout (each observation's n values contiguous, the unit the kernels tile
over) and kept in its own precision -- float32 input stays float32 in HBM (the reference
upcasts to a float64 copy, dense.py:82; the kernels convert in-register, which is exact).
The device copy is cached on the object, keyed by identity, like the reference caches nothing
but recomputes nothing either: V is immutable after construction.
"""

from __future__ import annotations

import threading

import numpy as np

from . import _native


class ObservationSet:
    """A set of p weighted observations of an n-vector (reference dense.py:60-114)."""

    def __init__(self, V, nu=None, labels=None, *, device: int | None = None):
        src = V
        if _is_torch_tensor(src):
            raise TypeError("use ObservationSet.from_device for torch tensors")
        arr = np.asarray(src)
        if arr.dtype != np.float32:
            arr = np.asarray(arr, dtype=float)
        if arr.ndim != 2:
            raise ValueError(f"V must be a 2-D matrix, got ndim={arr.ndim}")
        n, p = arr.shape
        if n < 1 or p < 1:
            raise ValueError(f"V must be at least 1x1, got shape {arr.shape}")
        if not np.isfinite(arr).all():
            raise ValueError("V contains non-finite entries")
        self._Vsrc = arr
        self._V64 = arr if arr.dtype == np.float64 else None
        self._n, self._p = n, p
        self._uniform_default = nu is None
        self.nu = _check_nu(nu, p)
        self.labels = _check_labels(labels, p)
        self._device = device
        self._dev = None
        self._dev_lock = threading.Lock()
        self._dev_obs = None  # (torch tensor, ...) when constructed from device memory
        self._host_obs = None  # (p x n) host array when constructed observation-major

    @classmethod
    def from_device(cls, V_obs_major, nu=None, labels=None, *, p_total: int | None = None,
                    release: bool = False):
        """Wrap a CUDA tensor holding observations row-wise (p x n, each row one v_l).

        This is the layout the kernels use, so nothing is transposed or copied to the host;
        the tensor is validated and uploaded device-to-device.  ``p_total`` (row shards only)
        sets the uniform weight to 1/p_total instead of 1/p.  ``release=True`` drops this
        object's reference to the tensor once it is uploaded (HBM for very large sets: the
        context keeps its own copy), after which ``V`` is no longer available.
        """
        import torch

        if not (_is_torch_tensor(V_obs_major) and V_obs_major.is_cuda):
            raise TypeError("from_device expects a CUDA tensor")
        if V_obs_major.ndim != 2:
            raise ValueError(f"V must be a 2-D matrix, got ndim={V_obs_major.ndim}")
        if V_obs_major.dtype not in (torch.float32, torch.float64):
            raise ValueError("V must be float32 or float64")
        p, n = V_obs_major.shape
        if n < 1 or p < 1:
            raise ValueError(f"V must be at least 1x1, got shape {(n, p)}")
        self = cls.__new__(cls)
        self._Vsrc = None
        self._V64 = None
        self._n, self._p = int(n), int(p)
        self._uniform_default = nu is None
        self.nu = _check_nu(nu, p) if nu is not None else None
        self._nu_const = 1.0 / float(p_total if p_total is not None else p)
        self.labels = _check_labels(labels, p)
        self._device = V_obs_major.device.index or 0
        self._dev = None
        self._dev_lock = threading.Lock()
        self._dev_obs = V_obs_major.contiguous()
        self._release = bool(release)
        return self

    @classmethod
    def from_obs_major_host(cls, V_pn, nu=None, labels=None, *, p_total: int | None = None,
                            device: int | None = None):
        """Wrap a host (p x n) observation-major array (e.g. a memory-mapped MOMV payload).

        Nothing is copied or validated on the host: the upload copies the rows into HBM and
        checks finiteness on the device (ValueError on failure, like dense.py:87-88).
        """
        V_pn = np.asarray(V_pn) if not isinstance(V_pn, np.memmap) else V_pn
        if V_pn.ndim != 2:
            raise ValueError(f"V must be a 2-D matrix, got ndim={V_pn.ndim}")
        p, n = V_pn.shape
        if n < 1 or p < 1:
            raise ValueError(f"V must be at least 1x1, got shape {(n, p)}")
        self = cls.__new__(cls)
        self._Vsrc = None
        self._V64 = None
        self._host_obs = V_pn
        self._n, self._p = int(n), int(p)
        self._uniform_default = nu is None
        self.nu = _check_nu(nu, p) if nu is not None else None
        self._nu_const = 1.0 / float(p_total if p_total is not None else p)
        self.labels = _check_labels(labels, p)
        self._device = device
        self._dev = None
        self._dev_lock = threading.Lock()
        self._dev_obs = None
        return self

    # -- reference surface ----------------------------------------------------------------
    @property
    def V(self) -> np.ndarray:
        """The (n, p) float64 observation matrix (host), as the reference exposes it."""
        if self._V64 is None:
            if self._Vsrc is not None:
                self._V64 = np.asarray(self._Vsrc, dtype=float)
            elif getattr(self, "_host_obs", None) is not None:
                self._V64 = np.asarray(self._host_obs, dtype=float).T
            else:
                if getattr(self, "_released", False):
                    raise RuntimeError("V was released after the upload (from_device(release=True))")
                self._V64 = self._dev_obs.double().t().cpu().numpy()
        return self._V64

    @property
    def n(self) -> int:
        return self._n

    @property
    def p(self) -> int:
        return self._p

    def has_uniform_weights(self, rtol: float = 1e-14) -> bool:
        nu = self.weights()
        return bool(np.allclose(nu, 1.0 / self.p, rtol=rtol, atol=0.0))

    def weights(self) -> np.ndarray:
        if self.nu is None:
            self.nu = np.full(self._p, self._nu_const)
        return self.nu

    # -- device side ----------------------------------------------------------------------
    def device_context(self) -> _native.Context:
        """The mcp context holding this set in HBM (created and uploaded on first call)."""
        with self._dev_lock:
            if self._dev is None:
                dev = self._device
                if dev is None:
                    dev = _current_device()
                ctx = _native.Context(dev)
                if self._dev_obs is not None:
                    t = self._dev_obs
                    code = _native.MCP_F64 if t.element_size() == 8 else _native.MCP_F32
                    nu_ptr = None
                    self._nu_dev = None
                    if self.nu is not None and not self._uniform_default:
                        import torch

                        self._nu_dev = torch.as_tensor(self.nu, dtype=torch.float64,
                                                       device=t.device)
                        nu_ptr = self._nu_dev.data_ptr()
                    ctx.load_obs_device(t.data_ptr(), code, _native.MCP_OBS_MAJOR, self._n,
                                        self._p, t.stride(0), nu_ptr, self._nu_const)
                    if getattr(self, "_release", False):
                        import torch

                        torch.cuda.synchronize(t.device)
                        self._dev_obs = None
                        self._released = True
                elif getattr(self, "_host_obs", None) is not None:
                    nu = None if self._uniform_default else self.nu
                    ctx.load_obs_host(self._host_obs, _native.MCP_OBS_MAJOR, nu, self._nu_const)
                else:
                    nu = None if self._uniform_default else self.nu
                    ctx.load_obs_host(self._Vsrc, _native.MCP_VAR_MAJOR, nu, 1.0 / self._p)
                self._dev = ctx
            return self._dev


def _current_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except ImportError:  # torch is plumbing only; the library works without it
        pass
    return 0


def _is_torch_tensor(x) -> bool:
    t = type(x)
    return t.__module__.startswith("torch") and t.__name__ == "Tensor"


def _check_nu(nu, p: int) -> np.ndarray:
    if nu is None:
        return np.full(p, 1.0 / p)
    nu = np.asarray(nu, dtype=float)
    if nu.shape != (p,):
        raise ValueError(f"nu must have length p={p}, got shape {nu.shape}")
    if not np.isfinite(nu).all() or np.any(nu <= 0.0):
        raise ValueError("nu entries must be finite and strictly positive")
    return nu


def _check_labels(labels, p: int):
    if labels is None:
        return None
    labels = np.asarray(labels)
    if labels.shape != (p,):
        raise ValueError(f"labels must have length p={p}")
    return labels
