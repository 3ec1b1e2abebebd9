"""ctypes binding of the C ABI in ``include/momentcp_b200.h`` (``_lib/libmomentcp_b200.so``).

There is no CPU fallback: if the shared library is missing, or no B200 is visible, every entry
point raises.  Argument errors reported by the library (``MCP_ERR_ARG``) surface as
``ValueError`` -- the exception the reference raises for the same conditions
(pkg/src/momentcp/objective.py:38-48, pkg/src/momentcp/implicit.py:102-105) -- and CUDA failures
as ``RuntimeError``.  ctypes releases the GIL for the duration of each call; the library
serialises calls per context, so pool threads may share one observation set
(pkg/src/momentcp/optimize.py:484-493).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

LIB_PATH = os.environ.get("MCP_LIBRARY") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "_lib", "libmomentcp_b200.so")  # env: A/B builds

MCP_OK, MCP_ERR_ARG, MCP_ERR_CUDA, MCP_ERR_STATE = 0, 1, 2, 3
MCP_F64, MCP_F32 = 0, 1
MCP_VAR_MAJOR, MCP_OBS_MAJOR = 0, 1
MODES = {"fp64": 0, "tf32x3": 1}
MCP_OPT_FUSED_TAIL = 1
MCP_OPT_SMALL_KERNEL = 2

# name -> (restype, argtypes); every symbol include/momentcp_b200.h declares
_c_void_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
# void (*)(const double* x, int64_t len, void* user)  (mcp_iterate_hook)
IterateHook = ctypes.CFUNCTYPE(None, ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.c_void_p)

# int (*)(int64_t* idx, int64_t count, void* user)  (mcp_sample_fn)
SampleFn = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
                            ctypes.c_void_p)

SIGNATURES = {
    "mcp_abi_version": (ctypes.c_int, []),
    "mcp_last_error": (ctypes.c_char_p, [_c_void_p]),
    "mcp_create": (ctypes.c_int, [ctypes.POINTER(_c_void_p), ctypes.c_int]),
    "mcp_destroy": (ctypes.c_int, [_c_void_p]),
    "mcp_device_sms": (ctypes.c_int, [_c_void_p]),
    "mcp_load_obs": (ctypes.c_int, [_c_void_p, _c_void_p, ctypes.c_int, ctypes.c_int, _i64, _i64,
                                    _i64, _c_void_p, ctypes.c_double]),
    "mcp_load_obs_device": (ctypes.c_int, [_c_void_p, _c_void_p, ctypes.c_int, ctypes.c_int, _i64,
                                           _i64, _i64, _c_void_p, ctypes.c_double]),
    "mcp_obs_shape": (ctypes.c_int, [_c_void_p, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "mcp_fg": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, _c_void_p, _c_void_p,
                              ctypes.c_double, ctypes.c_int, _dp, _c_void_p, _c_void_p]),
    "mcp_fg_packed": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, _c_void_p,
                                     ctypes.c_double, ctypes.c_int, _dp, _c_void_p]),
    "mcp_fg_batch": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_void_p,
                                    ctypes.c_double, ctypes.c_int, _c_void_p, _c_void_p]),
    "mcp_ttsv_batch": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, _c_void_p,
                                      ctypes.c_int, _c_void_p]),
    "mcp_data_norm_sq": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, _dp]),
    "mcp_data_norm_sq_part": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, _dp]),
    "mcp_data_norm_sq_cross": (ctypes.c_int, [_c_void_p, _c_void_p, _i64, _c_void_p,
                                              ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]),
    "mcp_obs_device_view": (ctypes.c_int, [_c_void_p, ctypes.POINTER(_c_void_p),
                                           ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                           ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(_c_void_p),
                                           ctypes.POINTER(ctypes.c_double)]),
    "mcp_fg_partial_device": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, _c_void_p,
                                             ctypes.c_int, _c_void_p, _c_void_p]),
    "mcp_fg_finish_device": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, _c_void_p,
                                            _c_void_p, ctypes.c_double, _c_void_p, _c_void_p]),
    "mcp_fg_device": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, _c_void_p,
                                     ctypes.c_double, ctypes.c_int, _c_void_p, _c_void_p]),
    "mcp_set_kernel_timing": (ctypes.c_int, [_c_void_p, ctypes.c_int]),
    "mcp_set_option": (ctypes.c_int, [_c_void_p, ctypes.c_int, _i64]),
    "mcp_kernel_time_ms": (ctypes.c_int, [_c_void_p, _dp, ctypes.POINTER(ctypes.c_int),
                                          ctypes.c_int]),
    "mcp_lbfgs": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                 ctypes.c_int, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _dp,
                                 _c_void_p, _c_void_p, _i64, _c_void_p, IterateHook, _c_void_p]),
    "mcp_lbfgs_batch": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_double, ctypes.c_int, _c_void_p, _c_void_p,
                                       _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
                                       _i64, _c_void_p]),
    "mcp_lbfgs_batch_errors": (ctypes.c_char_p, []),
    "mcp_gather_rows": (ctypes.c_int, [_c_void_p, _c_void_p, _i64, _c_void_p, _i64, ctypes.c_int]),
    "mcp_adam": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _c_void_p,
                                _c_void_p, _c_void_p, _i64, SampleFn, _c_void_p, _c_void_p,
                                _c_void_p, _dp, _c_void_p, _c_void_p, _i64, _c_void_p]),
    "mcp_peer_signal": (ctypes.c_int, [_c_void_p, _c_void_p, ctypes.c_int, ctypes.c_int, _i64,
                                       _c_void_p]),
    "mcp_fg_partial_signal_device": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int,
                                                    _c_void_p, ctypes.c_int, _c_void_p, _c_void_p,
                                                    ctypes.c_int, ctypes.c_int, _i64, _c_void_p]),
    "mcp_peer_reduce_finish": (ctypes.c_int, [_c_void_p, ctypes.c_int, ctypes.c_int, _c_void_p,
                                              _c_void_p, _c_void_p, ctypes.c_int, _i64,
                                              ctypes.c_double, _c_void_p, _c_void_p, _c_void_p]),
    "mcp_last_launch_count": (ctypes.c_int, [_c_void_p]),
    "mcp_last_variant": (ctypes.c_char_p, [_c_void_p]),
}

_lib = None
_lib_lock = threading.Lock()


def load_library():
    """Load (once) and type the C ABI; raises if the native build is missing."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"native library not built: {LIB_PATH} is missing "
                    "(run `python -c 'import __graft_entry__ as g; g.build()'`); "
                    "there is no CPU fallback for this path"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                # an A/B build selected with MCP_LIBRARY may predate newer entry points
                fn = getattr(lib, name, None)
                if fn is None and os.environ.get("MCP_LIBRARY"):
                    continue
                if fn is None:
                    raise RuntimeError(f"{LIB_PATH} does not export {name}")
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def mode_code(mode: str | None) -> int:
    if mode is None:
        mode = "fp64"
    try:
        return MODES[mode]
    except KeyError:
        raise ValueError(f"unknown mode {mode!r}; expected one of {sorted(MODES)}") from None


def stream_handle(torch_stream) -> int:
    """C-ABI stream argument for a torch stream: torch reports the legacy default stream as 0,
    which the ABI reserves for "the context's own stream", so map it to cudaStreamLegacy (1)."""
    h = int(torch_stream.cuda_stream)
    return h if h != 0 else 1


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Context:
    """One device context holding one observation set (mcp_ctx*)."""

    def __init__(self, device: int = 0):
        self._lib = load_library()
        h = ctypes.c_void_p()
        rc = self._lib.mcp_create(ctypes.byref(h), int(device))
        if rc != MCP_OK:
            msg = self._lib.mcp_last_error(None).decode()
            raise RuntimeError(f"mcp_create(device={device}) failed: {msg}")
        self._h = h
        self.device = int(device)
        self.dtype_code = None  # set by the load calls

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.mcp_destroy(h)
            except Exception:  # noqa: BLE001 -- interpreter teardown
                pass
            self._h = None

    # -- error mapping --------------------------------------------------------------------
    def _check(self, rc: int, what: str) -> None:
        if rc == MCP_OK:
            return
        msg = self._lib.mcp_last_error(self._h).decode()
        if rc == MCP_ERR_ARG:
            raise ValueError(msg)
        raise RuntimeError(f"{what}: {msg}")

    @property
    def sms(self) -> int:
        return int(self._lib.mcp_device_sms(self._h))

    @property
    def last_launch_count(self) -> int:
        return int(self._lib.mcp_last_launch_count(self._h))

    @property
    def last_variant(self) -> str:
        return self._lib.mcp_last_variant(self._h).decode()

    def set_option(self, key: int, value: int) -> None:
        """mcp_set_option (e.g. MCP_OPT_FUSED_TAIL)."""
        self._check(self._lib.mcp_set_option(self._h, int(key), int(value)), "mcp_set_option")

    # -- kernel timing (bench) ------------------------------------------------------------
    def set_kernel_timing(self, enable, every: int = 1) -> None:
        """enable: time K1/K5 launches with CUDA events; every > 1 samples one launch in every."""
        code = (max(int(every), 1) if every > 1 else 1) if enable else 0
        self._check(self._lib.mcp_set_kernel_timing(self._h, code), "timing")

    def kernel_time_ms(self, reset: bool = True) -> tuple[float, int]:
        ms = ctypes.c_double()
        k = ctypes.c_int()
        rc = self._lib.mcp_kernel_time_ms(self._h, ctypes.byref(ms), ctypes.byref(k), int(reset))
        self._check(rc, "mcp_kernel_time_ms")
        return ms.value, k.value

    # -- observation upload ---------------------------------------------------------------
    def load_obs_host(self, V: np.ndarray, layout: int, nu: np.ndarray | None, nu_const: float):
        if V.dtype == np.float32:
            dt = MCP_F32
        elif V.dtype == np.float64 and V.dtype.byteorder in ("=", "<", "|"):
            dt = MCP_F64
        else:
            V = np.ascontiguousarray(V, dtype=np.float64)
            dt = MCP_F64
        if not (isinstance(V, np.memmap) and V.flags.c_contiguous):
            V = np.ascontiguousarray(V)
        if layout == MCP_VAR_MAJOR:
            n, p = V.shape
            ld = p
        else:
            p, n = V.shape
            ld = n
        nu_arr = None if nu is None else np.ascontiguousarray(nu, dtype=np.float64)
        rc = self._lib.mcp_load_obs(self._h, _ptr(V), dt, layout, n, p, ld,
                                    None if nu_arr is None else _ptr(nu_arr), float(nu_const))
        self._check(rc, "mcp_load_obs")
        self.dtype_code = dt

    def load_obs_device(self, V_ptr: int, dtype_code: int, layout: int, n: int, p: int, ld: int,
                        nu_ptr: int | None, nu_const: float):
        rc = self._lib.mcp_load_obs_device(self._h, ctypes.c_void_p(V_ptr), dtype_code, layout,
                                           n, p, ld,
                                           None if nu_ptr is None else ctypes.c_void_p(nu_ptr),
                                           float(nu_const))
        self._check(rc, "mcp_load_obs_device")
        self.dtype_code = int(dtype_code)

    # -- evaluations (host buffers) --------------------------------------------------------
    def fg_packed(self, x: np.ndarray, n: int, d: int, r: int, alpha: float, mode: str | None):
        # hot path of every solver step: raw addresses (ints) instead of ctypes pointer objects;
        # the library checks finiteness while staging x
        x = np.ascontiguousarray(x, dtype=np.float64)
        g = np.empty(r + n * r, dtype=np.float64)
        f = ctypes.c_double()
        rc = self._lib.mcp_fg_packed(self._h, d, r, x.ctypes.data, alpha, mode_code(mode),
                                     ctypes.byref(f), g.ctypes.data)
        if rc:
            self._check(rc, "mcp_fg_packed")
        return f.value, g

    def fg(self, lam: np.ndarray, A_fortran: np.ndarray, d: int, alpha: float, mode: str | None):
        n, r = A_fortran.shape
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        A_fortran = np.asfortranarray(A_fortran, dtype=np.float64)
        g_lam = np.empty(r, dtype=np.float64)
        g_A = np.empty((n, r), dtype=np.float64, order="F")
        f = ctypes.c_double()
        rc = self._lib.mcp_fg(self._h, int(d), int(r), _ptr(lam), _ptr(A_fortran), float(alpha),
                              mode_code(mode), ctypes.byref(f), _ptr(g_lam), _ptr(g_A))
        self._check(rc, "mcp_fg")
        return f.value, g_lam, g_A

    def fg_batch(self, X: np.ndarray, n: int, d: int, r: int, alpha: float, mode: str | None):
        X = np.ascontiguousarray(X, dtype=np.float64)
        k = X.shape[0]
        F = np.empty(k, dtype=np.float64)
        G = np.empty_like(X)
        rc = self._lib.mcp_fg_batch(self._h, int(d), int(r), int(k), _ptr(X), float(alpha),
                                    mode_code(mode), _ptr(F), _ptr(G))
        self._check(rc, "mcp_fg_batch")
        return F, G

    def lbfgs(self, x0: np.ndarray, n: int, d: int, r: int, alpha: float, mode: str | None,
              opts, hook=None) -> dict:
        """Device-resident L-BFGS (mcp_lbfgs); opts = (memory, pgtol, max_iters,
        max_total_iters, c1, c2, max_line_steps)."""
        N = r + n * r
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        if x0.shape != (N,):
            raise ValueError(f"expected packed length {N}, got {x0.shape}")
        o = np.array([float(v) for v in opts], dtype=np.float64)
        cap = int(min(o[2], o[3])) + 1
        x = np.empty(N)
        g = np.empty(N)
        tf = np.empty(cap)
        tt = np.empty(cap)
        info = np.zeros(4, dtype=np.int64)
        f = ctypes.c_double()
        err: list[BaseException] = []

        def _hook(xp, length, _user):
            if err:
                return
            try:
                hook(np.ctypeslib.as_array(xp, shape=(length,)).copy())
            except BaseException as exc:  # re-raised after the native call returns
                err.append(exc)

        cb = IterateHook(_hook) if hook is not None else IterateHook()
        rc = self._lib.mcp_lbfgs(self._h, int(d), int(r), float(alpha), mode_code(mode), _ptr(x0),
                                 _ptr(o), _ptr(x), _ptr(g), ctypes.byref(f), _ptr(tf), _ptr(tt),
                                 cap, _ptr(info), cb, None)
        if err:
            raise err[0]
        self._check(rc, "mcp_lbfgs")
        k = int(info[3])
        return {"x": x, "g": g, "f": f.value, "n_fg": int(info[0]), "n_steps": int(info[1]),
                "reason": ("tolerance", "iteration cap", "line-search failure")[int(info[2])],
                "trace": list(zip(tf[:k].tolist(), tt[:k].tolist()))}

    def lbfgs_batch(self, X0: np.ndarray, n: int, d: int, r: int, alpha: float, mode, opts):
        """k lock-step device L-BFGS solves (mcp_lbfgs_batch); returns one dict per start."""
        X0 = np.ascontiguousarray(X0, dtype=np.float64)
        k, N = X0.shape
        if N != r + n * r:
            raise ValueError(f"expected packed length {r + n * r}, got {N}")
        o = np.array([float(v) for v in opts], dtype=np.float64)
        cap = int(min(o[2], o[3])) + 1
        X = np.empty_like(X0)
        G = np.empty_like(X0)
        F = np.empty(k)
        tf = np.empty((k, cap))
        tt = np.empty((k, cap))
        info = np.zeros((k, 4), dtype=np.int64)
        rc = self._lib.mcp_lbfgs_batch(self._h, int(k), int(d), int(r), float(alpha),
                                       mode_code(mode), _ptr(X0), _ptr(o), _ptr(X), _ptr(G),
                                       _ptr(F), _ptr(tf), _ptr(tt), cap, _ptr(info))
        self._check(rc, "mcp_lbfgs_batch")
        errs = {}
        for line in (self._lib.mcp_lbfgs_batch_errors() or b"").decode().splitlines():
            head, _, msg = line.partition(": ")
            errs[int(head.split()[1])] = msg
        reasons = ("tolerance", "iteration cap", "line-search failure", "error")
        out = []
        for s_ in range(k):
            nt = int(info[s_, 3])
            out.append({"x": X[s_].copy(), "g": G[s_].copy(), "f": float(F[s_]),
                        "n_fg": int(info[s_, 0]), "n_steps": int(info[s_, 1]),
                        "reason": reasons[int(info[s_, 2])], "error": errs.get(s_),
                        "trace": list(zip(tf[s_, :nt].tolist(), tt[s_, :nt].tolist()))})
        return out

    def gather_rows(self, idx: np.ndarray, dst_ptr: int, ld: int, dtype_code: int) -> None:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        rc = self._lib.mcp_gather_rows(self._h, _ptr(idx), int(idx.size), ctypes.c_void_p(dst_ptr),
                                       int(ld), int(dtype_code))
        self._check(rc, "mcp_gather_rows")

    def adam(self, x0: np.ndarray, n: int, d: int, r: int, mode: str | None, opts,
             est_idx: np.ndarray, sample) -> dict:
        """Device-resident Adam (mcp_adam); sample(count) -> int64 indices for one epoch."""
        N = r + n * r
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        o = np.array([float(v) for v in opts], dtype=np.float64)
        est_idx = np.ascontiguousarray(est_idx, dtype=np.int64)
        cap = int(o[7]) + 1
        x = np.empty(N)
        g = np.empty(N)
        tf = np.empty(cap)
        tt = np.empty(cap)
        info = np.zeros(4, dtype=np.int64)
        f = ctypes.c_double()
        err: list[BaseException] = []

        def _sample(buf, count, _user):
            try:
                np.ctypeslib.as_array(buf, shape=(count,))[:] = sample(int(count))
                return 0
            except BaseException as exc:  # re-raised after the native call returns
                err.append(exc)
                return 1

        cb = SampleFn(_sample)
        rc = self._lib.mcp_adam(self._h, int(d), int(r), mode_code(mode), _ptr(x0), _ptr(o),
                                _ptr(est_idx), int(est_idx.size), cb, None, _ptr(x), _ptr(g),
                                ctypes.byref(f), _ptr(tf), _ptr(tt), cap, _ptr(info))
        if err:
            raise err[0]
        self._check(rc, "mcp_adam")
        k = int(info[2])
        return {"x": x, "g": g, "f": f.value, "n_iter": int(info[0]), "unused_draws": int(info[3]),
                "reason": ("iteration cap", "learning-rate exhausted")[int(info[1])],
                "trace": list(zip(tf[:k].tolist(), tt[:k].tolist()))}

    def peer_signal(self, flag_ptrs_dev: int, rank: int, world: int, epoch: int, stream_ptr):
        rc = self._lib.mcp_peer_signal(self._h, ctypes.c_void_p(flag_ptrs_dev), int(rank),
                                       int(world), int(epoch), ctypes.c_void_p(stream_ptr))
        self._check(rc, "mcp_peer_signal")

    def fg_partial_signal_device(self, d, r, dx_ptr, mode, dYw_ptr, flag_ptrs_dev, rank, world,
                                 epoch, stream_ptr):
        rc = self._lib.mcp_fg_partial_signal_device(
            self._h, int(d), int(r), ctypes.c_void_p(dx_ptr), mode_code(mode),
            ctypes.c_void_p(dYw_ptr), ctypes.c_void_p(flag_ptrs_dev), int(rank), int(world),
            int(epoch), ctypes.c_void_p(stream_ptr))
        self._check(rc, "mcp_fg_partial_signal_device")

    def peer_reduce_finish(self, d, r, dx_ptr, part_ptrs_dev, my_flags_ptr, world, epoch, alpha,
                           dout_ptr, derr_ptr, stream_ptr):
        rc = self._lib.mcp_peer_reduce_finish(
            self._h, int(d), int(r), ctypes.c_void_p(dx_ptr), ctypes.c_void_p(part_ptrs_dev),
            ctypes.c_void_p(my_flags_ptr), int(world), int(epoch), float(alpha),
            ctypes.c_void_p(dout_ptr), ctypes.c_void_p(derr_ptr), ctypes.c_void_p(stream_ptr))
        self._check(rc, "mcp_peer_reduce_finish")

    def ttsv_batch(self, A_fortran: np.ndarray, d: int, mode: str | None) -> np.ndarray:
        n, r = A_fortran.shape
        A_fortran = np.asfortranarray(A_fortran, dtype=np.float64)
        Y = np.empty((n, r), dtype=np.float64, order="F")
        rc = self._lib.mcp_ttsv_batch(self._h, int(d), int(r), _ptr(A_fortran), mode_code(mode),
                                      _ptr(Y))
        self._check(rc, "mcp_ttsv_batch")
        return Y

    def data_norm_sq(self, d: int, mode: str | None, part: int = 0, nparts: int = 1) -> float:
        out = ctypes.c_double()
        if nparts == 1:
            rc = self._lib.mcp_data_norm_sq(self._h, int(d), mode_code(mode), ctypes.byref(out))
        else:
            rc = self._lib.mcp_data_norm_sq_part(self._h, int(d), mode_code(mode), int(part),
                                                 int(nparts), ctypes.byref(out))
        self._check(rc, "mcp_data_norm_sq")
        return out.value

    def data_norm_sq_cross(self, dVJ: int, p_pad_J: int, dnuJ: int | None, nu_const_J: float,
                           d: int, mode: str | None, part: int = 0, nparts: int = 1,
                           pair_order: int = 0) -> float:
        out = ctypes.c_double()
        rc = self._lib.mcp_data_norm_sq_cross(self._h, ctypes.c_void_p(dVJ), int(p_pad_J),
                                              None if not dnuJ else ctypes.c_void_p(dnuJ),
                                              float(nu_const_J), int(d), mode_code(mode),
                                              int(pair_order), int(part), int(nparts),
                                              ctypes.byref(out))
        self._check(rc, "mcp_data_norm_sq_cross")
        return out.value

    def obs_device_view(self) -> dict:
        """The resident observation buffer: ptr, ldv, p_pad (elements), dtype code, nu ptr."""
        dv, nu = ctypes.c_void_p(), ctypes.c_void_p()
        ldv, p_pad = ctypes.c_int64(), ctypes.c_int64()
        dt = ctypes.c_int()
        nc = ctypes.c_double()
        rc = self._lib.mcp_obs_device_view(self._h, ctypes.byref(dv), ctypes.byref(ldv),
                                           ctypes.byref(p_pad), ctypes.byref(dt),
                                           ctypes.byref(nu), ctypes.byref(nc))
        if rc != MCP_OK:
            raise RuntimeError("mcp_obs_device_view: no observation set loaded")
        return {"ptr": dv.value or 0, "ldv": ldv.value, "p_pad": p_pad.value, "dtype": dt.value,
                "nu": nu.value or 0, "nu_const": nc.value}

    # -- evaluations (device pointers, caller's stream) ------------------------------------
    def fg_partial_device(self, d, r, dx_ptr, mode, dYw_ptr, stream_ptr):
        rc = self._lib.mcp_fg_partial_device(self._h, int(d), int(r), ctypes.c_void_p(dx_ptr),
                                             mode_code(mode), ctypes.c_void_p(dYw_ptr),
                                             ctypes.c_void_p(stream_ptr))
        self._check(rc, "mcp_fg_partial_device")

    def fg_finish_device(self, d, r, dx_ptr, dYw_ptr, alpha, dout_ptr, stream_ptr):
        rc = self._lib.mcp_fg_finish_device(self._h, int(d), int(r), ctypes.c_void_p(dx_ptr),
                                            ctypes.c_void_p(dYw_ptr), float(alpha),
                                            ctypes.c_void_p(dout_ptr), ctypes.c_void_p(stream_ptr))
        self._check(rc, "mcp_fg_finish_device")

    def fg_device(self, d, r, dx_ptr, alpha, mode, dout_ptr, stream_ptr):
        rc = self._lib.mcp_fg_device(self._h, int(d), int(r), ctypes.c_void_p(dx_ptr),
                                     float(alpha), mode_code(mode), ctypes.c_void_p(dout_ptr),
                                     ctypes.c_void_p(stream_ptr))
        self._check(rc, "mcp_fg_device")
