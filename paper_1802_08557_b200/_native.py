"""ctypes binding of libblp.so (include/blp.h).

The CUDA library is the product: there is no CPU fallback.  If the shared
object is missing, or no CUDA device is visible, every solve raises
``NativeUnavailable`` instead of silently computing on the host.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("BLP_LIBRARY", PKG_DIR / "libblp.so"))

BLP_OK = 0
ERRORS = {-1: "invalid arguments", -2: "CUDA error", -3: "LP shape too large"}


class NativeUnavailable(RuntimeError):
    """libblp.so cannot be loaded or no CUDA device is usable."""


class NativeError(RuntimeError):
    """libblp.so returned an error code."""


class Limits(ctypes.Structure):
    """blp_limits (include/blp.h) = SolverLimits (simplex.py:34-60)."""

    _fields_ = [("max_iterations", ctypes.c_int32),
                ("anti_cycling", ctypes.c_int32),
                ("degenerate_limit", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


_lib = None

# Every function include/blp.h declares; tests/test_native_abi.py checks the exports.
EXPORTS = ("blp_solve_batch_device", "blp_solve_batch_host", "blp_solve_batch_gather", "blp_shape_supported",
           "blp_kernel_variant", "blp_kernel_variant_mode", "blp_launch_count", "blp_last_error", "blp_abi_version",
           "blp_probe_smem_gbs", "blp_probe_fp64_gflops", "blp_box_solve_device", "blp_box_solve_host",
           "blp_certify_batch_device", "blp_certify_batch_host", "blp_certify_reprice_device",
           "blp_certify_reprice_host")


def load():
    """Load libblp.so (no CUDA call is made here)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeUnavailable(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(str(LIB_PATH))
    P = ctypes.c_void_p
    sig = [P, P, P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
           ctypes.POINTER(Limits), P, P, P, P, P]
    lib.blp_solve_batch_device.argtypes = sig + [P]
    lib.blp_solve_batch_device.restype = ctypes.c_int
    lib.blp_solve_batch_host.argtypes = sig + [ctypes.c_int32]
    lib.blp_solve_batch_host.restype = ctypes.c_int
    lib.blp_solve_batch_gather.argtypes = [P, P, P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.POINTER(Limits), P, P, P, P, P, ctypes.c_int32]
    lib.blp_solve_batch_gather.restype = ctypes.c_int
    lib.blp_shape_supported.argtypes = [ctypes.c_int32, ctypes.c_int32]
    lib.blp_shape_supported.restype = ctypes.c_int
    lib.blp_kernel_variant.argtypes = [ctypes.c_int32, ctypes.c_int32]
    lib.blp_kernel_variant.restype = ctypes.c_char_p
    lib.blp_kernel_variant_mode.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
    lib.blp_kernel_variant_mode.restype = ctypes.c_char_p
    lib.blp_launch_count.argtypes = []
    lib.blp_launch_count.restype = ctypes.c_int64
    lib.blp_last_error.argtypes = []
    lib.blp_last_error.restype = ctypes.c_char_p
    lib.blp_probe_smem_gbs.argtypes = [ctypes.c_int32]
    lib.blp_probe_smem_gbs.restype = ctypes.c_double
    lib.blp_probe_fp64_gflops.argtypes = [ctypes.c_int32]
    lib.blp_probe_fp64_gflops.restype = ctypes.c_double
    lib.blp_abi_version.argtypes = []
    lib.blp_abi_version.restype = ctypes.c_int
    box = [P, P, P, ctypes.c_int64, ctypes.c_int32, P, P, P]
    lib.blp_box_solve_device.argtypes = box + [P]
    lib.blp_box_solve_device.restype = ctypes.c_int
    lib.blp_box_solve_host.argtypes = box + [ctypes.c_int32]
    lib.blp_box_solve_host.restype = ctypes.c_int
    cert = [P, P, P, P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, ctypes.c_double,
            P, P, P, P]
    lib.blp_certify_batch_device.argtypes = cert + [P]
    lib.blp_certify_batch_device.restype = ctypes.c_int
    lib.blp_certify_batch_host.argtypes = cert + [ctypes.c_int32]
    lib.blp_certify_batch_host.restype = ctypes.c_int
    rep = [P, P, P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P]
    lib.blp_certify_reprice_device.argtypes = rep + [P]
    lib.blp_certify_reprice_device.restype = ctypes.c_int
    lib.blp_certify_reprice_host.argtypes = rep + [ctypes.c_int32]
    lib.blp_certify_reprice_host.restype = ctypes.c_int
    _lib = lib
    return lib


def box_solve_host(lower: np.ndarray, upper: np.ndarray, direction: np.ndarray, device: int = 0) -> dict:
    """Packed hyper-rectangle LPs [count, n] -> value, point, status (blp_box_solve_host)."""
    lib = load()
    _require_gpu()
    count, n = direction.shape
    out = dict(value=alloc_host((count,)), point=alloc_host((count, n)), status=alloc_host((count,), np.int32))
    _check(lib.blp_box_solve_host(_ptr(lower), _ptr(upper), _ptr(direction), count, n, _ptr(out["value"]),
                                  _ptr(out["point"]), _ptr(out["status"]), int(device)))
    return out


def certify_host(A, b, c, x, status, tol: float, *, shared_Ab: bool = False, device: int = 0) -> dict:
    """Batched certificates of packed LPs + points (blp_certify_batch_host)."""
    lib = load()
    _require_gpu()
    count, n = c.shape
    m = b.shape[-1]
    out = dict(max_reduced_cost=np.empty(count), max_violation=np.empty(count), max_negativity=np.empty(count),
               needs_prices=np.empty(count, np.int8))
    _check(lib.blp_certify_batch_host(_ptr(A), _ptr(b), _ptr(c), _ptr(x), count, m, n, int(shared_Ab),
                                      _ptr(status), float(tol), _ptr(out["max_reduced_cost"]),
                                      _ptr(out["max_violation"]), _ptr(out["max_negativity"]),
                                      _ptr(out["needs_prices"]), int(device)))
    return out


def certify_reprice_host(A, c, y, mask, max_reduced_cost, *, shared_Ab: bool = False, device: int = 0) -> None:
    """In place: max_reduced_cost[k] = max(c - A^T y_k, -y_k) where mask[k] (blp_certify_reprice_host)."""
    lib = load()
    _require_gpu()
    count, n = c.shape
    m = y.shape[-1]
    _check(lib.blp_certify_reprice_host(_ptr(A), _ptr(c), _ptr(y), count, m, n, int(shared_Ab), _ptr(mask),
                                        _ptr(max_reduced_cost), int(device)))


def _check(rc: int) -> None:
    if rc != BLP_OK:
        msg = load().blp_last_error().decode(errors="replace")
        raise NativeError(f"libblp: {ERRORS.get(rc, rc)}: {msg}")


def _require_gpu() -> None:
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device is visible; the batched simplex runs only on the GPU")


def make_limits(max_iterations=None, anti_cycling=True, degenerate_pivot_limit=None) -> Limits:
    return Limits(0 if max_iterations is None else int(max_iterations),
                  1 if anti_cycling else 0,
                  -1 if degenerate_pivot_limit is None else int(degenerate_pivot_limit), 0)


def kernel_variant(m: int, n: int, shared_Ab: bool = False) -> str:
    return load().blp_kernel_variant_mode(m, n, 1 if shared_Ab else 0).decode()


def probe_smem_gbs(device: int = 0) -> float:
    """Measured LDS+STS bandwidth of one GPU (GB/s)."""
    _require_gpu()
    v = float(load().blp_probe_smem_gbs(int(device)))
    if v < 0:
        raise NativeError("smem probe failed: " + load().blp_last_error().decode())
    return v


def probe_fp64_gflops(device: int = 0) -> float:
    """Measured unfused FP64 rate of one GPU (GFLOP/s, DMUL and DADD one flop each)."""
    _require_gpu()
    v = float(load().blp_probe_fp64_gflops(int(device)))
    if v < 0:
        raise NativeError("fp64 probe failed: " + load().blp_last_error().decode())
    return v


def launch_count() -> int:
    return int(load().blp_launch_count())


def solve_host(A: np.ndarray, b: np.ndarray, c: np.ndarray, limits: Limits, *, shared_Ab: bool = False,
               device: int = 0, out: dict | None = None) -> dict:
    """Host arrays in, host arrays out (blp_solve_batch_host).  A/b/c must be C-contiguous fp64."""
    lib = load()
    _require_gpu()
    count, n = c.shape
    m = b.shape[-1]
    if out is None:
        out = alloc_outputs(count, n)
    _check(lib.blp_solve_batch_host(_ptr(A), _ptr(b), _ptr(c), count, m, n, 1 if shared_Ab else 0,
                                    ctypes.byref(limits), _ptr(out["status"]), _ptr(out["objective"]),
                                    _ptr(out["x"]), _ptr(out["it1"]), _ptr(out["it2"]), int(device)))
    return out


def solve_gather(ptrs: bytes, count: int, m: int, n: int, limits: Limits, *, device: int = 0,
                 out: dict | None = None, first: int = 0) -> dict:
    """One pointer per LP array (blp_solve_batch_gather): `ptrs` is int64[3][total] (A, b, c
    addresses, _pyobj.collect); LPs [first, first + count) are solved into `out`."""
    lib = load()
    _require_gpu()
    if out is None:
        out = alloc_outputs(count, n)
    if count == 0:
        return out
    total = len(ptrs) // 24
    base = ctypes.cast(ctypes.c_char_p(ptrs), ctypes.c_void_p).value
    pa, pb, pc = (base + 8 * (first + k * total) for k in range(3))
    _check(lib.blp_solve_batch_gather(pa, pb, pc, count, m, n, ctypes.byref(limits), _ptr(out["status"]),
                                      _ptr(out["objective"]), _ptr(out["x"]), _ptr(out["it1"]), _ptr(out["it2"]),
                                      int(device)))
    return out


def alloc_host(shape, dtype=np.float64) -> np.ndarray:
    """Page-locked host array when a GPU is visible (torch's caching pinned allocator), else plain."""
    import torch
    if torch.cuda.is_available():
        tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32,
               np.dtype(np.int8): torch.int8}[np.dtype(dtype)]
        return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
    return np.empty(shape, dtype)


def alloc_outputs(count: int, n: int) -> dict:
    """Result arrays in page-locked host memory (torch's caching pinned allocator), so the
    library's device->host copies stay asynchronous and overlap the next sub-batch."""
    import torch

    def pinned(shape, dtype):
        if torch.cuda.is_available():
            return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()
        return np.empty(shape, dtype=torch.empty(0, dtype=dtype).numpy().dtype)

    return dict(status=pinned((count,), torch.int8), objective=pinned((count,), torch.float64),
                x=pinned((count, n), torch.float64), it1=pinned((count,), torch.int32),
                it2=pinned((count,), torch.int32))


def solve_device(A, b, c, limits: Limits, out: dict, *, shared_Ab: bool = False, stream=None) -> None:
    """torch CUDA tensors in/out (blp_solve_batch_device); enqueued on `stream`, not synchronised."""
    import torch
    lib = load()
    count, n = c.shape
    m = b.shape[-1]
    if stream is None:
        stream = torch.cuda.current_stream(c.device)
    _check(lib.blp_solve_batch_device(A.data_ptr(), b.data_ptr(), c.data_ptr(), count, m, n,
                                      1 if shared_Ab else 0, ctypes.byref(limits),
                                      out["status"].data_ptr(), out["objective"].data_ptr(),
                                      out["x"].data_ptr(), out["it1"].data_ptr(), out["it2"].data_ptr(),
                                      ctypes.c_void_p(stream.cuda_stream)))


def _ptr(a) -> int:
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    return a.data_ptr()  # torch tensor (pinned host or device)
