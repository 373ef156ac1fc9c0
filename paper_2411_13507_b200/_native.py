"""ctypes binding of libbzg.so (the C ABI declared in include/bzg.h).

Loading fails loudly: there is no CPU fallback for the graph stage.  The
library is built in-tree by ``paper_2411_13507_b200._build`` (or
``__graft_entry__.build()``) and loaded from this directory only.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libbzg.so"

BZG_OK, BZG_EINVAL, BZG_ENODEV, BZG_ECUDA, BZG_EUNSUPPORTED, BZG_ENOMEM = 0, -1, -2, -3, -4, -5


class BzgError(RuntimeError):
    """A libbzg call failed; ``code`` is the BZG_E* value."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"libbzg error {code}: {msg}")
        self.code = code


class BzgValueError(BzgError, ValueError):
    """BZG_EINVAL: invalid input, where the reference raises ValueError."""


class BuildDesc(C.Structure):
    _fields_ = [
        ("m", C.c_int32), ("gamma", C.c_int32), ("p", C.c_int32), ("n_F", C.c_int32),
        ("F", C.c_void_p), ("G", C.c_void_p), ("eps_geo", C.c_double), ("D", C.c_void_p),
        ("N", C.c_int64),
        ("pcg_state_hi", C.c_uint64), ("pcg_state_lo", C.c_uint64),
        ("pcg_inc_hi", C.c_uint64), ("pcg_inc_lo", C.c_uint64),
        ("sample_lo", C.c_void_p), ("sample_hi", C.c_void_p),
        ("xd_rows", C.c_int32), ("xd_A", C.c_void_p), ("xd_b", C.c_void_p),
        ("n_include", C.c_int64), ("include", C.c_void_p),
        ("vertices", C.c_void_p),
        ("row_begin", C.c_int64), ("row_end", C.c_int64),
        ("n_regions", C.c_int32), ("region_row_off", C.c_void_p), ("region_F", C.c_void_p),
        ("region_G", C.c_void_p), ("region_box_lo", C.c_void_p), ("region_box_hi", C.c_void_p),
        ("k_nearest", C.c_int64),
    ]

    def __init__(self, *args, **kw):
        super().__init__(*args, **kw)
        if "k_nearest" not in kw:
            self.k_nearest = -1  # prefilter off


class CutConfigC(C.Structure):
    _fields_ = [
        ("eps_cut", C.c_double), ("heur_margin", C.c_double), ("eps_geo", C.c_double),
        ("qp_max_iter", C.c_int32),
        ("qp_eps_abs", C.c_double), ("qp_eps_rel", C.c_double), ("qp_rho", C.c_double),
        ("qp_sigma", C.c_double), ("qp_alpha", C.c_double), ("qp_eps_pinf", C.c_double),
        ("qp_polish", C.c_int32),
    ]


class RegionSampler(C.Structure):
    """bzg_region_sampler (include/bzg.h): the keep-in sampler of a planner."""
    _fields_ = [("n_regions", C.c_int32), ("N", C.c_void_p), ("pcg", C.c_void_p), ("lo", C.c_void_p),
                ("hi", C.c_void_p), ("row_off", C.c_void_p), ("A", C.c_void_p), ("b", C.c_void_p)]


_P = C.c_void_p
_SIGS = {
    "bzg_abi_version": ([], C.c_int),
    "bzg_last_error": ([], C.c_char_p),
    "bzg_ctx_create": ([C.c_int, _P, C.POINTER(_P)], C.c_int),
    "bzg_ctx_destroy": ([_P], C.c_int),
    "bzg_ctx_stream": ([_P, C.POINTER(_P)], C.c_int),
    "bzg_ctx_synchronize": ([_P], C.c_int),
    "bzg_ctx_set_profiling": ([_P, C.c_int], C.c_int),
    "bzg_ctx_profile_only": ([_P, C.c_char_p], C.c_int),
    "bzg_ctx_stats": ([_P, C.POINTER(C.c_longlong), C.c_int, C.c_char_p, _P, _P, C.POINTER(C.c_int)], C.c_int),
    "bzg_ctx_reset_stats": ([_P], C.c_int),
    "bzg_build_graph": ([_P, C.POINTER(BuildDesc), C.POINTER(_P)], C.c_int),
    "bzg_sample_states": ([_P, C.POINTER(BuildDesc), _P], C.c_int),
    "bzg_graph_eps_band": ([_P, C.POINTER(BuildDesc), C.c_double, _P], C.c_int),
    "bzg_graph_from_edges": ([_P, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int64, _P, C.c_int64, _P, _P, _P,
                              C.c_int, C.POINTER(_P)], C.c_int),
    "bzg_graph_with_edges": ([_P, C.c_int64, _P, _P, _P, C.c_int, C.POINTER(_P)], C.c_int),
    "bzg_graph_set_edges": ([_P, C.c_int64, _P, _P, _P, C.c_int], C.c_int),
    "bzg_graph_set_cut_cache": ([_P, C.c_int32], C.c_int),
    "bzg_graph_destroy": ([_P], C.c_int),
    "bzg_graph_info": ([_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                        C.POINTER(C.c_int64)], C.c_int),
    "bzg_graph_copy_vertices": ([_P, _P], C.c_int),
    "bzg_graph_copy_edges": ([_P, _P, _P], C.c_int),
    "bzg_graph_copy_points": ([_P, _P], C.c_int),
    "bzg_graph_copy_csr": ([_P, _P, _P], C.c_int),
    "bzg_graph_export_device": ([_P, _P, _P, _P], C.c_int),
    "bzg_check_edges": ([_P, C.c_int32, C.c_int32, _P, _P, C.c_double, C.c_int64, _P, _P, _P], C.c_int),
    "bzg_cut_graph": ([_P, _P, C.c_int32, _P, _P, _P, _P, _P, _P, C.POINTER(CutConfigC), C.POINTER(_P)], C.c_int),
    "bzg_sample_region_states": ([_P, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _P, _P, C.c_double, _P], C.c_int),
    "bzg_cut_points": ([_P, C.c_int32, C.c_int32, C.c_int64, _P, _P, C.c_int32, _P, _P, _P, _P, _P, _P,
                        C.POINTER(CutConfigC), C.c_int32, _P, _P, _P], C.c_int),
    "bzg_mask_destroy": ([_P], C.c_int),
    "bzg_mask_copy": ([_P, _P, _P, _P], C.c_int),
    "bzg_mask_info": ([_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
    "bzg_mask_qp_count": ([_P, C.POINTER(C.c_int64)], C.c_int),
    "bzg_mask_copy_qp": ([_P, _P, _P, _P, _P, _P], C.c_int),
    "bzg_mask_from_arrays": ([_P, _P, _P, _P, _P, C.c_int, C.POINTER(_P)], C.c_int),
    "bzg_mask_export_device": ([_P, _P, _P], C.c_int),
    "bzg_find_path": ([_P, _P, _P, _P, _P, _P, _P, C.c_double, C.c_int, C.c_int, _P, C.c_int64,
                       C.POINTER(C.c_int64), C.POINTER(C.c_double)], C.c_int),
    "bzg_query_create": ([_P, _P, _P, _P, _P, C.c_double, C.c_int, C.c_int, C.POINTER(_P)], C.c_int),
    "bzg_query_run": ([_P, _P, _P, _P, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_double)], C.c_int),
    "bzg_query_kernels": ([_P, C.POINTER(C.c_int64)], C.c_int),
    "bzg_query_destroy": ([_P], C.c_int),
    "bzg_replanner_create": ([_P, _P, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_double, C.c_int,
                              C.c_int, C.POINTER(_P)], C.c_int),
    "bzg_replanner_run": ([_P, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int64, C.POINTER(C.c_int64),
                           C.POINTER(C.c_double), _P, C.POINTER(C.c_int32)], C.c_int),
    "bzg_replanner_mask": ([_P, C.POINTER(_P)], C.c_int),
    "bzg_replanner_info": ([_P, _P], C.c_int),
    "bzg_replanner_destroy": ([_P], C.c_int),
    "bzg_planner_create": ([_P, _P, _P, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_double, C.c_int,
                            C.c_int, C.POINTER(_P)], C.c_int),
    "bzg_planner_run": ([_P, _P, _P, C.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int64, C.POINTER(C.c_int64),
                         C.POINTER(C.c_double), _P, C.POINTER(C.c_int64), C.POINTER(C.c_int32)], C.c_int),
    "bzg_planner_result": ([_P, C.POINTER(_P), C.POINTER(_P)], C.c_int),
    "bzg_planner_info": ([_P, _P], C.c_int),
    "bzg_planner_destroy": ([_P], C.c_int),
    "bzg_project_on_path": ([_P, C.c_int32, C.c_int32, C.c_double, _P, C.c_int64, _P, C.c_double, C.c_int32, _P,
                             C.POINTER(C.c_double)], C.c_int),
    "bzg_probe_fp64": ([_P, C.c_int, C.POINTER(C.c_double)], C.c_int),
}
EXPORTS = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load(path: Path | str | None = None):
    """Load libbzg.so and declare every exported signature.  Raises if absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise ImportError(
                f"{p} is missing: build the CUDA library first "
                "(python -m paper_2411_13507_b200._build); there is no CPU fallback")
        lib = C.CDLL(str(p))
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.bzg_abi_version() != 1:
            raise ImportError("libbzg ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != BZG_OK:
        msg = _lib.bzg_last_error().decode(errors="replace") if _lib is not None else "?"
        raise (BzgValueError if rc == BZG_EINVAL else BzgError)(rc, msg)


def ptr(a: np.ndarray | None):
    """Raw data pointer of a C-contiguous array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays crossing the C ABI must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


class Context:
    """One libbzg context: a CUDA device and a stream (bzg_ctx_create)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.lib = load()
        h = C.c_void_p()
        check(self.lib.bzg_ctx_create(int(device), C.c_void_p(stream) if stream else None, C.byref(h)))
        self.handle = h
        self.device = device

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        check(self.lib.bzg_ctx_stream(self.handle, C.byref(s)))
        return int(s.value or 0)

    def synchronize(self):
        check(self.lib.bzg_ctx_synchronize(self.handle))

    def set_profiling(self, on: bool):
        check(self.lib.bzg_ctx_set_profiling(self.handle, int(bool(on))))

    def profile_only(self, kernel: str | None):
        check(self.lib.bzg_ctx_profile_only(self.handle, kernel.encode() if kernel else None))

    def reset_stats(self):
        check(self.lib.bzg_ctx_reset_stats(self.handle))

    def stats(self) -> tuple[int, dict]:
        """(launch count, {kernel: (total_ms, launches)}) since the last reset."""
        cap = 128
        names = C.create_string_buffer(64 * cap)
        ms = np.zeros(cap)
        cnt = np.zeros(cap, dtype=np.int64)
        n = C.c_int()
        launches = C.c_longlong()
        check(self.lib.bzg_ctx_stats(self.handle, C.byref(launches), cap, names, ptr(ms), ptr(cnt), C.byref(n)))
        out = {}
        for i in range(min(n.value, cap)):
            nm = names.raw[64 * i: 64 * i + 64].split(b"\0", 1)[0].decode()
            out[nm] = (float(ms[i]), int(cnt[i]))
        return launches.value, out

    def probe_fp64(self, use_fma: bool = True) -> float:
        """Measured FP64 instruction issue rate (instructions/s) of this device."""
        r = C.c_double()
        check(self.lib.bzg_probe_fp64(self.handle, int(bool(use_fma)), C.byref(r)))
        return r.value

    def close(self):
        if getattr(self, "handle", None):
            self.lib.bzg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    """Process-wide context on the current CUDA device (LOCAL_RANK when set)."""
    global _default_ctx
    if _default_ctx is None:
        import os

        dev = int(os.environ.get("BZG_DEVICE", os.environ.get("LOCAL_RANK", "0")))
        _default_ctx = Context(dev)
    return _default_ctx


def set_default_context(ctx: Context | None) -> None:
    global _default_ctx
    _default_ctx = ctx
