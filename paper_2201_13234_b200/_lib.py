"""ctypes binding of the C-ABI in include/voxellate_b200.h.

This is the reference-side FFI a Python caller would bind.
The shared library is built in-tree by ``__graft_entry__.build()``; there is
no fallback of any kind: if it is missing, importing the package fails.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# VX_LIB=debug: the bounds-checked build; VX_LIB_PATH: an explicit library (A/B timing of builds)
LIB_PATH = os.environ.get("VX_LIB_PATH") or os.path.join(
    HERE, "libvoxellate_b200_debug.so" if os.environ.get("VX_LIB") == "debug" else "libvoxellate_b200.so")

VX_OK, VX_EINVAL, VX_ECUDA, VX_ENOMEM, VX_EUNSUPPORTED, VX_EIO = 0, 1, 2, 3, 4, 5
VX_MAX_DIM = 16


class vx_problem(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("dim", C.c_int32),
        ("periodic", C.c_int32),
        ("reserved0", C.c_int32),
        ("counts", C.c_int64 * VX_MAX_DIM),
        ("lengths", C.c_double * VX_MAX_DIM),
        ("n_sites", C.c_int64),
        ("positions", C.c_void_p),
        ("times", C.c_void_p),
        ("weights", C.c_void_p),
        ("growth", C.c_double),
    ]


class vx_options(C.Structure):
    _fields_ = [
        ("prune", C.c_int32),
        ("has_override", C.c_int32),
        ("override_param", C.c_double),
        ("device", C.c_int32),
        ("device_pointers", C.c_int32),
        ("stream", C.c_void_p),
        ("asynchronous", C.c_int32),
        ("profile_stages", C.c_int32),
        ("distances_out", C.c_void_p),
        ("histogram_out", C.c_void_p),
        ("slab_begin", C.c_int64),
        ("slab_end", C.c_int64),
        ("ball_scale", C.c_double),
        ("n_gpus", C.c_int32),
        ("reserved", C.c_int32),
    ]


class vx_stats(C.Structure):
    _fields_ = [
        ("param", C.c_double),
        ("n_voxels", C.c_int64),
        ("n_sites_kept", C.c_int64),
        ("n_unresolved", C.c_int64),
        ("ball_evals", C.c_uint64),
        ("shell_evals", C.c_uint64),
        ("engine", C.c_int32),
        ("kernel_launches", C.c_int32),
        ("overflow_bricks", C.c_uint64),
        ("stage_ms", C.c_float * 8),
    ]


STAGES = ("ingest", "bin", "params", "ball", "shell", "d2h")


def stats_dict(st: "vx_stats") -> dict:
    d = {k: getattr(st, k) for k, _ in vx_stats._fields_ if k != "stage_ms"}
    d["stage_ms"] = {name: float(st.stage_ms[i]) for i, name in enumerate(STAGES)}
    return d


class vx_validation(C.Structure):
    _fields_ = [
        ("voxels_checked", C.c_int64),
        ("label_mismatches", C.c_int64),
        ("value_mismatches", C.c_int64),
        ("n_examples", C.c_int64),
        ("examples", C.c_int64 * 16),
    ]


# every function include/voxellate_b200.h declares: name -> (restype, argtypes)
_P = C.c_void_p
SIGNATURES = {
    "vx_abi_version": (C.c_uint32, []),
    "vx_version_string": (C.c_char_p, []),
    "vx_last_error": (C.c_char_p, []),
    "vx_last_d2h_bytes": (C.c_uint64, []),
    "vx_options_init": (None, [C.POINTER(vx_options)]),
    "vx_context_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "vx_context_destroy": (None, [_P]),
    "vx_context_workspace_bytes": (C.c_int64, [_P]),
    "vx_context_stage_ms": (C.c_int, [_P, C.POINTER(C.c_float)]),
    "vx_tessellate": (C.c_int, [_P, C.POINTER(vx_problem), C.POINTER(vx_options), _P,
                                C.POINTER(vx_stats)]),
    "vx_tessellate_brute": (C.c_int, [_P, C.POINTER(vx_problem), C.POINTER(vx_options), _P,
                                      C.POINTER(vx_stats)]),
    "vx_prune": (C.c_int, [_P, C.POINTER(vx_problem), _P, C.POINTER(C.c_int64)]),
    "vx_validate_partition": (C.c_int, [_P, C.POINTER(vx_problem), _P, _P, C.c_int64, C.c_uint64,
                                        C.POINTER(vx_validation)]),
    "vx_optimal_r0": (C.c_int, [C.c_int64, C.c_int, _P, C.POINTER(C.c_double)]),
    "vx_generate_uniform_sites": (C.c_int, [C.c_int, _P, C.c_int64, C.c_int, C.c_double, C.c_double,
                                            C.c_uint64, _P, _P]),
    "vx_slab_bounds": (None, [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64),
                              C.POINTER(C.c_int64)]),
    "vx_label_fingerprint": (C.c_uint64, [_P, C.c_int64]),
    "vx_probe_pipe_rates": (C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "vx_probe_exact_arith": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_double, C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64)]),
    "vx_probe_h2d": (C.c_int, [C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_float)]),
    "vx_tessellate_to_files": (C.c_int, [_P, C.POINTER(vx_problem), C.POINTER(vx_options), C.c_char_p,
                                         C.c_char_p, C.c_int64, C.POINTER(vx_stats)]),
    "vx_write_image": (C.c_int, [C.c_char_p, C.c_int, C.c_int, _P, _P, C.c_int, C.c_int, C.c_int64,
                                 C.c_int64, _P]),
    "vx_read_image": (C.c_int, [C.c_char_p, C.c_int, _P, _P, _P, _P, C.c_int64]),
    "vx_write_image_sidecar": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, _P, _P, C.c_int, C.c_int,
                                         C.c_int64, C.c_int64, C.c_uint64]),
    "vx_image_sidecar_text": (C.c_int, [C.c_char_p, C.c_int, _P, _P, C.c_int, C.c_int, C.c_int64,
                                        C.c_int64, C.c_uint64, C.c_char_p, C.c_int64]),
}

_lib = None


def lib():
    """Load libvoxellate_b200.so (built by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (the CUDA engine has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name, None)
            if f is None:
                if os.environ.get("VX_LIB_PATH"):  # an older build under A/B timing
                    continue
                raise ImportError(f"{LIB_PATH} does not export {name}: rebuild it")
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class VxError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == VX_OK:
        return
    msg = lib().vx_last_error().decode()
    if rc == VX_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    raise VxError(rc, msg)
