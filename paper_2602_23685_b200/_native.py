"""Loader for the C-ABI library ``lib/libvrprpd.so`` (include/vrp_rpd.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every device entry point raises :class:`NativeUnavailable`.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
# VRP_LIB overrides the library path (side builds for ablation experiments)
LIB_PATH = Path(os.environ["VRP_LIB"]) if os.environ.get("VRP_LIB") else PKG / "lib" / "libvrprpd.so"

VRP_OK, VRP_CAPACITY, VRP_DEADLOCK, VRP_MALFORMED = 0, 1, 2, 3
VRP_EINVAL, VRP_ECUDA, VRP_EUNSUPPORTED = 1, 2, 3
MODE_EXACT, MODE_EVALUATE, MODE_TWO_PASS = 0, 1, 2


class NativeUnavailable(RuntimeError):
    """libvrprpd.so is not built or cannot run here (no CUDA device)."""


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero error code."""


_lib = None


def _declare(L):
    P, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "vrp_version": ([P, P], C.c_int),
        "vrp_last_error": ([], C.c_char_p),
        "vrp_instance_create": ([i32, i32, i32, P, P, P], C.c_int),
        "vrp_instance_destroy": ([P], C.c_int),
        "vrp_instance_info": ([P, P, P, P, P], C.c_int),
        "vrp_makespan_batch": ([P, P, i32, i64, P, i64, i32, P, P, P, P, P], C.c_int),
        "vrp_evaluate_records": ([P, P, i64, P, i64, P, P, P, P, P, P, P], C.c_int),
        "vrp_decode_batch": ([P, P, i64, i64, i32, f64, P, P, P, P, P, i32, i64, P, P], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def lib(require_device: bool = True):
    """The loaded library.  Raises NativeUnavailable when it cannot be used."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeUnavailable(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(str(LIB_PATH))
        _declare(L)
        declare_k4(L)
        _lib = L
    if require_device:
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device visible: the B200 path has no CPU fallback")
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib(require_device=False).vrp_last_error().decode(errors="replace")
        raise NativeError(f"{what or 'libvrprpd'} failed (code {rc}): {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def declare_k4(L):
    P, i64, f64 = C.c_void_p, C.c_int64, C.c_double
    L.vrp_fitness_order.argtypes = [P, i64, P, P]
    L.vrp_evolve.argtypes = [P, P, i64, i64, f64, f64, f64, P, P, P, P, P]
    L.vrp_best_update.argtypes = [P, i64, i64, P, i64, P, P, P, P, P]
    L.vrp_repair_batch.argtypes = [P, P, i64, P, P, i64, P, P, P, P, i64, P, P, i64, P]
    L.vrp_destroy_batch.argtypes = [P, P, i64, P, P, P, C.c_int32, P, P, i64, P, P, i64, P, i64, P]
    L.vrp_alns_iterate.argtypes = [P, P, P, C.c_int32, P, P, P, P, P, i64, i64, i64, P, P, i64, P, P,
                                   i64, P]
    L.vrp_ls_build.argtypes = [P, C.c_int32, P, P, P, P, i64, P, i64, i64, P, C.c_int32, P, P]
    L.vrp_random_fill.argtypes = [P, i64, P, P]
    L.vrp_sa_exp.argtypes = [P, P, i64, P]
    L.vrp_remove_batch.argtypes = [P, P, i64, P, P, i64, P, P, i64, P, P, i64, P, i64, P]
    L.vrp_removal_gains.argtypes = [P, P, i64, P, P, i64, i64, P]
    L.vrp_ls_entries.argtypes = [P, C.c_int32, P, P, P, P, P, C.c_int32, P, P, P, P, P, P, P]
    L.vrp_ls_topk.argtypes = [P, P, i64, P, P, P, P, i64, P, P, P, C.c_int32, C.c_int32, P, P, P, P]
    for name in ("vrp_fitness_order", "vrp_evolve", "vrp_best_update", "vrp_repair_batch",
                 "vrp_destroy_batch", "vrp_alns_iterate", "vrp_ls_build", "vrp_random_fill",
                 "vrp_sa_exp", "vrp_remove_batch", "vrp_removal_gains", "vrp_ls_topk",
                 "vrp_ls_entries"):
        getattr(L, name).restype = C.c_int
