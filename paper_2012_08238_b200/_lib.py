"""ctypes binding of libsfft_b200.so (the C-ABI in include/sfft_b200.h).

The product path has no CPU fallback: if the library is missing, importing a
compute entry point raises ``LibraryMissing``; if no CUDA device is present,
every compute call raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# SFFT_LIB_PATH: an alternative build of the same library (A/B measurements only)
LIB_PATH = os.environ.get("SFFT_LIB_PATH") or os.path.join(HERE, "libsfft_b200.so")

_lock = threading.Lock()
_lib = None

i32, i64, f64, vp, sz = C.c_int32, C.c_int64, C.c_double, C.c_void_p, C.c_size_t
P_i32 = vp
P_i64 = vp
P_f64 = vp

# name -> (restype, argtypes); mirrors include/sfft_b200.h
SIGNATURES = {
    "sfft_version": (C.c_int, []),
    "sfft_last_error": (C.c_char_p, []),
    "sfft_twiddles": (C.c_int, [vp, i64, vp]),
    "sfft_flat_taps": (C.c_int, [P_f64, i64, i64, f64, vp]),
    "sfft_bucketize_ws_bytes": (sz, [i64, i64]),
    "sfft_build_gtable": (C.c_int, [P_f64, i64, i64, i64, vp, vp, P_f64, P_i64, vp, sz, vp]),
    "sfft_flat_bucketize": (C.c_int, [C.c_int, vp, i64, i64, P_f64, i64, i64, i64, P_i32, P_i64,
                                      P_i64, P_i64, P_i32, vp, vp, vp, sz, vp]),
    "sfft_spike_bucketize": (C.c_int, [C.c_int, vp, i64, i64, i64, i64, P_i32, P_i64, P_i32, vp,
                                       vp, vp, sz, vp]),
}


class LibraryMissing(ImportError):
    pass


def lib():
    """Load the library once (thread-safe) and declare every prototype."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().sfft_last_error()
        raise RuntimeError(f"{what} failed (rc={rc}): {msg.decode() if msg else ''}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_of(device) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def require_cuda(device=None):
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2012_08238_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

SIGNATURES.update({
    "sfft_access_mark": (C.c_int, [vp, i64, C.c_int, i64, i64, i64, P_i64, vp]),
    "sfft_count_nonzero": (C.c_int, [vp, i64, P_i64, vp]),
})
SIGNATURES.update({
    "sfft_noise_floor": (C.c_int, [vp, i64, i64, f64, P_f64, P_f64, vp]),
    "sfft_heavy_bitmap": (C.c_int, [vp, i64, i64, P_f64, i64, vp, P_i32, vp]),
    "sfft_votes_ws_bytes": (sz, [i64, i64, i64]),
    "sfft_vote_select": (C.c_int, [i64, i64, i64, i64, vp, P_i64, P_i64, i64, P_i64, P_i64, i64,
                                   i64, P_i64, P_i32, vp, sz, vp]),
    "sfft_vote_tally": (C.c_int, [i64, i64, P_i64, P_i64, vp, P_i64, P_i64, P_i32, P_i64, P_i64,
                                  vp]),
    "sfft_energy_estimates": (C.c_int, [vp, i64, vp, P_f64, i64, i64, P_i64, P_i64, P_i64, i64,
                                        vp, vp]),
    "sfft_trimmed_mean": (C.c_int, [vp, i64, i64, vp, vp]),
    "sfft_subtract_flat": (C.c_int, [vp, vp, i64, i64, P_i32, i64, vp, i64, P_i32, P_i64, P_i64,
                                     P_i64, vp, P_i32, i64, vp]),
})
SIGNATURES.update({
    "sfft_iterative_ws_bytes": (sz, [i64, i64, i64, i64, i64]),
    "sfft_run_iterative": (C.c_int, [C.c_int, vp, i64, i64, i64, i64, P_f64, i64, i64, vp, P_f64,
                                     vp, P_i64, P_i64, i64, i64, i64, i64, vp, i64, i32, i32,
                                     i64, P_i64,
                                     vp, P_i32, P_i32, P_i32, P_i64, P_i64, P_i32, vp, sz, vp]),
    "sfft_schedule_layout": (C.c_int, [vp, vp]),
    "sfft_dirichlet_ws_bytes": (sz, [i64, i64]),
    "sfft_dirichlet_bucketize": (C.c_int, [C.c_int, vp, i64, vp, i64, i64, i32, i64, i64, P_i64,
                                           vp, vp, vp, sz, vp]),
    "sfft_freqshift_estimate": (C.c_int, [C.c_int, vp, i64, P_i64, i64, i64, vp, vp, sz, vp]),
})
SIGNATURES.update({
    "sfft_launch_count": (i64, []),
    "sfft_prof_enable": (C.c_int, [C.c_int]),
    "sfft_prof_read": (C.c_int, [vp, vp, vp]),
})
SIGNATURES.update({
    "sfft_voting_ws_bytes": (sz, [i64, i64, i64, i64, i64, i64]),
    "sfft_run_voting": (C.c_int, [C.c_int, vp, i64, i64, i64, P_f64, i64, i64, vp, P_f64, vp,
                                  P_i64, P_i64, i64, i64, i64, i64, vp, P_i64, vp, P_i32, P_i64,
                                  P_i64, vp, sz, vp]),
})
SIGNATURES.update({
    "sfft_peeling_ws_bytes": (sz, [i64, i64, vp, i64, i64]),
    "sfft_run_peeling": (C.c_int, [C.c_int, vp, i64, i64, i64, vp, i64, vp, i64, P_i64, vp,
                                   P_i32, P_i32, P_i32, P_i32, P_i64, P_i64, vp, sz, vp]),
})
SIGNATURES.update({
    "sfft_oneshot_ws_bytes": (sz, [i64, i64, i64, i64, i64]),
    "sfft_run_oneshot": (C.c_int, [C.c_int, vp, i64, i64, i64, i64, i64, vp, i64, vp, i64, vp,
                                   i64, P_i64, vp, P_i32, P_i32, P_i32, P_i64, P_i64, vp, sz,
                                   vp]),
})
SIGNATURES.update({
    "sfft_set_avail": (C.c_int, [P_i32, C.c_int32, vp]),
})
