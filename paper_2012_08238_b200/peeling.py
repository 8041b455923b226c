"""Batched FFAST-style peeling runner (sfft/frameworks.py:614-699) on the device."""

from __future__ import annotations

import ctypes
import math

from ._lib import check, lib, ptr, stream_of
from .errors import ConfigMismatch, InvalidParameter
from .filters import twiddles


def peeling_batch(xs, k: int, cfg):
    import torch
    from .frameworks import BatchResult, _as_batch, _empty_batch, _sched_buffer, _WS
    cfg = cfg.validated()
    if cfg.framework != "peeling":
        raise ConfigMismatch(f"run_peeling got framework {cfg.framework!r}")
    X, _ = _as_batch(xs)
    S, n = X.shape
    dev = X.device
    factors = tuple(int(p) for p in cfg.coprime_factors)
    if any(p <= 1 for p in factors) or math.prod(factors) != n:
        raise ConfigMismatch(f"factors {factors} do not multiply to n={n}")
    for i, p in enumerate(factors):
        for q in factors[i + 1:]:
            if math.gcd(p, q) != 1:
                raise ConfigMismatch(f"factors {p} and {q} are not co-prime")
    if k <= 0:
        return _empty_batch(n, S, 0, dev, 0, True)
    m = len(factors)
    fac = (ctypes.c_int64 * m)(*factors)
    tws = [twiddles(n // p, dev) for p in factors]
    wst = (ctypes.c_void_p * m)(*[t.data_ptr() for t in tws])
    out_pos = torch.zeros((S, k), dtype=torch.int64, device=dev)
    out_coef = torch.zeros((S, k), dtype=torch.complex128, device=dev)
    out_n = torch.zeros(S, dtype=torch.int32, device=dev)
    out_it = torch.zeros(S, dtype=torch.int32, device=dev)
    out_cv = torch.zeros(S, dtype=torch.int32, device=dev)
    out_err = torch.zeros(S, dtype=torch.int32, device=dev)
    out_sm = torch.zeros(S, dtype=torch.int64, device=dev)
    sched = _sched_buffer(S, dev)
    L = lib()
    wsb = L.sfft_peeling_ws_bytes(n, S, fac, m, k)
    ws = _WS.get(wsb, dev, "peeling")
    dt = 0 if X.dtype == torch.complex64 else 1
    check(L.sfft_run_peeling(dt, ptr(X), n, X.stride(0), S, fac, m, wst, k, ptr(out_pos),
                             ptr(out_coef), ptr(out_n), ptr(out_it), ptr(out_cv), ptr(out_err),
                             ptr(out_sm), ptr(sched), ptr(ws), wsb, stream_of(dev)),
          "sfft_run_peeling")
    if bool(out_err.any()):
        raise InvalidParameter("1 moments cannot resolve a_max=1 (a factor of 2 gives a "
                               "one-shift stage)")
    return BatchResult(n, k, out_pos, out_coef, out_n, out_it, out_cv, out_sm, sched)
