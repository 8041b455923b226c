"""Batched one-shot framework (sfft/frameworks.py:216-311) on the device."""

from __future__ import annotations

import numpy as np

from ._lib import check, lib, ptr, stream_of
from .errors import ConfigMismatch, InvalidParameter
from .filters import twiddles


def oneshot_shifts(n: int, cfg) -> tuple[list, list]:
    """Measurement shifts and ladder of run_oneshot (sfft/frameworks.py:237-245):
    0..2a_max-1, the phase-ladder rungs not among them, then the pursuit
    shifts drawn from default_rng(cfg.seed) (the same numpy calls)."""
    from .frameworks import phase_ladder
    base = list(range(2 * cfg.a_max))
    ladder = phase_ladder(n)
    extra = [d for d in ladder if d not in base]
    rng = np.random.default_rng(cfg.seed)
    pursuit = [int(t) for t in rng.integers(0, n, size=cfg.pursuit_shifts)]
    return base + extra + pursuit, ladder


def oneshot_batch(xs, k: int, cfg):
    import torch
    from .frameworks import BatchResult, _as_batch, _empty_batch, _sched_buffer, _WS
    cfg = cfg.validated()
    if cfg.framework != "one_shot":
        raise ConfigMismatch(f"run_oneshot got framework {cfg.framework!r}")
    X, _ = _as_batch(xs)
    S, n = X.shape
    dev = X.device
    if k <= 0:
        return _empty_batch(n, S, 0, dev, 0, True)
    b = cfg.resolve_buckets(n, k)
    shifts, ladder = oneshot_shifts(n, cfg)
    if cfg.a_max > 8 or len(shifts) > 64 or k > 8192:
        raise InvalidParameter(f"one_shot on the device: a_max <= 8, <= 64 shifts and k <= 8192 "
                               f"(a_max={cfg.a_max}, {len(shifts)} shifts, k={k})")
    out_pos = torch.zeros((S, k), dtype=torch.int64, device=dev)
    out_coef = torch.zeros((S, k), dtype=torch.complex128, device=dev)
    out_n = torch.zeros(S, dtype=torch.int32, device=dev)
    out_it = torch.zeros(S, dtype=torch.int32, device=dev)
    out_cv = torch.zeros(S, dtype=torch.int32, device=dev)
    out_sm = torch.zeros(S, dtype=torch.int64, device=dev)
    sched = _sched_buffer(S, dev)
    L = lib()
    sh = np.asarray(shifts, dtype=np.int64)
    lad = np.asarray(ladder, dtype=np.int64)
    wsb = L.sfft_oneshot_ws_bytes(n, S, b, cfg.a_max, sh.size)
    ws = _WS.get(wsb, dev, "oneshot")
    dt = 0 if X.dtype == torch.complex64 else 1
    check(L.sfft_run_oneshot(dt, ptr(X), n, X.stride(0), S, b, cfg.a_max, sh.ctypes.data,
                             sh.size, lad.ctypes.data, lad.size, ptr(twiddles(b, dev)), k,
                             ptr(out_pos), ptr(out_coef), ptr(out_n), ptr(out_it), ptr(out_cv),
                             ptr(out_sm), ptr(sched), ptr(ws), wsb, stream_of(dev)),
          "sfft_run_oneshot")
    return BatchResult(n, k, out_pos, out_coef, out_n, out_it, out_cv, out_sm, sched)
