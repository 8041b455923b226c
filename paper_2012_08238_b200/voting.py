"""Batched voting runner (sfft/frameworks.py:354-417) on the device."""

from __future__ import annotations

import numpy as np

from ._lib import check, lib, ptr, stream_of
from .errors import ConfigMismatch, NonDivisorParameter
from .filters import make_flat_filter, twiddles
from .reconstruct import need_votes


def voting_batch(xs, k: int, cfg):
    import torch
    from .frameworks import BatchResult, _as_batch, _empty_batch, _sched_buffer, _WS, draw_perms
    cfg = cfg.validated()
    if cfg.framework != "voting":
        raise ConfigMismatch(f"run_voting got framework {cfg.framework!r}")
    X, _ = _as_batch(xs)
    S, n = X.shape
    dev = X.device
    if cfg.rounds <= 0 or k <= 0:
        return _empty_batch(n, S, max(k, 0), dev, 0, False)
    b = cfg.resolve_buckets(n, k)
    if cfg.rounds > 255:
        # scores are kept in 8 bits per position on the device
        raise NotImplementedError("device voting supports up to 255 rounds")
    filt = make_flat_filter(n, b, device=dev)
    bpre = 0
    if cfg.spike_prestage:
        bpre = n // max(2, cfg.prestage_width)
        if bpre <= 0 or n % bpre:
            raise NonDivisorParameter(f"num_buckets={bpre} does not divide n={n}")
    R = cfg.rounds
    sig, tau = draw_perms(n, cfg.seed, R)
    psig = torch.as_tensor(np.tile(sig, (S, 1)), device=dev)
    ptau = torch.as_tensor(np.tile(tau, (S, 1)), device=dev)
    out_pos = torch.zeros((S, k), dtype=torch.int64, device=dev)
    out_coef = torch.zeros((S, k), dtype=torch.complex128, device=dev)
    out_n = torch.zeros(S, dtype=torch.int32, device=dev)
    out_sm = torch.zeros(S, dtype=torch.int64, device=dev)
    sched = _sched_buffer(S, dev)
    L = lib()
    wsb = L.sfft_voting_ws_bytes(n, b, S, R, k, bpre)
    ws = _WS.get(wsb, dev, "voting")
    gmax = torch.tensor([filt.peak], dtype=torch.float64, device=dev)
    dt = 0 if X.dtype == torch.complex64 else 1
    check(L.sfft_run_voting(dt, ptr(X), n, X.stride(0), S, ptr(filt.kernel_taps), filt.support, b,
                            ptr(filt.gtable), ptr(gmax), ptr(twiddles(b, dev)), ptr(psig),
                            ptr(ptau), R, k, need_votes(cfg.min_vote_fraction, R), bpre,
                            ptr(twiddles(bpre, dev)) if bpre else None, ptr(out_pos),
                            ptr(out_coef), ptr(out_n), ptr(out_sm), ptr(sched), ptr(ws), wsb,
                            stream_of(dev)), "sfft_run_voting")
    its = torch.full((S,), R, dtype=torch.int32, device=dev)
    conv = torch.ones(S, dtype=torch.int32, device=dev)
    return BatchResult(n, k, out_pos, out_coef, out_n, its, conv, out_sm, sched)
