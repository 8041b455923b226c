"""Decode-stage drop-ins (sfft/reconstruct.py) on the device.

``robust_noise_floor`` (:119-133), ``vote_tally`` (:158-179) and
``select_by_votes`` (:182-194) keep their reference signatures; the heavy
sets, per-position vote scores and the (-score, position) selection run in
sm_100a kernels (decode.cu).  ``VoteTable.counts`` is a device int64 tensor.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from ._lib import check, lib, ptr, stream_of
from .errors import FilterKindMismatch, InvalidParameter
from .filters import FLAT

__all__ = ["VoteTable", "robust_noise_floor", "vote_tally", "select_by_votes",
           "noise_floors", "need_votes", "estimate_freqshift"]


def _dev_values(values, device=None):
    import torch
    if isinstance(values, torch.Tensor):
        t = values if values.is_cuda else values.cuda()
    else:
        from ._lib import require_cuda
        t = torch.as_tensor(np.asarray(values, dtype=np.complex128), device=require_cuda(device))
    if t.dtype != torch.complex128:
        t = t.to(torch.complex128)
    return t.contiguous()


def noise_floors(values, median_mult: float = 3.0, with_peak: bool = False):
    """Per-row floors of a [nsets][B] complex128 device tensor (device result)."""
    import torch
    v = _dev_values(values)
    if v.ndim == 1:
        v = v.unsqueeze(0)
    nsets, b = v.shape
    fl = torch.empty(nsets, dtype=torch.float64, device=v.device)
    pk = torch.empty(nsets, dtype=torch.float64, device=v.device) if with_peak else None
    if nsets and b:
        check(lib().sfft_noise_floor(ptr(v), nsets, b, float(median_mult), ptr(fl), ptr(pk),
                                     stream_of(v.device)), "sfft_noise_floor")
    return (fl, pk) if with_peak else fl


def robust_noise_floor(values, median_mult: float = 3.0) -> float:
    """max(min(3*median|v|, peak/4), 1e-9*peak, 1e-300); 0.0 for empty input."""
    v = _dev_values(values)
    if v.numel() == 0:
        return 0.0
    return float(noise_floors(v.reshape(1, -1), median_mult)[0].item())


@dataclass
class VoteTable:
    """Per-position vote counts accumulated over rounds (device int64)."""

    n: int
    rounds: int = 0
    counts: object = field(default=None)

    def __post_init__(self):
        if self.counts is None:
            import torch
            from ._lib import require_cuda
            self.counts = torch.zeros(self.n, dtype=torch.int64, device=require_cuda())

    @property
    def score(self):
        return self.counts

    def score_of(self, position: int) -> int:
        return int(self.counts[position % self.n].item())


def need_votes(min_fraction: float, rounds: int) -> int:
    """Smallest integer score meeting max(min_fraction*rounds, 1e-12)."""
    need = max(min_fraction * rounds, 1e-12)
    return max(1, math.ceil(need))


def vote_tally(rounds, heavy_count: int) -> VoteTable:
    """Per round, the ``heavy_count`` largest buckets at/above the round's
    threshold are heavy; each original position whose flat bucket is heavy
    gains one vote (evaluated per position on the device, no scatter)."""
    import torch
    rounds = list(rounds)
    if not rounds:
        return VoteTable(n=1, rounds=0)
    first = rounds[0][0]
    n, b = first.n, first.num_buckets
    for bs, _ in rounds:
        if bs.filter_kind != FLAT:
            raise FilterKindMismatch(f"device vote_tally supports flat bucket sets, got {bs.filter_kind}")
    dev = first.values.device
    R = len(rounds)
    vals = torch.stack([_dev_values(bs.values) for bs, _ in rounds])
    thr = torch.as_tensor([float(t) for _, t in rounds], dtype=torch.float64, device=dev)
    words = (b + 31) // 32
    bits = torch.zeros((R, words), dtype=torch.int32, device=dev)
    st = stream_of(dev)
    check(lib().sfft_heavy_bitmap(ptr(vals), R, b, ptr(thr), int(heavy_count), ptr(bits), None,
                                  st), "sfft_heavy_bitmap")
    sig = torch.as_tensor([bs.perm.sigma for bs, _ in rounds], dtype=torch.int64, device=dev)
    bp = torch.as_tensor([bs.perm.b_prime for bs, _ in rounds], dtype=torch.int64, device=dev)
    counts = torch.empty(n, dtype=torch.int64, device=dev)
    wsb = lib().sfft_votes_ws_bytes(n, 1, R)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    check(lib().sfft_vote_select(n, b, R, 1, ptr(bits), ptr(sig), ptr(bp), first.center_shift,
                                 None, ptr(counts), 1, 0, None, None, ptr(ws), wsb, st),
          "sfft_vote_select")
    return VoteTable(n=n, rounds=R, counts=counts)


def select_by_votes(table: VoteTable, keep: int, min_fraction: float) -> list:
    """Up to ``keep`` positions with score >= min_fraction*rounds, highest
    score first, ties to the lower position."""
    import torch
    if table.rounds == 0 or keep <= 0:
        return []
    counts = table.counts
    if not isinstance(counts, torch.Tensor) or not counts.is_cuda:
        counts = _dev_values(np.zeros(1)).new_tensor(np.asarray(counts, dtype=np.int64))
    counts = counts.to(torch.int64).contiguous()
    dev = counts.device
    n = table.n
    R = table.rounds
    cand = torch.empty(keep, dtype=torch.int64, device=dev)
    ncand = torch.zeros(1, dtype=torch.int32, device=dev)
    wsb = lib().sfft_votes_ws_bytes(n, 1, R)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    check(lib().sfft_vote_select(n, n, R, 1, None, None, None, 0, ptr(counts), None,
                                 need_votes(min_fraction, R), keep, ptr(cand), ptr(ncand),
                                 ptr(ws), wsb, stream_of(dev)), "sfft_vote_select")
    k = int(ncand.item())
    return [int(p) for p in cand[:k].cpu().tolist()]


def estimate_freqshift(x, f: int, t: int, seed=0) -> complex:
    """Coefficient at ``f`` by shift-to-DC random sampling (sfft/reconstruct.py:356-371):
    mean of x[i] w^{f i} over t positions drawn exactly as the reference draws
    them (numpy Generator on the host), or all N positions when t >= N."""
    import torch
    if t < 1:
        raise InvalidParameter(f"t={t} must be >= 1")
    n = x.n
    if t >= n:
        idx = np.arange(n, dtype=np.int64)
    else:
        rng = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
        idx = rng.integers(0, n, size=t)
    xs = x.samples
    dev = xs.device
    it = torch.as_tensor(np.asarray(idx, dtype=np.int64), device=dev)
    out = torch.empty(1, dtype=torch.complex128, device=dev)
    ws = torch.empty(4096, dtype=torch.uint8, device=dev)
    dt = 0 if xs.dtype == torch.complex64 else 1
    check(lib().sfft_freqshift_estimate(dt, ptr(xs), n, ptr(it), int(it.numel()), int(f),
                                        ptr(out), ptr(ws), 4096, stream_of(dev)),
          "sfft_freqshift_estimate")
    x.record(("list", it))
    return complex(out.item())
