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
from .filters import FLAT, SPIKE

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
    threshold are heavy; each original position whose bucket under that
    round's hash view is heavy gains one vote (sfft/reconstruct.py:158-179).
    Bucket sets of any kind (flat, spike, Dirichlet), width and centre shift
    mix freely; the heavy sets and the per-position scores run on the device
    (per-position evaluation of the preimage scatter, no atomics)."""
    import torch
    rounds = list(rounds)
    if not rounds:
        return VoteTable(n=1, rounds=0)
    first = rounds[0][0]
    n = first.n
    dev = first.values.device if hasattr(first.values, "device") else None
    R = len(rounds)
    # heavy bitmaps: one launch per distinct bucket count, each group's rounds
    # packed contiguously (bit_offset per round)
    by_b = {}
    for r, (bs, _) in enumerate(rounds):
        if bs.n != n:
            raise InvalidParameter(f"bucket sets of different lengths ({bs.n} != {n})")
        by_b.setdefault(bs.num_buckets, []).append(r)
    offs = np.zeros(R, dtype=np.int64)
    total = 0
    for b, idx in by_b.items():
        for r in idx:
            offs[r] = total
            total += (b + 31) // 32
    dev = _dev_values(first.values, dev).device
    bits = torch.zeros(max(total, 1), dtype=torch.int32, device=dev)
    st = stream_of(dev)
    for b, idx in by_b.items():
        vals = torch.stack([_dev_values(rounds[r][0].values, dev) for r in idx])
        thr = torch.as_tensor([float(rounds[r][1]) for r in idx], dtype=torch.float64, device=dev)
        check(lib().sfft_heavy_bitmap(ptr(vals), len(idx), b, ptr(thr), int(heavy_count),
                                      ptr(bits[int(offs[idx[0]]):]), None, st),
              "sfft_heavy_bitmap")
    kinds = []
    for bs, _ in rounds:
        if bs.filter_kind == SPIKE:
            kinds.append(1)
        elif bs.filter_kind == FLAT or bs.half_offset:
            kinds.append(0)
        else:
            kinds.append(2)
    i64 = lambda v: torch.as_tensor(np.asarray(v, dtype=np.int64), device=dev)
    nb = i64([bs.num_buckets for bs, _ in rounds])
    sig = i64([bs.perm.sigma for bs, _ in rounds])
    bp = i64([bs.perm.b_prime for bs, _ in rounds])
    cs = i64([bs.center_shift for bs, _ in rounds])
    kd = torch.as_tensor(np.asarray(kinds, dtype=np.int32), device=dev)
    counts = torch.empty(n, dtype=torch.int64, device=dev)
    check(lib().sfft_vote_tally(n, R, ptr(nb), ptr(i64(offs)), ptr(bits), ptr(sig), ptr(bp),
                                ptr(kd), ptr(cs), ptr(counts), st), "sfft_vote_tally")
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
