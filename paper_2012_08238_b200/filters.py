"""The flat (Gaussian x sinc) window, built on the device.

Mirrors sfft/filters.py:114-151 (``default_gauss_sigma``, ``default_flat_support``,
``make_flat_filter``) and ``WindowFilter.bucket_weight`` (:102-111).  The
N-point response G is kept as the transposed table T[rho][j] = G[rho + j*L]
(L = N/B rows of B buckets): row rho is the B-point transform of the taps
modulated by w_N^{rho*i}, so the table is built by the same fold+FFT kernel as
a bucketization and every per-tone weight vector a
subtraction needs is one contiguous circular row.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass

from .errors import InvalidParameter, NonDivisorParameter
from ._lib import check, lib, ptr, require_cuda, stream_of

__all__ = ["WindowFilter", "FLAT", "SPIKE", "DIRICHLET", "default_gauss_sigma",
           "default_flat_support", "make_flat_filter", "make_dirichlet_bank",
           "filter_freq_shift", "twiddles"]

FLAT = "flat"
SPIKE = "spike_train"
DIRICHLET = "dirichlet_bank"

_cache_lock = threading.Lock()
_tw_cache: dict = {}
_filt_cache: dict = {}


def twiddles(B: int, device):
    """Device table W[e] = w_B^e, cached per (device, B)."""
    import torch
    key = (str(device), int(B))
    with _cache_lock:
        t = _tw_cache.get(key)
    if t is None:
        t = torch.empty(B, dtype=torch.complex128, device=device)
        check(lib().sfft_twiddles(ptr(t), B, stream_of(device)), "sfft_twiddles")
        with _cache_lock:
            t = _tw_cache.setdefault(key, t)
    return t


def default_gauss_sigma(n: int, num_buckets: int) -> float:
    return num_buckets * math.sqrt(math.log2(n))


def default_flat_support(n: int, num_buckets: int) -> int:
    """Smallest even support >= 4*B*sqrt(log2 N), capped at N."""
    omega = math.ceil(4.0 * default_gauss_sigma(n, num_buckets))
    omega += omega % 2
    return min(omega, n - (n % 2))


@dataclass(frozen=True, eq=False)
class WindowFilter:
    """A flat window (device taps + transposed response table) or a Dirichlet
    bank (device complex box taps + natural-order response)."""

    kind: str
    n: int
    num_buckets: int
    bucket_width: int
    support: int
    taps: object            # flat: torch float64 [support]; Dirichlet: complex128 [L]
    gtable: object          # flat: torch complex128 [L][B], gtable[r, j] = G[r + j*L]
    peak: float             # max |G|
    gauss_sigma: float = 0.0
    center_offset: int = 0
    half_bucket_offset: bool = True
    response: object = None  # Dirichlet: complex128 [N] unnormalised box transform
    base_taps: object = None  # frequency-shifted flat window: the real taps the kernels use
                              # (``taps`` then holds taps * w^(-f0 i), as in the reference)

    @property
    def device(self):
        return self.taps.device

    @property
    def kernel_taps(self):
        """The real flat taps (a shifted window's modulation w^(-f0 i) rides on
        the kernels' per-item phase term)."""
        return self.taps if self.base_taps is None else self.base_taps

    @property
    def freq_response(self):
        """G over [0, N) in natural order (device tensor)."""
        if self.gtable is None:
            return self.response
        g = self.gtable.transpose(0, 1).reshape(self.n)
        if self.kind == FLAT and self.center_offset:
            import torch
            g = torch.roll(g, self.center_offset)  # G'[f] = G[f - f0]
        return g

    def bucket_centers(self):
        """Position-space passband centers, one per bucket (sfft/filters.py:92-100)."""
        import numpy as np
        base = 0 if self.half_bucket_offset else self.bucket_width // 2
        c = self.bucket_width * np.arange(self.num_buckets, dtype=np.int64) + base
        if self.kind == DIRICHLET:
            c = c + self.center_offset
        elif self.kind == FLAT:
            c = c - self.center_offset
        return c % self.n

    def bucket_weight(self, bucket: int, position):
        """Complex weight of spectrum ``position`` in ``bucket`` (sfft/filters.py:102-111):
        flat G[(bucket*L - m) mod N]; Dirichlet response[(m - center) mod N]."""
        import numpy as np
        import torch
        m = np.asarray(position, dtype=np.int64)
        if self.kind == DIRICHLET:
            base = 0 if self.half_bucket_offset else self.bucket_width // 2
            e = (m - (bucket * self.bucket_width + base)) % self.n
            return self.response[torch.as_tensor(e, device=self.device)]
        e = (bucket * self.bucket_width - m - self.center_offset) % self.n
        r = torch.as_tensor(e % self.bucket_width, device=self.device)
        j = torch.as_tensor(e // self.bucket_width, device=self.device)
        return self.gtable[r, j]

    def tap_positions(self):
        import torch
        return torch.arange(self.support, dtype=torch.int64, device=self.device)


def make_flat_filter(n: int, num_buckets: int, support: int | None = None,
                     gauss_sigma: float | None = None, device=None) -> WindowFilter:
    """Gaussian-windowed sinc taps and their response, built and cached on the
    device (sfft/filters.py:125-151)."""
    if num_buckets <= 0 or n % num_buckets != 0:
        raise InvalidParameter(f"num_buckets={num_buckets} does not divide n={n}")
    if support is None:
        support = default_flat_support(n, num_buckets)
    if gauss_sigma is None:
        gauss_sigma = default_gauss_sigma(n, num_buckets)
    if support % 2 != 0 or not 0 < support <= n:
        raise InvalidParameter(f"support={support} must be even and in (0, {n}]")
    import torch
    dev = require_cuda(device)
    key = (str(dev), n, num_buckets, int(support), float(gauss_sigma))
    with _cache_lock:
        hit = _filt_cache.get(key)
    if hit is not None:
        return hit
    b = num_buckets
    L = n // b
    st = stream_of(dev)
    taps = torch.empty(support, dtype=torch.float64, device=dev)
    check(lib().sfft_flat_taps(ptr(taps), support, b, float(gauss_sigma), st), "sfft_flat_taps")
    W = twiddles(b, dev)
    gt = torch.empty((L, b), dtype=torch.complex128, device=dev)
    gmax = torch.zeros(1, dtype=torch.float64, device=dev)
    rows = torch.arange(L, dtype=torch.int64, device=dev)
    wsb = lib().sfft_bucketize_ws_bytes(b, L)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    check(lib().sfft_build_gtable(ptr(taps), support, n, b, ptr(W), ptr(gt), ptr(gmax),
                                  ptr(rows), ptr(ws), wsb, st), "sfft_build_gtable")
    filt = WindowFilter(kind=FLAT, n=n, num_buckets=b, bucket_width=L, support=support,
                        taps=taps, gtable=gt, peak=float(gmax.item()),
                        gauss_sigma=float(gauss_sigma))
    with _cache_lock:
        filt = _filt_cache.setdefault(key, filt)
    return filt


def make_dirichlet_bank(n: int, bucket_width: int, num_buckets: int, half_offset: bool = True,
                        device=None) -> WindowFilter:
    """Bank of B modulated boxes of width L (sfft/filters.py:168-187): taps
    sqrt(N)/L, unnormalised response; per-bucket modulation happens in the
    bucketizer."""
    L, b = bucket_width, num_buckets
    if L * b != n:
        raise NonDivisorParameter(f"bucket_width*num_buckets = {L}*{b} != n={n}")
    import torch
    dev = require_cuda(device)
    taps = torch.full((L,), math.sqrt(n) / L, dtype=torch.complex128, device=dev)
    pad = torch.zeros(n, dtype=torch.complex128, device=dev)
    pad[:L] = taps
    resp = torch.fft.fft(pad)  # setup only; the hot path never evaluates the response
    return WindowFilter(kind=DIRICHLET, n=n, num_buckets=b, bucket_width=L, support=L,
                        taps=taps, gtable=None, peak=float(resp.abs().max().item()),
                        half_bucket_offset=half_offset, response=resp)


def filter_freq_shift(f: WindowFilter, f0: int) -> WindowFilter:
    """Move the passband centre(s) by f0 bins: taps *= w^(-f0 * position),
    center_offset += f0 (sfft/filters.py:190-200).  A flat window keeps its
    real taps for the kernels (``base_taps``): the modulation is the same
    per-sample phase term a permutation's b' uses, so ``bucketize_flat`` folds
    the shift into it, and the response is the unshifted table rolled by f0."""
    from dataclasses import replace
    import numpy as np
    import torch
    from .signal import phase_factor
    f0 = int(f0)
    if f.kind == FLAT:
        off = (f.center_offset + f0) % f.n
        base = f.kernel_taps
        pos = np.arange(f.support, dtype=np.int64)
        taps = base * phase_factor(f.n, -off * pos, device=f.device)
        return replace(f, taps=taps, base_taps=base, center_offset=off)
    if f.kind != DIRICHLET:
        raise NotImplementedError("filter_freq_shift: flat windows and Dirichlet banks")
    pos = np.arange(f.support, dtype=np.int64)
    taps = f.taps * phase_factor(f.n, -f0 * pos, device=f.device)
    pad = torch.zeros(f.n, dtype=torch.complex128, device=f.device)
    pad[:f.support] = taps
    resp = torch.fft.fft(pad)
    return replace(f, taps=taps, response=resp, peak=float(resp.abs().max().item()),
                   center_offset=(f.center_offset + f0) % f.n)
