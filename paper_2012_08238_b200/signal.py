"""Signal containers: a device-resident TimeSignal with an access schedule,
plus the host-side permutation parameters and sparse result container.

Mirrors sfft/signal.py (TimeSignal :60-112, SparseSpectrum :115-156,
PermutationParams :159-210, phase_factor :50-57).  Differences, by design:

* ``TimeSignal.samples`` is a CUDA tensor (complex128, or complex64 for the
  rounded-input mode) that stays resident in HBM across calls;
* reads are not recorded as a bool map written during the gather.  Each read
  appends its *index schedule* (flat: sigma, tau_tot, Omega; spike: stride,
  tau, B; explicit index lists) and ``access_count`` evaluates the union on
  the device — the hot gather never issues bookkeeping stores.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import InvalidParameter, NonInvertibleScaling

__all__ = ["TimeSignal", "SparseSpectrum", "PermutationParams", "phase_factor"]

_DTYPES = {"complex128": 1, "c128": 1, "complex64": 0, "c64": 0}


def _torch():
    import torch
    return torch


def phase_factor(n: int, exponents, device=None):
    """w_n^e (w_n = exp(-2*pi*i/n)) on the device, exponent reduced in int64
    first (sfft/signal.py:50-57)."""
    from ._lib import require_cuda
    torch = _torch()
    dev = require_cuda(device)
    e = torch.remainder(torch.as_tensor(np.asarray(exponents, dtype=np.int64), device=dev), n)
    th = (-2.0 * math.pi) * e.to(torch.float64) / n
    return torch.polar(torch.ones_like(th), th)


class TimeSignal:
    """Length-N complex samples resident on a CUDA device, with counted reads.

    ``dtype`` selects the kernel input precision: ``"complex128"`` (default,
    like the reference) or ``"complex64"`` (input rounded once, all
    accumulation in fp64).  ``fresh_copy`` shares the device buffer and starts
    an empty access schedule (sfft/signal.py:104-106).
    """

    __slots__ = ("samples", "_log", "_count_cache")

    def __init__(self, samples, accessed: list | None = None, dtype: str | None = None,
                 device=None):
        from ._lib import require_cuda
        torch = _torch()
        dev = require_cuda(device if device is not None else
                           (samples.device if isinstance(samples, torch.Tensor)
                            and samples.is_cuda else None))
        if dtype is None:
            dtype = ("complex64" if isinstance(samples, torch.Tensor)
                     and samples.dtype == torch.complex64 else "complex128")
        if dtype not in _DTYPES:
            raise InvalidParameter(f"dtype {dtype!r} not in {sorted(_DTYPES)}")
        tdt = torch.complex64 if _DTYPES[dtype] == 0 else torch.complex128
        if isinstance(samples, torch.Tensor):
            t = samples.to(device=dev, dtype=tdt)
        else:
            arr = np.asarray(samples)
            if arr.dtype.kind not in "biufc":
                raise InvalidParameter("samples must be numeric")
            # complex64 input is uploaded as it is (widening it on the host first
            # doubled the bytes over PCIe and cost ~10 ms for 2^22 samples); any
            # other numeric type goes through complex128 like the reference
            host = (np.ascontiguousarray(arr) if arr.dtype == np.complex64
                    else np.ascontiguousarray(arr, dtype=np.complex128))
            t = torch.as_tensor(host, device=dev).to(tdt)
        if t.ndim != 1 or t.numel() == 0:
            raise InvalidParameter("samples must be a nonempty 1-d sequence")
        self.samples = t.contiguous()
        self._log = [] if accessed is None else accessed
        self._count_cache = None

    # -- properties --------------------------------------------------------
    @property
    def n(self) -> int:
        return int(self.samples.numel())

    @property
    def dtype_code(self) -> int:
        return 0 if self.samples.dtype == _torch().complex64 else 1

    @property
    def device(self):
        return self.samples.device

    def __len__(self) -> int:
        return self.n

    def __repr__(self) -> str:
        return f"TimeSignal(n={self.n}, dtype={self.samples.dtype}, reads={len(self._log)})"

    # -- reads -------------------------------------------------------------
    def record(self, rec: tuple) -> None:
        """Append one read schedule (used by the bucketizers)."""
        self._log.append(rec)
        self._count_cache = None

    def take(self, indices):
        """Gather ``samples[indices mod N]`` on the device and record the read."""
        torch = _torch()
        idx = torch.remainder(torch.as_tensor(np.asarray(indices, dtype=np.int64)
                                              if not isinstance(indices, torch.Tensor)
                                              else indices, device=self.device), self.n)
        self.record(("list", idx.to(torch.int64)))
        return self.samples[idx]

    def read_all(self):
        self.record(("all",))
        return self.samples

    @property
    def access_count(self) -> int:
        if self._count_cache is None:
            from .access import count_schedule
            self._count_cache = count_schedule(self.n, self._log, self.device)
        return self._count_cache

    def accessed_indices(self) -> np.ndarray:
        from .access import schedule_map
        m = schedule_map(self.n, self._log, self.device)
        return _torch().nonzero(m).flatten().cpu().numpy()

    @property
    def access_counter(self) -> frozenset:
        return frozenset(self.accessed_indices().tolist())

    def fresh_copy(self) -> "TimeSignal":
        t = TimeSignal.__new__(TimeSignal)
        t.samples = self.samples
        t._log = []
        t._count_cache = None
        return t

    def to_numpy(self) -> np.ndarray:
        return self.samples.detach().cpu().numpy().astype(np.complex128)


@dataclass
class SparseSpectrum:
    """Finite map from frequency position to complex coefficient
    (sfft/signal.py:115-156)."""

    n: int
    entries: dict = field(default_factory=dict)

    def __post_init__(self):
        clean: dict = {}
        for pos, coeff in self.entries.items():
            p = int(pos)
            if not 0 <= p < self.n:
                raise InvalidParameter(f"position {p} outside [0, {self.n})")
            if p in clean:
                raise InvalidParameter(f"duplicate position {p}")
            clean[p] = complex(coeff)
        self.entries = clean

    def to_dense(self) -> np.ndarray:
        out = np.zeros(self.n, dtype=np.complex128)
        for p, c in self.entries.items():
            out[p] = c
        return out

    def support(self) -> set:
        return set(self.entries)

    def top_k(self, k: int) -> "SparseSpectrum":
        """k largest magnitudes, ties to the smaller index (sfft/signal.py:142-145)."""
        ranked = sorted(self.entries.items(), key=lambda it: (-abs(it[1]), it[0]))
        return SparseSpectrum(self.n, dict(ranked[:max(k, 0)]))

    @classmethod
    def from_dense(cls, dense, k: int | None = None) -> "SparseSpectrum":
        dense = np.asarray(dense)
        n = dense.size
        if k is None:
            pos = np.flatnonzero(dense)
        else:
            order = np.lexsort((np.arange(n), -np.abs(dense)))
            pos = np.sort(order[:max(k, 0)])
        return cls(n, {int(p): complex(dense[p]) for p in pos})


@dataclass(frozen=True)
class PermutationParams:
    """(sigma, tau, b'): x'_i = x_{sigma(i - tau)} w^{b' sigma i}
    (sfft/signal.py:159-210).  Host integers; the kernels receive them as
    int64 arrays."""

    n: int
    sigma: int = 1
    tau: int = 0
    b_prime: int = 0

    def __post_init__(self):
        if math.gcd(self.sigma % self.n, self.n) != 1:
            raise NonInvertibleScaling(f"gcd(sigma={self.sigma}, n={self.n}) != 1")
        object.__setattr__(self, "sigma", self.sigma % self.n)
        object.__setattr__(self, "tau", self.tau % self.n)
        object.__setattr__(self, "b_prime", self.b_prime % self.n)

    @property
    def b(self) -> int:
        return (self.b_prime * self.sigma) % self.n

    @property
    def sigma_inv(self) -> int:
        return pow(self.sigma, -1, self.n)

    def permuted_position(self, freq):
        f = np.asarray(freq, dtype=np.int64)
        return (self.sigma * (f - self.b_prime)) % self.n

    def original_position(self, permuted):
        m = np.asarray(permuted, dtype=np.int64)
        return (self.sigma_inv * m + self.b_prime) % self.n

    @classmethod
    def identity(cls, n: int) -> "PermutationParams":
        return cls(n=n)

    @classmethod
    def random(cls, n: int, rng: np.random.Generator, use_b: bool = False) -> "PermutationParams":
        """Same draws, in the same order, as the reference: sigma by rejection
        on gcd, then tau, then b' when requested."""
        sigma = int(rng.integers(1, n))
        while math.gcd(sigma, n) != 1:
            sigma = int(rng.integers(1, n))
        tau = int(rng.integers(0, n))
        b_prime = int(rng.integers(0, n)) if use_b else 0
        return cls(n=n, sigma=sigma, tau=tau, b_prime=b_prime)
