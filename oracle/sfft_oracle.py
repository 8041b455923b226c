"""CPU oracle for the sparse-FFT bucketization hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference algorithm
(`sparsefft`, /root/reference/pkg/src/sparsefft) for the rows of SURVEY.md §8:
flat/spike bucketization, the robust noise floor, heavy-bucket voting, vote
selection, bucket-energy estimation, the trimmed mean over rounds, the
bucket-domain forward-model subtraction and the voting / iterative (phase) /
peeling runners.  Every function cites the reference lines it restates.

It is the *checker*, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it.
The product path (``paper_2012_08238_b200``) never imports this module and has
no CPU fallback.

Parity pin: ``tests/golden/make_golden.py`` runs the real reference (importable
in the build container only) on seeded inputs and stores its outputs under
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this module
against every one of those vectors, so the oracle is pinned, not free-standing.

Index conventions (as in the reference, `sfft/signal.py:1-21`): forward DFT
carries 1/N, w_N = exp(-2*pi*i/N).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "OracleError", "unit_root", "Access", "draw_perm", "flat_support", "flat_sigma",
    "FlatWindow", "flat_window", "flat_buckets", "spike_buckets", "noise_floor",
    "vote_counts", "pick_votes", "energy_est", "robust_mean", "model_subtract",
    "ladder", "unwrap", "Cfg", "Outcome", "resolve_b", "voting", "iterative",
    "peeling", "synth", "keep_top", "n_buckets_for",
]


class OracleError(Exception):
    """Raised where the reference raises a SparseFFTError subclass; ``kind``
    carries the reference exception name."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ---------------------------------------------------------------- primitives

def unit_root(n: int, e) -> np.ndarray:
    """w_n^e with the exponent reduced in int64 first (sfft/signal.py:50-57)."""
    red = np.mod(np.asarray(e, dtype=np.int64), n)
    return np.exp(-2j * np.pi * red / n)


class Access:
    """Distinct-index bookkeeping of one signal read (sfft/signal.py:60-106)."""

    def __init__(self, samples):
        self.x = np.ascontiguousarray(samples, dtype=np.complex128)
        self.seen = np.zeros(self.x.size, dtype=bool)

    @property
    def n(self) -> int:
        return self.x.size

    def read(self, idx) -> np.ndarray:
        i = np.mod(np.asarray(idx, dtype=np.int64), self.n)
        self.seen[i] = True
        return self.x[i]

    def count(self) -> int:
        return int(np.count_nonzero(self.seen))


def draw_perm(n: int, rng: np.random.Generator, use_b: bool = False):
    """(sigma, tau, b') drawn exactly like PermutationParams.random
    (sfft/signal.py:202-210): rejection on gcd, then tau, then optional b'."""
    sigma = int(rng.integers(1, n))
    while math.gcd(sigma, n) != 1:
        sigma = int(rng.integers(1, n))
    tau = int(rng.integers(0, n))
    bp = int(rng.integers(0, n)) if use_b else 0
    return sigma % n, tau % n, bp % n


# ---------------------------------------------------------------- flat window

def flat_sigma(n: int, b: int) -> float:
    """sfft/filters.py:114-115."""
    return b * math.sqrt(math.log2(n))


def flat_support(n: int, b: int) -> int:
    """Even ceil(4*sigma_g), capped at N (sfft/filters.py:118-122)."""
    w = math.ceil(4.0 * flat_sigma(n, b))
    if w % 2:
        w += 1
    return min(w, n - (n % 2))


@dataclass
class FlatWindow:
    n: int
    b: int
    support: int
    taps: np.ndarray          # float64[support] (reference stores them as complex)
    response: np.ndarray      # complex128[n], B-normalised transform of the taps
    center: int = 0           # passband offset in bins (flat_shift)

    @property
    def width(self) -> int:
        return self.n // self.b


def flat_window(n: int, b: int, support: int | None = None,
                gauss_sigma: float | None = None) -> FlatWindow:
    """Gaussian x sinc taps and their response (sfft/filters.py:125-151)."""
    if b <= 0 or n % b:
        raise OracleError("InvalidParameter", f"B={b} does not divide n={n}")
    w = flat_support(n, b) if support is None else support
    sg = flat_sigma(n, b) if gauss_sigma is None else gauss_sigma
    if w % 2 or not 0 < w <= n:
        raise OracleError("InvalidParameter", f"support {w}")
    u = np.arange(w, dtype=float) - w / 2
    with np.errstate(divide="ignore", invalid="ignore"):
        core = np.where(u == 0, 1.0 / b, np.sin(np.pi * u / b) / (np.pi * u))
    taps = core * np.exp(-0.5 * (u / sg) ** 2)
    line = np.zeros(n, dtype=np.complex128)
    line[:w] = taps
    return FlatWindow(n, b, w, taps, np.fft.fft(line) / b)


def flat_shift(win: FlatWindow, f0: int) -> FlatWindow:
    """Passband moved by f0 bins: taps *= w^(-f0 i), response recomputed
    (sfft/filters.py:190-200).  ``center`` accumulates the offset."""
    i = np.arange(win.support, dtype=np.int64)
    taps = win.taps * unit_root(win.n, -f0 * i)
    line = np.zeros(win.n, dtype=np.complex128)
    line[:win.support] = taps
    return FlatWindow(win.n, win.b, win.support, taps, np.fft.fft(line) / win.b,
                      (win.center + f0) % win.n)


# ---------------------------------------------------------------- encode

def flat_buckets(acc: Access, win: FlatWindow, sigma: int, tau: int,
                 bprime: int = 0, tau_extra: int = 0) -> np.ndarray:
    """Permuted gather, window, fold mod B, B-point DFT / B
    (sfft/bucketize.py:142-161, fold :135-139)."""
    n, b = acc.n, win.b
    tt = (tau + tau_extra) % n
    i = np.arange(win.support, dtype=np.int64)
    z = win.taps.astype(np.complex128) * acc.read((sigma * (i - tt)) % n) \
        * unit_root(n, bprime * sigma * i)
    rows = -(-z.size // b)
    folded = np.zeros(rows * b, dtype=np.complex128)
    folded[:z.size] = z
    return np.fft.fft(folded.reshape(rows, b).sum(axis=0)) / b


def spike_buckets(acc: Access, b: int, tau: int = 0) -> np.ndarray:
    """Stride-(N/B) subsample behind a shift, B-point DFT / B
    (sfft/bucketize.py:164-178)."""
    n = acc.n
    if b <= 0 or n % b:
        raise OracleError("NonDivisorParameter", f"B={b} does not divide n={n}")
    step = n // b
    return np.fft.fft(acc.read((step * np.arange(b, dtype=np.int64) - tau) % n)) / b


# ---------------------------------------------------------------- Dirichlet bank

@dataclass(frozen=True)
class DirichletBank:
    """make_dirichlet_bank (sfft/filters.py:168-187) [+ filter_freq_shift :190-200]."""
    n: int
    width: int            # L
    b: int
    half: bool
    taps: np.ndarray      # complex128[L]
    response: np.ndarray  # complex128[n], unnormalised transform of the padded taps
    center: int = 0       # center_offset


def dirichlet_bank(n: int, width: int, b: int, half: bool = True) -> DirichletBank:
    if width * b != n:
        raise OracleError("NonDivisorParameter", f"{width}*{b} != n={n}")
    taps = np.full(width, math.sqrt(n) / width, dtype=np.complex128)
    pad = np.zeros(n, dtype=np.complex128)
    pad[:width] = taps
    return DirichletBank(n, width, b, half, taps, np.fft.fft(pad))


def dirichlet_shift(bank: DirichletBank, f0: int) -> DirichletBank:
    """filter_freq_shift for a Dirichlet bank: taps *= w^{-f0 pos}, response
    recomputed unnormalised, center_offset += f0 (sfft/filters.py:190-200)."""
    pos = np.arange(bank.width, dtype=np.int64)
    taps = bank.taps * unit_root(bank.n, -f0 * pos)
    pad = np.zeros(bank.n, dtype=np.complex128)
    pad[pos] = taps
    return DirichletBank(bank.n, bank.width, bank.b, bank.half, taps, np.fft.fft(pad),
                         (bank.center + f0) % bank.n)


def dirichlet_buckets(acc: Access, bank: DirichletBank, offsets) -> np.ndarray:
    """Box windows at each sample offset t: L consecutive samples x[t - i],
    fold mod B, B * inverse transform, de-rotate by w^{-c t} at each bucket
    center, average over offsets (sfft/bucketize.py:181-211)."""
    n, b, L = acc.n, bank.b, bank.width
    offsets = tuple(int(t) for t in offsets)
    if not offsets:
        raise OracleError("NonDivisorParameter", "at least one sample offset is required")
    base = 0 if bank.half else L // 2
    centers = (L * np.arange(b, dtype=np.int64) + base + bank.center) % n
    pos = np.arange(L, dtype=np.int64)
    half_mod = unit_root(n, -(L // 2) * pos) if not bank.half else np.ones(L, dtype=np.complex128)
    total = np.zeros(b, dtype=np.complex128)
    for t in offsets:
        win = bank.taps * acc.read((t - pos) % n) * half_mod
        pad = (-win.size) % b
        z = np.concatenate([win, np.zeros(pad, dtype=win.dtype)]) if pad else win
        v = b * np.fft.ifft(z.reshape(-1, b).sum(axis=0))
        total += v * unit_root(n, centers * t)
    return total / len(offsets)


def freqshift_estimate(acc: Access, f: int, t: int, seed=0) -> complex:
    """Mean of x[i] w^{f i} over t random (or all N) positions
    (sfft/reconstruct.py:356-371)."""
    if t < 1:
        raise OracleError("InvalidParameter", f"t={t} must be >= 1")
    n = acc.n
    if t >= n:
        idx = np.arange(n, dtype=np.int64)
    else:
        rng = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
        idx = rng.integers(0, n, size=t)
    return complex(np.mean(acc.read(idx) * unit_root(n, f * idx)))


# ---------------------------------------------------------------- decode

def noise_floor(values, mult: float = 3.0) -> float:
    """max(min(3*median, peak/4), 1e-9*peak, 1e-300) (sfft/reconstruct.py:119-133)."""
    mag = np.abs(np.asarray(values))
    if mag.size == 0:
        return 0.0
    top = float(mag.max())
    return float(max(min(mult * np.median(mag), 0.25 * top), 1e-9 * top, 1e-300))


def _flat_bucket_of(n: int, b: int, sigma: int, bprime: int, pos, cshift: int = 0):
    """Flat hash (sfft/bucketize.py:85-94): round-to-nearest passband."""
    L = n // b
    m = (sigma * (np.asarray(pos, dtype=np.int64) - bprime)) % n
    return (((m - cshift + L // 2) % n) // L) % b


def _heavy_order(values, thr: float) -> np.ndarray:
    """Buckets at/above max(thr, 0) ordered by (-|v|, index)
    (sfft/reconstruct.py:171-175)."""
    mag = np.abs(values)
    ok = np.flatnonzero(mag >= max(thr, 0.0))
    return ok[np.lexsort((ok, -mag[ok]))]


def vote_counts(rounds, heavy_count: int, n: int) -> np.ndarray:
    """Per-position vote counts.  ``rounds`` = [(values, thr, sigma, bprime)].

    Restates vote_tally (sfft/reconstruct.py:158-179) as a per-position
    evaluation: position f scores one in round r iff its flat bucket under
    round r's permutation is among that round's heavy buckets — the same set
    the reference reaches by scattering bucket preimages
    (sfft/bucketize.py:108-118)."""
    counts = np.zeros(n, dtype=np.int64)
    f = np.arange(n, dtype=np.int64)
    for values, thr, sigma, bprime in rounds:
        b = len(values)
        heavy = np.zeros(b, dtype=bool)
        heavy[_heavy_order(values, thr)[:heavy_count]] = True
        counts += heavy[_flat_bucket_of(n, b, sigma, bprime, f)]
    return counts


def pick_votes(counts: np.ndarray, nrounds: int, keep: int, min_fraction: float) -> list:
    """sfft/reconstruct.py:182-194: score >= max(frac*R, 1e-12), (-score, pos)."""
    if nrounds == 0 or keep <= 0:
        return []
    need = max(min_fraction * nrounds, 1e-12)
    pos = np.flatnonzero(counts >= need)
    pos = pos[np.lexsort((pos, -counts[pos]))]
    return [int(p) for p in pos[:keep]]


def energy_est(values, win: FlatWindow, sigma: int, tau: int, cands,
               floor_frac: float = 0.05) -> np.ndarray:
    """Bucket value / (weight * phase), NaN under the response floor
    (sfft/frameworks.py:321-332)."""
    n, L = win.n, win.width
    m = (sigma * np.asarray(cands, dtype=np.int64)) % n
    bk = ((m + L // 2) % n) // L
    w = win.response[(bk * L - m) % n]
    with np.errstate(divide="ignore", invalid="ignore"):
        est = values[bk] / (w * unit_root(n, tau * m))
    est[np.abs(w) < floor_frac * np.abs(win.response).max()] = np.nan
    return est


def robust_mean(est: np.ndarray) -> np.ndarray:
    """Trimmed mean around the coordinatewise median over rounds
    (sfft/frameworks.py:335-351)."""
    with np.errstate(all="ignore"):
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            centre = np.nanmedian(est.real, axis=0) + 1j * np.nanmedian(est.imag, axis=0)
            dist = np.abs(est - centre[None, :])
            q1 = np.nanquantile(dist, 0.25, axis=0)
            lim = np.maximum(4.0 * q1, 1e-8 * (np.abs(centre) + 1e-300))
            kept = np.where(dist <= lim[None, :], est, np.nan)
            re = np.nanmean(np.where(np.isnan(kept), np.nan, kept.real), axis=0)
            im = np.nanmean(np.where(np.isnan(kept), np.nan, kept.imag), axis=0)
    return re + 1j * im


def model_subtract(values, win: FlatWindow, sigma: int, tau: int, tau_extra: int,
                   tones) -> np.ndarray:
    """y[b] - sum_f c_f * G[(bL - sigma f) mod N] * w^(tau_tot * sigma f), tones in
    order (sfft/frameworks.py:423-436).  ``tones`` is an iterable of (f, c)."""
    tones = list(tones.items()) if isinstance(tones, dict) else list(tones)
    if not tones:
        return values
    n, b, L = win.n, win.b, win.width
    out = np.array(values, dtype=np.complex128, copy=True)
    tt = (tau + tau_extra) % n
    bl = np.arange(b, dtype=np.int64) * L
    for f, c in tones:
        m = (sigma * f) % n
        out -= c * win.response[(bl - m) % n] * unit_root(n, tt * m)
    return out


# ---------------------------------------------------------------- config

_FRAMEWORKS = ("one_shot", "voting", "iterative", "peeling", "dense")


@dataclass(frozen=True)
class Cfg:
    """The AlgorithmConfig fields the hot-path runners read
    (sfft/frameworks.py:67-122)."""
    framework: str
    num_buckets: int | None = None
    coprime_factors: tuple | None = None
    location_method: str | None = None
    branching: int = 2
    rounds: int = 10
    max_iterations: int = 10
    spike_prestage: bool = False
    prestage_width: int = 32
    min_vote_fraction: float = 0.5
    a_max: int = 4
    pursuit_shifts: int = 8
    seed: int = 0


def resolve_b(framework: str, num_buckets, n: int, k: int) -> int:
    """sfft/frameworks.py:111-122."""
    b = num_buckets
    if b is None:
        mult = 8 if framework == "one_shot" else 4
        b = 1 << max(3, math.ceil(math.log2(max(mult * max(k, 1), 8))))
        while b > max(n // 2, 1):
            b //= 2
    if n % b:
        raise OracleError("ConfigMismatch", f"B={b} does not divide n={n}")
    return b


def n_buckets_for(n: int, k: int) -> int:
    """Config-5 rule from BASELINE.json: next power of two >= sqrt(N K)."""
    return 1 << math.ceil(math.log2(math.sqrt(n * k)))


@dataclass
class Outcome:
    entries: dict = field(default_factory=dict)
    samples_read: int = 0
    iterations: int = 0
    converged: bool = False


def keep_top(entries: dict, k: int) -> dict:
    """Drop exact zeros, keep k largest |c|, ties to smaller f
    (sfft/frameworks.py:151-155; sfft/signal.py:142-145)."""
    nz = [(int(f), complex(c)) for f, c in entries.items() if c != 0]
    nz.sort(key=lambda t: (-abs(t[1]), t[0]))
    return dict(nz[:max(k, 0)])


def _finish(acc: Access, entries, k, iters, conv) -> Outcome:
    return Outcome(keep_top(entries, k), acc.count(), iters, conv)


# ---------------------------------------------------------------- voting

def voting(acc: Access, k: int, cfg: Cfg) -> Outcome:
    """Randomised rounds, top-2K heavy votes, energy estimates, trimmed mean and
    two candidate-model refinement passes (sfft/frameworks.py:354-417)."""
    n = acc.n
    if cfg.rounds <= 0 or k <= 0:
        return _finish(acc, {}, max(k, 0), 0, False)
    b = resolve_b("voting", cfg.num_buckets, n, k)
    win = flat_window(n, b)
    rng = np.random.default_rng(cfg.seed)

    allowed = None
    if cfg.spike_prestage:
        bpre = n // max(2, cfg.prestage_width)
        pv = spike_buckets(acc, bpre, 0)
        top = _heavy_order(pv, noise_floor(pv))[:2 * k]
        step = n // bpre
        if top.size:
            allowed = np.unique(np.concatenate(
                [np.sort(int(i) + bpre * np.arange(step, dtype=np.int64)) for i in top]))
        else:
            allowed = np.zeros(0, dtype=np.int64)

    perms, vals, rounds = [], [], []
    for _ in range(cfg.rounds):
        s, t, bp = draw_perm(n, rng)
        y = flat_buckets(acc, win, s, t, bp, 0)
        perms.append((s, t))
        vals.append(y)
        rounds.append((y, noise_floor(y), s, bp))

    counts = vote_counts(rounds, 2 * k, n)
    cands = np.array(pick_votes(counts, cfg.rounds, 2 * k, cfg.min_vote_fraction),
                     dtype=np.int64)
    if allowed is not None and cands.size:
        cands = cands[np.isin(cands, allowed)]
    if cands.size == 0:
        return _finish(acc, {}, k, cfg.rounds, True)

    est = np.vstack([energy_est(y, win, s, t, cands) for y, (s, t) in zip(vals, perms)])
    coef = robust_mean(est)
    for _ in range(2):
        safe = np.where(np.isfinite(coef), coef, 0.0)
        model = [(int(f), complex(c)) for f, c in zip(cands, safe)]
        est = np.vstack([energy_est(model_subtract(y, win, s, t, 0, model), win, s, t, cands)
                         for y, (s, t) in zip(vals, perms)])
        coef = safe + robust_mean(est)
    ent = {int(f): complex(c) for f, c in zip(cands, coef)
           if np.isfinite(c.real) and np.isfinite(c.imag)}
    return _finish(acc, ent, k, cfg.rounds, True)


# ---------------------------------------------------------------- iterative (phase)

def ladder(n: int) -> list:
    """1, 8, 64, ... below N/16, then N/16 (sfft/frameworks.py:199-213)."""
    top = max(n // 16, 1)
    out, d = [], 1
    while d < top:
        out.append(d)
        d *= 8
    out.append(top)
    return out


def unwrap(y0, ys: dict, n: int):
    """Coarse-to-fine phase unwrapping over the ladder (sfft/frameworks.py:179-196)."""
    if abs(y0) == 0 or 1 not in ys:
        return None
    q = (np.angle(ys[1] / y0) * (-n / (2.0 * np.pi))) % n
    for d in sorted(ys):
        if d == 1:
            continue
        phi = (np.angle(ys[d] / y0) * (-n / (2.0 * np.pi))) % n
        period = n / d
        base = phi / d
        q = base + np.round((q - base) / period) * period
    return int(np.round(q)) % n


class Ambiguous(Exception):
    """AmbiguousSplit (sfft/errors.py)."""


def split_search(sub, bucket: int, width: int, branching: int, noise_floor: float) -> int:
    """Iterated class splits of the in-bucket offset (sfft/reconstruct.py:197-215):
    digit by digit, the `branching` class sums mod step = scale*branching are
    compared by magnitude; a top-two gap below the noise floor is ambiguous."""
    digits = round(np.log(width) / np.log(branching))
    if branching < 2 or branching ** digits != width:
        raise OracleError("InvalidParameter", f"width {width} is not a power of {branching}")
    r, scale = 0, 1
    for _ in range(digits):
        step = scale * branching
        mags = np.array([abs(sub(bucket, r + d * scale, step)) for d in range(branching)])
        top = np.sort(mags)[::-1]
        if top[0] - top[1] < noise_floor:
            raise Ambiguous(f"{top[0]:.3g} vs {top[1]:.3g}")
        r += scale * int(np.argmax(mags))
        scale = step
    return r


def iterative(acc: Access, k: int, cfg: Cfg) -> Outcome:
    """Iterative framework (sfft/frameworks.py:439-570) with phase location
    (:493-516) or binary / multiscale class-split location (:517-554), plus the
    residual polish (:573-608)."""
    loc = cfg.location_method or "phase"
    if loc not in ("phase", "binary", "multiscale"):
        raise OracleError("ConfigMismatch", f"iterative cannot use location {loc}")
    n = acc.n
    if k <= 0:
        return _finish(acc, {}, 0, 0, True)
    b = resolve_b("iterative", cfg.num_buckets, n, k)
    win = flat_window(n, b)
    L = win.width
    rng = np.random.default_rng(cfg.seed)
    rec: dict = {}
    conv, its = False, 0
    peak = np.abs(win.response).max()
    sref, last = 0.0, np.inf
    rungs = ladder(n)

    for its in range(1, cfg.max_iterations + 1):
        s, t, bp = draw_perm(n, rng)
        sinv = pow(s, -1, n)
        memo: dict = {}

        def meas(d):
            d %= n
            if d not in memo:
                memo[d] = model_subtract(flat_buckets(acc, win, s, t, bp, d), win, s, t, d, rec)
            return memo[d]

        y0 = meas(0)
        mag = np.abs(y0)
        sref = max(sref, mag.max())
        fl = max(noise_floor(y0), 1e-9 * sref)
        if mag.max() < 1.3 * fl:
            conv, last = True, float(mag.max())
            its -= 1
            break
        hv = np.flatnonzero(mag >= fl)
        hv = hv[np.lexsort((hv, -mag[hv]))]
        new: dict = {}
        if loc == "phase":
            ys = {d: meas(d) for d in rungs}
            for bi in hv:
                q = unwrap(y0[bi], {d: ys[d][bi] for d in rungs}, n)
                if q is None:
                    continue
                lo = (bi * L - L // 2) % n
                if (q - lo) % n >= L:
                    continue
                tol = max(3.0 * fl, 0.15 * abs(y0[bi]))
                if any(abs(ys[d][bi] - y0[bi] * unit_root(n, d * q)) > tol for d in rungs):
                    continue
                w = win.response[(bi * L - q) % n]
                if abs(w) < 0.05 * peak:
                    continue
                sh = np.array([0] + rungs, dtype=np.int64)
                v = np.array([y0[bi]] + [ys[d][bi] for d in rungs])
                c = complex(np.mean(v * unit_root(n, -(t + sh) * q)) / w)
                f = int((sinv * q + bp) % n)
                new[f] = new.get(f, 0.0) + c
        else:
            br = 2 if loc == "binary" else cfg.branching
            digits = round(math.log(L, br))
            if br ** digits != L:
                raise OracleError("ConfigMismatch", f"bucket width {L} is not a power of {br}")

            def sub(bi, off, step):
                # class-sum measurement from `step` shifted bucketizations
                base = (bi * L - L // 2) % n
                qc = (base + off) % step
                dd = np.arange(step, dtype=np.int64)
                vals = np.array([meas(int(tt))[bi] for tt in dd * (n // step)])
                return complex(np.mean(vals * np.exp(2j * np.pi * dd * qc / step)))

            for bi in hv:
                try:
                    r = split_search(sub, int(bi), L, br, fl / 2)
                except Ambiguous:
                    continue
                q = (bi * L - L // 2 + r) % n
                meas(1), meas(3)  # whole-window alias check shifts
                tol = max(3.0 * fl, 0.15 * abs(y0[bi]))
                checks = [tt for tt in sorted(memo) if tt != 0]
                if any(abs(memo[tt][bi] - y0[bi] * unit_root(n, tt * q)) > tol for tt in checks):
                    continue
                w = win.response[(bi * L - q) % n]
                if abs(w) < 0.05 * peak:
                    continue
                c = complex(y0[bi] * unit_root(n, -t * q) / w)
                f = int((sinv * q + bp) % n)
                new[f] = new.get(f, 0.0) + c
        for f, c in new.items():
            rec[f] = rec.get(f, 0.0) + c
        if len(rec) >= k and new:
            r = model_subtract(y0, win, s, t, 0, new)
            if np.abs(r).max() < 1.3 * fl:
                conv, last = True, float(np.abs(r).max())
                break

    if conv and rec and last < 0.01 * sref:
        _polish(acc, win, rng, rec)
    return _finish(acc, rec, k, its, conv)


def _polish(acc: Access, win: FlatWindow, rng, rec: dict) -> None:
    """Residual corrections at fresh permutations, 2 epochs x <=3 passes x
    shifts (0,1,2); only non-collided tones are corrected
    (sfft/frameworks.py:573-608)."""
    n, b, L = win.n, win.b, win.width
    peak = np.abs(win.response).max()
    for _ in range(2):
        todo = set(rec)
        for _ in range(3):
            if not todo:
                break
            s, t, bp = draw_perm(n, rng)
            res = {d: model_subtract(flat_buckets(acc, win, s, t, bp, d), win, s, t, d, rec)
                   for d in (0, 1, 2)}
            fs = sorted(rec)
            m = (s * np.asarray(fs, dtype=np.int64)) % n
            bk = ((m + L // 2) % n) // L
            occ = np.bincount(bk, minlength=b)
            for f, mi, bi in zip(fs, m, bk):
                if f not in todo or occ[bi] != 1:
                    continue
                w = win.response[(bi * L - mi) % n]
                if abs(w) < 0.05 * peak:
                    continue
                v = np.array([res[d][bi] * unit_root(n, -(t + d) * mi) for d in (0, 1, 2)])
                rec[f] += complex(np.mean(v) / w)
                todo.discard(f)


# ---------------------------------------------------------------- peeling

_ZERO, _SINGLE, _MULTI = 0, 1, 2


def _nearest(raw: float, cands: np.ndarray, n: int) -> int:
    """Circular nearest candidate, ties to the smaller (sfft/reconstruct.py:136-140)."""
    d = np.abs((cands.astype(float) - raw + n / 2) % n - n / 2)
    return int(cands[np.lexsort((cands, d))[0]])


def _classify(mom: np.ndarray, bucket: int, b: int, n: int, fl: float):
    """a_max=1 classification (sfft/reconstruct.py:412-440 with :143-155)."""
    if mom.size < 2:
        raise OracleError("InvalidParameter", f"{mom.size} moments cannot resolve a_max=1")
    if float(np.mean(np.abs(mom))) < fl:
        return (_ZERO, None, None)
    if abs(mom[0]) < fl:
        return (_MULTI, None, None)
    if abs(mom[0]) <= 0.0:
        raise OracleError("ZeroTonBucket", "empty reference moment")
    raw = (np.angle(mom[1] / mom[0]) * (-n / (2 * np.pi))) % n
    L = n // b
    f = _nearest(raw, (bucket + b * np.arange(L, dtype=np.int64)) % n, n)
    car = unit_root(n, np.arange(mom.size, dtype=np.int64) * f)
    if np.abs(mom - mom[0] * car).max() < max(fl, 0.05 * abs(mom[0])):
        return (_SINGLE, f, complex(np.mean(mom * car.conj())))
    return (_MULTI, None, None)


def peeling(acc: Access, k: int, cfg: Cfg) -> Outcome:
    """Co-prime spike stages, classification, two-tier FIFO single-ton peeling
    (sfft/frameworks.py:614-699)."""
    n = acc.n
    ps = tuple(int(p) for p in (cfg.coprime_factors or ()))
    if not ps:
        raise OracleError("ConfigMismatch", "peeling requires coprime_factors")
    if any(p <= 1 for p in ps) or math.prod(ps) != n:
        raise OracleError("ConfigMismatch", f"factors {ps} vs n={n}")
    for i, p in enumerate(ps):
        for q in ps[i + 1:]:
            if math.gcd(p, q) != 1:
                raise OracleError("ConfigMismatch", f"{p},{q} not co-prime")
    if k <= 0:
        return _finish(acc, {}, 0, 0, True)

    st = []
    for p in ps:
        b = n // p
        ns = 3 if p > 3 else max(p - 1, 1)
        mm = np.vstack([spike_buckets(acc, b, t) for t in range(ns)])
        st.append(dict(b=b, ns=ns, m=mm, fl=noise_floor(mm[0]), ver=ns >= 3, cls={}))

    def cls_of(sg, bk):
        col = sg["m"][:, bk]
        if np.abs(col).mean() < sg["fl"]:
            return (_ZERO, None, None)
        return _classify(col, bk, sg["b"], n, sg["fl"])

    qs = {True: [], False: []}
    for si, sg in enumerate(st):
        for bk in np.flatnonzero(np.abs(sg["m"]).mean(axis=0) >= sg["fl"]):
            c = cls_of(sg, int(bk))
            sg["cls"][int(bk)] = c
            if c[0] == _SINGLE:
                qs[sg["ver"]].append((si, int(bk)))

    rec: dict = {}
    budget = k + sum(sg["b"] for sg in st)
    peels = 0
    while peels < budget:
        hit = None
        for tier in (True, False):
            while qs[tier]:
                si, bk = qs[tier].pop(0)
                c = st[si]["cls"].get(bk)
                if c is not None and c[0] == _SINGLE:
                    hit = c
                    break
            if hit is not None:
                break
        if hit is None:
            break
        f, c = hit[1], hit[2]
        rec[f] = rec.get(f, 0.0) + c
        peels += 1
        for si, sg in enumerate(st):
            bk = f % sg["b"]
            sg["m"][:, bk] -= c * unit_root(n, np.arange(sg["ns"], dtype=np.int64) * f)
            c2 = cls_of(sg, bk)
            sg["cls"][bk] = c2
            if c2[0] == _SINGLE:
                qs[sg["ver"]].append((si, bk))
    stuck = any(c[0] == _MULTI for sg in st for c in sg["cls"].values())
    return _finish(acc, rec, k, peels, not stuck)


# ---------------------------------------------------------------- inputs

def synth(n: int, k: int, snr_db, seed: int, positions=None, magnitudes=None):
    """Seeded K-sparse test signal, restating gen_signal (sfft/harness.py:93-124):
    positions without replacement (sorted), phases U[0,2pi), synthesis without
    1/N, complex AWGN scaled to the mean signal power.  Returns (x, truth)."""
    rng = np.random.default_rng(seed)
    if positions is None:
        positions = np.sort(rng.choice(n, size=k, replace=False))
    else:
        positions = np.asarray(positions, dtype=np.int64)
    mags = np.ones(k) if magnitudes is None else np.asarray(magnitudes)
    coefs = mags * np.exp(1j * rng.uniform(0.0, 2.0 * np.pi, size=k))
    spec = np.zeros(n, dtype=np.complex128)
    spec[positions] = coefs
    x = np.fft.ifft(spec) * n
    if snr_db is not None:
        p = float(np.mean(np.abs(x) ** 2))
        if p > 0:
            sd = math.sqrt(p / (10.0 ** (snr_db / 10.0)) / 2.0)
            x = x + (rng.normal(0.0, sd, n) + 1j * rng.normal(0.0, sd, n))
    return x, {int(f): complex(c) for f, c in zip(positions, coefs)}


# ---------------------------------------------------------------- one-shot

class _Singular(Exception):
    """SingularMomentMatrix / RankDeficient (sfft/errors.py)."""


def _hankel_counts(moms: np.ndarray, a_max: int) -> np.ndarray:
    """count_collisions (sfft/reconstruct.py:245-267): pooled singular values of
    the per-bucket a_max x a_max moment Hankel matrices.  moms: [2 a_max][B]."""
    b = moms.shape[1]
    if b == 0:
        return np.zeros(0, dtype=np.int64)
    h = np.empty((b, a_max, a_max), dtype=np.complex128)
    for i in range(b):
        m = moms[:, i]
        for r in range(a_max):
            h[i, r, :] = m[r:r + a_max]
    svals = np.linalg.svd(h, compute_uv=False)
    pooled = np.sort(svals.ravel())[::-1]
    cutoff = pooled[min(2 * b, pooled.size) - 1]
    floor = max(3.0 * np.median(pooled), 1e-12 * pooled[0]) if pooled[0] > 0 else np.inf
    counts = np.zeros(b, dtype=np.int64)
    for i in range(b):
        sv = svals[i]
        ok = (sv >= cutoff) & (sv >= 0.1 * sv[0]) & (sv > floor)
        counts[i] = min(int(ok.sum()), a_max)
    return counts


def _prony_positions(m: np.ndarray, a: int, bucket: int, b: int, n: int) -> list:
    """locate_prony (sfft/reconstruct.py:270-302): linear prediction by lstsq,
    companion roots on the unit circle, nearest admissible positions."""
    rows = m.size - a
    mat = np.empty((rows, a), dtype=np.complex128)
    for r in range(rows):
        mat[r] = m[r:r + a]
    rhs = -m[a:a + rows]
    coeffs, _, rank, sv = np.linalg.lstsq(mat, rhs, rcond=None)
    if rank < a or sv[0] <= 0 or sv[-1] < 1e-10 * sv[0]:
        raise _Singular("moment system rank")
    roots = np.roots(np.concatenate([[1.0], coeffs[::-1]]))
    mags = np.abs(roots)
    if np.any(mags < 1e-12):
        raise _Singular("vanishing root magnitude")
    roots = roots / mags
    cand = (bucket + b * np.arange(n // b, dtype=np.int64)) % n
    out = []
    for z in roots:
        raw = (-np.angle(z) * n / (2 * np.pi)) % n
        out.append(_nearest(raw, cand, n))
    return sorted(out)


def _prony_coeffs(positions, shifts, values, n: int) -> np.ndarray:
    """estimate_prony without `keep` (sfft/reconstruct.py:374-409)."""
    positions = np.asarray(positions, dtype=np.int64)
    a = positions.size
    if a == 0:
        return np.zeros(0, dtype=np.complex128)
    if shifts.size < a:
        raise _Singular("too few measurements")
    vand = unit_root(n, np.outer(shifts, positions))
    sol, _, rank, _ = np.linalg.lstsq(vand, values, rcond=None)
    if rank < a:
        raise _Singular("measurement matrix rank")
    return sol


def one_shot(acc: Access, k: int, cfg: Cfg) -> Outcome:
    """run_oneshot (sfft/frameworks.py:216-311): spike-train moments at shifts
    0..2a_max-1, ladder rungs and random pursuit shifts; Hankel collision
    counts; single-tons by phase unwrapping, collisions by Prony with
    escalation and a partner-subtraction refinement; least-squares
    coefficients."""
    n = acc.n
    if k <= 0:
        return _finish(acc, {}, 0, 0, True)
    b = resolve_b("one_shot", cfg.num_buckets, n, k)
    a_max = cfg.a_max
    rng = np.random.default_rng(cfg.seed)
    base = list(range(2 * a_max))
    lad = ladder(n)
    extra = [d for d in lad if d not in base]
    pursuit = [int(t) for t in rng.integers(0, n, size=cfg.pursuit_shifts)]
    shifts = np.array(base + extra + pursuit, dtype=np.int64)
    meas = np.vstack([spike_buckets(acc, b, int(t)) for t in shifts])
    rows = {d: meas[len(base) + j] for j, d in enumerate(extra)}
    for d in lad:
        if d in base:
            rows[d] = meas[d]
    moms = meas[:2 * a_max]
    floor = noise_floor(np.abs(moms[0]))
    counts = _hankel_counts(moms, a_max)
    energy = np.abs(moms).mean(axis=0)

    def solve(i, positions):
        c = _prony_coeffs(positions, shifts, meas[:, i], n)
        model = unit_root(n, np.outer(shifts, positions)) @ c
        return c, float(np.abs(meas[:, i] - model).max())

    def refine(i, positions, coeffs):
        out = []
        for j, f in enumerate(positions):
            others = [(g, c) for l, (g, c) in enumerate(zip(positions, coeffs)) if l != j]
            y0 = moms[0, i] - sum(c for _, c in others)
            ys = {d: rows[d][i] - sum(c * unit_root(n, d * g) for g, c in others) for d in lad}
            q = unwrap(y0, ys, n)
            out.append(int(i + round((q - i) / b) * b) % n if q is not None else f)
        return sorted(set(out))

    entries: dict = {}
    for i in range(b):
        if counts[i] == 0 or energy[i] < floor:
            continue
        tol = max(float(floor), 0.05 * float(energy[i]))
        best = None
        if counts[i] == 1:
            q = unwrap(moms[0, i], {d: rows[d][i] for d in lad}, n)
            if q is not None:
                pos = [int(i + round((q - i) / b) * b) % n]
                try:
                    c, r = solve(i, pos)
                    best = (r, pos, c)
                except _Singular:
                    best = None
        if best is None or best[0] >= tol:
            for a in range(max(int(counts[i]), 2), a_max + 1):
                try:
                    pos = sorted(set(_prony_positions(moms[:, i], a, i, b, n)))
                    pos = refine(i, pos, _prony_coeffs(pos, shifts, meas[:, i], n))
                    c, r = solve(i, pos)
                except _Singular:
                    continue
                if best is None or r < best[0]:
                    best = (r, pos, c)
                if r < tol:
                    break
        if best is None:
            try:
                pos = sorted(set(_prony_positions(moms[:, i], 1, i, b, n)))
                c, r = solve(i, pos)
                best = (r, pos, c)
            except _Singular:
                continue
        for f, c in zip(best[1], best[2]):
            entries[f] = entries.get(f, 0.0) + complex(c)
    return _finish(acc, entries, k, 1, True)
