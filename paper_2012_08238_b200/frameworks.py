"""Runner drop-ins (sfft/frameworks.py) backed by device-resident engines.

``AlgorithmConfig`` / ``RecoveryResult`` / ``run_algorithm`` keep the
reference's fields, validation and dispatch (:67-155, :704-715).
``run_voting`` / ``run_iterative`` / ``run_peeling`` keep their signatures
``(x, k, cfg) -> RecoveryResult``; each is the one-signal case of a batched
``*_batch(xs, k, cfg)`` that runs many independent signals through one
sequence of sm_100a kernels (csrc/voting.cu, iterative.cu, peeling.cu).

Randomness: the host draws every permutation with the reference's own
generator calls (``np.random.default_rng(cfg.seed)`` then
PermutationParams.random in order) and uploads them, so the device consumes
exactly the reference's stream.
"""

from __future__ import annotations

import hashlib
import json
import math
from dataclasses import asdict, dataclass, replace

import numpy as np

from ._lib import check, lib, ptr, stream_of
from .errors import ConfigMismatch
from .filters import FLAT, SPIKE, make_flat_filter, twiddles
from .signal import PermutationParams, SparseSpectrum, TimeSignal

__all__ = ["AlgorithmConfig", "RecoveryResult", "BatchResult", "FRAMEWORKS", "run_algorithm",
           "run_voting", "run_iterative", "run_peeling", "run_voting_batch",
           "run_iterative_batch", "run_peeling_batch", "phase_ladder", "draw_perms"]

FRAMEWORKS = ("one_shot", "voting", "iterative", "peeling", "dense")

_LOCATIONS = {"one_shot": {"prony"}, "voting": {"statistics"},
              "iterative": {"phase", "binary", "multiscale"}, "peeling": {"phase"},
              "dense": {"direct"}}
_DEFAULT_LOCATION = {"one_shot": "prony", "voting": "statistics", "iterative": "phase",
                     "peeling": "phase", "dense": "direct"}
_FILTERS = {"one_shot": SPIKE, "voting": FLAT, "iterative": FLAT, "peeling": SPIKE,
            "dense": "none"}
_ESTIMATIONS = {"one_shot": {"prony"}, "voting": {"energy"}, "iterative": {"energy"},
                "peeling": {"energy"}, "dense": {"direct"}}
_DEFAULT_ESTIMATION = {"one_shot": "prony", "voting": "energy", "iterative": "energy",
                       "peeling": "energy", "dense": "direct"}


@dataclass(frozen=True)
class AlgorithmConfig:
    """Same fields, validation, JSON round trip and digest as the reference
    (sfft/frameworks.py:67-138), so records are interchangeable."""

    framework: str
    filter_kind: str | None = None
    num_buckets: int | None = None
    coprime_factors: tuple | None = None
    location_method: str | None = None
    estimation_method: str | None = None
    rounds: int = 10
    max_iterations: int = 10
    a_max: int = 4
    branching: int = 2
    pursuit_shifts: int = 8
    spike_prestage: bool = False
    prestage_width: int = 32
    min_vote_fraction: float = 0.5
    seed: int = 0

    def validated(self) -> "AlgorithmConfig":
        if self.framework not in FRAMEWORKS:
            raise ConfigMismatch(f"unknown framework {self.framework!r}")
        fk = self.filter_kind or _FILTERS[self.framework]
        if fk != _FILTERS[self.framework]:
            raise ConfigMismatch(
                f"{self.framework} requires the {_FILTERS[self.framework]} filter, got {fk}")
        loc = self.location_method or _DEFAULT_LOCATION[self.framework]
        if loc not in _LOCATIONS[self.framework]:
            raise ConfigMismatch(f"{self.framework} cannot use location {loc!r}")
        est = self.estimation_method or _DEFAULT_ESTIMATION[self.framework]
        if est not in _ESTIMATIONS[self.framework]:
            raise ConfigMismatch(f"{self.framework} cannot use estimation {est!r}")
        if self.framework == "peeling" and not self.coprime_factors:
            raise ConfigMismatch("peeling requires coprime_factors")
        if self.a_max < 1:
            raise ConfigMismatch(f"a_max={self.a_max} must be >= 1")
        return replace(self, filter_kind=fk, location_method=loc, estimation_method=est)

    def resolve_buckets(self, n: int, k: int) -> int:
        b = self.num_buckets
        if b is None:
            mult = 8 if self.framework == "one_shot" else 4
            b = 1 << max(3, math.ceil(math.log2(max(mult * max(k, 1), 8))))
            while b > max(n // 2, 1):
                b //= 2
        if n % b != 0:
            raise ConfigMismatch(f"num_buckets={b} does not divide n={n}")
        return b

    def to_json(self) -> str:
        d = asdict(self)
        if d["coprime_factors"] is not None:
            d["coprime_factors"] = list(d["coprime_factors"])
        return json.dumps(d, sort_keys=True)

    @classmethod
    def from_json(cls, text: str) -> "AlgorithmConfig":
        d = json.loads(text)
        if d.get("coprime_factors") is not None:
            d["coprime_factors"] = tuple(d["coprime_factors"])
        return cls(**d)

    def digest(self) -> str:
        return hashlib.sha1(self.to_json().encode()).hexdigest()[:12]


@dataclass
class RecoveryResult:
    spectrum: SparseSpectrum
    samples_read: int
    iterations: int
    converged: bool


@dataclass
class BatchResult:
    """Device outputs of a batched run: pos/coef [S][k] in (-|c|, f) order,
    count/iterations/converged/samples_read [S]."""

    n: int
    k: int
    pos: object
    coef: object
    count: object
    iterations: object
    converged: object
    samples_read: object
    schedule: object = None   # int64 [S][groups][words] read schedule (see schedule_records)

    def schedule_records(self, s: int) -> list:
        """Read records of signal s in TimeSignal-log form."""
        if self.schedule is None:
            return []
        out = []
        for row in self.schedule[s].cpu().numpy():
            kind = int(row[0])
            if kind < 0:
                break
            a, tau, cnt, nsh = (int(v) for v in row[1:5])
            if kind == 0:
                for d in row[5:5 + nsh]:
                    out.append(("flat", a, (tau + int(d)) % self.n, cnt))
            elif kind == 2:  # split location: shifts j * row[5], j < nsh
                step = int(row[5])
                for j in range(nsh):
                    out.append(("flat", a, (tau + j * step) % self.n, cnt))
            else:
                out.append(("spike", a, tau % self.n, cnt))
        return out

    def to_results(self) -> list:
        pos = self.pos.cpu().numpy()
        coef = self.coef.cpu().numpy()
        cnt = self.count.cpu().numpy()
        its = self.iterations.cpu().numpy()
        conv = self.converged.cpu().numpy()
        smp = self.samples_read.cpu().numpy()
        out = []
        for s in range(pos.shape[0]):
            c = int(cnt[s])
            ent = {int(p): complex(v) for p, v in zip(pos[s, :c], coef[s, :c])}
            out.append(RecoveryResult(SparseSpectrum(self.n, ent), int(smp[s]), int(its[s]),
                                      bool(conv[s])))
        return out


def phase_ladder(n: int) -> list:
    """1, 8, 64, ... below N/16, then N/16 (sfft/frameworks.py:199-213)."""
    ladder, delta, top = [], 1, max(n // 16, 1)
    while delta < top:
        ladder.append(delta)
        delta *= 8
    ladder.append(top)
    return ladder


def draw_perms(n: int, seed: int, count: int):
    """The first ``count`` permutations of default_rng(seed) (sigma, tau)."""
    rng = np.random.default_rng(seed)
    sig = np.empty(count, dtype=np.int64)
    tau = np.empty(count, dtype=np.int64)
    for i in range(count):
        p = PermutationParams.random(n, rng)
        sig[i], tau[i] = p.sigma, p.tau
    return sig, tau


def _sched_buffer(S, dev):
    import ctypes
    import torch
    g, w = ctypes.c_int32(), ctypes.c_int32()
    lib().sfft_schedule_layout(ctypes.byref(g), ctypes.byref(w))
    return torch.empty((S, g.value, w.value), dtype=torch.int64, device=dev)


def _as_batch(xs):
    """[S][N] CUDA tensor (complex64/complex128) from a tensor, a TimeSignal
    or a list of TimeSignals."""
    import torch
    if isinstance(xs, TimeSignal):
        return xs.samples.unsqueeze(0), [xs]
    if isinstance(xs, (list, tuple)):
        sigs = list(xs)
        return torch.stack([s.samples for s in sigs]), sigs
    t = xs if xs.ndim == 2 else xs.unsqueeze(0)
    return t.contiguous(), None


def _empty_batch(n, S, k, dev, iterations, converged):
    import torch
    kk = max(k, 1)
    return BatchResult(n, max(k, 0), torch.zeros((S, kk), dtype=torch.int64, device=dev),
                       torch.zeros((S, kk), dtype=torch.complex128, device=dev),
                       torch.zeros(S, dtype=torch.int32, device=dev),
                       torch.full((S,), iterations, dtype=torch.int32, device=dev),
                       torch.full((S,), int(converged), dtype=torch.int32, device=dev),
                       torch.zeros(S, dtype=torch.int64, device=dev))


class _WS:
    """Grow-only device scratch handed to the library (caller-owned memory),
    keyed by (device, current stream, tag): a buffer is only ever used by the
    launches of the stream it was allocated on, so calls on different streams
    never share scratch, and the torch caching allocator's stream-ordered reuse
    keeps an evicted buffer safe.  At most ``cap`` buffers are kept (least
    recently used evicted), so pooled side streams cannot pin unbounded
    GB-scale workspaces."""
    buf: dict = {}
    cap: int = 8

    @classmethod
    def get(cls, nbytes, device, tag: str = ""):
        import torch
        dev = torch.device(device)
        key = (str(dev), torch.cuda.current_stream(dev).cuda_stream, tag)
        t = cls.buf.pop(key, None)
        if t is None or t.numel() < nbytes:
            t = None  # release before allocating the larger one
            t = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=dev)
        cls.buf[key] = t  # most recently used last
        while len(cls.buf) > cls.cap:
            cls.buf.pop(next(iter(cls.buf)))
        return t


# ------------------------------------------------------------------ iterative

DEFAULT_SLOTS = 128


def run_iterative_batch(xs, k: int, cfg: AlgorithmConfig, slots: int | None = None,
                        avail=None, engines: int = 1) -> BatchResult:
    """run_iterative (phase, binary or multiscale location) for every row of ``xs``.

    The device engine keeps ``slots`` signals in flight (default
    min(len(xs), 128)) and refills a slot from the queue as soon as its signal
    finishes, so long-running signals never idle the GPU.  ``avail`` (device
    int32 scalar) enables streaming admission (see run_iterative_stream).
    ``engines`` > 1 splits the queue over that many engines on their own CUDA
    streams (host threads; ctypes releases the GIL), so one engine's
    memory-bound gathers overlap another's FP64 subtraction kernels."""
    if engines > 1 and avail is None:
        return _iterative_engines(xs, k, cfg, slots, engines)
    import torch
    cfg = cfg.validated()
    if cfg.framework != "iterative":
        raise ConfigMismatch(f"run_iterative got framework {cfg.framework!r}")
    X, _ = _as_batch(xs)
    S, n = X.shape
    dev = X.device
    if k <= 0:
        return _empty_batch(n, S, 0, dev, 0, True)
    b = cfg.resolve_buckets(n, k)
    split = cfg.location_method in ("binary", "multiscale")
    if split:
        # class-split location (frameworks.py:517-522): n/B = branching^digits
        br = 2 if cfg.location_method == "binary" else cfg.branching
        width = n // b
        digits = round(math.log(width, br)) if br >= 2 and width >= 1 else 0
        if br < 2 or br ** digits != width:
            raise ConfigMismatch(f"bucket width {width} is not a power of branching {br}")
        ladder, M = [], width + 2
        # every loop keeps n/B + 2 bucketizations per slot: bound the slots by memory
        slot_cap = max(1, (8 << 30) // (M * b * 16))
    else:
        br = 0
        ladder = phase_ladder(n)
        M = 1 + len(ladder)
        slot_cap = S
    filt = make_flat_filter(n, b, device=dev)
    P = cfg.max_iterations + 6
    sig, tau = draw_perms(n, cfg.seed, P)
    psig = torch.as_tensor(sig, device=dev)    # one stream shared by all signals
    ptau = torch.as_tensor(tau, device=dev)
    nslots = min(S, slots or DEFAULT_SLOTS, slot_cap)
    cap = cfg.max_iterations * b
    out_pos = torch.zeros((S, k), dtype=torch.int64, device=dev)
    out_coef = torch.zeros((S, k), dtype=torch.complex128, device=dev)
    out_n = torch.zeros(S, dtype=torch.int32, device=dev)
    out_it = torch.zeros(S, dtype=torch.int32, device=dev)
    out_cv = torch.zeros(S, dtype=torch.int32, device=dev)
    out_sm = torch.zeros(S, dtype=torch.int64, device=dev)
    sched = _sched_buffer(S, dev)
    L = lib()
    wsb = L.sfft_iterative_ws_bytes(n, b, nslots, M, cap)
    ws = _WS.get(wsb, dev, "iterative")
    import ctypes
    lad = (ctypes.c_int64 * len(ladder))(*ladder) if ladder else None
    dt = 0 if X.dtype == torch.complex64 else 1
    gmax = torch.tensor([filt.peak], dtype=torch.float64, device=dev)
    check(L.sfft_run_iterative(dt, ptr(X), n, X.stride(0), S, nslots, ptr(filt.kernel_taps),
                               filt.support, b, ptr(filt.gtable), ptr(gmax),
                               ptr(twiddles(b, dev)), ptr(psig), ptr(ptau), P, 0, k,
                               cfg.max_iterations, lad, len(ladder), 1 if split else 0, br,
                               cap,
                               ptr(out_pos), ptr(out_coef), ptr(out_n), ptr(out_it), ptr(out_cv),
                               ptr(out_sm), ptr(sched), ptr(avail), ptr(ws), wsb,
                               stream_of(dev)), "sfft_run_iterative")
    return BatchResult(n, k, out_pos, out_coef, out_n, out_it, out_cv, out_sm, sched)


def _iterative_engines(xs, k, cfg, slots, engines):
    import threading

    import torch
    X, _ = _as_batch(xs)
    S = X.shape[0]
    dev = X.device
    parts = [(i * S // engines, (i + 1) * S // engines) for i in range(engines)]
    parts = [p for p in parts if p[1] > p[0]]
    per_slots = max(1, (slots or DEFAULT_SLOTS) // len(parts))
    main = torch.cuda.current_stream(dev)
    streams = [torch.cuda.Stream(dev) for _ in parts]
    out = [None] * len(parts)
    err = []

    def work(i):
        try:
            with torch.cuda.device(dev), torch.cuda.stream(streams[i]):
                streams[i].wait_stream(main)
                lo, hi = parts[i]
                out[i] = run_iterative_batch(X[lo:hi], k, cfg, slots=per_slots)
        except Exception as e:  # re-raised on the caller's thread
            err.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(parts))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    for s in streams:
        main.wait_stream(s)
    cat = lambda f: torch.cat([getattr(o, f) for o in out])
    return BatchResult(out[0].n, out[0].k, cat("pos"), cat("coef"), cat("count"),
                       cat("iterations"), cat("converged"), cat("samples_read"),
                       cat("schedule"))


def run_iterative_stream(host_x, k: int, cfg: AlgorithmConfig, slots: int | None = None,
                         chunk: int = 64, out=None) -> BatchResult:
    """End-to-end batch from host memory: rows of ``host_x`` (pinned CPU tensor
    [Q][N], complex64/complex128) are copied to the device chunk by chunk on a
    side stream while the engine already works on the rows that arrived
    (streaming admission), so the transfer overlaps the compute."""
    import torch
    from ._lib import require_cuda
    dev = require_cuda()
    Q, n = host_x.shape
    X = out if out is not None else torch.empty((Q, n), dtype=host_x.dtype, device=dev)
    avail = torch.zeros(1, dtype=torch.int32, device=dev)
    cs = torch.cuda.Stream(dev)
    cs.wait_stream(torch.cuda.current_stream(dev))
    L = lib()
    with torch.cuda.stream(cs):
        for c0 in range(0, Q, chunk):
            c1 = min(Q, c0 + chunk)
            X[c0:c1].copy_(host_x[c0:c1], non_blocking=True)
            check(L.sfft_set_avail(ptr(avail), c1, cs.cuda_stream), "sfft_set_avail")
    br = run_iterative_batch(X, k, cfg, slots=slots, avail=avail)
    torch.cuda.current_stream(dev).wait_stream(cs)
    return br


def run_iterative(x: TimeSignal, k: int, cfg: AlgorithmConfig) -> RecoveryResult:
    """Permute, bucketize, locate single-tons (phase ladder or binary /
    multiscale class splits), subtract, repeat (sfft/frameworks.py:439-570),
    then polish (:573-608)."""
    return _single(run_iterative_batch, x, k, cfg)


def _single(batch_fn, x, k, cfg) -> RecoveryResult:
    br = batch_fn(x, k, cfg)
    res = br.to_results()[0]
    if isinstance(x, TimeSignal):
        had = bool(x._log)
        for rec in br.schedule_records(0):
            x.record(rec)
        if had:
            # the access counter only grows: earlier reads of x count too
            res.samples_read = x.access_count
    return res


# ------------------------------------------------------------------ dispatch

def run_voting_batch(xs, k: int, cfg: AlgorithmConfig) -> BatchResult:
    from .voting import voting_batch
    return voting_batch(xs, k, cfg)


def run_voting(x: TimeSignal, k: int, cfg: AlgorithmConfig) -> RecoveryResult:
    """Randomised rounds, heavy-bucket votes, energy estimates, trimmed mean and
    two model-refinement passes (sfft/frameworks.py:354-417)."""
    return _single(run_voting_batch, x, k, cfg)


def run_peeling_batch(xs, k: int, cfg: AlgorithmConfig) -> BatchResult:
    from .peeling import peeling_batch
    return peeling_batch(xs, k, cfg)


def run_peeling(x: TimeSignal, k: int, cfg: AlgorithmConfig) -> RecoveryResult:
    """Co-prime spike stages decoded by single-ton peeling
    (sfft/frameworks.py:614-699)."""
    return _single(run_peeling_batch, x, k, cfg)


def run_oneshot_batch(xs, k: int, cfg: AlgorithmConfig) -> BatchResult:
    from .oneshot import oneshot_batch
    return oneshot_batch(xs, k, cfg)


def run_oneshot(x: TimeSignal, k: int, cfg: AlgorithmConfig) -> RecoveryResult:
    """Single spike-train encoding, Hankel collision counts, single-ton phase
    unwrapping / Prony location with refinement, least-squares estimation
    (sfft/frameworks.py:216-311)."""
    return _single(run_oneshot_batch, x, k, cfg)


_RUNNERS = {"one_shot": run_oneshot, "voting": run_voting, "iterative": run_iterative,
            "peeling": run_peeling}


def run_algorithm(x: TimeSignal, k: int, cfg: AlgorithmConfig) -> RecoveryResult:
    cfg = cfg.validated()
    if cfg.framework not in _RUNNERS:
        raise NotImplementedError(
            f"{cfg.framework!r} is outside the device hot path (SURVEY.md §2: the dense "
            "baseline is not rebuilt)")
    return _RUNNERS[cfg.framework](x, k, cfg)
