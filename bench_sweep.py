"""Config-5 sweep for roofline plots (BASELINE.json configs[4]) on one B200.

Voting (sFFT1.0/2.0 style) with B = next_pow2(sqrt(N K)) and rounds = 10 over
the grid N in {2^14, ..., 2^24} at K = 50 and K in {8, 32, 128, 512, 2048} at
N = 2^22, each at SNR in {inf, 40, 10} dB, a batch of seeded signals per
point, complex64.  Per point: device-resident transforms/s, the bucketization
kernel's algorithmic GB/s (Omega*8 + B*16 per bucketization over the summed
kernel time, CUDA events) against the measured HBM copy bandwidth, and a
parity spot check against the CPU oracle where the oracle finishes in seconds.

Inputs: gen_signal's positions and phases (numpy default_rng(seed)), unit
magnitudes, synthesis by inverse FFT without 1/N and complex AWGN drawn on the
device (a different noise stream than numpy's, same distribution); the spot
checks run the oracle on the exact device input (rounded to complex64).

  python bench_sweep.py [--signals 256] [--reps 2] [--points all|quick] > sweep.jsonl
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GRID_N = [(1 << e, 50) for e in (14, 16, 18, 20, 22, 24)]
GRID_K = [(1 << 22, k) for k in (8, 32, 128, 512, 2048)]
SNRS = [None, 40.0, 10.0]


def n_buckets(n: int, k: int) -> int:
    return 1 << math.ceil(math.log2(math.sqrt(n * k)))


def make_batch(n, k, snr, S, base_seed, dev):
    import numpy as np
    import torch
    X = torch.empty((S, n), dtype=torch.complex64, device=dev)
    g = torch.Generator(device=dev)
    for i in range(S):
        seed = base_seed + i
        rng = np.random.default_rng(seed)
        pos = np.sort(rng.choice(n, size=k, replace=False))
        ph = rng.uniform(0.0, 2.0 * np.pi, size=k)
        spec = torch.zeros(n, dtype=torch.complex128, device=dev)
        spec[torch.as_tensor(pos, device=dev)] = torch.as_tensor(np.exp(1j * ph), device=dev)
        x = torch.fft.ifft(spec) * n
        if snr is not None:
            p = float((x.abs() ** 2).mean())
            sd = math.sqrt(p / (10.0 ** (snr / 10.0)) / 2.0)
            g.manual_seed(seed)
            noise = torch.randn((2, n), dtype=torch.float64, device=dev, generator=g) * sd
            x = x + torch.complex(noise[0], noise[1])
        X[i] = x.to(torch.complex64)
    return X


def run_point(n, k, snr, S, reps, check):
    import numpy as np
    import torch
    import paper_2012_08238_b200 as sb
    from paper_2012_08238_b200._lib import lib
    from paper_2012_08238_b200.filters import default_flat_support
    dev = torch.device("cuda", 0)
    B = n_buckets(n, k)
    X = make_batch(n, k, snr, S, 5000, dev)
    cfg = sb.AlgorithmConfig(framework="voting", num_buckets=B, rounds=10)
    br = sb.run_voting_batch(X, k, cfg)
    torch.cuda.synchronize()
    L = lib()
    L.sfft_prof_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        br = sb.run_voting_batch(X, k, cfg)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pm, pl, pi = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
    L.sfft_prof_read(ctypes.byref(pm), ctypes.byref(pl), ctypes.byref(pi))
    L.sfft_prof_enable(0)
    omega = default_flat_support(n, B)
    gbs = pi.value * (omega * 8 + B * 16) / (pm.value * 1e-3) / 1e9 if pm.value else 0.0
    ok = 0
    res = br.to_results() if check else []
    if check:
        from oracle import sfft_oracle as O
        for s in range(check):
            x = X[s].cpu().numpy().astype(np.complex128)
            want = O.voting(O.Access(x), k, O.Cfg(framework="voting", num_buckets=B, rounds=10))
            ok += set(res[s].spectrum.entries) == set(want.entries)
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    return {"n": n, "k": k, "snr": snr, "B": B, "omega": omega, "signals": S,
            "transforms_per_s": S / (ms * 1e-3), "ms_per_batch": ms, "bucketize_gbs": gbs,
            "frac_of_measured_hbm": gbs / peak, "frac_of_8tbs": gbs / 8000.0,
            "support_identical": f"{ok}/{check}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--signals", type=int, default=256)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--points", default="all", choices=["all", "quick"])
    args = ap.parse_args()
    grid = GRID_N + [p for p in GRID_K if p not in GRID_N]
    snrs = SNRS if args.points == "all" else [40.0]
    for n, k in grid:
        for snr in snrs:
            S = args.signals
            if n * S > (1 << 32):  # keep a batch under 32 GB of complex64
                S = max(8, (1 << 32) // n)
            # the oracle finishes in seconds up to N = 2^20 and K = 512
            check = 2 if (n <= (1 << 20) and k <= 512) else 0
            t0 = time.time()
            r = run_point(n, k, snr, S, args.reps, check)
            r["wall_s"] = time.time() - t0
            print(json.dumps(r), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
