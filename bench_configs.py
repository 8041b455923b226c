"""Per-config throughput table (BASELINE.json configs C1-C5) for BASELINE.md §5.

Not the driver's bench contract (that is bench.py, config C3); this measures
every BASELINE config on one GPU with the batched device runners: device-
resident transforms/s, the bucketization kernel's algorithmic GB/s and its
fraction of the measured HBM copy bandwidth, plus a parity spot check of a few
signals against the CPU oracle.

  python bench_configs.py [--signals S] [--configs C1,C2,...]
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

CONFIGS = {
    # name: (framework, n, k, snr, cfg kwargs, dtype, magnitudes)
    "C1": ("iterative", 1 << 16, 16, None, dict(num_buckets=256), "complex128", False),
    "C2": ("voting", 1 << 20, 64, 20.0, dict(num_buckets=1024, rounds=20), "complex64", False),
    "C3": ("iterative", 1 << 22, 256, 30.0, dict(num_buckets=4096), "complex64", True),
    "C4": ("peeling", 3_888_000, 200, None, dict(coprime_factors=(128, 125, 243)), "complex64",
           False),
    "C5a": ("voting", 1 << 22, 50, 40.0, dict(num_buckets=1 << 14, rounds=10), "complex64", False),
    "C5b": ("voting", 1 << 22, 512, 10.0, dict(num_buckets=1 << 16, rounds=10), "complex64",
            False),
    # class-split location (n/B shifted bucketizations per loop)
    "C1bin": ("iterative", 1 << 16, 16, None, dict(num_buckets=256, location_method="binary"),
              "complex128", False),
    "C1ms4": ("iterative", 1 << 16, 16, 30.0,
              dict(num_buckets=256, location_method="multiscale", branching=4), "complex128",
              False),
    "C3bin": ("iterative", 1 << 22, 256, 30.0, dict(num_buckets=4096, location_method="binary"),
              "complex64", True),
    # one-shot (spike moments, Hankel counts, Prony, least squares)
    "C1os": ("one_shot", 1 << 16, 16, None, dict(), "complex128", False),
    "C3os": ("one_shot", 1 << 22, 256, 30.0, dict(), "complex64", True),
}


def make_batch(name, S, dev):
    """Exact gen_signal restatement for every signal (numpy), uploaded."""
    import numpy as np
    import torch
    from oracle import sfft_oracle as O
    fwk, n, k, snr, kw, dtype, mags = CONFIGS[name]
    xs = []
    for s in range(S):
        m = 10 ** np.random.default_rng(s + 1000).uniform(0, 1, k) if mags else None
        x, _ = O.synth(n, k, snr, s, magnitudes=m)
        xs.append(torch.as_tensor(x))
    tdt = torch.complex64 if dtype == "complex64" else torch.complex128
    return torch.stack(xs).to(dev, tdt)


def omega_of(fwk, n, kw):
    from paper_2012_08238_b200.filters import default_flat_support
    if fwk in ("peeling", "one_shot"):
        return None
    return default_flat_support(n, kw["num_buckets"])


def run(name, S, reps, check):
    import numpy as np
    import torch
    import paper_2012_08238_b200 as sb
    from paper_2012_08238_b200._lib import lib
    from oracle import sfft_oracle as O
    fwk, n, k, snr, kw, dtype, mags = CONFIGS[name]
    dev = torch.device("cuda", 0)
    X = make_batch(name, S, dev)
    cfg = sb.AlgorithmConfig(framework=fwk, **kw)
    runner = {"voting": sb.run_voting_batch, "iterative": sb.run_iterative_batch,
              "peeling": sb.run_peeling_batch, "one_shot": sb.run_oneshot_batch}[fwk]
    br = runner(X, k, cfg)  # warm-up (filter tables, workspaces)
    torch.cuda.synchronize()
    L = lib()
    L.sfft_prof_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        br = runner(X, k, cfg)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pm, pl, pi = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
    L.sfft_prof_read(ctypes.byref(pm), ctypes.byref(pl), ctypes.byref(pi))
    L.sfft_prof_enable(0)
    sin = 8 if dtype == "complex64" else 16
    om = omega_of(fwk, n, kw)
    if kw.get("location_method") in ("binary", "multiscale") and n > (1 << 16):
        check = 0  # the oracle needs minutes per split-location transform at this size
    if fwk == "one_shot":  # spike: B samples gathered and B buckets written per item
        per_item = cfg.resolve_buckets(n, k) * (sin + 16)
    elif om is None:  # spike: B_j samples gathered and written per item, mixed sizes
        per_item = sum(3 * (n // p) * (sin + 16) for p in kw["coprime_factors"]) / 9
    else:
        per_item = om * sin + kw["num_buckets"] * 16
    gbs = pi.value * per_item / (pm.value * 1e-3) / 1e9 if pm.value else 0.0
    res = br.to_results()
    ok, err = 0, 0.0
    for s in range(min(check, S)):
        x = X[s].cpu().numpy().astype(np.complex128)
        ocfg = O.Cfg(framework=fwk, **kw)
        want = {"voting": O.voting, "iterative": O.iterative, "peeling": O.peeling,
                "one_shot": O.one_shot}[fwk](
            O.Access(x), k, ocfg)
        got = res[s].spectrum.entries
        if set(got) == set(want.entries):
            ok += 1
            if want.entries:
                err = max(err, max(abs(got[f] - c) / abs(c) for f, c in want.entries.items()))
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    return {"config": name, "framework": fwk, "n": n, "k": k, "dtype": dtype, "signals": S,
            "transforms_per_s": S / (ms * 1e-3), "ms_per_batch": ms,
            "bucketize_gbs": gbs, "frac_of_measured_hbm": gbs / peak,
            "frac_of_8tbs": gbs / 8000.0,
            "support_identical": f"{ok}/{min(check, S)}", "max_rel_coeff_err": err,
            "converged": sum(r.converged for r in res)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--signals", type=int, default=256)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--check", type=int, default=4)
    ap.add_argument("--configs", default=",".join(CONFIGS))
    args = ap.parse_args()
    out = []
    for name in args.configs.split(","):
        S = args.signals if CONFIGS[name][1] <= (1 << 20) else max(1, args.signals // 2)
        if name == "C5b":
            S = min(S, 64)
        if name == "C3bin":
            S = min(S, 32)
        t0 = time.time()
        r = run(name, S, args.reps, args.check)
        r["wall_s"] = time.time() - t0
        print(json.dumps(r), flush=True)
        out.append(r)
    return 0


if __name__ == "__main__":
    sys.exit(main())
