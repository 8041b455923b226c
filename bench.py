"""Headline benchmark: sFFT transforms/s at N=2^22, K=256 (BASELINE.json config 3)
and the gather-fold bucketization bandwidth against the HBM roofline, on B200.

One step = one batch of S independent seeded signals through the
device-resident iterative (phase-location) sFFT runner — every
bucketization, subtraction, location, polish and the samples_read count.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch S] [--impl ours|reference]

Under torchrun (N > 1) each rank runs its own batch (replicas, no
collective; the path shards by signal): value = all ranks' transforms / the
max over ranks of the device-timed region.  ``--impl reference`` times the
reference algorithm's CPU path (the numpy oracle port, oracle/sfft_oracle.py)
on the host cores, on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N = 1 << 22
K = 256
B = 4096
SNR_DB = 30.0
WORKLOAD = "C3 iterative/phase sFFT, N=2^22, K=256, B=2^12, SNR 30 dB, log-uniform |a| in [1,10]"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=2048, help="signals per step (queue length)")
    ap.add_argument("--slots", type=int, default=2048, help="device slots kept in flight")
    ap.add_argument("--engines", type=int, default=1, help="concurrent engines (streams)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="signals in the CPU-baseline sample (0: one per host core, max 32)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


KERNEL_DESC = ("bucketization launches of the step: k_gf_prep + k_group_fold (item groups of a "
               "slot's permutations; one gather per sample of a permutation window into shared "
               "memory, every shift folded from there) + k_fft_rows (in-place radix-8 row FFT); "
               "later-round misses the same way")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ CPU side

def _cpu_worker(args):
    seed, memo = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import functools

    import numpy as np
    from oracle import sfft_oracle as O
    if memo and not hasattr(O.flat_window, "cache_info"):
        # the reference builds the filter inside every runner call
        # (sfft/frameworks.py:457); "memo" times the path with it cached
        O.flat_window = functools.lru_cache(maxsize=4)(O.flat_window)
        O.flat_window(N, B)
    mags = 10 ** np.random.default_rng(seed + 1000).uniform(0, 1, K)
    x, _ = O.synth(N, K, SNR_DB, seed, magnitudes=mags)
    cfg = O.Cfg(framework="iterative", num_buckets=B, max_iterations=10)
    t0 = time.perf_counter()
    out = O.iterative(O.Access(x), K, cfg)
    dt = time.perf_counter() - t0
    return dt, (dict(out.entries), out.samples_read, out.iterations, out.converged)


def cpu_baseline(nsig: int, memo: bool = False, want_results: bool = False):
    """Oracle port of the reference CPU path, one single-threaded process per
    host core; throughput = transforms / (summed per-transform CPU seconds /
    workers) -- conservative against wall time, which also counts signal
    generation and process start-up (reported in ``sample``)."""
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    nsig = nsig or min(cores, 32)
    workers = min(cores, nsig)
    env_old = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS",
                                              "MKL_NUM_THREADS")}
    for k in env_old:
        os.environ[k] = "1"
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(workers) as pool:
        res = pool.map(_cpu_worker, [(i, memo) for i in range(nsig)], chunksize=1)
    wall = time.perf_counter() - t0
    for k, v in env_old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    secs = [r[0] for r in res]
    value = nsig / (sum(secs) / workers)
    out = {"value": value, "unit": "transforms/s", "cores": workers,
           "kind": "port",
           "sample": f"{nsig} seeded C3 signals (seeds 0..{nsig - 1}, exact gen_signal "
                     f"restatement, complex128), oracle iterative runner "
                     f"{'with the filter cached (D13)' if memo else 'as-is (filter built per call)'}, "
                     f"{workers} single-threaded numpy processes; median "
                     f"{statistics.median(secs):.2f} s/transform; wall {wall:.1f} s incl. "
                     f"generation; rate = transforms / (summed transform seconds / workers)"}
    if want_results:
        return out, [r[1] for r in res]
    return out


def gpu_parity(sb, cfg, results, dev):
    """The CPU-baseline signals (exact gen_signal inputs, complex128) through
    the GPU arm in complex64 (rounded once), against the oracle's results on
    the unrounded signals: the north_star criterion (identical support,
    values within 1e-4) plus identical samples_read / iterations / converged."""
    import numpy as np
    import torch
    from oracle import sfft_oracle as O
    xs = []
    for seed in range(len(results)):
        mags = 10 ** np.random.default_rng(seed + 1000).uniform(0, 1, K)
        xs.append(O.synth(N, K, SNR_DB, seed, magnitudes=mags)[0])
    X = torch.as_tensor(np.stack(xs)).to(torch.complex64).to(dev)
    got = sb.run_iterative_batch(X, K, cfg).to_results()
    same_support, diag, err = 0, 0, 0.0
    for g, (ent, smp, its, conv) in zip(got, results):
        e = g.spectrum.entries
        if set(e) == set(ent):
            same_support += 1
            if ent:
                err = max(err, max(abs(e[f] - c) / abs(c) for f, c in ent.items()))
        diag += (g.samples_read, g.iterations, g.converged) == (smp, its, conv)
    return {"signals": len(results), "support_identical": same_support,
            "diagnostics_identical": diag, "max_rel_err": err, "tol": 1e-4,
            "inputs": "the cpu_baseline seeds (exact gen_signal), complex64 on the GPU vs "
                      "complex128 oracle"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(args.cpu_sample)
        if i >= args.warmup:
            steps.append(cb["value"])
    value = statistics.median(steps)
    cb["value"] = value
    line = {"metric": "sFFT transforms/s (N=2^22, K=256, C3)", "value": value,
            "unit": "transforms/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * (args.cpu_sample or min(
                len(os.sched_getaffinity(0)), 32)) / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "n": N, "k": K, "num_buckets": B},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": "transforms/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ GPU side

class Clocks:
    """nvidia-smi sampling during the timed region."""

    def __init__(self, index: int):
        self.p = None
        self.index = index

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except Exception:
                continue
            for name, v in zip(names, f[2:]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_signals(S, dev, base_seed):
    """C3 inputs: gen_signal's positions/phases (numpy default_rng(seed)),
    magnitudes 10**U(0,1) from default_rng(seed+1000), synthesis by inverse FFT
    without 1/N, complex AWGN at 30 dB drawn on the device (Philox, seeded)."""
    import numpy as np
    import torch
    X = torch.empty((S, N), dtype=torch.complex64, device=dev)
    g = torch.Generator(device=dev)
    for i in range(S):
        seed = base_seed + i
        rng = np.random.default_rng(seed)
        pos = np.sort(rng.choice(N, size=K, replace=False))
        ph = rng.uniform(0.0, 2.0 * np.pi, size=K)
        mags = 10 ** np.random.default_rng(seed + 1000).uniform(0, 1, K)
        spec = torch.zeros(N, dtype=torch.complex128, device=dev)
        spec[torch.as_tensor(pos, device=dev)] = torch.as_tensor(mags * np.exp(1j * ph), device=dev)
        x = torch.fft.ifft(spec) * N
        p = float((x.abs() ** 2).mean())
        sd = math.sqrt(p / (10.0 ** (SNR_DB / 10.0)) / 2.0)
        g.manual_seed(seed)
        noise = torch.randn((2, N), dtype=torch.float64, device=dev, generator=g) * sd
        X[i] = (x + torch.complex(noise[0], noise[1])).to(torch.complex64)
    return X


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    import paper_2012_08238_b200 as sb
    from paper_2012_08238_b200._lib import lib

    S = args.batch
    cfg = sb.AlgorithmConfig(framework="iterative", location_method="phase", num_buckets=B,
                             max_iterations=10)
    X = make_signals(S, dev, base_seed=1_000_000 * rank)
    torch.cuda.synchronize()
    L = lib()
    st = torch.cuda.current_stream(dev)

    def step(xs):
        return sb.run_iterative_batch(xs, K, cfg, slots=args.slots, engines=args.engines)

    for _ in range(args.warmup):
        br = step(X)
    torch.cuda.synchronize()

    # ---- device-resident throughput (value) with live bucketization timing
    L.sfft_prof_enable(1)
    l0 = L.sfft_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(st)
        for _ in range(args.steps):
            br = step(X)
        e1.record(st)
        torch.cuda.synchronize()
    launches = L.sfft_launch_count() - l0
    ms = e0.elapsed_time(e1)
    import ctypes
    pm, pl, pi = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
    L.sfft_prof_read(ctypes.byref(pm), ctypes.byref(pl), ctypes.byref(pi))
    L.sfft_prof_enable(0)
    from paper_2012_08238_b200.replicas import combine
    ms, total = combine(ms, S * args.steps, dev)
    res = br.to_results()
    conv = sum(r.converged for r in res)
    exact = sum(len(r.spectrum.entries) == K for r in res)

    # roofline of the bucketization (gather-fold + FFT) launches: algorithmic
    # bytes per item as SURVEY §8(d) defines them, Omega*s + B*s with s = 8
    # (complex64); the bucket values are stored as complex128 (B*16), which is
    # also reported
    omega = sb.default_flat_support(N, B)
    item_bytes = omega * 8 + B * 8
    item_bytes_c128_out = omega * 8 + B * 16
    kern_ms = pm.value
    achieved = (pi.value * item_bytes) / (kern_ms * 1e-3) / 1e9 if kern_ms > 0 else 0.0
    peak, peak_kind = peaks()
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture
    # (profiles/r2_k_group_fold_ncu_raw.json: the C3 first-round group-fold
    # launch at 512 slots, "items" bucketizations)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r2_k_group_fold_ncu_raw.json")) as f:
            raw = json.load(f)
        unit = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        rd = float(raw["dram__bytes_read.sum"][0]) * unit[raw["dram__bytes_read.sum"][1]]
        wr = float(raw["dram__bytes_write.sum"][0]) * unit[raw["dram__bytes_write.sum"][1]]
        traffic = (rd + wr) / float(raw.get("items", 1024))  # per item, like bytes_per_item
    except Exception:
        traffic = None

    value = total / (ms * 1e-3)

    # ---- end to end through the public API from pinned host buffers: the
    # streaming entry point copies chunks on a side stream while the engine
    # admits the signals that have arrived; results are read back to host.
    e2e = None
    if not args.no_e2e:
        # one rank: the whole batch; several ranks on one node: at most 512
        # signals per rank (16 GB of pinned host memory each instead of 69 GB;
        # the path is PCIe-bound per GPU, so the rate is the same)
        Se = S if world == 1 else min(S, 512)
        Xh = torch.empty((Se, N), dtype=X.dtype, pin_memory=True)
        Xh.copy_(X[:Se])
        Xd = torch.empty_like(Xh, device=dev)
        h2d = Xh.numel() * Xh.element_size()

        def e2e_step():
            br = sb.run_iterative_stream(Xh, K, cfg, slots=args.slots, chunk=64, out=Xd)
            return (br.pos.cpu(), br.coef.cpu(), br.count.cpu(), br.iterations.cpu(),
                    br.converged.cpu(), br.samples_read.cpu())
        for _ in range(2):
            host = e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        for _ in range(args.steps):
            host = e2e_step()
        a1.record(st)
        torch.cuda.synchronize()
        ems, etot = combine(a0.elapsed_time(a1), Se * args.steps, dev)
        d2h = sum(t.numel() * t.element_size() for t in host)
        # the streamed results must be the resident batch's, row for row
        ref_rows = (br.pos[:Se].cpu(), br.coef[:Se].cpu(), br.count[:Se].cpu(),
                    br.iterations[:Se].cpu(), br.converged[:Se].cpu(),
                    br.samples_read[:Se].cpu())
        same = all(torch.equal(a, b) for a, b in zip(host, ref_rows))
        e2e = {"value": etot / (ems * 1e-3), "unit": "transforms/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": ems / args.steps,
               "path": "run_iterative_stream (pinned host rows, H2D overlapped with compute)",
               "identical_to_resident": bool(same)}
        del Xh, Xd
        torch.cuda.empty_cache()

    # ---- single-signal drop-in latency through the public API (host numpy
    # signal -> TimeSignal upload -> run_algorithm -> RecoveryResult), the
    # call a reference user makes after plugin.install()
    dropin = None
    if rank == 0 and not args.no_e2e:
        x1 = X[0].cpu().numpy()
        lat = []
        for i in range(6):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r1 = sb.run_algorithm(sb.TimeSignal(x1, dtype="complex64"), K, cfg)
            lat.append(time.perf_counter() - t0)
        dropin = {"ms_median": 1e3 * statistics.median(lat[1:]), "samples": len(lat) - 1,
                  "path": "run_algorithm(TimeSignal(host c64 signal)) -> RecoveryResult, "
                          "one C3 transform, upload + result conversion included",
                  "entries": len(r1.spectrum.entries)}

    # ---- complex128 input mode (the reference's dtype), same workload
    c128 = None
    if rank == 0 and not args.no_e2e:
        S2 = min(S, 512)
        X2 = X[:S2].to(torch.complex128)
        step2 = lambda: sb.run_iterative_batch(X2, K, cfg, slots=min(args.slots, S2))
        step2()
        torch.cuda.synchronize()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(st)
        for _ in range(2):
            step2()
        b1.record(st)
        torch.cuda.synchronize()
        c128 = {"value": 2 * S2 / (b0.elapsed_time(b1) * 1e-3), "unit": "transforms/s",
                "signals": S2, "note": "same signals widened to complex128 (16-byte gathers)"}
        del X2

    cb = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cb, results = cpu_baseline(args.cpu_sample, want_results=True)
        cbm = cpu_baseline(args.cpu_sample, memo=True)
        cb["value_filter_cached"] = cbm["value"]
        cb["sample_filter_cached"] = cbm["sample"]
        parity = gpu_parity(sb, cfg, results, dev)

    if rank == 0:
        line = {
            "metric": "sFFT transforms/s (N=2^22, K=256, C3)", "value": value,
            "unit": "transforms/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c64",
            "data": "synthetic (seeded gen_signal positions/phases, device AWGN)",
            "config": {"workload": WORKLOAD, "batch_per_gpu": S, "slots": args.slots, "engines": args.engines, "n": N, "k": K,
                       "num_buckets": B, "omega": omega, "parallelism": f"replicas{world}",
                       "l2": "inputs larger than L2 (%.1f GB per GPU)" % (S * N * 8 / 1e9)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind,
                         "traffic": traffic,
                         "traffic_unit": "DRAM read+write bytes per item of k_group_fold (ncu --set full, profiles/r2_k_group_fold_ncu_raw.json)",
                         "kernel": KERNEL_DESC,
                         "bytes_per_item": item_bytes,
                         "bytes_per_item_def": "SURVEY 8(d): Omega*8 gathered + B*8 buckets (c64)",
                         "frac_c128_outputs": (pi.value * item_bytes_c128_out) /
                         (kern_ms * 1e-3) / 1e9 / peak if kern_ms > 0 else None,
                         "items": pi.value,
                         "launches": pl.value, "kernel_ms": kern_ms,
                         "kernel_share_of_step": kern_ms / ms if ms else None},
            "cpu_baseline": cb,
            "parity": parity,
            "e2e": e2e,
            "dropin_latency": dropin,
            "c128": c128,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "check": {"converged": conv, "with_k_entries": exact, "signals": S},
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
