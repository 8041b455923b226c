"""Small-shape driver for compute-sanitizer: every kernel family
of the hot path once, at sizes memcheck/racecheck/synccheck finish in minutes.

  compute-sanitizer --tool memcheck  python tests/sanitize_driver.py
  compute-sanitizer --tool racecheck python tests/sanitize_driver.py
  compute-sanitizer --tool synccheck python tests/sanitize_driver.py

Covers: the one-CTA fused path (C1, B=256), the 8-CTA cluster gather-fold
k_cluster with its DSMEM exchange (B=4096, small N), the fold pass + four-step
FFT (B=8192), the permutation-run fold (k_run_fold + in-place cluster FFT),
the shared-memory radix selects (floor / heavy / decide), voting (C2-small),
peeling (the toy fixture and a small co-prime case), one-shot, and the split
(binary) location.  Prints one line per stage; exits non-zero on any error.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import numpy as np
    import torch

    import paper_2012_08238_b200 as sb
    from oracle import sfft_oracle as O

    dev = torch.device("cuda:0")

    def run(name, fn):
        fn()
        torch.cuda.synchronize()
        print(f"sanitize: {name} ok", flush=True)

    x16 = O.synth(1 << 16, 16, None, 0)[0]
    run("flat fused B=256", lambda: sb.bucketize_flat(
        sb.TimeSignal(x16, device=dev), sb.make_flat_filter(1 << 16, 256, device=dev),
        sb.PermutationParams(n=1 << 16, sigma=40503, tau=777), 3).values_host())
    run("flat cluster B=4096", lambda: sb.bucketize_flat(
        sb.TimeSignal(x16, dtype="complex64", device=dev),
        sb.make_flat_filter(1 << 16, 4096, device=dev),
        sb.PermutationParams(n=1 << 16, sigma=12345, tau=99), 0).values_host())
    x18 = O.synth(1 << 18, 32, 30.0, 1)[0]
    run("flat four-step B=8192", lambda: sb.bucketize_flat(
        sb.TimeSignal(x18, dtype="complex64", device=dev),
        sb.make_flat_filter(1 << 18, 8192, device=dev),
        sb.PermutationParams(n=1 << 18, sigma=777, tau=5), 1).values_host())
    run("iterative C1", lambda: sb.run_iterative(
        sb.TimeSignal(x16, device=dev), 16,
        sb.AlgorithmConfig(framework="iterative", num_buckets=256)))
    xs = torch.as_tensor(np.stack([O.synth(1 << 16, 16, 30.0, 3 + j)[0] for j in range(3)]))
    for rf, sf in (("0", "1"), ("1", "0"), ("1", "1")):
        os.environ["SFFT_ROW_CACHE"] = "1"
        os.environ["SFFT_RUN_FOLD"] = rf
        os.environ["SFFT_STREAM_FOLD"] = sf
        run(f"iterative row cache B=4096 run_fold={rf} stream_fold={sf}",
            lambda: sb.run_iterative_batch(
                xs.to(torch.complex64).to(dev), 16,
                sb.AlgorithmConfig(framework="iterative", num_buckets=4096), slots=2).to_results())
    run("iterative row cache B=256 stream fold c128", lambda: sb.run_iterative_batch(
        xs.to(dev), 16, sb.AlgorithmConfig(framework="iterative", num_buckets=256),
        slots=2).to_results())
    os.environ.pop("SFFT_ROW_CACHE", None)
    os.environ.pop("SFFT_RUN_FOLD", None)
    os.environ.pop("SFFT_STREAM_FOLD", None)
    x14 = O.synth(1 << 14, 8, None, 4)[0]
    run("iterative binary", lambda: sb.run_iterative(
        sb.TimeSignal(x14, device=dev), 8,
        sb.AlgorithmConfig(framework="iterative", num_buckets=64, location_method="binary")))
    x20 = O.synth(1 << 18, 16, 20.0, 5)[0]
    run("voting", lambda: sb.run_voting(
        sb.TimeSignal(x20, dtype="complex64", device=dev), 16,
        sb.AlgorithmConfig(framework="voting", num_buckets=1024, rounds=12)))
    toy = np.fft.ifft(np.array([0, 1.0, 0, 0.8, 0, 1.2, 0, 0, 0, 0, 0.9, 0, 0, 1.1, 0, 0, 0, 0,
                                0, 0], dtype=complex)) * 20
    run("peeling toy", lambda: sb.run_peeling(
        sb.TimeSignal(toy, device=dev), 5,
        sb.AlgorithmConfig(framework="peeling", coprime_factors=(4, 5))))
    x1155 = O.synth(1155, 12, None, 77)[0]
    run("peeling 1155", lambda: sb.run_peeling(
        sb.TimeSignal(x1155, device=dev), 12,
        sb.AlgorithmConfig(framework="peeling", coprime_factors=(3, 5, 7, 11))))
    x12 = O.synth(1 << 12, 4, None, 6)[0]
    run("one-shot", lambda: sb.run_oneshot(
        sb.TimeSignal(x12, device=dev), 4,
        sb.AlgorithmConfig(framework="one_shot", num_buckets=64)))
    return 0


if __name__ == "__main__":
    sys.exit(main())
