"""Seeded parity sweep: many signals per BASELINE config through the batched
device runners, each compared with the CPU oracle (pinned to the reference by
tests/golden) on the same input.  Oracle runs in a process pool.

Criteria as in test_gpu_runners: identical support; coefficients within 1e-10
(complex128) / 1e-4 (complex64 vs the complex128 oracle on the unrounded
signal); samples_read / iterations / converged identical (noisy configs in
complex64 mode, every config in complex128 mode)."""

import os
import multiprocessing as mp

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _signal(n, k, snr, seed, mags_seed):
    from oracle import sfft_oracle as O
    mags = None if mags_seed is None else 10 ** np.random.default_rng(mags_seed).uniform(0, 1, k)
    x, _ = O.synth(n, k, snr, seed, magnitudes=mags)
    return x


def _oracle_job(args):
    fwk, n, k, snr, seed, mags_seed, cfgkw = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import sfft_oracle as O
    x = _signal(n, k, snr, seed, mags_seed)
    run = {"voting": O.voting, "iterative": O.iterative, "peeling": O.peeling}[fwk]
    out = run(O.Access(x), k, O.Cfg(framework=fwk, **cfgkw))
    return out.entries, out.samples_read, out.iterations, out.converged


SWEEP = [
    # name, framework, n, k, snr, seeds, mags?, cfg, dtype
    ("C1", "iterative", 1 << 16, 16, None, range(100, 148), False,
     dict(num_buckets=256), "complex128"),
    ("C2", "voting", 1 << 20, 64, 20.0, range(100, 112), False,
     dict(num_buckets=1024, rounds=20), "complex64"),
    ("C3", "iterative", 1 << 22, 256, 30.0, range(100, 112), True,
     dict(num_buckets=4096, max_iterations=10), "complex64"),
    ("C4", "peeling", 3_888_000, 200, None, range(100, 116), False,
     dict(coprime_factors=(128, 125, 243)), "complex64"),
    ("C5", "voting", 1 << 16, 50, 40.0, range(100, 124), False,
     dict(num_buckets=2048, rounds=10), "complex64"),
]


@pytest.fixture(scope="module")
def sb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2012_08238_b200 as sb
    return sb


@pytest.mark.parametrize("case", SWEEP, ids=[c[0] for c in SWEEP])
def test_parity_sweep(sb, case):
    import torch
    name, fwk, n, k, snr, seeds, mags, cfgkw, dtype = case
    seeds = list(seeds)
    jobs = [(fwk, n, k, snr, s, (s + 1000) if mags else None, cfgkw) for s in seeds]
    with mp.get_context("spawn").Pool(min(len(jobs), os.cpu_count() or 4)) as pool:
        want = pool.map(_oracle_job, jobs)
    X = torch.stack([torch.as_tensor(_signal(n, k, snr, s, (s + 1000) if mags else None))
                     for s in seeds]).to("cuda", torch.complex64 if dtype == "complex64"
                                         else torch.complex128)
    cfg = sb.AlgorithmConfig(framework=fwk, **cfgkw)
    runner = {"voting": sb.run_voting_batch, "iterative": sb.run_iterative_batch,
              "peeling": sb.run_peeling_batch}[fwk]
    got = runner(X, k, cfg).to_results()
    tol = 1e-10 if dtype == "complex128" else 1e-4
    diag = dtype == "complex128" or snr is not None
    for s, (ent, smp, its, conv), res in zip(seeds, want, got):
        g = res.spectrum.entries
        assert set(g) == set(ent), (name, s, sorted(set(g) ^ set(ent))[:8])
        if ent:
            err = max(abs(g[f] - c) / abs(c) for f, c in ent.items())
            assert err <= tol, (name, s, err)
        if diag:
            assert (res.samples_read, res.iterations, res.converged) == (smp, its, conv), (name, s)
