"""The reference's acceptance criterion 3 (tests/test_acceptance.py:131-160 of the
reference: 100 seeded noiseless trials per framework, n = 4096 / 1155 / 15015,
K = 16, config seed = trial index) run through the device runners and checked
trial by trial against the CPU oracle (pinned bit-exactly to the reference by
tests/golden): identical support, samples_read, iterations and converged,
coefficients within 1e-10; plus the criterion's own exact-recovery counts."""

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TRIALS = 100


@pytest.fixture(scope="module")
def sb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2012_08238_b200 as sb
    return sb


def _check(res, want, name):
    assert set(res.spectrum.entries) == set(want.entries), name
    if want.entries:
        err = max(abs(res.spectrum.entries[f] - c) / abs(c) for f, c in want.entries.items())
        assert err <= 1e-10, (name, err)
    assert (res.samples_read, res.iterations, res.converged) == \
        (want.samples_read, want.iterations, want.converged), name


CASES = [("iterative", 4096, None, 10_000, TRIALS), ("one_shot", 4096, None, 10_000, TRIALS - 1),
         ("voting", 4096, None, 10_000, TRIALS - 1),
         ("peeling", 1155, (3, 5, 7, 11), 20_000, TRIALS),
         ("peeling", 15015, (3, 5, 7, 11, 13), 20_000, TRIALS)]


@pytest.mark.parametrize("fw,n,factors,base,need", CASES,
                         ids=[f"{c[0]}_{c[1]}" for c in CASES])
def test_criterion3_exact_recovery(sb, fw, n, factors, base, need):
    from oracle import sfft_oracle as O
    run = {"iterative": O.iterative, "one_shot": O.one_shot, "voting": O.voting,
           "peeling": O.peeling}[fw]
    hits = 0
    for s in range(TRIALS):
        x, truth = O.synth(n, 16, None, base + s)
        kw = dict(framework=fw, seed=s)
        if factors:
            kw["coprime_factors"] = factors
        want = run(O.Access(x), 16, O.Cfg(**kw))
        res = sb.run_algorithm(sb.TimeSignal(x), 16, sb.AlgorithmConfig(**kw))
        _check(res, want, f"{fw} n={n} trial {s}")
        hits += set(res.spectrum.entries) == set(truth)
    assert hits >= need, (fw, n, hits)
