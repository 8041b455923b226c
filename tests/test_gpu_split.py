"""Binary / multiscale class-split location of the iterative runner on the
device (sfft/frameworks.py:517-554) against golden vectors of the real
reference (tests/golden/split.npz, make_golden.py split_runners).

Criteria as for the other runners: identical support, samples_read,
iterations and converged; coefficients within 1e-10 relative (complex128)."""

import numpy as np
import pytest

from conftest import regen_signal, runner_cases
from test_gpu_runners import _cfg, check_case, check_rounded, sb  # noqa: F401

pytestmark = pytest.mark.gpu

SPLIT = runner_cases("split")


@pytest.mark.parametrize("case", SPLIT, ids=[c[0]["name"] for c in SPLIT])
def test_split_golden_c128(sb, case):  # noqa: F811
    rec, arr = case
    check_case(sb, rec, arr, "complex128", 1e-10)


@pytest.mark.parametrize("case", [c for c in SPLIT if c[0]["n"] >= 4096],
                         ids=[c[0]["name"] for c in SPLIT if c[0]["n"] >= 4096])
def test_split_rounded_c64(sb, case):  # noqa: F811
    """complex64 mode vs the oracle on the same rounded input."""
    check_rounded(sb, *case)


def test_split_batched_slots(sb):  # noqa: F811
    """Many signals through few slots (continuous batching) == one at a time."""
    import torch
    from oracle import sfft_oracle as O
    cases = [c for c in SPLIT if c[0]["name"].startswith("search_binary")]
    xs = np.stack([regen_signal(*c) for c in cases])
    rec = cases[0][0]
    cfg = _cfg(sb, rec)
    br = sb.run_iterative_batch(torch.as_tensor(xs, device="cuda"), rec["k"], cfg, slots=3)
    res = br.to_results()
    for (rc, arr), r in zip(cases, res):
        want = O.iterative(O.Access(regen_signal(rc, arr)), rc["k"],
                           O.Cfg(framework="iterative", location_method="binary",
                                 num_buckets=16, branching=2, seed=rec["cfg"]["seed"]))
        assert set(r.spectrum.entries) == set(want.entries)
        assert r.samples_read == want.samples_read
        assert r.iterations == want.iterations
        assert r.converged == want.converged


def test_split_schedule_matches_access_count(sb):  # noqa: F811
    """The exported read schedule (arithmetic shift groups) reproduces
    samples_read through the TimeSignal access map."""
    rec, arr = next(c for c in SPLIT if c[0]["name"] == "split_binary2_n12_k8_s0")
    xs = sb.TimeSignal(regen_signal(rec, arr))
    res = sb.run_algorithm(xs, rec["k"], _cfg(sb, rec))
    assert res.samples_read == xs.access_count == rec["samples_read"]


def test_split_schedule_groups_partial(sb):  # noqa: F811
    """Coarse split depths read a strict subset of the signal: a converge-at-
    first-look signal logs only shift 0 (Omega samples)."""
    import torch
    n = 4096
    x = np.zeros(n, dtype=np.complex128)
    cfg = sb.AlgorithmConfig(framework="iterative", location_method="binary",
                             num_buckets=64, seed=1)
    xs = sb.TimeSignal(x)
    res = sb.run_algorithm(xs, 4, cfg)
    from oracle import sfft_oracle as O
    want = O.iterative(O.Access(x), 4, O.Cfg(framework="iterative", location_method="binary",
                                             num_buckets=64, seed=1))
    assert res.samples_read == want.samples_read == xs.access_count
    assert res.converged == want.converged and res.iterations == want.iterations
    del torch
