"""Config 5 at its large grid points: voting with
B = next_pow2(sqrt(N K)) = 2^13 .. 2^17 (the fold pass + four-step FFT route
and the shared-memory floor/heavy select at B > 4096), against golden vectors
the real reference wrote (tests/golden/make_golden.py c5grid; reference
sfft/frameworks.py:354-417, :111-122).

The three SNR variants of a grid point run as ONE batch of three signals
(every signal its own queue entry, one shared permutation stream), so the
batched path is what is checked.  Criteria (north_star): identical support;
coefficients within 1e-10 (complex128) / 1e-4 (complex64, against the
complex128 reference on the unrounded signal); identical samples_read.
"""

import numpy as np
import pytest

from conftest import regen_signal, runner_cases

pytestmark = pytest.mark.gpu

CASES = runner_cases("c5grid")


def _points():
    pts = {}
    for rec, arr in CASES:
        g = rec["gen"]
        pts.setdefault((g["n"], g["k"]), []).append((rec, arr))
    return sorted(pts.items())


POINTS = _points()


@pytest.fixture(scope="module")
def sb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2012_08238_b200 as sb
    return sb


@pytest.mark.parametrize("point", POINTS, ids=[f"n{int(np.log2(n))}_k{k}" for (n, k), _ in POINTS])
@pytest.mark.parametrize("dtype,tol", [("complex64", 1e-4), ("complex128", 1e-10)])
def test_c5_grid_voting(sb, point, dtype, tol):
    import torch
    (n, k), cases = point
    cfg = sb.AlgorithmConfig(**cases[0][0]["cfg"])
    tdt = torch.complex64 if dtype == "complex64" else torch.complex128
    X = torch.stack([torch.as_tensor(regen_signal(r, a)).to(tdt) for r, a in cases]).cuda()
    got = sb.run_voting_batch(X, k, cfg).to_results()
    del X
    for (rec, arr), res in zip(cases, got):
        want = dict(zip(arr["pos"].tolist(), arr["coef"].tolist()))
        ent = res.spectrum.entries
        assert set(ent) == set(want), (rec["name"], sorted(set(ent) ^ set(want))[:10])
        err = max(abs(ent[f] - c) / abs(c) for f, c in want.items())
        assert err <= tol, (rec["name"], err)
        assert res.samples_read == rec["samples_read"], rec["name"]
        assert (res.iterations, res.converged) == (rec["iterations"], rec["converged"])
