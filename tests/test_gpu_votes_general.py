"""Drop-in generality of the vote stage and the voting runner (golden vectors
from the real reference, tests/golden/make_golden.py votegen):

* vote_tally over mixed bucket-set kinds in one tally -- flat sets with b' != 0,
  spike trains of two widths, Dirichlet banks with and without half offsets and
  with a frequency shift (non-zero centre shift) -- exactly the reference's
  counts (sfft/reconstruct.py:158-179, preimages sfft/bucketize.py:108-118);
* run_voting beyond 64 rounds (80, 200) and with heavy bitmaps larger than
  shared memory (B = 2^16, 30 rounds: read from global memory).
"""

import json

import numpy as np
import pytest

from conftest import load_golden, regen_signal, runner_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2012_08238_b200 as sb
    return sb


def test_vote_tally_mixed_kinds(sb):
    import torch
    from paper_2012_08238_b200.bucketize import BucketSet
    from paper_2012_08238_b200.reconstruct import vote_tally
    z = load_golden("votegen")
    kinds = json.loads(str(z["vt_kinds"]))
    n = 4096
    vals = z["vt_values"]
    sets, o = [], 0
    for (b, _, half, cs, sg, tau, bp), kind in zip(z["vt_meta"].tolist(), kinds):
        v = torch.as_tensor(vals[o:o + b]).cuda()
        o += b
        sets.append(BucketSet(values=v, filter_kind=kind,
                              perm=sb.PermutationParams(n=n, sigma=sg, tau=tau, b_prime=bp),
                              tau_extra=0, n=n, num_buckets=b, bucket_width=n // b,
                              half_offset=bool(half), center_shift=cs))
    table = vote_tally(zip(sets, z["vt_thr"].tolist()), heavy_count=12)
    assert table.rounds == int(z["vt_rounds"])
    np.testing.assert_array_equal(table.counts.cpu().numpy(), z["vt_counts"])


CASES = runner_cases("votegen")


@pytest.mark.parametrize("case", CASES, ids=[c[0]["name"] for c in CASES])
@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-10), ("complex64", 1e-4)])
def test_voting_many_rounds(sb, case, dtype, tol):
    rec, arr = case
    x = regen_signal(rec, arr)
    res = sb.run_algorithm(sb.TimeSignal(x, dtype=dtype), rec["k"],
                           sb.AlgorithmConfig(**rec["cfg"]))
    want = dict(zip(arr["pos"].tolist(), arr["coef"].tolist()))
    got = res.spectrum.entries
    assert set(got) == set(want), rec["name"]
    err = max(abs(got[f] - c) / abs(c) for f, c in want.items())
    assert err <= tol, (rec["name"], err)
    assert (res.samples_read, res.iterations, res.converged) == \
        (rec["samples_read"], rec["iterations"], rec["converged"])
