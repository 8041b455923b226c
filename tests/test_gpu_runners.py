"""End-to-end parity of the device runners with the reference (golden
vectors generated from the real reference by tests/golden/make_golden.py).

Criteria (BASELINE.json north_star): identical support,
identical samples_read / iterations / converged, coefficients within 1e-10
relative (complex128 input) or 1e-4 (complex64 input, compared with the
complex128 reference on the unrounded signal)."""

import numpy as np
import pytest

from conftest import regen_signal, runner_cases

pytestmark = pytest.mark.gpu

CASES = runner_cases()


@pytest.fixture(scope="module")
def sb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2012_08238_b200 as sb
    return sb


def _cfg(sb, rec):
    kw = dict(rec["cfg"])
    if "coprime_factors" in kw:
        kw["coprime_factors"] = tuple(kw["coprime_factors"])
    return sb.AlgorithmConfig(**kw)


def check_case(sb, rec, arr, dtype, tol):
    x = regen_signal(rec, arr)
    xs = sb.TimeSignal(x, dtype=dtype)
    cfg = _cfg(sb, rec)
    if rec["error"]:
        err = getattr(sb, rec["error"])
        with pytest.raises(err):
            sb.run_algorithm(xs, rec["k"], cfg)
        return
    res = sb.run_algorithm(xs, rec["k"], cfg)
    want = dict(zip(arr["pos"].tolist(), arr["coef"].tolist()))
    got = res.spectrum.entries
    assert set(got) == set(want), (rec["name"], sorted(set(got) ^ set(want))[:10])
    if want:
        err = max(abs(got[f] - c) / abs(c) for f, c in want.items())
        assert err <= tol, (rec["name"], err)
    assert res.samples_read == rec["samples_read"], rec["name"]
    assert res.iterations == rec["iterations"], rec["name"]
    assert res.converged == rec["converged"], rec["name"]


def _select(fw):
    return [c for c in CASES if c[0]["cfg"]["framework"] == fw]


ITER = _select("iterative")


@pytest.mark.parametrize("case", ITER, ids=[c[0]["name"] for c in ITER])
@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-10), ("complex64", 1e-4)])
def test_iterative_golden(sb, case, dtype, tol):
    rec, arr = case
    if dtype == "complex64" and rec["gen"] is None and rec["name"].startswith("fix"):
        pass
    check_case(sb, rec, arr, dtype, tol)
