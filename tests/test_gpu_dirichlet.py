"""Dirichlet-bank bucketization and the freq-shift estimate on the device
against golden vectors of the real reference (tests/golden/stage_dirichlet.npz,
make_golden.py stage_dirichlet): values within 1e-10 relative, identical
access counts and error types."""

import json

import numpy as np
import pytest

from conftest import load_golden, sig_checksum, stage_signal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2012_08238_b200 as sb
    return sb


def _cases():
    z = load_golden("stage_dirichlet")
    off = yo = 0
    out = []
    for i, (n, L, b, half, f0, no, cshift) in enumerate(z["meta"]):
        out.append((i, int(n), int(L), int(b), bool(half), int(f0),
                    tuple(int(t) for t in z["offsets"][off:off + no]), int(cshift),
                    z["y"][yo:yo + b], int(z["access"][i]), z["checksum"][i]))
        off += no
        yo += b
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"d{c[0]}")
@pytest.mark.parametrize("dtype", ["complex128", "complex64"])
def test_dirichlet_golden(sb, case, dtype):
    i, n, L, b, half, f0, offs, cshift, want, acc, chk = case
    x = stage_signal(20240904 + i, n)
    np.testing.assert_array_equal(sig_checksum(x), chk)
    bank = sb.make_dirichlet_bank(n, L, b, half_offset=half)
    if f0:
        bank = sb.filter_freq_shift(bank, f0)
    xs = sb.TimeSignal(x, dtype=dtype)
    bs = sb.bucketize_dirichlet(xs, bank, offs)
    got = bs.values_host()
    if dtype == "complex128":
        ref = want
    else:  # against the oracle on the same rounded input
        from oracle import sfft_oracle as O
        ob = O.dirichlet_bank(n, L, b, half)
        if f0:
            ob = O.dirichlet_shift(ob, f0)
        ref = O.dirichlet_buckets(O.Access(x.astype(np.complex64).astype(np.complex128)), ob,
                                  offs)
    scale = max(np.abs(ref).max(), 1e-300)
    assert np.abs(got - ref).max() / scale < 1e-10
    assert xs.access_count == acc
    assert bs.center_shift == cshift and bs.sample_offsets == offs
    assert bs.filter_kind == "dirichlet_bank" and bs.half_offset == half


def test_freqshift_golden(sb):
    z = load_golden("stage_dirichlet")
    for j, (n, f, t, seed) in enumerate(z["est_specs"]):
        xs = sb.TimeSignal(stage_signal(20240950 + j, int(n)))
        got = sb.estimate_freqshift(xs, int(f), int(t), seed=int(seed))
        want = complex(z["est"][j])
        assert abs(got - want) <= 1e-12 * max(abs(want), 1.0)
        assert xs.access_count == z["est_access"][j]


def test_dirichlet_errors(sb):
    z = load_golden("stage_dirichlet")
    errs = json.loads(str(z["errors"]))
    xs = sb.TimeSignal(stage_signal(1, 2048))
    with pytest.raises(getattr(sb, errs["kind"])):
        sb.bucketize_dirichlet(xs, sb.make_flat_filter(2048, 16), (0,))
    with pytest.raises(getattr(sb, errs["nooffset"])):
        sb.bucketize_dirichlet(xs, sb.make_dirichlet_bank(2048, 128, 16), ())
    with pytest.raises(getattr(sb, errs["bank"])):
        sb.make_dirichlet_bank(2048, 100, 16)
    with pytest.raises(getattr(sb, errs["t0"])):
        sb.estimate_freqshift(xs, 3, 0)
    assert xs.access_count == 0


def test_dirichlet_weighted_spectrum(sb):
    """Single offset at t=0: each bucket equals the response-weighted spectrum
    sum (reference tests/test_bucketize.py:193-205)."""
    n = 2048
    x = stage_signal(99, n)
    xhat = np.fft.fft(x) / n  # dft_dense (sfft/signal.py:216-222)
    f = np.arange(n)
    for half in (True, False):
        bank = sb.make_dirichlet_bank(n, 128, 16, half_offset=half)
        got = sb.bucketize_dirichlet(sb.TimeSignal(x), bank, (0,)).values_host()
        pred = np.array([np.sum(bank.bucket_weight(b, f).cpu().numpy() * xhat) for b in range(16)])
        assert np.abs(got - pred).max() / np.abs(pred).max() < 1e-9
