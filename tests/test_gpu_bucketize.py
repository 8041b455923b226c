"""Parity of the sm_100a bucketization kernels with the reference (golden
vectors) and the CPU oracle.  Tolerances: complex128 input 1e-12 relative to
max|y| (fp64 fold + FFT; only the FFT rounding differs from pocketfft);
complex64 input 1e-4 (BASELINE.json north_star), compared with the complex128
oracle on the unrounded signal."""

import numpy as np
import pytest

from conftest import load_golden, sig_checksum, stage_signal
from oracle import sfft_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2012_08238_b200 as sb
    return sb


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-12), ("complex64", 1e-4)])
def test_flat_golden(sb, dtype, tol):
    z = load_golden("stage_flat")
    off = 0
    for i, (n, b, sup, s, t, bp, te) in enumerate(z["meta"]):
        n, b = int(n), int(b)
        x = stage_signal(20240901 + i, n)
        xs = sb.TimeSignal(x, dtype=dtype)
        filt = sb.make_flat_filter(n, b, int(sup))
        perm = sb.PermutationParams(n=n, sigma=int(s), tau=int(t), b_prime=int(bp))
        bs = sb.bucketize_flat(xs, filt, perm, int(te))
        assert rel(bs.values_host(), z["y"][off:off + b]) < tol, (i, n, b)
        assert xs.access_count == z["access"][i]
        off += b


@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-12), ("complex64", 1e-4)])
def test_flat_freq_shift_golden(sb, dtype, tol):
    """filter_freq_shift of a flat window (sfft/filters.py:190-200) and flat
    bucketizations through it, against the reference: modulated taps, rolled
    response, passband centres, bucket weights, bucket values, centre shift,
    reads and the hash view (incl. composed shifts, f0 = 0, N and negative)."""
    from paper_2012_08238_b200.bucketize import hash_view_for
    z = load_golden("stage_flatshift")
    for i, row in enumerate(z["meta"]):
        n, b, ns, s, t, bp, te, center, cshift, access, step = (int(v) for v in row[:11])
        f = sb.make_flat_filter(n, b)
        for f0 in row[11:11 + ns]:
            f = sb.filter_freq_shift(f, int(f0))
        assert f.center_offset == center
        assert rel(f.taps.cpu().numpy(), z[f"{i}_taps"]) < 1e-13
        assert rel(f.freq_response.cpu().numpy()[::step], z[f"{i}_resp"]) < 1e-13
        assert np.array_equal(f.bucket_centers(), z[f"{i}_centers"])
        m = (np.arange(40, dtype=np.int64) * 997 + 3) % n
        got_w = np.stack([f.bucket_weight(bq, m).cpu().numpy() for bq in (0, 1, b - 1)])
        assert np.abs(got_w - z[f"{i}_weight"]).max() < 1e-13 * np.abs(z[f"{i}_resp"]).max()
        xs = sb.TimeSignal(stage_signal(20241001 + i, n), dtype=dtype)
        perm = sb.PermutationParams(n=n, sigma=s, tau=t, b_prime=bp)
        bs = sb.bucketize_flat(xs, f, perm, te)
        assert rel(bs.values_host(), z[f"{i}_y"]) < tol, (i, n, b)
        assert bs.center_shift == cshift and xs.access_count == access
        hv = hash_view_for(f, perm)
        assert np.array_equal(np.asarray(hv.bucket_of(m)), z[f"{i}_bucket_of"])
        assert np.array_equal(hv.preimage(b // 2), z[f"{i}_pre"])
        assert np.array_equal(np.asarray(bs.hash_map().bucket_of(m)), z[f"{i}_bucket_of"])


def test_filter_response_matches_oracle(sb):
    z = load_golden("stage_filter")
    for n, b in [(2048, 16), (3000, 24), (65536, 256)]:
        f = sb.make_flat_filter(n, b)
        taps = f.taps.cpu().numpy()
        np.testing.assert_allclose(taps, z[f"taps_{n}_{b}"], rtol=1e-14, atol=1e-17)
        resp = f.freq_response.cpu().numpy()
        want = z[f"resp_{n}_{b}"]
        got = resp if n < 10000 else resp[::37]
        assert rel(got, want) < 1e-13
        assert abs(f.peak - np.abs(O.flat_window(n, b).response).max()) < 1e-14


@pytest.mark.parametrize("n,b", [(1 << 16, 256), (1 << 20, 1024), (1 << 22, 4096),
                                 (1 << 18, 1 << 13), (1 << 22, 1 << 14), (1 << 22, 1 << 17)])
@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-12), ("complex64", 1e-4)])
def test_flat_config_shapes(sb, n, b, dtype, tol):
    rng = np.random.default_rng(n + b)
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    xs = sb.TimeSignal(x, dtype=dtype)
    filt = sb.make_flat_filter(n, b)
    win = O.flat_window(n, b)
    for _ in range(2):
        s, t, _bp = O.draw_perm(n, rng)
        te = int(rng.integers(0, 5))
        got = sb.bucketize_flat(xs, filt, sb.PermutationParams(n, s, t), te).values_host()
        want = O.flat_buckets(O.Access(x), win, s, t, 0, te)
        assert rel(got, want) < tol


@pytest.mark.parametrize("dtype,tol", [("complex128", 1e-12), ("complex64", 1e-4)])
def test_spike_golden(sb, dtype, tol):
    z = load_golden("stage_spike")
    off = 0
    for i, (n, b, t) in enumerate(z["meta"]):
        n, b = int(n), int(b)
        x = stage_signal(20240902 + i, n)
        assert np.allclose(sig_checksum(x), z["checksum"][i])
        xs = sb.TimeSignal(x, dtype=dtype)
        bs = sb.bucketize_spike(xs, b, int(t))
        assert rel(bs.values_host(), z["y"][off:off + b]) < tol, (n, b, t)
        assert xs.access_count == z["access"][i]
        off += b


@pytest.mark.parametrize("n,b", [(3_888_000, 30375), (3_888_000, 31104), (3_888_000, 16000),
                                 (1 << 20, 1 << 15), (17 * 64, 17 * 4)])
def test_spike_large_and_mixed_radix(sb, n, b):
    rng = np.random.default_rng(b)
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    xs = sb.TimeSignal(x)
    for t in (0, 1, 2):
        got = sb.bucketize_spike(xs, b, t).values_host()
        want = O.spike_buckets(O.Access(x), b, t)
        assert rel(got, want) < 1e-12


def test_batched_items_match_single(sb):
    import torch
    n, b = 1 << 16, 256
    rng = np.random.default_rng(3)
    xs = [rng.normal(size=n) + 1j * rng.normal(size=n) for _ in range(3)]
    X = torch.as_tensor(np.stack(xs)).cuda()
    filt = sb.make_flat_filter(n, b)
    perms = [O.draw_perm(n, rng) for _ in range(5)]
    item_sig = [0, 1, 2, 1, 0]
    out = sb.bucketize_flat_batch(X, filt, [p[0] for p in perms], [p[1] for p in perms],
                                  item_sig=item_sig).cpu().numpy()
    for i, (s, t, _) in enumerate(perms):
        want = O.flat_buckets(O.Access(xs[item_sig[i]]), O.flat_window(n, b), s, t)
        assert rel(out[i], want) < 1e-12


def test_closed_form_frequency_sum(sb):
    """Bucket value == sum_m G[(iL - m) mod N] * xhat_p[m] (reference
    tests/test_bucketize.py:98-111), at 1e-9."""
    n, b = 2048, 16
    rng = np.random.default_rng(12345)
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    filt = sb.make_flat_filter(n, b, 516)
    s, t, bp, te = 171, 9, 23, 2
    vals = sb.bucketize_flat(sb.TimeSignal(x), filt, sb.PermutationParams(n, s, t, bp),
                             te).values_host()
    tt = (t + te) % n
    i = np.arange(n)
    xp = x[(s * (i - tt)) % n] * O.unit_root(n, bp * s * i)
    xp_hat = np.fft.fft(xp) / n
    resp = filt.freq_response.cpu().numpy()
    m = np.arange(n)
    pred = np.array([np.sum(resp[(j * (n // b) - m) % n] * xp_hat) for j in range(b)])
    assert np.linalg.norm(vals - pred) / np.linalg.norm(pred) < 1e-9


def test_errors(sb):
    x = sb.TimeSignal(np.ones(100, dtype=complex))
    with pytest.raises(sb.NonDivisorParameter):
        sb.bucketize_spike(x, 7)
    with pytest.raises(sb.InvalidParameter):
        sb.make_flat_filter(100, 7)
