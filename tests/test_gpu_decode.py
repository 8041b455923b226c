"""Parity of the decode-stage kernels (floor, heavy sets, votes, selection,
energy estimates, trimmed mean, subtraction) with the reference's golden
vectors.  Discrete outputs must be identical; fp64 values agree to 1e-12
relative (the kernels differ from numpy only in rounding order)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import sfft_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2012_08238_b200 as sb
    return sb


@pytest.fixture(scope="module")
def z():
    return load_golden("stage_decode")


def test_noise_floor(sb, z):
    from paper_2012_08238_b200.reconstruct import robust_noise_floor
    off = 0
    for ln, want in zip(z["floor_lens"], z["floor_out"]):
        got = robust_noise_floor(z["floor_in"][off:off + ln])
        assert got == pytest.approx(want, rel=1e-15, abs=0), (ln, got, want)
        off += ln


def test_noise_floor_random_sizes(sb):
    from paper_2012_08238_b200.reconstruct import noise_floors
    rng = np.random.default_rng(7)
    for B in (1, 2, 3, 8, 255, 256, 4096, 4097, 1 << 14, 1 << 17):
        v = rng.normal(size=(3, B)) + 1j * rng.normal(size=(3, B))
        v[1, : B // 2] = 0  # heavy ties at zero
        v[2] = np.round(v[2], 1)  # many equal magnitudes
        got = noise_floors(v).cpu().numpy()
        want = [O.noise_floor(r) for r in v]
        np.testing.assert_array_equal(got, want)


def _bucket_sets(sb, z):
    from paper_2012_08238_b200.bucketize import BucketSet
    n, k, b, R = (int(v) for v in z["vote_meta"])
    filt = sb.make_flat_filter(n, b)
    sets = []
    for (s, t), y in zip(z["vote_perms"], z["vote_y"]):
        sets.append(BucketSet(values=__import__("torch").as_tensor(y).cuda(), filter_kind="flat",
                              perm=sb.PermutationParams(n, int(s), int(t)), tau_extra=0, n=n,
                              num_buckets=b, bucket_width=n // b))
    return n, k, b, R, filt, sets


def test_votes_and_selection(sb, z):
    from paper_2012_08238_b200.reconstruct import select_by_votes, vote_tally
    n, k, b, R, filt, sets = _bucket_sets(sb, z)
    table = vote_tally(zip(sets, z["vote_thr"]), heavy_count=2 * k)
    np.testing.assert_array_equal(table.counts.cpu().numpy(), z["vote_counts"])
    cands = select_by_votes(table, keep=2 * k, min_fraction=0.5)
    assert cands == z["vote_cands"].tolist()


def test_select_tie_rules(sb):
    import torch
    from paper_2012_08238_b200.reconstruct import VoteTable, select_by_votes
    t = VoteTable(n=64, rounds=9, counts=torch.zeros(64, dtype=torch.int64).cuda())
    t.counts[40], t.counts[8], t.counts[55] = 7, 7, 7
    assert select_by_votes(t, keep=2, min_fraction=0.5) == [8, 40]
    t.counts[:] = 0
    t.counts[10], t.counts[20], t.counts[30] = 9, 9, 4
    assert select_by_votes(t, keep=4, min_fraction=0.5) == [10, 20]
    # many candidates across chunks: (-count, position) order, keep cut
    rng = np.random.default_rng(1)
    n, R = 50000, 12
    c = rng.integers(0, R + 1, size=n)
    t = VoteTable(n=n, rounds=R, counts=torch.as_tensor(c).cuda())
    got = select_by_votes(t, keep=3000, min_fraction=0.5)
    pos = np.flatnonzero(c >= 6)
    want = pos[np.lexsort((pos, -c[pos]))][:3000].tolist()
    assert got == want


def test_heavy_bitmap_ties(sb):
    import torch
    from paper_2012_08238_b200._lib import lib, ptr, stream_of
    rng = np.random.default_rng(5)
    B = 1000
    v = np.round(rng.normal(size=(4, B)), 1) + 0j
    thr = np.array([0.0, 0.5, 1.0, 10.0])
    vt = torch.as_tensor(v).cuda()
    tt = torch.as_tensor(thr).cuda()
    bits = torch.zeros((4, (B + 31) // 32), dtype=torch.int32).cuda()
    assert lib().sfft_heavy_bitmap(ptr(vt), 4, B, ptr(tt), 37, ptr(bits), None,
                                   stream_of(vt.device)) == 0
    got = bits.cpu().numpy().view(np.uint32)
    for r in range(4):
        mag = np.abs(v[r])
        ok = np.flatnonzero(mag >= max(thr[r], 0))
        order = ok[np.lexsort((ok, -mag[ok]))][:37]
        want = np.zeros(B, dtype=bool)
        want[order] = True
        have = np.array([(got[r, i >> 5] >> (i & 31)) & 1 for i in range(B)], dtype=bool)
        np.testing.assert_array_equal(have, want)


def test_energy_trimmed_subtract(sb, z):
    import torch
    from paper_2012_08238_b200._lib import lib, ptr, stream_of
    n, k, b, R, filt, sets = _bucket_sets(sb, z)
    dev = torch.device("cuda")
    y = torch.as_tensor(z["vote_y"]).to(dev)
    sig = torch.as_tensor(z["vote_perms"][:, 0]).to(dev)
    tau = torch.as_tensor(z["vote_perms"][:, 1]).to(dev)
    cand = torch.as_tensor(z["vote_cands"]).to(dev)
    C = cand.numel()
    est = torch.empty((R, C), dtype=torch.complex128, device=dev)
    gmax = torch.tensor([filt.peak], dtype=torch.float64, device=dev)
    st = stream_of(dev)
    assert lib().sfft_energy_estimates(ptr(y), b, ptr(filt.gtable), ptr(gmax), n, R, ptr(sig),
                                       ptr(tau), ptr(cand), C, ptr(est), st) == 0
    got = est.cpu().numpy()
    want = z["vote_est"]
    np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
    fin = np.isfinite(want)
    assert np.abs(got[fin] - want[fin]).max() <= 1e-12 * np.abs(want[fin]).max()
    tm = torch.empty(C, dtype=torch.complex128, device=dev)
    assert lib().sfft_trimmed_mean(ptr(torch.as_tensor(want).to(dev)), R, C, ptr(tm), st) == 0
    np.testing.assert_allclose(tm.cpu().numpy(), z["vote_tm"], rtol=1e-13, atol=0)
    e = torch.as_tensor(z["tm_in"]).to(dev)
    tm2 = torch.empty(e.shape[1], dtype=torch.complex128, device=dev)
    assert lib().sfft_trimmed_mean(ptr(e), e.shape[0], e.shape[1], ptr(tm2), st) == 0
    np.testing.assert_allclose(tm2.cpu().numpy(), z["tm_out"], rtol=1e-13, atol=0)
    # subtraction: model = candidates with finite trimmed means
    coef = np.where(np.isfinite(z["vote_tm"]), z["vote_tm"], 0)
    tp = torch.as_tensor(z["vote_cands"]).to(dev)
    tc = torch.as_tensor(coef).to(dev)
    cnt = torch.tensor([C], dtype=torch.int32, device=dev)
    out = torch.empty((2, b), dtype=torch.complex128, device=dev)
    taus = torch.tensor([int(z["vote_perms"][0, 1]), (int(z["vote_perms"][1, 1]) + 3) % n],
                        dtype=torch.int64, device=dev)
    item_sig = torch.zeros(2, dtype=torch.int32, device=dev)
    assert lib().sfft_subtract_flat(ptr(y[:2].contiguous()), ptr(out), b, b, None, 2,
                                    ptr(filt.gtable), n, ptr(item_sig), ptr(sig[:2].contiguous()),
                                    ptr(taus), ptr(tp), ptr(tc), ptr(cnt), 0, st) == 0
    o = out.cpu().numpy()
    for i, key in enumerate(["vote_sub0", "vote_sub1_t3"]):
        assert np.abs(o[i] - z[key]).max() <= 1e-12 * np.abs(z[key]).max()
