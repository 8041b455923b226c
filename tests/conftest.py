import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def stage_signal(seed, n):
    """Matches tests/golden/make_golden.py:stage_signal."""
    rng = np.random.default_rng(seed)
    return rng.normal(size=n) + 1j * rng.normal(size=n)


def sig_checksum(x):
    x = np.asarray(x)
    return np.array([x.sum(), (x * np.arange(x.size) / x.size).sum(), x[0], x[-1]],
                    dtype=np.complex128)


def runner_cases(name="runners"):
    import json
    z = load_golden(name)
    index = json.loads(str(z["index_json"]))
    out = []
    for rec in index:
        i = rec["id"]
        arr = {key.split("_", 1)[1]: z[key] for key in z.files if key.startswith(f"{i}_")}
        out.append((rec, arr))
    return out


def regen_signal(rec, arr):
    """Input of a golden runner case: stored samples or the seeded generator."""
    from oracle import sfft_oracle as O
    if "x" in arr:
        return np.asarray(arr["x"])
    g = rec["gen"]
    mags = None
    if g.get("mags_seed") is not None:
        mags = 10 ** np.random.default_rng(g["mags_seed"]).uniform(0, 1, g["k"])
    x, _ = O.synth(g["n"], g["k"], g["snr"], g["seed"], magnitudes=mags)
    return x


def oracle_cfg(rec):
    from oracle import sfft_oracle as O
    kw = dict(rec["cfg"])
    fwk = kw.pop("framework")
    if "coprime_factors" in kw:
        kw["coprime_factors"] = tuple(kw["coprime_factors"])
    return fwk, O.Cfg(framework=fwk, **kw)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
