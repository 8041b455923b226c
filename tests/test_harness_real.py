"""The harness plug-in against the REAL reference harness (SURVEY.md §8(f) #3,
sfft/harness.py:170-275, CSV schema :32-33).

Runs only where the reference package is importable (the build container,
/root/reference/pkg/src); it is never shipped.  No GPU here, so the device
TimeSignal and the device runner are stand-ins that run the reference's own
stock runner on the uploaded samples and report the indices it read: what is
checked is the plumbing a user flips with ``plugin.install()`` — dispatch
through ``frameworks._RUNNERS``, config round trip, access-map marking,
result conversion, error translation into ``converged=false`` rows — through
the unmodified ``run_experiment`` / ``run_sweep``, whose rows must equal the
rows without the plug-in apart from the runtime column.
"""

import csv
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present (build container only)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        import sparsefft  # noqa: F401
        from sparsefft import frameworks, harness
    except Exception as exc:  # pragma: no cover
        pytest.skip(f"reference not importable: {exc}")
    return frameworks, harness


@pytest.fixture
def stub_device(ref, monkeypatch):
    """Device TimeSignal / runners replaced by the reference's stock runners
    on the uploaded samples (the wrapper code under test is unchanged)."""
    frameworks, _ = ref
    import paper_2012_08238_b200.signal as sig
    from paper_2012_08238_b200.errors import SparseFFTError as DevError
    import paper_2012_08238_b200.errors as dev_errors
    from paper_2012_08238_b200.frameworks import RecoveryResult, SparseSpectrum
    stock = dict(frameworks._RUNNERS)
    calls = []

    class StubSignal:
        def __init__(self, samples, dtype=None, device=None):
            self.samples = np.asarray(samples)
            self.read = None

        def accessed_indices(self):
            return self.read

    monkeypatch.setattr(sig, "TimeSignal", StubSignal)

    def make(name):
        def run(xs, k, cfg):
            calls.append((name, k, cfg.framework))
            import sparsefft
            rx = sparsefft.TimeSignal(xs.samples)
            try:
                out = stock[name](rx, k, sparsefft.AlgorithmConfig.from_json(cfg.to_json()))
            except sparsefft.SparseFFTError as exc:  # surfaces as the device error type
                raise getattr(dev_errors, type(exc).__name__, DevError)(str(exc)) from exc
            xs.read = np.flatnonzero(rx._accessed)
            return RecoveryResult(SparseSpectrum(rx.n, dict(out.spectrum.entries)),
                                  out.samples_read, out.iterations, out.converged)
        run.__name__ = f"device_{name}"
        return run

    from paper_2012_08238_b200 import frameworks as dev
    for name, attr in (("voting", "run_voting"), ("iterative", "run_iterative"),
                       ("peeling", "run_peeling"), ("one_shot", "run_oneshot")):
        monkeypatch.setattr(dev, attr, make(name))
    return calls


def _row(rec):
    r = rec.to_row()
    return r[:5] + r[6:]  # everything but runtime_s


def test_csv_header_is_the_reference_schema(ref):
    _, harness = ref
    assert harness.CSV_HEADER == ["algorithm", "n", "k", "snr_db", "seed", "runtime_s",
                                  "sampling_fraction", "l0", "l1", "l2", "converged",
                                  "config_digest"]


def test_run_experiment_rows_equal_with_plugin(ref, stub_device):
    frameworks, harness = ref
    from paper_2012_08238_b200 import plugin
    cases = [
        (frameworks.AlgorithmConfig(framework="iterative", num_buckets=64, seed=2),
         harness.SignalSpec(4096, 8, None, 3)),
        (frameworks.AlgorithmConfig(framework="voting", num_buckets=64, rounds=9, seed=1),
         harness.SignalSpec(4096, 8, 20.0, 4)),
        (frameworks.AlgorithmConfig(framework="peeling", coprime_factors=(3, 5, 7, 11)),
         harness.SignalSpec(1155, 8, None, 5)),
        (frameworks.AlgorithmConfig(framework="one_shot", num_buckets=64),
         harness.SignalSpec(4096, 4, None, 6)),
        # a framework error: both paths must give the same converged=false row
        (frameworks.AlgorithmConfig(framework="peeling", coprime_factors=(2, 10)),
         harness.SignalSpec(20, 3, None, 0)),
    ]
    want = [_row(harness.run_experiment(c, s, repeats=1)) for c, s in cases]
    prev = plugin.install(frameworks)
    try:
        got = [_row(harness.run_experiment(c, s, repeats=1)) for c, s in cases]
    finally:
        plugin.uninstall(prev, frameworks)
    assert got == want
    # every case went through the device seam (the error case raises inside it)
    assert [c[0] for c in stub_device] == ["iterative", "voting", "peeling", "one_shot",
                                           "peeling"]
    assert want[-1][-2] == "false"  # converged column of the error row


def test_run_sweep_csv_equal_with_plugin(ref, stub_device, tmp_path):
    frameworks, harness = ref
    from paper_2012_08238_b200 import plugin
    base = [("iter", frameworks.AlgorithmConfig(framework="iterative", num_buckets=32)),
            ("vote", frameworks.AlgorithmConfig(framework="voting", num_buckets=32, rounds=7))]

    def sweep(path):
        harness.run_sweep("k_sweep", [2, 4], base, path, n=2048, k=4, snr_db=None,
                          seed=1, repeats=1)
        with open(path) as fh:
            rows = list(csv.reader(fh))
        return rows[0], sorted(r[:5] + r[6:] for r in rows[1:])

    hdr0, rows0 = sweep(tmp_path / "ref.csv")
    prev = plugin.install(frameworks)
    try:
        hdr1, rows1 = sweep(tmp_path / "dev.csv")
    finally:
        plugin.uninstall(prev, frameworks)
    assert hdr0 == hdr1 == harness.CSV_HEADER
    assert rows1 == rows0 and len(rows1) == 4
    assert len(stub_device) == 4
