"""The harness plug-in (paper_2012_08238_b200.plugin) against a stand-in for
the reference's frameworks module: registration, error-type translation,
access-map marking and result conversion.  The device runner is replaced by
a stub so this runs without a GPU (the GPU runners have their own parity
suites)."""

import sys
import types

import numpy as np
import pytest


def _fake_reference():
    pkg = types.ModuleType("fakeref")
    errors = types.ModuleType("fakeref.errors")

    class SparseFFTError(Exception):
        pass

    class ConfigMismatch(SparseFFTError):
        pass

    errors.SparseFFTError = SparseFFTError
    errors.ConfigMismatch = ConfigMismatch
    fw = types.ModuleType("fakeref.frameworks")

    class SparseSpectrum:
        def __init__(self, n, entries):
            self.n, self.entries = n, entries

    class RecoveryResult:
        def __init__(self, spectrum, samples_read, iterations, converged):
            self.spectrum, self.samples_read = spectrum, samples_read
            self.iterations, self.converged = iterations, converged

    fw.SparseSpectrum, fw.RecoveryResult = SparseSpectrum, RecoveryResult
    fw._RUNNERS = {"one_shot": "o", "voting": "v", "iterative": "i", "peeling": "p",
                    "dense": "d"}
    sys.modules.update({"fakeref": pkg, "fakeref.errors": errors, "fakeref.frameworks": fw})
    return fw, errors


class _RefSignal:
    def __init__(self, samples):
        self.samples = np.asarray(samples, dtype=np.complex128)
        self._accessed = np.zeros(self.samples.size, dtype=bool)

    @property
    def n(self):
        return self.samples.size

    @property
    def access_count(self):
        return int(self._accessed.sum())


def test_install_and_uninstall():
    from paper_2012_08238_b200 import plugin
    fw, _ = _fake_reference()
    prev = plugin.install(fw, frameworks=("voting", "iterative"))
    assert set(prev) == {"voting", "iterative"}
    assert callable(fw._RUNNERS["voting"]) and fw._RUNNERS["peeling"] == "p"
    plugin.uninstall(prev, fw)
    assert fw._RUNNERS["voting"] == "v" and fw._RUNNERS["iterative"] == "i"
    with pytest.raises(ValueError):
        plugin.install(fw, frameworks=("dense",))


def test_wrapper_converts_results_and_errors(monkeypatch):
    from paper_2012_08238_b200 import plugin
    import paper_2012_08238_b200.signal as sig
    from paper_2012_08238_b200.errors import ConfigMismatch
    from paper_2012_08238_b200.frameworks import AlgorithmConfig, RecoveryResult, SparseSpectrum
    fw, errors = _fake_reference()

    class StubSignal:  # stands in for the device TimeSignal (no GPU here)
        def __init__(self, samples, dtype=None, device=None):
            self.samples = samples

        def accessed_indices(self):
            return np.array([1, 5, 9])

    monkeypatch.setattr(sig, "TimeSignal", StubSignal)

    def ok_run(x, k, cfg):
        assert cfg.framework == "iterative" and k == 2
        return RecoveryResult(SparseSpectrum(16, {3: 1 + 2j}), 3, 4, True)

    def bad_run(x, k, cfg):
        raise ConfigMismatch("nope")

    class Cfg:
        def to_json(self):
            return AlgorithmConfig(framework="iterative").to_json()

    x = _RefSignal(np.zeros(16))
    r = plugin.wrap_runner(ok_run, fw, errors)(x, 2, Cfg())
    assert isinstance(r, fw.RecoveryResult)
    assert r.spectrum.entries == {3: 1 + 2j} and r.samples_read == 3 == x.access_count
    assert r.iterations == 4 and r.converged
    with pytest.raises(errors.ConfigMismatch):
        plugin.wrap_runner(bad_run, fw, errors)(_RefSignal(np.zeros(16)), 2, Cfg())


@pytest.mark.gpu
def test_wrapper_on_device_runner():
    """Real device runner behind the wrapper: entries, samples_read and the
    reference-side access map agree with the oracle (C1-like small case)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import sfft_oracle as O
    from paper_2012_08238_b200 import frameworks as dev
    from paper_2012_08238_b200 import plugin
    from paper_2012_08238_b200.frameworks import AlgorithmConfig
    fw, errors = _fake_reference()
    x, _ = O.synth(4096, 8, None, 3)
    cfg = AlgorithmConfig(framework="iterative", num_buckets=64, seed=2)
    ref = _RefSignal(x)
    r = plugin.wrap_runner(dev.run_iterative, fw, errors)(ref, 8, cfg)
    want = O.iterative(O.Access(x), 8, O.Cfg(framework="iterative", num_buckets=64, seed=2))
    assert set(r.spectrum.entries) == set(want.entries)
    assert r.samples_read == ref.access_count == want.samples_read
