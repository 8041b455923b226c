"""Plug the device runners into the reference harness.

The reference dispatches every run through ``frameworks._RUNNERS``
(sfft/frameworks.py:704-715), and ``run_experiment`` / ``run_sweep`` / the CLI
(sfft/harness.py:170-275, sfft/cli.py:53-87) call ``run_algorithm``.
``install()`` swaps the one-shot / voting / iterative / peeling entries for wrappers that
upload the reference ``TimeSignal``, run the device runner, mark the indices
the device read in the reference signal's access map (so ``samples_read`` and
the CSV's sampling fraction stay exact), re-raise library errors as the
reference's exception types (so ``run_experiment`` still turns them into
``converged=false`` rows), and return the reference's ``RecoveryResult``.
Bench rows then come out in the reference's own CSV schema, with device timings.
"""

from __future__ import annotations

import importlib

__all__ = ["install", "uninstall", "wrap_runner"]

_DEVICE = ("one_shot", "voting", "iterative", "peeling")


def wrap_runner(run, fw, errors, dtype: str = "complex128", device=None):
    """A reference-signature runner (x, k, cfg) backed by the device runner ``run``."""
    import numpy as np

    from .errors import SparseFFTError
    from .frameworks import AlgorithmConfig
    from .signal import TimeSignal

    def runner(x, k, cfg):
        xs = TimeSignal(np.asarray(x.samples), dtype=dtype, device=device)
        try:
            res = run(xs, k, AlgorithmConfig.from_json(cfg.to_json()))
        except SparseFFTError as exc:
            ref_exc = getattr(errors, type(exc).__name__, errors.SparseFFTError)
            raise ref_exc(str(exc)) from exc
        x._accessed[xs.accessed_indices()] = True
        spec = fw.SparseSpectrum(x.n, {int(f): complex(c) for f, c in res.spectrum.entries.items()})
        return fw.RecoveryResult(spec, x.access_count, res.iterations, res.converged)

    runner.__name__ = getattr(run, "__name__", "device_runner")
    return runner


def install(fw=None, frameworks=_DEVICE, dtype: str = "complex128", device=None) -> dict:
    """Register the device runners in the reference's ``_RUNNERS`` (default:
    the importable ``sparsefft.frameworks``).  Returns the replaced entries
    for ``uninstall``."""
    from . import frameworks as dev
    if fw is None:
        fw = importlib.import_module("sparsefft.frameworks")
    errors = importlib.import_module(fw.__name__.rsplit(".", 1)[0] + ".errors")
    table = {"one_shot": dev.run_oneshot, "voting": dev.run_voting,
             "iterative": dev.run_iterative, "peeling": dev.run_peeling}
    previous = {}
    for name in frameworks:
        if name not in table:
            raise ValueError(f"no device runner for framework {name!r}")
        previous[name] = fw._RUNNERS[name]
        fw._RUNNERS[name] = wrap_runner(table[name], fw, errors, dtype=dtype, device=device)
    return previous


def uninstall(previous: dict, fw=None) -> None:
    if fw is None:
        fw = importlib.import_module("sparsefft.frameworks")
    fw._RUNNERS.update(previous)
