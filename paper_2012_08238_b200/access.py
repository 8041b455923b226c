"""Union of read schedules on the device (samples_read, sfft/signal.py:82-94)."""

from __future__ import annotations

from ._lib import check, lib, ptr, stream_of


def schedule_map(n: int, log: list, device):
    """uint8[n] map of every index read by the records in ``log``."""
    import torch
    m = torch.zeros(n, dtype=torch.uint8, device=device)
    st = stream_of(device)
    L = lib()
    for rec in log:
        kind = rec[0]
        if kind == "flat":
            _, sigma, tau, omega = rec
            check(L.sfft_access_mark(ptr(m), n, 0, sigma, tau, omega, None, st), "access_mark")
        elif kind == "spike":
            _, step, tau, count = rec
            check(L.sfft_access_mark(ptr(m), n, 1, step, tau, count, None, st), "access_mark")
        elif kind == "all":
            check(L.sfft_access_mark(ptr(m), n, 2, 0, 0, 0, None, st), "access_mark")
        elif kind == "list":
            idx = rec[1]
            check(L.sfft_access_mark(ptr(m), n, 3, 0, 0, idx.numel(), ptr(idx), st),
                  "access_mark")
        else:
            raise ValueError(f"unknown read record {kind!r}")
    return m


def count_schedule(n: int, log: list, device) -> int:
    import torch
    if not log:
        return 0
    m = schedule_map(n, log, device)
    out = torch.zeros(1, dtype=torch.int64, device=device)
    check(lib().sfft_count_nonzero(ptr(m), n, ptr(out), stream_of(device)), "count_nonzero")
    return int(out.item())
