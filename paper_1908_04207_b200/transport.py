"""Imbalance injection (transport.py:98-149, 504-506 of the reference).

The message layer of the reference (Message/Tag, SimTransport, SocketTransport)
is gone -- peers talk through NVLink-mapped control blocks (world.py).  What
remains is the delay model that drives the imbalance benchmarks, bit-identical
to the reference's seeded schedules, and two ways to realise a delay on
hardware: a host sleep (`Sleep`, handled by `collectives.drive`) or a device
spin kernel on the compute stream (`device_delay`), which models a rank whose
GPU is still computing its gradient.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DELAY_KINDS = ("none", "constant", "linear_skew", "random_subset")


@dataclass
class Sleep:
    """A process yields Sleep(us) to idle (transport.py:59-61)."""
    us: int


@dataclass(frozen=True)
class DelayModel:
    """transport.py:101-124

    none           no delay anywhere
    constant       every rank sleeps unit_ms each round
    linear_skew    rank r sleeps (r + 1) * unit_ms each round
    random_subset  k distinct ranks, drawn per round from `seed`, sleep unit_ms
    """

    kind: str = "none"
    unit_ms: float = 0.0
    k: int = 1
    seed: int = 0

    def __post_init__(self):
        if self.kind not in DELAY_KINDS:
            raise ValueError(f"unknown delay kind {self.kind!r}")
        if self.unit_ms < 0:
            raise ValueError("unit_ms must be >= 0")
        if self.k < 0:
            raise ValueError("k must be >= 0")


def delayed_ranks(model: DelayModel, rnd: int, p: int) -> tuple:
    """transport.py:127-134: pure function of (seed, rnd, p)."""
    k = min(model.k, p)
    rng = np.random.default_rng([model.seed, rnd])
    return tuple(int(r) for r in rng.choice(p, size=k, replace=False))


def inject_delay(rank: int, rnd: int, model: DelayModel, p: int) -> int:
    """transport.py:137-149: microseconds `rank` idles before round `rnd`."""
    if model.kind == "none":
        return 0
    if model.kind == "constant":
        return int(round(model.unit_ms * 1000))
    if model.kind == "linear_skew":
        return int(round((rank + 1) * model.unit_ms * 1000))
    if model.kind == "random_subset":
        if rank in delayed_ranks(model, rnd, p):
            return int(round(model.unit_ms * 1000))
        return 0
    raise ValueError(model.kind)


def delays_for_round(model: DelayModel, rnd: int, p: int) -> list:
    """transport.py:504-506"""
    return [inject_delay(r, rnd, model, p) for r in range(p)]


def delay_table(model: DelayModel, p: int, rounds: int) -> np.ndarray:
    """[p, rounds] int64 microseconds (harness.py:198-203)."""
    d = np.zeros((p, rounds), dtype=np.int64)
    for t in range(rounds):
        for r in range(p):
            d[r, t] = inject_delay(r, t, model, p)
    return d


def device_delay(us: int, stream=None) -> None:
    """Spin the GPU for `us` microseconds on `stream` (default: current), the
    device-side form of the injected computation delay (%globaltimer loop)."""
    import torch

    from ._lib import call
    if us <= 0:
        return
    s = stream if stream is not None else torch.cuda.current_stream()
    call("ec_spin", int(us) * 1000, s.cuda_stream)
