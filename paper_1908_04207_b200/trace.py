"""Run-trace records in the reference's wire format (trace.py:15-109).

GPU runs emit the same `RoundRecord` / `SnapshotRecord` / `LatencyRecord`
shapes so that offline checkers written against the reference (e.g.
`eagercoll.verify.check_round_contracts`) consume them unchanged; `u` and
snapshot data are torch tensors here and become lists in the JSONL dump.
Times are host microseconds since import (the reference uses simulated time).
"""

from __future__ import annotations

import json
import threading
from dataclasses import dataclass, field

import numpy as np


def _as_list(x):
    if x is None:
        return None
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    return [float(v) for v in np.asarray(x).ravel()]


@dataclass
class RoundRecord:
    rank: int
    rnd: int
    u: object              # already divided by p (torch tensor or None)
    included: int          # bitmask of contributing ranks
    nap: int
    flavor: str
    initiator: int         # -1 when the flavor has no designated initiator
    t_done: int


@dataclass
class SnapshotRecord:
    rank: int
    rnd: int
    data: object           # contribution consumed from the send buffer (None if null)
    fresh: bool
    t: int


@dataclass
class LatencyRecord:
    rank: int
    rnd: int
    t_enter: int
    t_exit: int

    @property
    def latency_us(self) -> int:
        return self.t_exit - self.t_enter


@dataclass
class TraceRecorder:
    """trace.py:48-109.  Thread-safe (emulated worlds record from P threads)."""

    level: str = "results"
    rounds: list = field(default_factory=list)
    snapshots: list = field(default_factory=list)
    latencies: list = field(default_factory=list)
    op_events: list = field(default_factory=list)
    gradients: dict = field(default_factory=dict)
    weights: dict = field(default_factory=dict)
    losses: dict = field(default_factory=dict)
    _lock: threading.Lock = field(default_factory=threading.Lock, repr=False)

    def op_fired(self, t, rank, cid, gen, oid, label) -> None:
        if self.level == "ops":
            with self._lock:
                self.op_events.append((t, rank, cid, gen, oid, label))

    def round_done(self, rec: RoundRecord) -> None:
        with self._lock:
            self.rounds.append(rec)

    def snapshot(self, rec: SnapshotRecord) -> None:
        with self._lock:
            self.snapshots.append(rec)

    def latency(self, rec: LatencyRecord) -> None:
        with self._lock:
            self.latencies.append(rec)

    def rounds_by_key(self) -> dict:
        return {(r.rank, r.rnd): r for r in self.rounds}

    def dump_jsonl(self, path: str) -> None:
        with open(path, "w") as f:
            for r in self.rounds:
                f.write(json.dumps({
                    "kind": "round", "rank": r.rank, "round": r.rnd, "u": _as_list(r.u),
                    "included": r.included, "nap": r.nap, "flavor": r.flavor,
                    "initiator": r.initiator, "t_done": r.t_done,
                }) + "\n")
            for s in self.snapshots:
                f.write(json.dumps({
                    "kind": "snapshot", "rank": s.rank, "round": s.rnd,
                    "data": _as_list(s.data), "fresh": s.fresh, "t": s.t,
                }) + "\n")
            for lat in self.latencies:
                f.write(json.dumps({
                    "kind": "latency", "rank": lat.rank, "round": lat.rnd,
                    "t_enter": lat.t_enter, "t_exit": lat.t_exit,
                }) + "\n")
            for ev in self.op_events:
                t, rank, cid, gen, oid, label = ev
                f.write(json.dumps({
                    "kind": "op", "t": t, "rank": rank, "cid": cid, "gen": gen,
                    "op": oid, "label": label,
                }) + "\n")


class DeliveryLedger:
    """Per-gradient bookkeeping (the reference's verify.py:44-108 ledger): when
    was each (rank, round) gradient folded into a completed collective sum.
    Delivered at most once, ever.  Thread-safe."""

    def __init__(self):
        self._delivered: dict = {}
        self._order: list = []
        self._violations: list = []
        self._lock = threading.Lock()

    def generated(self, rank: int, rnd: int) -> None:
        with self._lock:
            key = (rank, rnd)
            if key in self._delivered:
                self._violations.append(("double-generation", rnd, rank))
                return
            self._delivered[key] = None
            self._order.append(key)

    def delivered(self, rank: int, generated_round: int, delivered_round: int) -> None:
        with self._lock:
            key = (rank, generated_round)
            if key not in self._delivered:
                self._violations.append(("unknown-gradient", delivered_round, rank))
                return
            if self._delivered[key] is not None:
                self._violations.append(("double-delivery", delivered_round, rank))
                return
            self._delivered[key] = delivered_round

    def entries(self) -> list:
        return [(r, g, self._delivered[(r, g)]) for r, g in self._order]

    def as_dict(self) -> dict:
        return dict(self._delivered)

    def staleness_of(self, rank: int, rnd: int):
        d = self._delivered.get((rank, rnd))
        return None if d is None else d - rnd

    def max_staleness(self) -> int:
        ages = [d - g for (_, g), d in self._delivered.items() if d is not None]
        return max(ages, default=0)

    def audit(self, tau=None, allow_pending_after=None) -> list:
        out = list(self._violations)
        for (rank, g), d in self._delivered.items():
            if d is None:
                if allow_pending_after is None or g <= allow_pending_after:
                    out.append(("undelivered", g, rank))
            elif d < g:
                out.append(("time-travel", g, rank))
            elif tau is not None and d - g > tau:
                out.append(("staleness", g, rank))
        return out
