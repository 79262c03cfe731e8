"""The reference's analytic latency / NAP oracles for the imbalance bench
(pkg/tests/test_harness.py:41-76) on the device, through harness.bench_flavor:
P=4, per-round skew (r+1)*unit.  A sync round closes when rank 3 arrives, so
rank r waits (3-r)*unit inside the call; a solo round is over before anyone
else arrives (latency ~0, nap 1); a majority round closes when its designated
initiator arrives: rank r waits max(0, init-r)*unit and nap = init+1.

Real clocks replace the simulator's: unit = 20 ms (a host thread on a shared
box can oversleep by several ms, which must not reorder arrivals); masks and naps are checked
exactly for every round, latencies per rank as the median over its rounds
within a host-jitter tolerance (host threads on a shared box occasionally
oversleep by a few ms -- a single round's latency is not an oracle)."""

import threading

import numpy as np
import pytest
import torch

from paper_1908_04207_b200 import EmulatedWorld, initiator_for_round
from paper_1908_04207_b200.harness import bench_flavor, summarize
from paper_1908_04207_b200.transport import DelayModel

pytestmark = pytest.mark.gpu

UNIT_US = 20000
TOL_US = 2000


def _run(flavor, rounds, p=4, seed=1234):
    world = EmulatedWorld(p)
    model = DelayModel("linear_skew", unit_ms=UNIT_US / 1000)
    bar = threading.Barrier(p)
    out, errors = {}, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = bench_flavor(world, r, p, flavor, model, rounds=rounds, vector_len=8,
                                  seed=seed, barrier=bar.wait, close=False, cid=7)
        except BaseException as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(p)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    world.close()
    assert not errors, errors[0]
    return [b for r in range(p) for b in out[r]]


def _median_error_per_rank(recs, expected):
    out = {}
    for r in sorted({b.rank for b in recs}):
        out[r] = float(np.median([b.latency_us - expected(b) for b in recs if b.rank == r]))
    return out


def test_sync_latency_matches_the_arrival_math():
    recs = _run("sync", rounds=6)
    assert all(b.nap == 4 for b in recs)
    err = _median_error_per_rank(recs, lambda b: (3 - b.rank) * UNIT_US)
    assert all(abs(e) < TOL_US for e in err.values()), err


def test_solo_latency_is_near_zero_and_nap_one_under_strict_skew():
    recs = _run("solo", rounds=6)
    assert all(b.nap == 1 for b in recs)
    err = _median_error_per_rank(recs, lambda b: 0)
    assert all(e < TOL_US for e in err.values()), err


def test_majority_latency_tracks_the_initiator():
    recs = _run("majority", rounds=8)
    for b in recs:
        init = initiator_for_round(1234, b.round, 4)
        assert b.initiator == init
        assert b.nap == init + 1, b
    err = _median_error_per_rank(
        recs, lambda b: max(0, initiator_for_round(1234, b.round, 4) - b.rank) * UNIT_US)
    assert all(abs(e) < TOL_US for e in err.values()), err


def test_flavor_ordering_under_skew():
    recs = _run("sync", 4) + _run("solo", 4) + _run("majority", 4)
    s = summarize(recs)
    lat = {f: s["flavors"][f]["mean_latency_us"] for f in ("sync", "solo", "majority")}
    assert lat["solo"] < lat["majority"] < lat["sync"]
    assert s["flavors"]["solo"]["mean_nap"] == 1.0 and s["flavors"]["sync"]["mean_nap"] == 4.0
