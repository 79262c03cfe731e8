"""CPU tests of the reference-compatible record formats: trace JSONL, the
eagercoll-bench-v1 CSV, summarize(), the delivery ledger and the EGW1
checkpoint (trace.py, harness.py:347-425, verify.py:44-108,
eagersgd.py:281-299 of the reference)."""

import json

import numpy as np
import pytest

from paper_1908_04207_b200.eagersgd import load_weights, save_weights
from paper_1908_04207_b200.harness import BenchRecord, summarize, write_bench_csv
from paper_1908_04207_b200.trace import (DeliveryLedger, LatencyRecord, RoundRecord,
                                         SnapshotRecord, TraceRecorder)


def test_trace_jsonl_roundtrip(tmp_path):
    rec = TraceRecorder()
    rec.round_done(RoundRecord(0, 3, np.array([1.5, 2.0]), 0b11, 2, "solo", -1, 10))
    rec.snapshot(SnapshotRecord(1, 3, None, False, 5))
    rec.latency(LatencyRecord(0, 3, 1, 9))
    path = tmp_path / "t.jsonl"
    rec.dump_jsonl(str(path))
    rows = [json.loads(x) for x in path.read_text().splitlines()]
    assert rows[0] == {"kind": "round", "rank": 0, "round": 3, "u": [1.5, 2.0], "included": 3,
                       "nap": 2, "flavor": "solo", "initiator": -1, "t_done": 10}
    assert rows[1]["kind"] == "snapshot" and rows[1]["data"] is None and rows[1]["fresh"] is False
    assert rows[2] == {"kind": "latency", "rank": 0, "round": 3, "t_enter": 1, "t_exit": 9}
    assert rec.latencies[0].latency_us == 8
    assert rec.rounds_by_key()[(0, 3)].nap == 2


def test_bench_csv_schema_and_summary(tmp_path):
    recs = [BenchRecord("sync", 0, r, 100 + r, 4) for r in range(4)] + \
           [BenchRecord("solo", 0, r, 10, 1) for r in range(4)]
    path = tmp_path / "b.csv"
    write_bench_csv(recs, str(path))
    lines = path.read_text().splitlines()
    assert lines[0] == "# eagercoll-bench-v1"
    assert lines[1] == "flavor,round,rank,latency_us,nap,initiator"
    assert lines[2] == "sync,0,0,100,4,-1"
    s = summarize(recs)
    assert s["flavors"]["sync"]["mean_latency_us"] == pytest.approx(101.5)
    assert s["flavors"]["solo"]["mean_nap"] == 1.0
    assert s["speedup_vs_sync"]["solo"] == pytest.approx(10.15)


def test_delivery_ledger_contracts():
    led = DeliveryLedger()
    for g in range(4):
        led.generated(0, g)
    led.delivered(0, 0, 0)
    led.delivered(0, 1, 3)
    led.delivered(0, 1, 3)          # double delivery
    led.delivered(0, 9, 3)          # unknown gradient
    kinds = sorted(v[0] for v in led.audit(tau=1))
    assert kinds == ["double-delivery", "staleness", "undelivered", "undelivered",
                     "unknown-gradient"]
    assert led.staleness_of(0, 1) == 2 and led.max_staleness() == 2
    assert led.entries()[:2] == [(0, 0, 0), (0, 1, 3)]
    assert not [v for v in led.audit(allow_pending_after=1) if v[0] == "undelivered"]


def test_egw1_checkpoint_roundtrip(tmp_path):
    w = np.random.default_rng(0).standard_normal(17)
    p = tmp_path / "w.egw"
    save_weights(str(p), w)
    raw = p.read_bytes()
    assert raw[:4] == b"EGW1" and len(raw) == 16 + 17 * 8
    assert np.array_equal(load_weights(str(p)), w)
    p.write_bytes(raw[:40])
    with pytest.raises(ValueError):
        load_weights(str(p))


def test_egs1_state_roundtrip(tmp_path):
    """Resumable eager-SGD state: weights, stash, momentum,
    pending rounds, ledger, step and generation survive bit for bit."""
    from paper_1908_04207_b200.eagersgd import read_state_file, write_state_file
    rng = np.random.default_rng(3)
    for dt in (np.float32, np.float64):
        rec = {"w": rng.standard_normal(1001).astype(dt), "t": 17, "generation": 17,
               "contributed_round": 15, "rank": 3, "resync_period": 8, "tau": None, "lr": 0.05,
               "mu": 0.9, "pending": [15, 16], "ledger": {3: 4, 7: 9},
               "stash": rng.standard_normal(1001).astype(dt),
               "momentum": rng.standard_normal(1001).astype(dt)}
        p = tmp_path / f"s{dt.__name__}.egs"
        write_state_file(str(p), rec)
        out = read_state_file(str(p))
        for k in ("w", "stash", "momentum"):
            assert out[k].dtype == dt and out[k].tobytes() == rec[k].tobytes()
        assert out["pending"] == [15, 16] and out["ledger"] == {3: 4, 7: 9}
        assert (out["t"], out["generation"], out["contributed_round"], out["tau"]) == (17, 17, 15, None)
        raw = p.read_bytes()
        assert raw[:4] == b"EGS1"
        p.write_bytes(raw[:-8])
        with pytest.raises(ValueError):
            read_state_file(str(p))
    rec["stash"] = rec["momentum"] = None
    rec["pending"], rec["tau"] = [], 4
    write_state_file(str(tmp_path / "n.egs"), rec)
    out = read_state_file(str(tmp_path / "n.egs"))
    assert out["stash"] is None and out["momentum"] is None and out["tau"] == 4
