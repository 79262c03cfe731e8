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


def test_train_csv_and_jsonl_mirror(tmp_path):
    """harness.py:393-407: eagercoll-train-v1 CSV (floats as repr) and its
    JSON-lines mirror with a schema header, identical fields and values."""
    from paper_1908_04207_b200.harness import emit_train, train_row
    rows = [train_row("solo", {"round": t, "epoch": t // 4, "rank": r, "loss": 0.1 * (t + r) + 1e-17,
                               "nap": 1 + r, "staleness_max": t % 2, "wall_or_sim_time": 10 * t})
            for t in range(3) for r in range(2)]
    emit_train(rows, str(tmp_path / "tr"))
    lines = (tmp_path / "tr.csv").read_text().splitlines()
    assert lines[0] == "# eagercoll-train-v1"
    assert lines[1] == "flavor,round,epoch,rank,loss,nap,staleness_max,t_us"
    assert lines[3] == f"solo,0,0,1,{rows[1]['loss']!r},2,0,0"
    js = [json.loads(x) for x in (tmp_path / "tr.jsonl").read_text().splitlines()]
    assert js[0] == {"schema": "eagercoll-train-v1"}
    assert js[1:] == rows
    for line, row in zip(lines[2:], rows):
        assert float(line.split(",")[4]) == row["loss"]      # repr round-trips


def test_read_bench_csv_roundtrip_and_schema_errors(tmp_path):
    """harness.py:410-424 read_bench_csv, harness.py:427-431 JSONL mirror."""
    from paper_1908_04207_b200.harness import ConfigError, emit_bench, read_bench_csv
    recs = [BenchRecord("majority", t, r, 7 * t + r, 1 + (t + r) % 3, (t * 5) % 4)
            for t in range(4) for r in range(4)]
    emit_bench(recs, str(tmp_path / "b"))
    assert read_bench_csv(str(tmp_path / "b.csv")) == recs
    js = [json.loads(x) for x in (tmp_path / "b.jsonl").read_text().splitlines()]
    assert js[0] == {"schema": "eagercoll-bench-v1"} and len(js) == 17
    assert js[5] == {"flavor": "majority", "round": 1, "rank": 0, "latency_us": 7, "nap": 2,
                     "initiator": 1}
    bad = tmp_path / "bad.csv"
    bad.write_text("# eagercoll-bench-v0\nflavor\n")
    with pytest.raises(ConfigError):
        read_bench_csv(str(bad))
    bad.write_text("# eagercoll-bench-v1\nflavor,round\n")
    with pytest.raises(ConfigError):
        read_bench_csv(str(bad))
    with pytest.raises(ValueError):
        BenchRecord("solo", 0, 0, -1, 1)
    with pytest.raises(ValueError):
        BenchRecord("solo", 0, 0, 1, 0)


def test_hyperplane_model_pinned_to_reference():
    """models.py:62-71 known answer (test_models.py:18-22), central
    differences (acceptance criterion 10) and -- against the reference's own
    config-1 run (tests/golden/c1_solo.npz) -- the dataset, the per-(rank, step)
    minibatch and the gradient at every epoch start, on CPU torch in f64."""
    import os

    import torch

    from paper_1908_04207_b200.models import gen_dataset, loss_and_grad, mse, sample_batch
    loss, grad = loss_and_grad(torch.tensor([2.0], dtype=torch.float64),
                               torch.tensor([[1.0]], dtype=torch.float64),
                               torch.tensor([0.0], dtype=torch.float64))
    assert float(loss) == 4.0 and grad.tolist() == [4.0]
    rng = np.random.default_rng(31337)
    worst = 0.0
    for _ in range(50):
        dim, b = int(rng.integers(1, 17)), int(rng.integers(1, 33))
        x = torch.as_tensor(rng.standard_normal((b, dim)))
        y = torch.as_tensor(rng.standard_normal(b))
        w = torch.as_tensor(rng.standard_normal(dim))
        _, g = loss_and_grad(w, x, y)
        for j in range(dim):
            e = torch.zeros(dim, dtype=torch.float64)
            e[j] = 1e-6
            fd = (mse(w + e, x, y) - mse(w - e, x, y)) / 2e-6
            worst = max(worst, abs(float(g[j]) - fd) / max(1.0, abs(fd)))
    assert worst <= 1e-6
    golden = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    tr = np.load(os.path.join(golden, "c1_solo.npz"))
    ds = gen_dataset(64, 4096, seed=99, device=torch.device("cpu"), dtype=torch.float64)
    spe = int(tr["steps_per_epoch"])
    for r in range(int(tr["p"])):
        for e in range(0, int(tr["epochs"]), 7):
            t = e * spe
            x, y = sample_batch(ds, 99, r, t, 128)
            loss, g = loss_and_grad(torch.as_tensor(tr["w_epoch"][r, e]), x, y)
            ref = tr["grads"][r, t]
            assert np.max(np.abs(g.numpy() - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
            assert abs(float(loss) - tr["losses"][r, t]) <= 1e-12 * max(1.0, tr["losses"][r, t])
