"""Workload side and wire formats on the device.

* Byte-identical reruns (test_acceptance.py:296-317): replaying the
  reference's config-1 schedule twice writes byte-identical eagercoll-train-v1
  CSV and JSONL files; the replayed losses (f64) equal the reference's.
* Null snapshots are recorded with the zero vector (trace.py:92-96).
* BASELINE config 4: the UCF101-shaped LSTM takes eager-SGD steps through the
  zero-copy bucket; the first step's weights equal w0 - lr * mean of the
  ranks' gradients (the fp32 restatement), and both ranks stay identical.
"""

import os
import threading

import numpy as np
import pytest
import torch

from oracle import restated as R
from paper_1908_04207_b200 import (AllreduceHandle, CollectiveConfig, EmulatedWorld, TrainState,
                                   TraceRecorder, finish_step, train_step_async)
from paper_1908_04207_b200.harness import emit_train
from paper_1908_04207_b200.models import gen_dataset, loss_and_grad, sample_batch
from paper_1908_04207_b200.replay import replay_training

pytestmark = pytest.mark.gpu


def test_replay_rerun_writes_byte_identical_train_csv(golden_dir, tmp_path):
    tr = np.load(os.path.join(golden_dir, "c1_solo.npz"))
    ds = gen_dataset(64, 4096, seed=99, device=torch.device("cuda", 0), dtype=torch.float64)

    def loss_fn(r, t, w):
        x, y = sample_batch(ds, 99, r, t, 128)
        return float(loss_and_grad(w.double(), x, y)[0])

    blobs = []
    for i, element in enumerate(("f8", "f8", "f4")):
        out = replay_training(tr, element, loss_fn=loss_fn, flavor="solo")
        stem = str(tmp_path / f"run{i}")
        emit_train(out["rows"], stem)
        blobs.append((open(stem + ".csv", "rb").read(), open(stem + ".jsonl", "rb").read()))
        if element == "f8":
            # f64 replay: the weights each step started from are the
            # reference's, so are the losses (numpy vs cuBLAS summation order)
            got = {(d["rank"], d["round"]): d["loss"] for d in out["rows"]}
            ref = tr["losses"]
            for (r, t), v in got.items():
                assert abs(v - ref[r, t]) <= 1e-12 * max(1.0, abs(ref[r, t]))
    assert blobs[0] == blobs[1]
    assert len(blobs[0][0]) > 1000 and blobs[0][0].startswith(b"# eagercoll-train-v1\n")
    assert blobs[2] != blobs[0]          # fp32 replay: same schedule, other bits


def test_null_snapshot_records_the_zero_vector():
    world = EmulatedWorld(2)
    cfg = CollectiveConfig(p=2, flavor="solo", vector_len=5, element="f4")
    rec = TraceRecorder()
    hs = [AllreduceHandle(cfg, r, world, recorder=rec) for r in range(2)]
    assert hs[0]._contribute(0, np.arange(5, dtype=np.float32), True, True)
    hs[0].wait_blocking(0)
    hs[1].wait_blocking(0)          # rank 1 never offered: its snapshot was null
    snaps = {(s.rank, s.rnd): s for s in rec.snapshots}
    assert snaps[(0, 0)].fresh and snaps[(0, 0)].data.cpu().tolist() == [0, 1, 2, 3, 4]
    assert not snaps[(1, 0)].fresh
    assert snaps[(1, 0)].data.cpu().tolist() == [0.0] * 5
    world.close()


def test_lstm_config4_eager_sgd_steps():
    from paper_1908_04207_b200.lstm import SyntheticUCF101, VideoLSTM, bind_flat, lstm_grad_step
    p, hidden, lr, steps = 2, 64, 0.01, 3
    world = EmulatedWorld(p)
    torch.manual_seed(1234)
    models = [VideoLSTM(hidden=hidden).cuda() for _ in range(p)]
    models[1].load_state_dict(models[0].state_dict())      # same w0 on both ranks
    n = sum(x.numel() for x in models[0].parameters())
    cfg = CollectiveConfig(p=p, flavor="solo", vector_len=n, element="f4", seed=1234)
    hs = [AllreduceHandle(cfg, r, world, cid=5) for r in range(p)]
    states = [TrainState.fresh(torch.zeros(n, device="cuda"), lr, rank=r, tau=None)
              for r in range(p)]
    for r in range(p):
        bind_flat(models[r], states[r].w, hs[r].grad_buffer())
    w0 = states[0].w.cpu().numpy().copy()
    data = SyntheticUCF101(batch=4, max_len=48)
    streams = [torch.cuda.Stream() for _ in range(p)]
    # a library's first use on a new stream (cuBLAS workspaces, autograd) may
    # synchronise the device: warm every rank's stream before an engine is
    # resident (library hazards)
    for r in range(p):
        with torch.cuda.stream(streams[r]):
            lstm_grad_step(models[r], hs[r].grad_buffer(), data.batch_for(r, 99))
    world.synchronize()
    g_first, w_first, losses, naps, errors = {}, {}, {}, {}, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(streams[r]):
                for t in range(steps):
                    loss = lstm_grad_step(models[r], hs[r].grad_buffer(), data.batch_for(r, t))
                    if t == 0:
                        g_first[r] = hs[r].grad_buffer().clone()
                    lo, res, gen = finish_step(states[r], hs[r],
                                               train_step_async(states[r], hs[r],
                                                                hs[r].grad_buffer(),
                                                                loss=loss, all_arrive=True))
                    losses[(r, t)] = float(lo.detach())
                    naps[(r, t)] = res.nap
                    if t == 0:
                        w_first[r] = states[r].w.clone()
                streams[r].synchronize()
        except BaseException as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(p)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    world.synchronize()
    assert not errors, errors[0]
    assert all(v == p for v in naps.values())
    assert all(np.isfinite(v) for v in losses.values())
    w = [st.w.cpu().numpy() for st in states]
    assert w[0].tobytes() == w[1].tobytes()                 # Lemma 1: same u everywhere
    assert not np.array_equal(w[0], w0)
    # first step against the restatement (fp32 tree order, / P, two roundings)
    u, _, _ = R.allreduce_round([g_first[r].cpu().numpy() for r in range(p)], [True] * p,
                                np.float32)
    assert np.isfinite(u).all()
    w1 = R.sgd_update(w0, u, lr)
    for r in range(p):
        assert w_first[r].cpu().numpy().tobytes() == w1.tobytes()
    world.close()
