"""The persistent engine on one GPU: P ranks of an EmulatedWorld (one engine
launch, one CTA group per rank) driven by P host threads.  Ports the
reference's known-answer tests (test_collectives.py, test_eagersgd.py) to the
device API, and replays the reference's config-1 schedules (tests/golden/c1_*)
bit for bit."""

import json
import os
import threading
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import restated as R  # noqa: E402
from paper_1908_04207_b200 import (  # noqa: E402
    AllreduceHandle, CollectiveConfig, EmulatedWorld, TraceRecorder, TrainState,
    attach_delivery_tracking, drive, initiator_for_round, run_allreduce, staleness_guard,
    train_step,
)
from paper_1908_04207_b200.replay import replay_training  # noqa: E402
from paper_1908_04207_b200.trace import DeliveryLedger  # noqa: E402


def _ka(golden_dir):
    with open(os.path.join(golden_dir, "known_answers.json")) as f:
        return json.load(f)


def _np(t):
    return t.detach().cpu().numpy()


def test_sync_pair_frozen_example():
    cfg = CollectiveConfig(p=2, flavor="sync", vector_len=2)
    res, _, world = run_allreduce(cfg, np.array([[2.0, 4.0], [4.0, 8.0]]))
    for r in range(2):
        assert _np(res[(r, 0)].u).tolist() == [3.0, 6.0]
        assert res[(r, 0)].included == 0b11 and res[(r, 0)].nap == 2
    world.close()


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8, 13])
def test_sync_matches_reference_bitwise(golden_dir, p):
    g = np.load(os.path.join(golden_dir, "tree_sums.npz"))
    contrib = g[f"sync_in_p{p}"]
    cfg = CollectiveConfig(p=p, flavor="sync", vector_len=8)
    res, _, world = run_allreduce(cfg, contrib, rounds=2)
    for r in range(p):
        for t in range(2):
            assert _np(res[(r, t)].u).tobytes() == g[f"sync_u_p{p}"].tobytes()
            assert res[(r, t)].nap == p
    world.close()


@pytest.mark.parametrize("p", [2, 3, 8])
@pytest.mark.parametrize("n", [1, 5, 1027, 300_001])
def test_sync_f32_matches_oracle(p, n):
    rng = np.random.default_rng(p * 1000 + n)
    contrib = rng.standard_normal((p, n)).astype(np.float32)
    cfg = CollectiveConfig(p=p, flavor="sync", vector_len=n, element="f4")
    res, _, world = run_allreduce(cfg, contrib, rounds=3)
    want, inc, nap = R.allreduce_round(list(contrib), [True] * p, np.float32)
    for r in range(p):
        for t in range(3):
            assert _np(res[(r, t)].u).tobytes() == want.tobytes()
            assert res[(r, t)].included == inc
    world.close()


def test_integer_element_divides_exactly(golden_dir):
    g = np.load(os.path.join(golden_dir, "tree_sums.npz"))
    cfg = CollectiveConfig(p=4, flavor="sync", vector_len=4, element="i8")
    res, _, world = run_allreduce(cfg, g["i8_in_p4"])
    assert res[(0, 0)].u.dtype == torch.int64
    assert _np(res[(0, 0)].u).tobytes() == g["i8_u_p4"].tobytes()
    world.close()


def test_solo_first_arrival_defines_the_round(golden_dir):
    ka = _ka(golden_dir)["solo_first_arrival"]
    contrib = np.array(ka["contrib"])
    cfg = CollectiveConfig(p=4, flavor="solo", vector_len=4)
    res, _, world = run_allreduce(cfg, contrib, delay_us=lambda r, t: 1000 * r, time_scale=20)
    for r in range(4):
        assert res[(r, 0)].included == ka["included"][r] == 0b0001
        assert _np(res[(r, 0)].u).tobytes() == np.array(ka["u"]).tobytes()
    world.close()


def test_solo_earliest_rank_need_not_be_rank_zero(golden_dir):
    ka = _ka(golden_dir)["solo_earliest_not_zero"]
    cfg = CollectiveConfig(p=4, flavor="solo", vector_len=2)
    contrib = np.random.default_rng(2).standard_normal((4, 2))
    res, _, world = run_allreduce(cfg, contrib, delay_us=lambda r, t: ka["delays_us"][r],
                                  time_scale=20)
    for r in range(4):
        assert res[(r, 0)].included == ka["included"] == 0b0100
    world.close()


def test_majority_round_zero_mask_is_an_arrival_prefix(golden_dir):
    ka = _ka(golden_dir)["majority_prefix"]
    for seed in (31, 32, 33, 34):
        p = 4
        cfg = CollectiveConfig(p=p, flavor="majority", vector_len=4, seed=seed)
        res, _, world = run_allreduce(cfg, lambda r, t: np.full(4, float(10 * r + t)),
                                      delay_us=lambda r, t: 1000 * r, time_scale=20)
        want = ka[str(seed)]
        assert initiator_for_round(seed, 0, p) == want["initiator"]
        for r in range(p):
            assert res[(r, 0)].included == want["included"]
            assert _np(res[(r, 0)].u).tolist() == want["u"]
        world.close()


def test_majority_multiround_agreement_and_initiator_freshness():
    p, rounds, seed = 4, 6, 31
    cfg = CollectiveConfig(p=p, flavor="majority", vector_len=4, seed=seed)
    rec = TraceRecorder()
    res, _, world = run_allreduce(cfg, lambda r, t: np.full(4, float(10 * r + t)), rounds=rounds,
                                  delay_us=lambda r, t: 1000 * r, recorder=rec, time_scale=5)
    by_gen = {}
    for row in rec.rounds:
        by_gen.setdefault(row.rnd, []).append(row)
    for g, rows in by_gen.items():
        init = initiator_for_round(seed, g, p)
        ref = rows[0]
        assert (ref.included >> init) & 1
        assert 1 <= ref.nap == bin(ref.included).count("1") <= p
        assert all(row.included == ref.included for row in rows)
        assert all(_np(row.u).tobytes() == _np(ref.u).tobytes() for row in rows)
    for r in range(p):
        gens = [res[(r, t)].rnd for t in range(rounds)]
        assert all(g >= t for t, g in enumerate(gens)) and gens == sorted(gens)
    world.close()


def test_solo_zero_skew_all_arrive():
    """With the bench's all-arrive barrier every contribution boards (nap = P)."""
    p = 8
    world = EmulatedWorld(p)
    cfg = CollectiveConfig(p=p, flavor="solo", vector_len=1000, element="f4")
    hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
    contrib = np.random.default_rng(3).standard_normal((p, 1000)).astype(np.float32)
    want, _, _ = R.allreduce_round(list(contrib), [True] * p, np.float32)
    out = {}

    def body(r):
        for t in range(3):
            hs[r]._contribute(t, contrib[r], fresh=True, activate=True, all_arrive=True)
            out[(r, t)] = hs[r].wait_blocking(t)

    th = [threading.Thread(target=body, args=(r,)) for r in range(p)]
    [x.start() for x in th]
    [x.join() for x in th]
    for r in range(p):
        for t in range(3):
            gen, res = out[(r, t)]
            assert gen == t and res.nap == p
            assert _np(res.u).tobytes() == want.tobytes()
    world.close()


def test_late_contribution_is_refused(golden_dir):
    ka = _ka(golden_dir)["late_refused"]
    world = EmulatedWorld(2)
    cfg = CollectiveConfig(p=2, flavor="solo", vector_len=2)
    hs = [AllreduceHandle(cfg, r, world) for r in range(2)]
    assert hs[0].try_contribute(0, np.array([1.0, 2.0])) is ka["accept0"] is True
    hs[0].activate(0)
    hs[0].wait_blocking(0)
    assert hs[0].round_done(0)
    assert hs[1].try_contribute(0, np.array([5.0, 5.0])) is ka["accept1"] is False
    gen, res = hs[1].latest_result()
    assert gen == ka["gen"] == 0 and res.included == ka["included"]
    assert _np(res.u).tolist() == ka["u"]
    world.close()


def test_out_of_order_round_is_an_error():
    world = EmulatedWorld(2)
    cfg = CollectiveConfig(p=2, flavor="solo", vector_len=2)
    hs = [AllreduceHandle(cfg, r, world) for r in range(2)]
    with pytest.raises(AssertionError):
        hs[0].try_contribute(1, np.array([1.0, 2.0]))
    world.close()


def test_wait_done_fast_path_returns_latest():
    cfg = CollectiveConfig(p=2, flavor="sync", vector_len=2)
    _, handles, world = run_allreduce(cfg, np.ones((2, 2)), rounds=3)
    world.resume()
    g = handles[0].wait_done(1)
    with pytest.raises(StopIteration) as ei:
        next(g)
    gen, res = ei.value.value
    assert gen == 2 and res.nap == 2
    world.close()


def test_pause_resume_allows_device_sync():
    world = EmulatedWorld(2)
    cfg = CollectiveConfig(p=2, flavor="sync", vector_len=16, element="f4")
    hs = [AllreduceHandle(cfg, r, world) for r in range(2)]
    out = {}

    def body(r, t):
        out[(r, t)] = drive(hs[r].call_round(t, np.full(16, r + 1.0, np.float32)))

    for t in range(2):
        th = [threading.Thread(target=body, args=(r, t)) for r in range(2)]
        [x.start() for x in th]
        [x.join() for x in th]
        world.synchronize()          # pause -> torch.cuda.synchronize -> resume
    assert _np(out[(0, 1)].u).tolist() == [1.5] * 16
    world.close()


def test_missed_round_folds_into_the_next_sum(golden_dir):
    """Fig. 7 (test_eagersgd.py:60-121): the slow rank misses round 0 and
    delivers both of its gradients in round 1."""
    ka = _ka(golden_dir)["fig7"]
    world = EmulatedWorld(2)
    cfg = CollectiveConfig(p=2, flavor="solo", vector_len=3)
    hs = [AllreduceHandle(cfg, r, world) for r in range(2)]
    states = [TrainState.fresh(np.zeros(3), lr=1.0, rank=r, dtype=torch.float64) for r in range(2)]
    ledger = DeliveryLedger()
    for r in range(2):
        attach_delivery_tracking(hs[r], states[r], ledger)
    gf = [torch.tensor(v, dtype=torch.float64, device="cuda") for v in ka["gf"]]
    gs = [torch.tensor(v, dtype=torch.float64, device="cuda") for v in ka["gs"]]
    seen = {}
    r0_done = threading.Event()
    slow_offered_1 = threading.Event()

    def fast():
        for t in range(2):
            if t == 1:
                slow_offered_1.wait(10)
            ledger.generated(0, t)
            _, res, gen = drive(train_step(states[0], None, hs[0], grad=gf[t], keep_u=True))
            seen[(0, t)] = res
            if t == 0:
                r0_done.set()

    def slow():
        r0_done.wait(10)          # round 0 completed: the bus is gone
        ledger.generated(1, 0)
        _, res, gen = drive(train_step(states[1], None, hs[1], grad=gs[0], keep_u=True))
        seen[(1, 0)] = res
        # round 1: fold g_s1 into the stash and offer it without activating; the
        # fast rank's offer boards before anyone activates (the link window)
        ledger.generated(1, 1)
        st = states[1]
        with hs[1].engine.lock:
            st.send_buf.fold(gs[1], 1)
            seq = hs[1]._post_contribute(1, 1)   # fresh, no activation
        assert hs[1]._reply(seq) == 1
        hs[1].contributed_round = 1
        hs[1]._fresh_gens.add(1)
        slow_offered_1.set()
        gen, res = hs[1].wait_blocking(1)
        seen[(1, 1)] = res

    th = [threading.Thread(target=fast), threading.Thread(target=slow)]
    [x.start() for x in th]
    [x.join() for x in th]
    r0 = seen[(0, 0)]
    assert r0.included == ka["r0_included"] and (_np(r0.u) * 2).tolist() == ka["r0_u_times_2"]
    for rank in range(2):
        r1 = seen[(rank, 1)]
        assert r1.included == ka["r1_included"]
        assert (_np(r1.u) * 2).tolist() == ka["r1_u_times_2"]
    assert ledger.staleness_of(1, 0) == 1
    assert ledger.staleness_of(1, 1) == 0
    assert ledger.staleness_of(0, 0) == 0
    assert not ledger.audit(tau=1)
    world.close()


@pytest.mark.parametrize("flavor", ["sync", "solo", "majority"])
def test_replay_c1_f64_bit_exact_vs_reference(golden_dir, flavor):
    tr = dict(np.load(os.path.join(golden_dir, f"c1_{flavor}.npz")))
    out = replay_training(tr, element="f8")
    assert out["accepted"].tolist() == tr["accepted"].tolist()
    assert out["masks"].tolist() == tr["masks"].tolist()
    assert out["w"].tobytes() == tr["final_w"].tobytes()
    led = {(int(r), int(g)): (None if d < 0 else int(d)) for r, g, d in tr["ledger"]}
    assert out["ledger"] == led


@pytest.mark.parametrize("flavor", ["sync", "solo", "majority"])
def test_replay_c1_f32_vs_oracle_and_reference(golden_dir, flavor):
    tr = dict(np.load(os.path.join(golden_dir, f"c1_{flavor}.npz")))
    out = replay_training(tr, element="f4")
    want = R.replay_run(tr, np.float32)
    assert out["w"].tobytes() == want["w"].tobytes()          # fixed order: bit-exact
    ref = tr["final_w"]
    rel = np.linalg.norm(out["w"].astype(np.float64) - ref) / np.linalg.norm(ref)
    assert rel < 1e-6                                          # north_star tolerance


def test_staleness_guard_holds_external_activation():
    """tau=1: rank 1 has a pending gradient of round 0; an external activation of
    round 1 is held until rank 1 itself contributes (eagersgd.py:89-110)."""
    world = EmulatedWorld(2)
    cfg = CollectiveConfig(p=2, flavor="solo", vector_len=4, element="f4")
    hs = [AllreduceHandle(cfg, r, world) for r in range(2)]
    st1 = TrainState.fresh(np.zeros(4), lr=0.1, rank=1, tau=1)
    staleness_guard(hs[1], st1)
    st1.send_buf.bind(hs[1])
    st1.send_buf.fold(torch.ones(4, device="cuda"), 0)   # pending round 0
    from paper_1908_04207_b200.eagersgd import _sync_hold
    _sync_hold(hs[1])                                    # hold generations >= 1
    # round 0 runs with rank 0 alone (not held: 0 + tau > 0)
    assert hs[0]._contribute(0, np.ones(4, np.float32), True, True)
    g, r0 = hs[0].wait_blocking(0)
    assert r0.included == 0b01
    # round 1: rank 0 activates, rank 1 holds
    assert hs[0]._contribute(1, np.ones(4, np.float32), True, True)
    time.sleep(0.05)
    assert not hs[0].round_done(1)
    assert hs[1]._contribute(1, np.full(4, 2.0, np.float32), True, False)
    g, r1 = hs[0].wait_blocking(1)
    assert r1.included == 0b11 and _np(r1.u).tolist() == [1.5] * 4
    world.close()


@pytest.mark.parametrize("p", [1, 3, 4])
def test_async_steps_match_oracle(p):
    """train_step_async (device-side fold mode, wait and update) gives the same
    bits as the oracle, with steps issued two ahead of reconciliation.  Each
    emulated rank needs its own stream: a device-side wait would otherwise sit
    in front of the peers' offers on a shared stream."""
    from collections import deque

    from paper_1908_04207_b200 import finish_step, train_step_async
    n, lr, steps = 100_003, 0.05, 5
    rng = np.random.default_rng(p)
    grads = rng.standard_normal((steps, p, n), dtype=np.float32)
    w0 = rng.standard_normal(n, dtype=np.float32)
    world = EmulatedWorld(p)
    cfg = CollectiveConfig(p=p, flavor="solo", vector_len=n, element="f4")
    hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
    states = [TrainState.fresh(w0, lr, rank=r, tau=None) for r in range(p)]
    gd = torch.as_tensor(grads, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(p)]
    torch.cuda.synchronize()
    out = {}

    def body(r):
        torch.cuda.set_device(0)
        torch.cuda.set_stream(streams[r])
        attach_delivery_tracking(hs[r], states[r])
        pend, res = deque(), []
        for t in range(steps):
            pend.append(train_step_async(states[r], hs[r], gd[t, r], all_arrive=True))
            if len(pend) > 2:
                res.append(finish_step(states[r], hs[r], pend.popleft()))
        while pend:
            res.append(finish_step(states[r], hs[r], pend.popleft()))
        torch.cuda.current_stream().synchronize()
        out[r] = res

    th = [threading.Thread(target=body, args=(r,)) for r in range(p)]
    [x.start() for x in th]
    [x.join() for x in th]
    w = w0.copy()
    for t in range(steps):
        u, inc, _ = R.allreduce_round(list(grads[t]), [True] * p, np.float32)
        w = R.sgd_update(w, u, lr)
        for r in range(p):
            _, res, gen = out[r][t]
            assert gen == t and res.included == inc
    for r in range(p):
        assert states[r].w.cpu().numpy().tobytes() == w.tobytes()
        assert states[r].send_buf.is_null
    world.close()


@pytest.mark.parametrize("flavor", ["sync", "solo", "majority"])
def test_training_process_config1_emulated(golden_dir, flavor):
    """BASELINE config 1 live (not replayed) on one GPU: 4 emulated ranks run the
    reference's training_process with its seeded random_subset delays, the
    staleness guard (tau = 8) and resync every 8 epochs.  Checks the run's
    contracts -- exactly-once, tau-bounded delivery, bit-identical weights after
    the final resync -- and that it converges to the reference's val MSE."""
    from paper_1908_04207_b200 import DelayModel, inject_delay, training_process
    from paper_1908_04207_b200.models import gen_dataset, init_weights
    p, epochs, spe = 4, 48, 4
    world = EmulatedWorld(p)
    ds = gen_dataset(64, 4096, seed=99)
    w0 = init_weights(64, seed=1234)
    model = DelayModel("random_subset", unit_ms=0.2, k=1, seed=11)
    cfg = CollectiveConfig(p=p, flavor=flavor, vector_len=64, element="f4", seed=1234)
    scfg = CollectiveConfig(p=p, flavor="sync", vector_len=64, element="f4")
    hs = [AllreduceHandle(cfg, r, world, cid=0) for r in range(p)]
    hr = [AllreduceHandle(scfg, r, world, cid=1) for r in range(p)]
    states = [TrainState.fresh(w0, 0.05, rank=r, resync_period=8, tau=8) for r in range(p)]
    ledger = DeliveryLedger()
    val, errors = {}, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            drive(training_process(r, states[r], hs[r], hr[r], ds, epochs=epochs,
                                   steps_per_epoch=spe, batch_per_rank=128, data_seed=99,
                                   delay_fn=lambda rank, t: inject_delay(rank, t, model, p),
                                   guard=True, ledger=ledger, val_out=val))
        except BaseException as e:
            errors.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(p)]
    [x.start() for x in th]
    [x.join() for x in th]
    assert not errors, errors
    # final resync at epoch 16: every rank holds the same bits
    ws = [s.w.cpu().numpy() for s in states]
    assert all(w.tobytes() == ws[0].tobytes() for w in ws)
    assert not ledger.audit(tau=8, allow_pending_after=epochs * spe - 9)
    tr = np.load(os.path.join(golden_dir, f"c1_{flavor}.npz"))
    final = np.mean([v for (r, e), v in val.items() if e == epochs - 1])
    assert abs(final - float(tr["final_val"])) < 0.002      # reference: 0.0105-0.0106
    world.close()


@pytest.mark.parametrize("p", [1, 4])
def test_zero_copy_offers_match_oracle(p):
    """Gradients written into the registered gradient bucket are offered in
    place (no fold) while the stash is null; results are the same bits."""
    from collections import deque

    from paper_1908_04207_b200 import finish_step, train_step_async
    n, lr, steps = 65_537, 0.05, 4
    rng = np.random.default_rng(10 + p)
    grads = rng.standard_normal((steps, p, n), dtype=np.float32)
    w0 = rng.standard_normal(n, dtype=np.float32)
    world = EmulatedWorld(p)
    cfg = CollectiveConfig(p=p, flavor="solo", vector_len=n, element="f4")
    hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
    states = [TrainState.fresh(w0, lr, rank=r, tau=None) for r in range(p)]
    gd = torch.as_tensor(grads, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(p)]
    bufs = [h.grad_buffer() for h in hs]
    torch.cuda.synchronize()

    def body(r):
        torch.cuda.set_device(0)
        torch.cuda.set_stream(streams[r])
        attach_delivery_tracking(hs[r], states[r])
        pend = deque()
        for t in range(steps):
            bufs[r].copy_(gd[t, r])                       # "backward" writes the bucket
            pend.append(train_step_async(states[r], hs[r], bufs[r], all_arrive=True))
            if len(pend) > 1:
                finish_step(states[r], hs[r], pend.popleft())
        while pend:
            finish_step(states[r], hs[r], pend.popleft())
        torch.cuda.current_stream().synchronize()

    th = [threading.Thread(target=body, args=(r,)) for r in range(p)]
    [x.start() for x in th]
    [x.join() for x in th]
    w = w0.copy()
    for t in range(steps):
        u, _, _ = R.allreduce_round(list(grads[t]), [True] * p, np.float32)
        w = R.sgd_update(w, u, lr)
    for r in range(p):
        assert states[r].w.cpu().numpy().tobytes() == w.tobytes()
    world.close()


@pytest.mark.parametrize("element,mu", [("f4", 0.0), ("f4", 0.9), ("f8", 0.0), ("f8", 0.9)])
def test_direct_fused_step_matches_oracle(element, mu):
    """World of one: decide + round + update run as ONE launch
    (ec_direct_step_kernel) that writes u to the slot and updates w from the
    register copy.  Same bits as the oracle's round followed by its (momentum)
    SGD update, for folded offers (arbitrary gradient tensor) and zero-copy
    offers (the registered bucket), ragged n, and the published u."""
    from collections import deque

    from paper_1908_04207_b200 import finish_step, train_step_async
    dt = np.float32 if element == "f4" else np.float64
    n, lr, steps = 100_003, 0.05, 6
    rng = np.random.default_rng(21)
    grads = rng.standard_normal((steps, n)).astype(dt)
    w0 = rng.standard_normal(n).astype(dt)
    world = EmulatedWorld(1)
    cfg = CollectiveConfig(p=1, flavor="solo", vector_len=n, element=element)
    h = AllreduceHandle(cfg, 0, world)
    st = TrainState.fresh(w0, lr, rank=0, tau=None, momentum=mu, dtype=cfg.torch_dtype)
    gd = torch.as_tensor(grads, device="cuda")
    bucket = h.grad_buffer()
    attach_delivery_tracking(h, st)
    pend = deque()
    for t in range(steps):
        if t % 2:
            bucket.copy_(gd[t])
            g = bucket                       # zero-copy offer
        else:
            g = gd[t]                        # folded into the stash
        pend.append(train_step_async(st, h, g, all_arrive=True))
        if len(pend) > 2:
            finish_step(st, h, pend.popleft())
    gens = []
    while pend:
        gens.append(finish_step(st, h, pend.popleft())[2])
    torch.cuda.synchronize()
    w, buf = w0.copy(), np.zeros_like(w0)
    for t in range(steps):
        u, inc, _ = R.allreduce_round([grads[t]], [True], dt)
        if mu:
            w, buf = R.momentum_update(w, buf, u, dt(lr), dt(mu))
        else:
            w = R.sgd_update(w, u, lr)
    assert gens[-1] == steps - 1
    assert st.w.cpu().numpy().tobytes() == w.tobytes()
    if mu:
        assert st.momentum_buf.cpu().numpy().tobytes() == buf.tobytes()
    gen, res = h.latest_result()
    assert gen == steps - 1 and _np(res.u).tobytes() == u.tobytes()
    assert st.send_buf.is_null
    world.close()


def test_direct_publication_stream_keeps_host_words_in_order():
    """World of one: a step's publication (replies, log, done_gen1) runs on the
    communicator's own stream, possibly after the next step already decided.
    Interleave pipelined async steps with plain rounds posted behind them
    (whose decide / round kernels answer on the caller's stream while earlier
    publications may still be pending) and a burst of 40 async steps: every
    reply and generation is reported in order, each plain round's result is
    its contribution, and w is the oracle's bits."""
    from collections import deque

    from paper_1908_04207_b200 import finish_step, train_step_async
    n, lr = 200_003, 0.05
    plan = ["a"] * 3 + ["r"] + ["a"] * 2 + ["r", "r"] + ["a"] * 40 + ["r"]
    rng = np.random.default_rng(33)
    grads = rng.standard_normal((len(plan), n)).astype(np.float32)
    w0 = rng.standard_normal(n).astype(np.float32)
    world = EmulatedWorld(1)
    h = AllreduceHandle(CollectiveConfig(p=1, flavor="solo", vector_len=n, element="f4"), 0, world)
    st = TrainState.fresh(w0, lr, rank=0, tau=None)
    gd = torch.as_tensor(grads, device="cuda")
    bucket = h.grad_buffer()
    pend, gens = deque(), []
    for t, kind in enumerate(plan):
        if kind == "a":
            bucket.copy_(gd[t])
            pend.append(train_step_async(st, h, bucket, all_arrive=True))
            if len(pend) > 3:
                gens.append(finish_step(st, h, pend.popleft())[2])
        else:
            # a plain round right behind pending (unreconciled) async steps,
            # no update; rounds are driven in order, so round t - 1 is done
            h.wait_blocking(t - 1)
            assert h._contribute(t, gd[t], fresh=True, activate=True)
            gen, res = h.wait_blocking(t)
            assert gen == t and res.included == 1 and res.nap == 1
            assert _np(res.u).tobytes() == grads[t].tobytes()
            while pend:
                gens.append(finish_step(st, h, pend.popleft())[2])
            gens.append(gen)
            st.t = t + 1
    while pend:
        gens.append(finish_step(st, h, pend.popleft())[2])
    torch.cuda.synchronize()
    assert gens == list(range(len(plan)))
    w = w0.copy()
    for t, kind in enumerate(plan):
        if kind == "a":
            u, _, _ = R.allreduce_round([grads[t]], [True], np.float32)
            w = R.sgd_update(w, u, lr)
    assert st.w.cpu().numpy().tobytes() == w.tobytes()
    gen, res = h.latest_result()
    assert gen == len(plan) - 1 and _np(res.u).tobytes() == grads[-1].tobytes()
    assert h.done_generation == len(plan) - 1
    world.close()


def test_direct_refused_step_takes_the_out_of_line_path():
    """World of one: a step whose offer arrives after its round already ran (a
    plain round took generation 0) is refused; the step kernel's out-of-line
    path applies generation 0 and keeps the zero-copy gradient in the stash,
    and its reply / report come from the publication kernel (no wait inside
    the step kernel).  The next step carries that gradient: u1 = 0 + (g0 + g1)."""
    from paper_1908_04207_b200 import finish_step, train_step_async
    n, lr = 70_001, 0.5
    rng = np.random.default_rng(8)
    v, g0, g1, w0 = (rng.standard_normal(n, dtype=np.float32) for _ in range(4))
    world = EmulatedWorld(1)
    h = AllreduceHandle(CollectiveConfig(p=1, flavor="solo", vector_len=n, element="f4"), 0, world)
    st = TrainState.fresh(w0, lr, rank=0, tau=None)
    assert h._contribute(0, v, fresh=True, activate=True)
    h.wait_blocking(0)
    bucket = h.grad_buffer()
    bucket.copy_(torch.as_tensor(g0, device="cuda"))
    _, res0, gen0 = finish_step(st, h, train_step_async(st, h, bucket, all_arrive=True))
    assert gen0 == 0
    w = w0 - np.float32(lr) * v
    assert st.w.cpu().numpy().tobytes() == w.tobytes()
    bucket.copy_(torch.as_tensor(g1, device="cuda"))
    _, res1, gen1 = finish_step(st, h, train_step_async(st, h, bucket, all_arrive=True))
    torch.cuda.synchronize()
    u1 = np.float32(0) + (g0 + g1)
    assert gen1 == 1 and res1.included == 1
    assert st.w.cpu().numpy().tobytes() == (w - np.float32(lr) * u1).tobytes()
    assert _np(h.latest_result()[1].u).tobytes() == u1.tobytes()
    world.close()


@pytest.mark.filterwarnings("ignore:The CUDA Graph is empty")
def test_async_step_refuses_graph_capture():
    """ec_step_async under stream capture fails loudly (EC_E_STATE) instead of
    baking one request sequence number into a graph that replays it; the
    communicator stays usable afterwards."""
    from paper_1908_04207_b200 import _lib, finish_step, train_step_async
    n = 4099
    world = EmulatedWorld(1)
    h = AllreduceHandle(CollectiveConfig(p=1, flavor="solo", vector_len=n, element="f4"), 0, world)
    st = TrainState.fresh(np.zeros(n, np.float32), 0.1, rank=0, tau=None)
    bucket = h.grad_buffer()
    bucket.fill_(1.0)
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with pytest.raises(_lib.EcError):
        with torch.cuda.graph(graph, stream=s):
            train_step_async(st, h, bucket)
    torch.cuda.synchronize()
    st.t = 0
    _, res, gen = finish_step(st, h, train_step_async(st, h, bucket))
    torch.cuda.synchronize()
    assert gen == 0 and res.nap == 1
    assert float(st.w[0]) == np.float32(-0.1)
    world.close()


@pytest.mark.parametrize("other_stream", [False, True])
def test_direct_zero_copy_folds_into_a_pending_stash(other_stream):
    """World of one: a zero-copy step that meets a pending (accepted, not yet
    reduced) stash folds the gradient into it inside the step kernel (no fold
    launch): u = 0 + (stash + g), the same bits as fold-then-round.  With
    other_stream the offer is posted from another stream than the step's (the
    step is ordered behind it, so its publication has nothing to wait for)."""
    from paper_1908_04207_b200 import finish_step, train_step_async
    n, lr = 50_001, 0.25
    rng = np.random.default_rng(5)
    v, g, w0 = (rng.standard_normal(n, dtype=np.float32) for _ in range(3))
    world = EmulatedWorld(1)
    h = AllreduceHandle(CollectiveConfig(p=1, flavor="solo", vector_len=n, element="f4"), 0, world)
    st = TrainState.fresh(w0, lr, rank=0, tau=None)
    attach_delivery_tracking(h, st)
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(side if other_stream else torch.cuda.current_stream()):
        assert h._contribute(0, v, fresh=True, activate=False)   # stash holds v, round 0 open
    bucket = h.grad_buffer()
    bucket.copy_(torch.as_tensor(g, device="cuda"))
    pend = train_step_async(st, h, bucket, all_arrive=True)
    _, res, gen = finish_step(st, h, pend)
    torch.cuda.synchronize()
    u = np.float32(0) + (v + g)
    assert gen == 0 and res.included == 1
    assert st.w.cpu().numpy().tobytes() == (w0 - np.float32(lr) * u).tobytes()
    assert _np(h.latest_result()[1].u).tobytes() == u.tobytes()
    world.close()


def test_zero_copy_refused_offer_is_kept_in_the_stash():
    """Fig. 7 with zero-copy offers: the slow rank's in-place offer for round 0
    is refused, the device copies that gradient into the stash, and round 1
    carries g_fast1 + (g_slow0 + g_slow1)."""
    from paper_1908_04207_b200 import finish_step, train_step_async
    world = EmulatedWorld(2)
    cfg = CollectiveConfig(p=2, flavor="solo", vector_len=5, element="f4")
    hs = [AllreduceHandle(cfg, r, world) for r in range(2)]
    st = [TrainState.fresh(np.zeros(5), 1.0, rank=r, tau=None) for r in range(2)]
    gf = [np.array([1, 0, 0, 0, 2], np.float32), np.array([0, 1, 0, 0, 2], np.float32)]
    gs = [np.array([0, 0, 4, 0, 2], np.float32), np.array([8, 0, 0, 0, 2], np.float32)]
    s = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    for r in range(2):
        attach_delivery_tracking(hs[r], st[r])
    res = {}
    # round 0: the fast rank alone (solo activation)
    with torch.cuda.stream(s[0]):
        hs[0].grad_buffer().copy_(torch.as_tensor(gf[0], device="cuda"))
        res[(0, 0)] = finish_step(st[0], hs[0], train_step_async(st[0], hs[0], hs[0].grad_buffer()))
    # the slow rank arrives late for round 0: refused, gradient preserved in the stash
    with torch.cuda.stream(s[1]):
        hs[1].grad_buffer().copy_(torch.as_tensor(gs[0], device="cuda"))
        res[(1, 0)] = finish_step(st[1], hs[1], train_step_async(st[1], hs[1], hs[1].grad_buffer()))
    assert res[(0, 0)][1].included == 0b01 and res[(1, 0)][1].included == 0b01
    assert not st[1].send_buf.is_null                     # g_slow0 is pending
    # round 1: both board (all-arrive), the slow rank's stash now also holds g_slow1
    p1 = {}
    for r, g in ((0, gf[1]), (1, gs[1])):
        with torch.cuda.stream(s[r]):
            hs[r].grad_buffer().copy_(torch.as_tensor(g, device="cuda"))
            p1[r] = train_step_async(st[r], hs[r], hs[r].grad_buffer(), all_arrive=True)
    for r in range(2):
        res[(r, 1)] = finish_step(st[r], hs[r], p1[r])
        assert res[(r, 1)][1].included == 0b11
    world.synchronize()          # never bare torch.cuda.synchronize() with engines resident
    # both ranks applied u0 = gf0/2 (the slow one as the latest result of its
    # step 0) and u1 = (gf1 + gs0 + gs1)/2
    want = -(gf[0] / 2 + (gf[1] + gs[0] + gs[1]) / 2)
    for r in range(2):
        assert np.allclose(st[r].w.cpu().numpy(), want)
    world.close()


@pytest.mark.parametrize("flavor", ["solo", "majority"])
def test_live_rounds_satisfy_lemma1_contracts(flavor):
    """Live (unforced) rounds under random skew checked with the reference's
    contract checker logic (verify.py:132-205): every rank returns every round
    it waits for, all ranks hold bit-identical (u, included), u equals the
    tree-ordered sum of exactly the flagged contributions / P (oracle), and
    nap = popcount(included) >= 1."""
    p, rounds, n = 4, 24, 1003
    rng = np.random.default_rng(42)
    vals = rng.standard_normal((rounds, p, n)).astype(np.float32)
    delays = rng.integers(0, 3000, size=(p, rounds))
    cfg = CollectiveConfig(p=p, flavor=flavor, vector_len=n, element="f4", seed=7)
    rec = TraceRecorder()
    res, _, world = run_allreduce(cfg, lambda r, t: vals[t, r], rounds=rounds,
                                  delay_us=lambda r, t: int(delays[r, t]), recorder=rec)
    by_gen = {}
    for row in rec.rounds:
        by_gen.setdefault(row.rnd, []).append(row)
    assert by_gen, "no rounds recorded"
    for g, rows in by_gen.items():
        ref = rows[0]
        for row in rows[1:]:
            assert row.included == ref.included
            assert _np(row.u).tobytes() == _np(ref.u).tobytes()
        fresh = [bool((ref.included >> r) & 1) for r in range(p)]
        want, inc, nap = R.allreduce_round([vals[g, r] if fresh[r] else None for r in range(p)],
                                           fresh, np.float32, n)
        assert _np(ref.u).tobytes() == want.tobytes(), g
        assert ref.nap == nap == bin(ref.included).count("1") >= 1
        if flavor == "majority":
            assert (ref.included >> initiator_for_round(7, g, p)) & 1
    for r in range(p):
        gens = [res[(r, t)].rnd for t in range(rounds)]
        assert all(g >= t for t, g in enumerate(gens)) and gens == sorted(gens)
    world.close()


def test_engine_budget_refuses_a_communicator_that_cannot_be_resident():
    """Every engine is a cooperative grid that must be co-resident with the
    running ones.  Eight emulated ranks fill the device (8 x 17 CTAs of 144 KB
    shared memory); a second collective gets an error, not a deadlock; after
    the first is released the same collective fits."""
    from paper_1908_04207_b200 import _lib
    world = EmulatedWorld(8)
    cfg = CollectiveConfig(p=8, flavor="sync", vector_len=1000, element="f4")
    h0 = [AllreduceHandle(cfg, r, world, cid=0) for r in range(8)]
    vec = np.arange(1000, dtype=np.float32)

    def sync_round(hs, t):
        out = [None] * len(hs)

        def body(r):
            out[r] = drive(hs[r].call_round(t, vec))

        th = [threading.Thread(target=body, args=(r,)) for r in range(len(hs))]
        [x.start() for x in th]
        [x.join() for x in th]
        return out

    assert all(o.nap == 8 for o in sync_round(h0, 0))
    with pytest.raises(_lib.EcError, match="no room for another engine"):
        AllreduceHandle(cfg, 0, world, cid=1)
    world.release(0)
    h1 = [AllreduceHandle(cfg, r, world, cid=1) for r in range(8)]
    assert all(o.nap == 8 for o in sync_round(h1, 0))
    world.close()


def test_torch_stream_creation_with_resident_engine():
    """Creating a torch stream while a persistent engine runs must not block
    (torch's stream pool is initialised when the world is built).  Run in a
    subprocess with a deadline: a regression fails instead of hanging."""
    import subprocess
    import sys
    script = os.path.join(os.path.dirname(__file__), "stream_late_check.py")
    res = subprocess.run([sys.executable, script], capture_output=True, text=True, timeout=180)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "stream created while the engine runs: True" in res.stdout


def test_checkpoint_resume_is_bit_exact(tmp_path):
    """save_state / load_state: two emulated ranks run 4 async
    steps (momentum, all-arrive), checkpoint, tear the world down, resume on a
    fresh world at the saved generation and run 4 more -- identical bits to 8
    uninterrupted steps, and the generations continue where they stopped."""
    from collections import deque

    from paper_1908_04207_b200 import finish_step, load_state, save_state, train_step_async
    p, n, lr, mu = 2, 70_001, 0.05, 0.9
    rng = np.random.default_rng(12)
    grads = torch.as_tensor(rng.standard_normal((8, p, n), dtype=np.float32), device="cuda")
    w0 = rng.standard_normal(n, dtype=np.float32)
    cfg = CollectiveConfig(p=p, flavor="solo", vector_len=n, element="f4")
    streams = [torch.cuda.Stream() for _ in range(p)]

    def run(world, hs, states, t_range):
        gens = {}

        def body(r):
            torch.cuda.set_device(0)
            torch.cuda.set_stream(streams[r])
            pend, out = deque(), []
            for t in t_range:
                pend.append(train_step_async(states[r], hs[r], grads[t, r], all_arrive=True))
                if len(pend) > 1:
                    out.append(finish_step(states[r], hs[r], pend.popleft())[2])
            while pend:
                out.append(finish_step(states[r], hs[r], pend.popleft())[2])
            torch.cuda.current_stream().synchronize()
            gens[r] = out

        th = [threading.Thread(target=body, args=(r,)) for r in range(p)]
        [x.start() for x in th]
        [x.join() for x in th]
        return gens

    world = EmulatedWorld(p)
    hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
    ref = [TrainState.fresh(w0, lr, rank=r, tau=None, momentum=mu) for r in range(p)]
    for r in range(p):
        attach_delivery_tracking(hs[r], ref[r])
    run(world, hs, ref, range(8))
    want = [(s.w.cpu().numpy().tobytes(), s.momentum_buf.cpu().numpy().tobytes()) for s in ref]
    world.close()

    world = EmulatedWorld(p)
    hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
    st = [TrainState.fresh(w0, lr, rank=r, tau=None, momentum=mu) for r in range(p)]
    for r in range(p):
        attach_delivery_tracking(hs[r], st[r])
    run(world, hs, st, range(4))
    for r in range(p):
        save_state(str(tmp_path / f"r{r}.egs"), st[r], hs[r])
    world.close()

    world = EmulatedWorld(p)
    hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
    st = [load_state(str(tmp_path / f"r{r}.egs"), hs[r]) for r in range(p)]
    for r in range(p):
        attach_delivery_tracking(hs[r], st[r])
        assert st[r].t == 4
    gens = run(world, hs, st, range(4, 8))
    assert gens[0] == gens[1] == [4, 5, 6, 7]
    for r in range(p):
        assert (st[r].w.cpu().numpy().tobytes(), st[r].momentum_buf.cpu().numpy().tobytes()) == want[r]
    world.close()


def test_zero_skew_trajectories_identical_across_flavors():
    """test_acceptance.py:168-185: with zero skew (every rank boards every
    round) sync, solo and majority produce the same trajectory, bit for bit,
    on every rank -- here through the async step path (progressive updates)."""
    from collections import deque

    from paper_1908_04207_b200 import finish_step, train_step_async
    p, n, lr, steps = 4, 50_003, 0.05, 4
    rng = np.random.default_rng(8)
    grads = torch.as_tensor(rng.standard_normal((steps, p, n), dtype=np.float32), device="cuda")
    w0 = rng.standard_normal(n, dtype=np.float32)
    streams = [torch.cuda.Stream() for _ in range(p)]
    finals = {}
    for flavor in ("sync", "solo", "majority"):
        world = EmulatedWorld(p)
        cfg = CollectiveConfig(p=p, flavor=flavor, vector_len=n, element="f4", seed=1234)
        hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
        st = [TrainState.fresh(w0, lr, rank=r, tau=None) for r in range(p)]
        naps = {}

        def body(r):
            torch.cuda.set_device(0)
            torch.cuda.set_stream(streams[r])
            attach_delivery_tracking(hs[r], st[r])
            pend, out = deque(), []
            for t in range(steps):
                pend.append(train_step_async(st[r], hs[r], grads[t, r], all_arrive=True))
                if len(pend) > 1:
                    out.append(finish_step(st[r], hs[r], pend.popleft())[1].nap)
            while pend:
                out.append(finish_step(st[r], hs[r], pend.popleft())[1].nap)
            torch.cuda.current_stream().synchronize()
            naps[r] = out

        th = [threading.Thread(target=body, args=(r,)) for r in range(p)]
        [x.start() for x in th]
        [x.join() for x in th]
        assert all(naps[r] == [p] * steps for r in range(p)), (flavor, naps)
        finals[flavor] = [s.w.cpu().numpy().tobytes() for s in st]
        world.close()
    w = w0.copy()
    for t in range(steps):
        u, _, _ = R.allreduce_round(list(grads[t].cpu().numpy()), [True] * p, np.float32)
        w = R.sgd_update(w, u, lr)
    for flavor, ws in finals.items():
        assert all(x == w.tobytes() for x in ws), flavor


def test_back_to_back_pinned_reads_and_concurrent_readers():
    """A host pin released in stream order (after the read's clone) must never
    clear a newer pin (advisor r1): a reader thread alternates latest_result()
    and wait_blocking() -- two pinned reads with no post between them -- on
    the handle its rank's driver also reads, while 300 sync rounds run on a
    3-slot ring.  Every u read must be its own generation's value (u = g)."""
    n = 1 << 16
    world = EmulatedWorld(2, ring_slots=3)
    cfg = CollectiveConfig(p=2, flavor="sync", vector_len=n, element="f4")
    hs = [AllreduceHandle(cfg, r, world) for r in range(2)]
    rounds = 300
    stop = threading.Event()
    bad: list = []
    errors: list = []

    def driver(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for t in range(rounds):
                    hs[r]._contribute(t, torch.full((n,), float(t), device="cuda"), True, True)
                    g, res = hs[r].wait_blocking(t)
                    if not bool((res.u == float(g)).all()):
                        bad.append(("driver", r, g))
        except BaseException as e:  # surfaced below
            errors.append(e)

    def reader():
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                while not stop.is_set():
                    g, res = hs[0].latest_result()
                    if g < 0:
                        continue
                    g2, res2 = hs[0].wait_blocking(g)
                    for gg, rr in ((g, res), (g2, res2)):
                        if not bool((rr.u == float(gg)).all()):
                            bad.append(("reader", gg))
        except BaseException as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=driver, args=(r,), daemon=True) for r in range(2)]
    rd = threading.Thread(target=reader, daemon=True)
    rd.start()
    for x in th:
        x.start()
    for x in th:
        x.join()
    stop.set()
    rd.join()
    world.close()
    assert not errors, errors[0]
    assert not bad, bad[:5]


@pytest.mark.parametrize("flavor", ["solo", "majority"])
def test_pipelined_rounds_with_two_in_flight(flavor):
    """Back-to-back rounds posted without waits (the nccl-tests pattern): the
    engine snapshots round g+1 and issues its command while round g's data
    phase runs (EcDesc::lead = 2).  Every round's mask is all-ones and the
    result is the tree-order sum; rounds publish in order."""
    from paper_1908_04207_b200.harness import _gen_times, rounds_pipelined
    p, n, k = 4, 300_001, 24
    world = EmulatedWorld(p)
    cfg = CollectiveConfig(p=p, flavor=flavor, vector_len=n, element="f4", seed=1234)
    hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
    rng = np.random.default_rng(5)
    x = rng.standard_normal((p, n)).astype(np.float32)
    for r in range(p):
        hs[r].send_buffer().copy_(torch.as_tensor(x[r], device="cuda"))
    streams = [torch.cuda.Stream() for _ in range(p)]
    world.synchronize()
    errors: list = []

    def body(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(streams[r]):
                rounds_pipelined(hs[r], 0, k)
        except BaseException as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(p)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[0]
    u, inc, _ = R.allreduce_round(list(x), [True] * p, np.float32)
    overlapped = 0
    for r in range(p):
        assert hs[r].done_generation == k - 1
        g, res = hs[r].wait_blocking(k - 1)
        assert g == k - 1 and res.included == inc and res.nap == p
        assert _np(res.u).tobytes() == u.tobytes()
        times = [_gen_times(hs[r], gg) for gg in range(k)]
        for gg in range(1, k):
            assert times[gg][3] >= times[gg - 1][3]            # published in order
            overlapped += times[gg][1] < times[gg - 1][3]      # g+1 issued before g published
    print(f"{flavor}: {overlapped} of {p * (k - 1)} rounds issued before the previous published")
    world.close()


def test_idle_park_lets_device_syncs_return():
    """A resident engine makes device-wide syncs wait for it.  After
    EC_IDLE_PARK_MS (100 ms) without work the library parks it, so a user's
    bare torch.cuda.synchronize() / empty_cache() between steps returns; the
    next step relaunches the engine and results stay bit-exact."""
    import ctypes as C

    from paper_1908_04207_b200 import finish_step, train_step_async
    from paper_1908_04207_b200._lib import call
    p, n, lr = 2, 10_007, 0.05
    world = EmulatedWorld(p)
    cfg = CollectiveConfig(p=p, flavor="solo", vector_len=n, element="f4")
    hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
    rng = np.random.default_rng(4)
    grads = rng.standard_normal((6, p, n)).astype(np.float32)
    w0 = rng.standard_normal(n).astype(np.float32)
    st = [TrainState.fresh(w0, lr, rank=r, tau=None) for r in range(p)]
    streams = [torch.cuda.Stream() for _ in range(p)]
    world.synchronize()

    def run(t0, k):
        errs = []

        def body(r):
            try:
                torch.cuda.set_device(0)
                with torch.cuda.stream(streams[r]):
                    for t in range(t0, t0 + k):
                        g = torch.as_tensor(grads[t, r], device="cuda")
                        finish_step(st[r], hs[r], train_step_async(st[r], hs[r], g,
                                                                    all_arrive=True))
                    streams[r].synchronize()
            except BaseException as e:  # surfaced below
                errs.append(e)

        th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(p)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        assert not errs, errs[0]

    run(0, 3)
    done = threading.Event()

    def user_sync():
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        done.set()

    t0 = time.time()
    th = threading.Thread(target=user_sync, daemon=True)
    th.start()
    th.join(timeout=15)
    assert done.is_set(), "device-wide sync did not return with an idle engine resident"
    waited = time.time() - t0
    parks, wakes, parked = C.c_uint64(), C.c_uint64(), C.c_int()
    call("ec_comm_idle_stats", hs[0].comm.ptr, C.byref(parks), C.byref(wakes), C.byref(parked))
    assert parks.value >= 1 and parked.value == 1
    run(3, 3)                                  # the next post relaunches the engine
    call("ec_comm_idle_stats", hs[0].comm.ptr, C.byref(parks), C.byref(wakes), C.byref(parked))
    assert wakes.value >= 1
    w = w0.copy()
    for t in range(6):
        u, _, _ = R.allreduce_round(list(grads[t]), [True] * p, np.float32)
        w = R.sgd_update(w, u, lr)
    world.synchronize()
    for r in range(p):
        assert st[r].w.cpu().numpy().tobytes() == w.tobytes()
    print(f"device sync returned after {waited * 1e3:.0f} ms (idle park)")
    world.close()


@pytest.mark.parametrize("seed", [31, 32, 33, 34])
def test_majority_quorum_waits_for_half_the_ranks(seed):
    """Opt-in majority_quorum (the north_star's "a randomly chosen initiator
    once at least half the ranks have arrived"): under skew r * 2 ms the mask
    is the arrival prefix up to max(initiator, ceil(P/2) - 1)."""
    p, n = 4, 16
    cfg = CollectiveConfig(p=p, flavor="majority", vector_len=n, element="f8", seed=seed,
                           majority_quorum=True)
    delays = np.array([[2000 * r] for r in range(p)])
    want = int(R.bench_masks("majority", delays, seed, quorum=(p + 1) // 2)[0])
    res, handles, world = run_allreduce(cfg, lambda r, t: np.full(n, 10.0 * r + t),
                                        delay_us=lambda r, t: 2000 * r)
    try:
        for r in range(p):
            assert res[(r, 0)].included == want, (seed, r, res[(r, 0)].included, want)
        vecs = [np.full(n, 10.0 * r) if (want >> r) & 1 else None for r in range(p)]
        u, _, _ = R.allreduce_round(vecs, [v is not None for v in vecs])
        assert _np(res[(0, 0)].u).tobytes() == u.tobytes()
    finally:
        world.close()


def test_nonfinite_gradient_leaves_a_pending_stash_intact():
    """eagersgd.py:145-147 (advisor r1): a non-finite gradient is refused with
    DivergenceError before it can poison a stash that still holds an earlier
    round's gradient -- the fold into a pending stash checks first and writes
    nothing; the pending rounds are unchanged and training can go on."""
    from paper_1908_04207_b200 import DivergenceError
    world = EmulatedWorld(2)
    cfg = CollectiveConfig(p=2, flavor="solo", vector_len=5, element="f4")
    hs = [AllreduceHandle(cfg, r, world) for r in range(2)]
    st = [TrainState.fresh(np.zeros(5, np.float32), 1.0, rank=r, tau=None) for r in range(2)]
    g0 = torch.tensor([1.0, 2.0, 3.0, 4.0, 5.0], device="cuda")
    drive(train_step(st[0], None, hs[0], grad=g0))               # round 0: rank 0 alone
    drive(train_step(st[1], None, hs[1], grad=g0 * 10))          # late: refused, pending
    assert st[1].send_buf.pending_rounds == [0]
    bad = torch.tensor([1.0, float("nan"), 0.0, 0.0, 0.0], device="cuda")
    with pytest.raises(DivergenceError):
        drive(train_step(st[1], None, hs[1], grad=bad))
    assert st[1].send_buf.pending_rounds == [0]
    assert _np(hs[1].send_buffer()).tolist() == [10.0, 20.0, 30.0, 40.0, 50.0]
    world.close()


@pytest.mark.parametrize("p,n", [(4, 1_000_003), (3, 77_777), (2, 2_000_001)])
def test_issued_nvlink_bytes_equal_the_bus_bytes(p, n):
    """The engine's own count of bytes it moves to/from other ranks
    (ec_comm_traffic): an all-arrive two-shot round issues exactly
    2(P-1) * S over all ranks -- each element pulled once from every other
    rank by its owner and pushed once to every other rank -- i.e. the bus
    bytes 2(P-1)/P * S per rank, nothing redundant.  One-shot rounds (small
    payloads) issue (P-1) * S pulls per rank and no pushes."""
    import ctypes as C

    from paper_1908_04207_b200._lib import call
    from paper_1908_04207_b200.harness import rounds_pipelined
    k = 5
    world = EmulatedWorld(p)
    cfg = CollectiveConfig(p=p, flavor="solo", vector_len=n, element="f4")
    hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
    streams = [torch.cuda.Stream() for _ in range(p)]

    def traffic():
        out = []
        for r in range(p):
            rx, tx = C.c_uint64(), C.c_uint64()
            call("ec_comm_traffic", hs[r].comm.ptr, r, C.byref(rx), C.byref(tx))
            out.append((rx.value, tx.value))
        return out

    world.synchronize()
    t0 = traffic()
    errs = []

    def body(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(streams[r]):
                rounds_pipelined(hs[r], 0, k)
        except BaseException as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(p)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs[0]
    world.synchronize()
    t1 = traffic()
    world.close()
    s = 4 * n
    rx = [(t1[r][0] - t0[r][0]) / k for r in range(p)]
    tx = [(t1[r][1] - t0[r][1]) / k for r in range(p)]
    oneshot = s <= (1 << 20 if p == 2 else 65536)
    if oneshot:
        assert all(x == (p - 1) * s for x in rx) and not any(tx)
    else:
        assert sum(rx) + sum(tx) == 2 * (p - 1) * s
        for r in range(p):        # per rank: the bus bytes, up to one chunk per owner
            assert abs(rx[r] + tx[r] - 2 * (p - 1) / p * s) <= 2 * (p - 1) * 16384
