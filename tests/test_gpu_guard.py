"""The staleness guard on every step path (eagersgd.py:89-110).

Acceptance criterion 7 of the reference (pkg/tests/test_acceptance.py:200-218):
tau = 1, P = 4, solo, 25 epochs x 4 steps, one rank per round delayed by the
seeded random_subset model (0.5 ms, k = 1, seed 5): every gradient is
delivered exactly once and at most one round late.  Here it runs live on the
device through the product's fast path (train_step_async / finish_step, the
gradient in the registered bucket, the delay a device spin on the rank's own
stream), so the guard must be enforced by the engine without a host round trip.
"""

import threading

import numpy as np
import pytest
import torch

from oracle import restated as R
from paper_1908_04207_b200 import (AllreduceHandle, CollectiveConfig, EmulatedWorld, TrainState,
                                   attach_delivery_tracking, finish_step, staleness_guard,
                                   train_step_async)
from paper_1908_04207_b200.trace import DeliveryLedger
from paper_1908_04207_b200.transport import device_delay

pytestmark = pytest.mark.gpu


def _run(tau, lag, rounds=100, p=4, unit_ms=0.5, dim=8, seed=5, time_scale=1.0):
    model = R.DelayModel("random_subset", unit_ms=unit_ms, k=1, seed=seed)
    delays = R.bench_delays(model, p, rounds)
    world = EmulatedWorld(p)
    cfg = CollectiveConfig(p=p, flavor="solo", vector_len=dim, element="f4", seed=21)
    hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
    rng = np.random.default_rng(22)
    grads = rng.standard_normal((p, rounds, dim)).astype(np.float32)
    states = [TrainState.fresh(np.zeros(dim, np.float32), 0.02, rank=r, tau=tau)
              for r in range(p)]
    ledger = DeliveryLedger()
    streams = [torch.cuda.Stream() for _ in range(p)]
    torch.cuda.synchronize()
    for r in range(p):
        staleness_guard(hs[r], states[r])
        attach_delivery_tracking(hs[r], states[r], ledger)
    naps: dict = {}
    errors: list = []
    go = threading.Barrier(p)

    def body(r):
        try:
            torch.cuda.set_device(0)
            h, st = hs[r], states[r]
            g_dev = torch.as_tensor(grads[r], device="cuda")
            pend = []
            with torch.cuda.stream(streams[r]):
                go.wait()
                for t in range(rounds):
                    d = int(delays[r, t] * time_scale)
                    if d:
                        device_delay(d)           # the rank's slow gradient, on its stream
                    ledger.generated(r, t)
                    h.grad_buffer().copy_(g_dev[t])
                    pend.append(train_step_async(st, h, h.grad_buffer()))
                    while len(pend) > lag:
                        _, res, gen = finish_step(st, h, pend.pop(0))
                        naps[(r, gen)] = res.nap
                while pend:
                    _, res, gen = finish_step(st, h, pend.pop(0))
                    naps[(r, gen)] = res.nap
                streams[r].synchronize()
        except BaseException as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(p)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    world.close()
    if errors:
        raise errors[0]
    return ledger, naps


@pytest.mark.parametrize("lag", [0, 2])
def test_criterion7_tau1_exactly_once_through_async_steps(lag):
    rounds, p = 100, 4
    ledger, naps = _run(tau=1, lag=lag, rounds=rounds, p=p)
    violations = ledger.audit(tau=1, allow_pending_after=rounds - 2)
    delivered = sum(1 for _, _, d in ledger.entries() if d is not None)
    assert not violations, violations[:10]
    assert ledger.max_staleness() <= 1
    assert delivered >= (rounds - 2) * p
    # the laggards really were late: some gradients travelled one round
    assert any(d is not None and d - g == 1 for _, g, d in ledger.entries())


def test_without_guard_the_tau_contract_breaks():
    """Control: the same schedule with the guard off (tau=None) and a longer
    delay: some laggard's gradient is delivered more than one round late or
    not at all within the run, i.e. the audit that passes above fails here."""
    rounds, p = 40, 4
    ledger, _ = _run(tau=None, lag=0, rounds=rounds, p=p, unit_ms=1.0)
    assert not [v for v in ledger.audit() if v[0] not in ("undelivered", "staleness")]
    assert ledger.audit(tau=1, allow_pending_after=rounds - 2)


@pytest.mark.parametrize("flavor,p,n", [("solo", 3, 200_003), ("majority", 3, 200_003),
                                        ("solo", 5, 9_001)])
def test_live_async_steps_under_random_skew_match_the_restatement(flavor, p, n):
    """Protocol stress in place of a race checker (compute-sanitizer is closed
    on this pool): P ranks issue async steps (lag 2, guard tau=2) with random
    device-side delays, so offers race snapshots, refused offers fold into the
    stash and zero-copy late offers are preserved.  Afterwards everything the
    device decided is taken as the schedule -- the masks it logged, the
    generation each step applied -- and the restatement recomputes every
    stash, every u and every rank's weights from it: bit-exact, ledger clean."""
    import ctypes as C

    from paper_1908_04207_b200._lib import call
    rounds, lr, tau = 40, 0.05, 2
    rng = np.random.default_rng(p * 100 + n % 97)
    spins = rng.integers(0, 400, size=(p, rounds))
    grads = rng.standard_normal((p, rounds, n)).astype(np.float32)
    w0 = rng.standard_normal(n).astype(np.float32)
    world = EmulatedWorld(p)
    cfg = CollectiveConfig(p=p, flavor=flavor, vector_len=n, element="f4", seed=3)
    hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
    states = [TrainState.fresh(w0, lr, rank=r, tau=tau) for r in range(p)]
    ledger = DeliveryLedger()
    streams = [torch.cuda.Stream() for _ in range(p)]
    torch.cuda.synchronize()
    for r in range(p):
        staleness_guard(hs[r], states[r])
        attach_delivery_tracking(hs[r], states[r], ledger)
    obs = np.zeros((p, rounds), np.int64)
    errors: list = []
    go = threading.Barrier(p)

    def body(r):
        try:
            torch.cuda.set_device(0)
            h, st = hs[r], states[r]
            gd = torch.as_tensor(grads[r], device="cuda")
            pend = []
            with torch.cuda.stream(streams[r]):
                go.wait()
                for t in range(rounds):
                    device_delay(int(spins[r, t]))
                    if t % 3:
                        h.grad_buffer().copy_(gd[t])
                        g = h.grad_buffer()
                    else:
                        g = gd[t]
                    ledger.generated(r, t)
                    pend.append(train_step_async(st, h, g))
                    while len(pend) > 2:
                        pt = pend[0].t
                        obs[r, pt] = finish_step(st, h, pend.pop(0))[2]
                while pend:
                    pt = pend[0].t
                    obs[r, pt] = finish_step(st, h, pend.pop(0))[2]
                streams[r].synchronize()
        except BaseException as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(p)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors[0]
    world.synchronize()
    last = int(obs.max())
    masks = []
    for g in range(last + 1):
        m, hm, nap = C.c_uint64(), C.c_uint64(), C.c_int()
        call("ec_gen_info", hs[0].comm.ptr, 0, g, C.byref(m), C.byref(hm), C.byref(nap))
        for r in range(1, p):            # Lemma 1: the same mask at every rank
            m2, hm2, nap2 = C.c_uint64(), C.c_uint64(), C.c_int()
            call("ec_gen_info", hs[r].comm.ptr, r, g, C.byref(m2), C.byref(hm2), C.byref(nap2))
            assert (m2.value, hm2.value) == (m.value, hm.value), (g, r)
        assert nap.value == bin(m.value).count("1") >= 1
        masks.append(m.value)
    ws = [st.w.cpu().numpy() for st in states]
    world.close()
    # the device's schedule, restated: an offer of step t boarded round t iff
    # bit r of mask[t] (a fresh snapshot of t consumes the stash)
    acc = np.array([[(masks[t] >> r) & 1 if t <= last else 0 for t in range(rounds)]
                    for r in range(p)], bool)
    contribs, led = R.replay_stashes(grads, acc, np.float32)
    u = [R.allreduce_round(contribs[t], [c is not None for c in contribs[t]], np.float32, n)[0]
         for t in range(last + 1)]
    for r in range(p):
        w = w0.copy()
        for t in range(rounds):
            assert obs[r, t] >= t
            w = R.sgd_update(w, u[int(obs[r, t])], lr)
        assert ws[r].tobytes() == w.tobytes(), (flavor, r)
    assert {k: v for k, v in led.items() if v is not None} == \
        {k: v for k, v in ledger.as_dict().items() if v is not None}
    assert not ledger.audit(tau=tau, allow_pending_after=rounds - 1 - tau)
