"""SPEC-level entry points on the device, with SPEC's
own examples: allreduce_sync / allreduce_solo / allreduce_majority as thin
wrappers over AllreduceHandle, and resync_models(states, period)."""

import threading

import numpy as np
import pytest
import torch

from oracle import restated as R
from paper_1908_04207_b200 import (AllreduceHandle, CollectiveConfig, EmulatedWorld, TrainState,
                                   allreduce_majority, allreduce_solo, allreduce_sync,
                                   resync_models)

pytestmark = pytest.mark.gpu

SPEC_OPS = {"sync": allreduce_sync, "solo": allreduce_solo, "majority": allreduce_majority}


@pytest.mark.parametrize("flavor", ["sync", "solo", "majority"])
def test_spec_two_term_average(flavor):
    """P=2, contributions [2,4] and [4,8] -> u=[3,6], included=11
    (solo / majority with zero skew behave as sync)."""
    cfg = CollectiveConfig(p=2, flavor=flavor, vector_len=2, seed=7)
    res = SPEC_OPS[flavor](cfg, [[2.0, 4.0], [4.0, 8.0]])
    assert res.u.cpu().tolist() == [3.0, 6.0]
    assert res.included == 0b11 and res.nap == 2


@pytest.mark.parametrize("flavor", ["sync", "solo", "majority"])
def test_spec_p1_identity(flavor):
    """SPEC.md:193 (P=1 -> u = contribution, included=1) and SPEC.md:212
    (majority at P=1: initiator 0 every round, nap=1)."""
    cfg = CollectiveConfig(p=1, flavor=flavor, vector_len=5)
    x = np.array([1.5, -2.0, 0.25, 7.0, -0.0])
    res = SPEC_OPS[flavor](cfg, x)
    assert res.u.cpu().numpy().tobytes() == (np.zeros(5) + x).tobytes()   # 0 + x leaf
    assert res.included == 1 and res.nap == 1


def test_spec_p8_matches_serial_sum():
    """P=8 random vectors -> u within 1e-12 of the serial sum, and
    bit-identical to the fixed tree order (Lemma 1 safety)."""
    rng = np.random.default_rng(8)
    x = rng.standard_normal((8, 1000))
    cfg = CollectiveConfig(p=8, flavor="sync", vector_len=1000)
    res = allreduce_sync(cfg, list(x))
    u = res.u.cpu().numpy()
    serial = np.zeros(1000)
    for r in range(8):
        serial = serial + x[r]
    serial = serial / 8
    assert np.max(np.abs(u - serial) / np.maximum(np.abs(serial), 1e-300)) < 1e-12
    want, inc, nap = R.allreduce_round(list(x), [True] * 8)
    assert u.tobytes() == want.tobytes() and res.included == inc == 0xFF


def test_spec_null_contribution_has_empty_flag():
    """SPEC.md:182-184 ContributionPayload: a null payload is the zero vector
    with an empty flag mask; u still divides by P."""
    cfg = CollectiveConfig(p=3, flavor="sync", vector_len=3, element="f4")
    res = allreduce_sync(cfg, [[3.0, 3.0, 3.0], None, [6.0, 0.0, 3.0]])
    assert res.included == 0b101 and res.nap == 2
    want, _, _ = R.allreduce_round([np.full(3, 3.0, np.float32), None,
                                    np.array([6, 0, 3], np.float32)], [True, False, True],
                                   np.float32)
    assert res.u.cpu().numpy().tobytes() == want.tobytes()


def test_spec_length_mismatch():
    cfg = CollectiveConfig(p=2, flavor="solo", vector_len=4)
    with pytest.raises(ValueError):
        allreduce_solo(cfg, [[1.0, 2.0, 3.0, 4.0], [1.0, 2.0]])
    with pytest.raises(ValueError):
        allreduce_solo(cfg, [[1.0, 2.0, 3.0, 4.0]])          # one row for P=2


def test_spec_per_rank_form_over_rounds():
    """The per-rank call form: every rank of a world calls allreduce_sync with
    its own handle; consecutive calls are consecutive rounds."""
    world = EmulatedWorld(2)
    cfg = CollectiveConfig(p=2, flavor="sync", vector_len=3, element="f4")
    hs = [AllreduceHandle(cfg, r, world) for r in range(2)]
    out = {}

    def body(r):
        torch.cuda.set_device(0)
        for t in range(3):
            out[(r, t)] = allreduce_sync(cfg, np.full(3, float(10 * r + t), np.float32),
                                         handle=hs[r])

    th = [threading.Thread(target=body, args=(r,)) for r in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for t in range(3):
        for r in range(2):
            res = out[(r, t)]
            assert res.rnd == t and res.included == 0b11
            assert res.u.cpu().tolist() == [(t + 10 + t) / 2] * 3
    with pytest.raises(ValueError):
        allreduce_solo(cfg, np.zeros(3, np.float32), handle=hs[0])   # a sync handle
    world.close()


def test_resync_models_spec_examples():
    """identical w -> unchanged; P=2 [0] and [2] -> both [1];
    the states form replaces every w with the fixed-tree-order average."""
    ws = [torch.tensor([0.0], dtype=torch.float64, device="cuda"),
          torch.tensor([2.0], dtype=torch.float64, device="cuda")]
    assert resync_models(ws).cpu().tolist() == [1.0]
    same = [torch.full((4,), 0.3, dtype=torch.float64, device="cuda")] * 3
    assert resync_models(same).cpu().tolist() == same[0].cpu().tolist()
    rng = np.random.default_rng(3)
    w = rng.standard_normal((5, 257)).astype(np.float32)
    states = [TrainState.fresh(w[r], 0.1, rank=r) for r in range(5)]
    out = resync_models(states, period=2, epoch=4)
    want = R.divide_by_p(R.engine_tree_sum(list(w), np.float32), 5)
    assert out is states
    for st in states:
        assert st.w.cpu().numpy().tobytes() == want.tobytes()
    # off-period epochs leave the models alone
    states2 = [TrainState.fresh(w[r], 0.1, rank=r) for r in range(5)]
    resync_models(states2, period=2, epoch=3)
    assert states2[1].w.cpu().numpy().tobytes() == w[1].tobytes()
