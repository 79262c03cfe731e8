"""Parity at the sizes the numbers are measured on (BASELINE configs 2/3).

* The bench's N=1 hot path exactly as bench.py runs it -- async steps with two
  in flight, the gradient in the registered bucket (zero-copy offer) and, as
  the pipelined e2e alternates, from a second buffer (folded offer) -- at
  N = 25,559,081: weights and the last reduced gradient bit-exact against the
  oracle restatement.
* The reference's own config-2/3 schedules (tests/golden/c2c3_bench.npz,
  recorded from its bench_flavor by oracle/gen_golden.py: solo under
  linear_skew 1 ms and random_subset k=1 0.2 ms seed 11 at P=2/4/8, majority
  seed 1234 and sync at P=8) replayed with forced masks on an emulated world
  at N = 25,559,081 fp32: masks, nap and accepted offers bit-exact, every
  observed result slot bit-exact against the fp32 restatement, and within
  1e-6 normwise of the same sum in f64 (north_star tolerance).
"""

import os

import numpy as np
import pytest
import torch

from oracle import restated as R
from paper_1908_04207_b200 import (AllreduceHandle, CollectiveConfig, EmulatedWorld, TrainState,
                                   finish_step, train_step_async)
from paper_1908_04207_b200.replay import replay_bench

pytestmark = pytest.mark.gpu

RESNET50_N = 25_559_081
LR = 0.05


def test_bench_direct_step_resnet50_bit_exact():
    """bench.py's N=1 step path at full size: lag 2, zero-copy from the bucket
    and folded offers from a second buffer, 6 steps; w and the last u
    bit-exact vs the restatement (eagersgd.py:55-57,165; collectives.py:254)."""
    n = RESNET50_N
    gen = torch.Generator(device="cuda").manual_seed(1234)
    w0 = torch.randn(n, device="cuda", generator=gen) * 0.01
    world = EmulatedWorld(1, 0)
    h = AllreduceHandle(CollectiveConfig(p=1, flavor="solo", vector_len=n, element="f4"), 0,
                        world)
    st = TrainState.fresh(w0, LR, rank=0, tau=None)
    bucket = h.grad_buffer()
    other = torch.empty_like(bucket)
    w = w0.cpu().numpy()
    pend, gens = [], []
    last_u = None
    for t in range(6):
        g = torch.randn(n, device="cuda", generator=gen)
        src = bucket if t % 3 != 2 else other      # every third step a folded offer
        src.copy_(g)
        pend.append(train_step_async(st, h, src))
        if len(pend) > 2:
            gens.append(finish_step(st, h, pend.pop(0))[2])
        u = R.divide_by_p(R.engine_tree_sum([g.cpu().numpy()], np.float32), 1)
        w = R.sgd_update(w, u, LR)
        last_u = u
    while pend:
        gens.append(finish_step(st, h, pend.pop(0))[2])
    torch.cuda.synchronize()
    assert gens == list(range(6))
    assert st.w.cpu().numpy().tobytes() == w.tobytes()
    assert h._slot(5).cpu().numpy().tobytes() == last_u.tobytes()
    world.close()


def _bench(golden_dir):
    return np.load(os.path.join(golden_dir, "c2c3_bench.npz"))


TRACES = ["solo_linear_p2", "solo_linear_p4", "solo_linear_p8", "solo_subset_p2",
          "solo_subset_p4", "solo_subset_p8", "majority_linear_p8", "majority_subset_p8",
          "sync_linear_p8"]


@pytest.mark.parametrize("name", TRACES)
def test_replay_reference_bench_schedule_at_resnet50_size(golden_dir, name):
    z = _bench(golden_dir)
    flavor = name.split("_")[0]
    p, rounds, seed = (int(x) for x in z[f"{name}/meta"])
    masks = z[f"{name}/masks"]
    acc = z[f"{name}/accepted"]
    obs = z[f"{name}/observed"]
    n = RESNET50_N
    # rank r's constant bench contribution (harness.py:222 np.full(.., r+1)),
    # here a seeded fp32 normal vector per rank
    host = [np.random.default_rng([seed, r]).standard_normal(n, dtype=np.float32)
            for r in range(p)]
    vecs = [torch.as_tensor(x, device="cuda") for x in host]
    expected: dict = {}
    sub = slice(0, n, 97)    # strided sample for the f64 tolerance check

    def expect(mask: int) -> torch.Tensor:
        if mask not in expected:
            contribs = [host[r] if (mask >> r) & 1 else None for r in range(p)]
            u32, inc, nap = R.allreduce_round(contribs, [c is not None for c in contribs],
                                              np.float32, n)
            assert inc == mask
            # north_star tolerance: the fp32 result vs the same sum in f64
            c64 = [None if c is None else c[sub].astype(np.float64) for c in contribs]
            u64 = R.divide_by_p(R.engine_tree_sum(c64, np.float64, len(range(0, n, 97))), p)
            rel = np.linalg.norm(u32[sub] - u64) / max(np.linalg.norm(u64), 1e-300)
            assert rel < 1e-6, (name, mask, rel)
            expected[mask] = torch.as_tensor(u32, device="cuda")
        return expected[mask]

    for m in set(int(x) for x in masks):
        expect(m)

    def verify(r, g, mask, slot):
        return mask == int(masks[g]) and torch.equal(slot, expected[mask])

    out = replay_bench(flavor, masks, acc, obs, vecs, element="f4", seed=seed, verify=verify)
    for r in range(p):
        o = out[r]
        assert o["accepted"] == [bool(a) for a in acc[r]], (name, r)
        assert o["masks_seen"] == [int(masks[g]) for g in obs[r]], (name, r)
        assert all(o["verified"]), (name, r, o["verified"].index(False))
