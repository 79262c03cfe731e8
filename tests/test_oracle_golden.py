"""The CPU oracle (oracle/restated.py) against fixtures the REFERENCE produced
(oracle/gen_golden.py).  This pins the oracle before it is trusted as the
checker of the GPU path."""

import json
import os

import numpy as np
import pytest

from oracle import restated as R


@pytest.fixture(scope="module")
def tree(golden_dir):
    return np.load(os.path.join(golden_dir, "tree_sums.npz"))


@pytest.fixture(scope="module")
def ka(golden_dir):
    with open(os.path.join(golden_dir, "known_answers.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def proto(golden_dir):
    with open(os.path.join(golden_dir, "protocol.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8, 13])
def test_engine_sum_matches_reference_allreduce(tree, p):
    u, inc, nap = R.allreduce_round(list(tree[f"sync_in_p{p}"]), [True] * p)
    assert u.tobytes() == tree[f"sync_u_p{p}"].tobytes()
    assert inc == (1 << p) - 1 and nap == p


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8, 13])
def test_fp32_matches_reference_tree_order_sum(tree, p):
    x = tree[f"f32_in_p{p}"]
    s = R.engine_tree_sum(list(x), np.float32)
    assert s.dtype == np.float32
    assert s.tobytes() == tree[f"f32_tree_p{p}"].tobytes()
    assert R.divide_by_p(s, p).tobytes() == tree[f"f32_u_p{p}"].tobytes()


def test_fp32_tree_order_differs_from_serial_order(tree):
    x = tree["f32_in_p8"]
    serial = x[0].copy()
    for r in range(1, 8):
        serial = serial + x[r]
    assert (R.engine_tree_sum(list(x), np.float32) != serial).mean() > 0.2


@pytest.mark.parametrize("p", [1, 2, 3])
def test_signed_zero_follows_the_engine(tree, p):
    u, _, _ = R.allreduce_round(list(tree[f"negzero_in_p{p}"]), [True] * p)
    assert u.tobytes() == tree[f"negzero_u_p{p}"].tobytes()
    assert not np.signbit(u[0])


def test_integer_floor_division(tree):
    u, _, _ = R.allreduce_round(list(tree["i8_in_p4"]), [True] * 4, np.int64)
    assert u.tobytes() == tree["i8_u_p4"].tobytes()


def test_known_answers(ka):
    u, inc, _ = R.allreduce_round([np.array([2.0, 4.0]), np.array([4.0, 8.0])], [True, True])
    assert u.tolist() == ka["sync_pair"]["u"] and inc == ka["sync_pair"]["included"]
    c = np.array(ka["solo_first_arrival"]["contrib"])
    u, inc, _ = R.allreduce_round([c[0], None, None, None], [True, False, False, False])
    assert u.tolist() == ka["solo_first_arrival"]["u"] and inc == 1
    for seed, want in ka["majority_prefix"].items():
        init = R.initiator_for_round(int(seed), 0, 4)
        assert init == want["initiator"]
        vecs = [np.full(4, float(10 * r)) if r <= init else None for r in range(4)]
        u, inc, _ = R.allreduce_round(vecs, [v is not None for v in vecs])
        assert inc == want["included"] and u.tolist() == want["u"]


def test_guard_truth_table(ka):
    for tau, pending, in_prog, contributed, gen, held in ka["guard_table"]:
        assert R.hold_policy(gen, contributed, pending, in_prog, tau) == held
        thr = R.hold_from(pending, in_prog, tau)
        # the device form: held <=> gen >= threshold and not yet contributed
        assert held == (thr is not None and gen >= thr and contributed < gen)


def test_protocol_tables(proto):
    for seed, vals in proto["initiator"].items():
        got = [R.initiator_for_round(int(seed), t, p) for p in (1, 2, 3, 4, 8) for t in range(64)]
        assert got == vals
    for key, rows in proto["delayed_ranks"].items():
        seed, k = map(int, key.split(","))
        m = R.DelayModel("random_subset", 0.2, k, seed)
        assert [list(R.delayed_ranks(m, rnd, 8)) for rnd in range(32)] == rows
    models = {"none": R.DelayModel("none"), "constant": R.DelayModel("constant", 0.5),
              "linear": R.DelayModel("linear_skew", 1.0),
              "subset": R.DelayModel("random_subset", 0.2, 1, 11)}
    for name, m in models.items():
        got = [[R.inject_delay(r, t, m, 8) for r in range(8)] for t in range(16)]
        assert got == proto["inject_delay"][name]


@pytest.mark.parametrize("flavor", ["sync", "solo", "majority"])
def test_replay_reproduces_reference_run_bitwise(golden_dir, flavor):
    tr = np.load(os.path.join(golden_dir, f"c1_{flavor}.npz"))
    out = R.replay_run(tr)
    assert out["w"].tobytes() == tr["final_w"].tobytes()
    assert out["w_epoch"].tobytes() == tr["w_epoch"].tobytes()
    assert out["u"].tobytes() == tr["u_by_gen"].tobytes()
    led = {(int(r), int(g)): (None if d < 0 else int(d)) for r, g, d in tr["ledger"]}
    assert out["ledger"] == led
    # fp32 restatement stays within the north_star tolerance of the f64 reference
    o32 = R.replay_run(tr, np.float32)
    rel = np.linalg.norm(o32["w"].astype(np.float64) - tr["final_w"]) / np.linalg.norm(tr["final_w"])
    assert rel < 1e-6


def test_replay_masks_are_consistent(golden_dir):
    for flavor in ("sync", "solo", "majority"):
        tr = np.load(os.path.join(golden_dir, f"c1_{flavor}.npz"))
        p, steps = int(tr["p"]), int(tr["steps"])
        for t in range(steps):
            bits = [bool((int(tr["masks"][t]) >> r) & 1) for r in range(p)]
            assert bits == [bool(a) for a in tr["accepted"][:, t]]
            assert any(bits)                       # Lemma 1: nap >= 1
        assert (tr["observed"] >= np.arange(steps)).all()
        if flavor == "sync":
            assert (tr["masks"] == (1 << p) - 1).all()


BENCH_DELAYS = {"linear": ("linear_skew", 1.0, 1, 0), "subset": ("random_subset", 0.2, 1, 11)}


def test_bench_schedules_match_the_restated_activation_rules(golden_dir):
    """The config-2/3 schedules recorded from the reference's bench_flavor
    (oracle/gen_golden.py) equal the restated activation rules: per round the
    fresh set is every rank that arrived by its activator's arrival, nap is its
    popcount, accepted offers are exactly the mask bits, and every rank saw its
    own round's result (the cadence leaves no lag)."""
    z = np.load(os.path.join(golden_dir, "c2c3_bench.npz"))
    names = sorted({k.split("/")[0] for k in z.files})
    assert len(names) == 9
    for name in names:
        flavor, kind, pp = name.split("_")
        p, rounds, seed = (int(x) for x in z[f"{name}/meta"])
        assert pp == f"p{p}"
        k, unit, kk, dseed = BENCH_DELAYS[kind]
        delays = R.bench_delays(R.DelayModel(k, unit, kk, dseed), p, rounds)
        masks = z[f"{name}/masks"]
        assert masks.tolist() == R.bench_masks(flavor, delays, seed).tolist(), name
        assert z[f"{name}/naps"].tolist() == [int(m).bit_count() for m in masks]
        acc = z[f"{name}/accepted"]
        for t in range(rounds):
            assert [bool(a) for a in acc[:, t]] == [bool((int(masks[t]) >> r) & 1)
                                                  for r in range(p)]
        assert (z[f"{name}/observed"] == np.arange(rounds)).all()
        if flavor == "majority":
            inits = z[f"{name}/initiator"]
            assert all((int(masks[t]) >> int(inits[t])) & 1 for t in range(rounds))


def test_majority_quorum_oracle_and_config():
    """The opt-in quorum rule (north_star: the initiator activates "once at
    least half the ranks have arrived"): under linear skew the fresh set is the
    arrival prefix up to max(initiator, ceil(P/2) - 1); the default is the
    reference's rule (no counting)."""
    from paper_1908_04207_b200.collectives import CollectiveConfig
    p = 8
    delays = R.bench_delays(R.DelayModel("linear_skew", 1.0), p, 64)
    plain = R.bench_masks("majority", delays, 1234)
    quor = R.bench_masks("majority", delays, 1234, quorum=(p + 1) // 2)
    for t in range(64):
        init = R.initiator_for_round(1234, t, p)
        assert int(plain[t]) == (1 << (init + 1)) - 1
        assert int(quor[t]) == (1 << (max(init, 3) + 1)) - 1
    assert CollectiveConfig(p=4, flavor="majority", vector_len=2).majority_quorum is False
    with pytest.raises(ValueError):
        CollectiveConfig(p=4, flavor="solo", vector_len=2, majority_quorum=True)
