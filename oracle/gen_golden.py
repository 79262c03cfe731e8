"""Generate the golden fixtures under tests/golden/ by running the REFERENCE itself.

TEST INFRASTRUCTURE ONLY.  This script imports the reference package
(`eagercoll`, pure Python/numpy) from /root/reference/pkg/src, which exists only
in the build container.  It runs the reference's own public API and records its
outputs as small fixtures that travel with the repo; the GPU box never reads
/root/reference.

Usage (container only):
    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py

Fixtures written:
  tree_sums.npz      run_allreduce(sync) outputs for P in {1..8,13} (f64) and the
                     reference's dtype-generic tree_order_sum on fp32 inputs
                     (collectives.py:385-403), plus signed-zero edge cases.
  known_answers.json hand-checked answers from the reference tests
                     (test_collectives.py:30-186, test_eagersgd.py:60-121).
  protocol.json      initiator_for_round / delayed_ranks / inject_delay tables
                     (collectives.py:78-88, transport.py:101-149).
  c1_<flavor>.npz    replay traces of BASELINE config 1 (hyperplane, p=4) per
                     flavor: per-generation masks, per-(rank, step) accepted
                     offers, observed generations, gradients, weights and the
                     delivery ledger (SURVEY.md Appendix A.4 recipe).
  c2c3_bench.npz     BASELINE configs 2/3 schedules at the bench cadence
                     (harness.py:206-241): solo under linear_skew 1 ms and
                     random_subset k=1 0.2 ms seed 11 at P=2/4/8, majority
                     seed 1234 and sync at P=8, 64 rounds each -- masks,
                     accepted offers, observed generations, latencies.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = os.environ.get("EAGERCOLL_REF_SRC", "/root/reference/pkg/src")
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _import_reference():
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import eagercoll.collectives as C  # noqa: F401
    import eagercoll.eagersgd as E  # noqa: F401
    import eagercoll.harness as H  # noqa: F401
    import eagercoll.transport as T  # noqa: F401
    import eagercoll.verify as V  # noqa: F401
    return C, E, H, T, V


def gen_tree_sums(C):
    out = {}
    for p in (1, 2, 3, 4, 5, 6, 7, 8, 13):
        # same inputs as test_collectives.py:39-49
        contrib = np.random.default_rng(p).standard_normal((p, 8))
        cfg = C.CollectiveConfig(p=p, flavor="sync", vector_len=8)
        res, _, _ = C.run_allreduce(cfg, contrib)
        out[f"sync_in_p{p}"] = contrib
        out[f"sync_u_p{p}"] = res[(0, 0)].u
        # dtype-generic oracle on fp32 data (collectives.py:385-403)
        c32 = np.random.default_rng(100 + p).standard_normal((p, 1027)).astype(np.float32)
        out[f"f32_in_p{p}"] = c32
        out[f"f32_tree_p{p}"] = C.tree_order_sum([c32[r] for r in range(p)])
        out[f"f32_u_p{p}"] = C.tree_order_sum([c32[r] for r in range(p)]) / np.float32(p)
    # signed zeros through the ENGINE (snapshot adds into a zeroed accumulator,
    # schedule.py:294-301,360-367): -0.0 contributions come out +0.0.
    for p in (1, 2, 3):
        contrib = np.zeros((p, 4))
        contrib[:, 0] = -0.0
        contrib[:, 1] = 1.5
        contrib[0, 2] = -0.0
        contrib[:, 3] = -2.25
        cfg = C.CollectiveConfig(p=p, flavor="sync", vector_len=4)
        res, _, _ = C.run_allreduce(cfg, contrib)
        out[f"negzero_in_p{p}"] = contrib
        out[f"negzero_u_p{p}"] = res[(0, 0)].u
    # integer element (test_collectives.py:52-57) plus negative floor division
    contrib = np.array([[8, -4, 100, -7]] * 3 + [[1, -1, 3, 0]], dtype=np.int64)
    cfg = C.CollectiveConfig(p=4, flavor="sync", vector_len=4, element="i8")
    res, _, _ = C.run_allreduce(cfg, contrib)
    out["i8_in_p4"] = contrib
    out["i8_u_p4"] = res[(0, 0)].u
    np.savez_compressed(os.path.join(OUT, "tree_sums.npz"), **out)


def gen_known_answers(C, E, T, V):
    ka = {}
    cfg = C.CollectiveConfig(p=2, flavor="sync", vector_len=2)
    res, _, _ = C.run_allreduce(cfg, np.array([[2.0, 4.0], [4.0, 8.0]]))
    ka["sync_pair"] = {"u": res[(0, 0)].u.tolist(), "included": res[(0, 0)].included}

    # solo: first arrival defines the round (test_collectives.py:60-69)
    cfg = C.CollectiveConfig(p=4, flavor="solo", vector_len=4)
    contrib = np.random.default_rng(1).standard_normal((4, 4))
    res, _, _ = C.run_allreduce(cfg, contrib, delay_us=lambda r, t: 1000 * r)
    ka["solo_first_arrival"] = {"contrib": contrib.tolist(),
                                "included": [res[(r, 0)].included for r in range(4)],
                                "u": res[(0, 0)].u.tolist()}
    delays = {0: 3000, 1: 2000, 2: 0, 3: 1000}
    res, _, _ = C.run_allreduce(C.CollectiveConfig(p=4, flavor="solo", vector_len=2),
                                np.random.default_rng(2).standard_normal((4, 2)),
                                delay_us=lambda r, t: delays[r])
    ka["solo_earliest_not_zero"] = {"delays_us": [delays[r] for r in range(4)],
                                    "included": res[(0, 0)].included}
    # majority: round-0 mask is an arrival prefix (test_collectives.py:94-111)
    maj = {}
    for seed in (31, 32, 33, 34):
        cfg = C.CollectiveConfig(p=4, flavor="majority", vector_len=4, seed=seed)
        res, _, _ = C.run_allreduce(cfg, lambda r, t: np.full(4, float(10 * r + t)),
                                    delay_us=lambda r, t: 1000 * r)
        maj[str(seed)] = {"initiator": C.initiator_for_round(seed, 0, 4),
                          "included": res[(0, 0)].included,
                          "u": res[(0, 0)].u.tolist()}
    ka["majority_prefix"] = maj
    # late contribution refused (test_collectives.py:165-176)
    sim = T.SimTransport(2)
    hs = [C.AllreduceHandle(C.CollectiveConfig(p=2, flavor="solo", vector_len=2), r, sim)
          for r in range(2)]
    a0 = hs[0].try_contribute(0, np.array([1.0, 2.0]))
    hs[0].activate(0)
    sim.run()
    a1 = hs[1].try_contribute(0, np.array([5.0, 5.0]))
    gen, r1 = hs[1].latest_result()
    ka["late_refused"] = {"accept0": a0, "accept1": a1, "gen": gen,
                          "included": r1.included, "u": r1.u.tolist()}

    # Fig. 7 missed-bus scenario (test_eagersgd.py:60-121), values only
    gf = [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]
    gs = [[0.0, 0.0, 4.0], [8.0, 0.0, 0.0]]
    ka["fig7"] = {"gf": gf, "gs": gs, "r0_included": 1, "r1_included": 3,
                  "r0_u_times_2": gf[0],
                  "r1_u_times_2": (np.array(gf[1]) + np.array(gs[0]) + np.array(gs[1])).tolist(),
                  "staleness": {"1,0": 1, "1,1": 0, "0,0": 0}}

    # staleness guard truth table (eagersgd.py:89-110; test_eagersgd.py:213-232)
    rows = []
    for tau in (1, 2, 4):
        for pending in ([], [0], [0, 1], [3]):
            for in_prog in (None, 2, 5):
                for contributed in (-1, 0, 3, 6):
                    for gen in range(0, 9):
                        st = E.TrainState.fresh(np.zeros(2), lr=0.1, tau=tau)
                        for g in pending:
                            st.send_buf.fold(np.ones(2), g)
                        st.in_progress = in_prog
                        sim = T.SimTransport(2)
                        h = C.AllreduceHandle(C.CollectiveConfig(p=2, flavor="solo",
                                                                 vector_len=2), 0, sim)
                        h.contributed_round = contributed
                        E.staleness_guard(h, st)
                        rows.append([tau, pending, in_prog, contributed, gen,
                                     bool(h.engine.hold_policy(gen))])
    ka["guard_table"] = rows
    with open(os.path.join(OUT, "known_answers.json"), "w") as f:
        json.dump(ka, f, indent=1, sort_keys=True)


def gen_protocol_tables(C, T):
    tab = {}
    tab["initiator"] = {str(seed): [C.initiator_for_round(seed, t, p) for p in (1, 2, 3, 4, 8)
                                    for t in range(64)]
                        for seed in (0, 1, 31, 77, 1234)}
    tab["delayed_ranks"] = {}
    for seed in (0, 11, 1234):
        for k in (0, 1, 2, 4):
            m = T.DelayModel("random_subset", unit_ms=0.2, k=k, seed=seed)
            tab["delayed_ranks"][f"{seed},{k}"] = [list(T.delayed_ranks(m, rnd, 8))
                                                   for rnd in range(32)]
    models = {
        "none": T.DelayModel("none"),
        "constant": T.DelayModel("constant", unit_ms=0.5),
        "linear": T.DelayModel("linear_skew", unit_ms=1.0),
        "subset": T.DelayModel("random_subset", unit_ms=0.2, k=1, seed=11),
    }
    tab["inject_delay"] = {name: [[T.inject_delay(r, t, m, 8) for r in range(8)]
                                  for t in range(16)] for name, m in models.items()}
    with open(os.path.join(OUT, "protocol.json"), "w") as f:
        json.dump(tab, f, sort_keys=True)


def c1_config(H, T, flavor: str, epochs: int = 48):
    """BASELINE.json config 1 / SURVEY.md §8(d)1: hyperplane, p=4."""
    return H.RunConfig(mode="train", flavors=(flavor,), p=4, epochs=epochs,
                       steps_per_epoch=4, dim=64, n_samples=4096, batch_per_rank=128,
                       lr=0.05, tau=8, resync_period=8,
                       delay=T.DelayModel("random_subset", unit_ms=0.2, k=1, seed=11),
                       link_latency_us=10, seed=1234, data_seed=99)


def gen_c1_traces(C, E, H, T):
    """Replay traces: wrap train_step to capture the
    generation each rank observed; everything else comes from the recorder."""
    for flavor in ("sync", "solo", "majority"):
        cfg = c1_config(H, T, flavor)
        orig = E.train_step
        obs = {}
        accepted = {}

        def wrapped(state, batch, handle, _orig=orig):
            t = state.t
            before = handle.contributed_round
            loss, res, gen = yield from _orig(state, batch, handle)
            obs[(state.rank, t)] = gen
            accepted[(state.rank, t)] = handle.contributed_round == t and before != t
            return loss, res, gen

        E.train_step = wrapped
        try:
            rep = H.run_training(cfg)
        finally:
            E.train_step = orig
        rec = rep.recorders[flavor]
        p = cfg.p
        steps = cfg.epochs * cfg.steps_per_epoch
        dim = cfg.dim
        masks = np.zeros(steps, dtype=np.int64)
        for r in rec.rounds:
            masks[r.rnd] = r.included
        grads = np.zeros((p, steps, dim))
        w_before = np.zeros((p, steps, dim))
        losses = np.zeros((p, steps))
        observed = np.zeros((p, steps), dtype=np.int64)
        acc = np.zeros((p, steps), dtype=np.int8)
        for r in range(p):
            for t in range(steps):
                grads[r, t] = rec.gradients[(r, t)]
                w_before[r, t] = rec.weights[(r, t)]
                losses[r, t] = rec.losses[(r, t)]
                observed[r, t] = obs[(r, t)]
                acc[r, t] = accepted[(r, t)]
        # every accepted offer is a fresh bit of that generation and vice versa
        for r in range(p):
            for t in range(steps):
                assert bool(acc[r, t]) == bool((masks[t] >> r) & 1), (flavor, r, t)
        final_w = np.stack([rep.weights[(flavor, r)] for r in range(p)])
        ledger = np.array([(r, g, -1 if d is None else d)
                           for r, g, d in rep.ledgers[flavor].entries()], dtype=np.int64)
        u_by_gen = np.zeros((steps, dim))
        for r in rec.rounds:
            if r.rank == 0:
                u_by_gen[r.rnd] = r.u
        np.savez_compressed(
            os.path.join(OUT, f"c1_{flavor}.npz"),
            p=p, steps=steps, epochs=cfg.epochs, steps_per_epoch=cfg.steps_per_epoch,
            dim=dim, lr=cfg.lr, tau=cfg.tau, resync_period=cfg.resync_period,
            seed=cfg.seed, masks=masks, accepted=acc, observed=observed,
            grads=grads, w_epoch=w_before[:, ::cfg.steps_per_epoch], losses=losses, final_w=final_w,
            ledger=ledger, u_by_gen=u_by_gen,
            w0=w_before[0, 0],  # w_epoch[r, e] = w at the first step of epoch e
            sim_time_us=rep.sim_time_us[flavor],
            final_val=rep.final_val(flavor))
        print(f"c1 {flavor}: nap hist",
              np.bincount([int(m).bit_count() for m in masks]).tolist(),
              "obs-lag hist", np.bincount((observed - np.arange(steps)).ravel()).tolist())


# BASELINE configs 2/3 at the bench cadence: the reference's
# own bench_flavor (harness.py:206-241) with the configs' injected delays.
# Participation is data-independent, so a small
# vector_len records the schedule that the GPU replays at ResNet-50 size.
BENCH_TRACES = {
    # name: (flavor, p, delay kind, unit_ms, k, delay seed)
    "solo_linear_p2": ("solo", 2, "linear_skew", 1.0, 1, 0),
    "solo_linear_p4": ("solo", 4, "linear_skew", 1.0, 1, 0),
    "solo_linear_p8": ("solo", 8, "linear_skew", 1.0, 1, 0),
    "solo_subset_p2": ("solo", 2, "random_subset", 0.2, 1, 11),
    "solo_subset_p4": ("solo", 4, "random_subset", 0.2, 1, 11),
    "solo_subset_p8": ("solo", 8, "random_subset", 0.2, 1, 11),
    "majority_linear_p8": ("majority", 8, "linear_skew", 1.0, 1, 0),
    "majority_subset_p8": ("majority", 8, "random_subset", 0.2, 1, 11),
    "sync_linear_p8": ("sync", 8, "linear_skew", 1.0, 1, 0),
}


def gen_bench_traces(C, H, T, rounds: int = 64):
    """Per trace: per-generation inclusion masks, per-(rank, round) accepted
    offers (a fresh snapshot of that round) and the generation each rank's
    call_round observed (collectives.py:334-345), from the reference run."""
    out = {}
    orig = C.AllreduceHandle.call_round
    for name, (flavor, p, kind, unit, k, dseed) in BENCH_TRACES.items():
        cfg = H.RunConfig(mode="bench", flavors=(flavor,), p=p, rounds=rounds, vector_len=8,
                          delay=T.DelayModel(kind, unit_ms=unit, k=k, seed=dseed),
                          link_latency_us=10, seed=1234)
        observed = np.full((p, rounds), -1, dtype=np.int64)

        def wrapped(self, t, vec, _orig=orig, _obs=observed):
            res = yield from _orig(self, t, vec)
            _obs[self.rank, t] = res.rnd
            return res

        C.AllreduceHandle.call_round = wrapped
        try:
            records, rec, _ = H.bench_flavor(cfg, flavor)
        finally:
            C.AllreduceHandle.call_round = orig
        masks = np.zeros(rounds, dtype=np.int64)
        naps = np.zeros(rounds, dtype=np.int64)
        for r in rec.rounds:
            masks[r.rnd] = r.included
            naps[r.rnd] = r.nap
        acc = np.zeros((p, rounds), dtype=np.int8)
        for sn in rec.snapshots:
            if sn.fresh:
                acc[sn.rank, sn.rnd] = 1
        assert (observed >= 0).all(), name
        for t in range(rounds):
            for r in range(p):
                assert bool(acc[r, t]) == bool((masks[t] >> r) & 1), (name, r, t)
        inits = np.array([C.initiator_for_round(cfg.seed, t, p) if flavor == "majority" else -1
                          for t in range(rounds)], dtype=np.int64)
        lat = np.zeros((p, rounds), dtype=np.int64)
        for b in records:
            lat[b.rank, b.round] = b.latency_us
        out[f"{name}/masks"] = masks
        out[f"{name}/naps"] = naps
        out[f"{name}/accepted"] = acc
        out[f"{name}/observed"] = observed
        out[f"{name}/initiator"] = inits
        out[f"{name}/latency_us"] = lat
        out[f"{name}/meta"] = np.array([p, rounds, cfg.seed], dtype=np.int64)
        print(f"bench {name}: nap hist {np.bincount(naps).tolist()}, "
              f"max obs lag {int((observed - np.arange(rounds)).max())}")
    np.savez_compressed(os.path.join(OUT, "c2c3_bench.npz"), **out)


def main():
    C, E, H, T, V = _import_reference()
    os.makedirs(OUT, exist_ok=True)
    gen_tree_sums(C)
    gen_known_answers(C, E, T, V)
    gen_protocol_tables(C, T)
    gen_c1_traces(C, E, H, T)
    gen_bench_traces(C, H, T)
    print("golden fixtures written to", os.path.normpath(OUT))


if __name__ == "__main__":
    main()
