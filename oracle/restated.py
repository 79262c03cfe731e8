"""numpy restatement of the reference partial-collective / eager-SGD path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites the
reference file:line it restates; paths are relative to
/root/reference/pkg/src/eagercoll/.  Dtype-generic: with float64 inputs the
results are bit-identical to the reference engine (pinned by
tests/test_oracle_golden.py against fixtures produced by the reference
itself, oracle/gen_golden.py); with float32 inputs they define the product's
fixed-order fp32 semantics.

Parity status: PINNED (f64 bit-exact vs the reference's own run_allreduce /
run_training outputs; f32 bit-exact vs the reference's dtype-generic
tree_order_sum).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SOLO, MAJORITY, SYNC = "solo", "majority", "sync"


# ---------------------------------------------------------------------------
# reduction order (collectives.py:91-96, 385-403; schedule.py:294-301,360-380)


def ceil_log2(p: int) -> int:
    """collectives.py:91-92"""
    return 0 if p <= 1 else (p - 1).bit_length()


def floor_pow2(p: int) -> int:
    """collectives.py:95-96"""
    return 1 << (p.bit_length() - 1)


def snapshot_leaf(x, like):
    """One rank's term as the ENGINE forms it.

    The snapshot adds the send buffer into an accumulator that replication
    zeroed (schedule.py:294-301 zeroes non-preserved buffers, collectives.py:150
    snap_sum = np.add(acc, send)), so a contribution enters the sum as
    (+0.0 + x): -0.0 becomes +0.0.  A rank that never contributed snapshots
    its zeroed send buffer (schedule.py:373-380), i.e. +0.0 everywhere.
    """
    z = np.zeros_like(like)
    if x is None:
        return z
    return z + np.asarray(x, dtype=like.dtype)


def engine_tree_sum(contribs, dtype=np.float64, n=None):
    """Sum of P snapshots in the butterfly's association.

    Leaves b < p2 are v_b (+ v_{b+p2}), then adjacent pairs combine
    (collectives.py:394-403); the butterfly produces exactly this order at
    every rank (collectives.py:15-20, test_collectives.py:39-49).
    `contribs[r]` is rank r's contributed vector or None for a null snapshot.
    """
    p = len(contribs)
    if p == 0:
        raise ValueError("no vectors")
    like = next((np.asarray(c, dtype=dtype) for c in contribs if c is not None), None)
    if like is None:
        if n is None:
            raise ValueError("need the vector length: at least one non-null contribution")
        like = np.zeros(n, dtype=dtype)
    c = [snapshot_leaf(v, like) for v in contribs]
    p2 = floor_pow2(p)
    leaves = []
    for b in range(p2):
        v = c[b].copy()
        if b + p2 < p:
            v = v + c[b + p2]
        leaves.append(v)
    while len(leaves) > 1:
        leaves = [leaves[i] + leaves[i + 1] for i in range(0, len(leaves), 2)]
    return leaves[0]


def divide_by_p(s, p: int):
    """collectives.py:254-260: always divides by the world size, never by nap;
    floats use true division, integers floor division."""
    if np.issubdtype(s.dtype, np.integer):
        return s // p
    return s / s.dtype.type(p)


def allreduce_round(contribs, fresh, dtype=np.float64, n=None):
    """One generation: (u, included, nap) for the given snapshots.

    `fresh[r]` is the rank's own flag bit (collectives.py:301-306); the mask is
    the OR of the flags (collectives.py:61-67,152-153) and nap its popcount
    (collectives.py:260).
    """
    p = len(contribs)
    s = engine_tree_sum(contribs, dtype, n)
    included = 0
    for r in range(p):
        if fresh[r]:
            included |= 1 << r
    return divide_by_p(s, p), included, included.bit_count()


# ---------------------------------------------------------------------------
# activation rules (collectives.py:78-88, 311-317)


def initiator_for_round(seed: int, t: int, p: int) -> int:
    """collectives.py:78-88: Philox4x64 keyed by the seed, round as counter."""
    if p < 1:
        raise ValueError("p must be >= 1")
    bitgen = np.random.Philox(key=np.uint64(seed), counter=[np.uint64(t), 0, 0, 0])
    return int(np.random.Generator(bitgen).integers(0, p))


def may_activate(flavor: str, rank: int, seed: int, t: int, p: int) -> bool:
    """collectives.py:311-317: majority activates only at the designated rank."""
    return flavor != MAJORITY or rank == initiator_for_round(seed, t, p)


# ---------------------------------------------------------------------------
# imbalance injection (transport.py:98-149, 504-506; harness.py:198-212)


DELAY_KINDS = ("none", "constant", "linear_skew", "random_subset")


@dataclass(frozen=True)
class DelayModel:
    """transport.py:101-124"""
    kind: str = "none"
    unit_ms: float = 0.0
    k: int = 1
    seed: int = 0


def delayed_ranks(model: DelayModel, rnd: int, p: int) -> tuple:
    """transport.py:127-134"""
    k = min(model.k, p)
    rng = np.random.default_rng([model.seed, rnd])
    return tuple(int(r) for r in rng.choice(p, size=k, replace=False))


def inject_delay(rank: int, rnd: int, model: DelayModel, p: int) -> int:
    """transport.py:137-149 (microseconds)"""
    if model.kind == "none":
        return 0
    if model.kind == "constant":
        return int(round(model.unit_ms * 1000))
    if model.kind == "linear_skew":
        return int(round((rank + 1) * model.unit_ms * 1000))
    if model.kind == "random_subset":
        if rank in delayed_ranks(model, rnd, p):
            return int(round(model.unit_ms * 1000))
        return 0
    raise ValueError(model.kind)


def bench_period_us(delays: np.ndarray, p: int, link_latency_us: int) -> int:
    """harness.py:211-212: round cadence of the latency bench."""
    hops = max(1, math.ceil(math.log2(p)))
    return int(delays.max()) + (3 * hops + 4) * link_latency_us + 1000


def bench_delays(model: DelayModel, p: int, rounds: int) -> np.ndarray:
    """harness.py:198-203: [p, rounds] injected microseconds."""
    d = np.zeros((p, rounds), dtype=np.int64)
    for t in range(rounds):
        for r in range(p):
            d[r, t] = inject_delay(r, t, model, p)
    return d


def bench_masks(flavor: str, delays: np.ndarray, seed: int, quorum: int = 0) -> np.ndarray:
    """Inclusion mask of every bench round (harness.py:206-241 with the
    activation rules of collectives.py:146-153, 311-317).

    The bench cadence gives every round its own slot, so rank r arrives at
    offset delays[r, t] and the round starts when its activator arrives: the
    first arrival (solo), the designated initiator (majority; with the opt-in
    quorum rule, not before the quorum-th arrival) or the last arrival (sync).  A rank is fresh iff it arrived no later than that moment
    (the injected offsets differ by >= 200 us, far above the few link hops the
    activation takes); everyone else's slot is snapshotted null."""
    p, rounds = delays.shape
    out = np.zeros(rounds, dtype=np.int64)
    for t in range(rounds):
        arr = delays[:, t]
        if flavor == SOLO:
            a = arr.min()
        elif flavor == MAJORITY:
            a = arr[initiator_for_round(seed, t, p)]
            if quorum:   # the opt-in quorum rule: also wait for the quorum-th arrival
                a = max(a, np.sort(arr)[quorum - 1])
        else:
            a = arr.max()
        out[t] = sum(1 << r for r in range(p) if arr[r] <= a)
    return out


# ---------------------------------------------------------------------------
# eager-SGD (eagersgd.py)


@dataclass
class GradientBuffer:
    """eagersgd.py:40-61 (dtype follows the inputs here; the reference's is f64)."""
    data: np.ndarray
    pending_rounds: list = field(default_factory=list)

    @classmethod
    def null(cls, dim: int, dtype=np.float64):
        return cls(data=np.zeros(dim, dtype=dtype))

    def fold(self, grad, rnd: int) -> None:
        self.data = self.data + grad          # eagersgd.py:56
        self.pending_rounds.append(rnd)

    def reset(self) -> None:
        self.data = np.zeros_like(self.data)  # eagersgd.py:60
        self.pending_rounds = []


def sgd_update(w, u, lr: float):
    """eagersgd.py:165: w - lr*u with numpy's weak-scalar promotion (lr is cast
    to the array dtype, two roundings, no fused multiply-add)."""
    return w - lr * u


def momentum_update(w, buf, u, lr: float, mu: float):
    """Opt-in extension (the reference is plain SGD):
    buf = mu*buf + u ; w = w - lr*buf (torch.optim.SGD, dampening 0)."""
    buf = mu * buf + u
    return w - lr * buf, buf


def hold_policy(gen: int, contributed_round: int, pending, in_progress, tau):
    """eagersgd.py:102-108 (tau=None disables the guard, eagersgd.py:97-100)."""
    if tau is None:
        return False
    if contributed_round >= gen:
        return False
    ages = list(pending)
    if in_progress is not None:
        ages.append(in_progress)
    return any(g + tau <= gen for g in ages)


def hold_from(pending, in_progress, tau):
    """The same policy as one threshold: generations >= this are held until the
    rank contributes (min age + tau); None when nothing can be held."""
    if tau is None:
        return None
    ages = list(pending) + ([] if in_progress is None else [in_progress])
    return None if not ages else min(ages) + tau


def replay_stashes(grads, accepted, dtype):
    """Per-rank stash evolution under forced offers.

    grads[r, t] is rank r's gradient of step t, accepted[r, t] whether its offer
    at step t boarded generation t (a fresh bit of mask[t]).  Folding and the
    offer happen under the engine lock (eagersgd.py:156-163); a fresh snapshot
    of generation t consumes the stash and delivers every pending gradient at
    t (eagersgd.py:117-124).  Returns (contribs[t][r] or None, ledger dict).
    """
    p, steps = accepted.shape
    contribs = [[None] * p for _ in range(steps)]
    ledger = {}
    for r in range(p):
        gb = GradientBuffer.null(grads.shape[-1], dtype)
        for t in range(steps):
            gb.fold(grads[r, t].astype(dtype), t)
            ledger[(r, t)] = None
            if accepted[r, t]:
                contribs[t][r] = gb.data.copy()
                for g in gb.pending_rounds:
                    ledger[(r, g)] = t
                gb.reset()
    return contribs, ledger


def replay_run(trace, dtype=np.float64, lr=None):
    """Replays a recorded eager-SGD run (oracle/gen_golden.py c1_* traces).

    The schedule-level events (accepted offers, observed generations) are
    inputs; this computes every generation's u, every rank's weights and the
    delivery ledger.  Mirrors training_process (eagersgd.py:187-226):
    per step w = w - lr * u_{observed}; at epoch ends with
    (epoch+1) % resync_period == 0 a sync allreduce averages w
    (eagersgd.py:177-184, 222-224).
    """
    p = int(trace["p"])
    steps = int(trace["steps"])
    epochs = int(trace["epochs"])
    spe = int(trace["steps_per_epoch"])
    lr = float(trace["lr"]) if lr is None else lr
    period = int(trace["resync_period"])
    grads = np.asarray(trace["grads"])
    accepted = np.asarray(trace["accepted"]).astype(bool)
    observed = np.asarray(trace["observed"])
    contribs, ledger = replay_stashes(grads, accepted, dtype)
    u = [allreduce_round(contribs[t], [c is not None for c in contribs[t]], dtype,
                         grads.shape[-1])[0] for t in range(steps)]
    w = [np.asarray(trace["w0"]).astype(dtype).copy() for _ in range(p)]
    w_epoch = np.zeros((p, epochs, grads.shape[-1]), dtype=dtype)
    for e in range(epochs):
        for r in range(p):
            w_epoch[r, e] = w[r]
        for s in range(spe):
            t = e * spe + s
            for r in range(p):
                w[r] = sgd_update(w[r], u[int(observed[r, t])], lr)
        if (e + 1) % period == 0:
            avg = divide_by_p(engine_tree_sum(w, dtype), p)
            w = [avg.copy() for _ in range(p)]
    return {"u": np.stack(u), "w": np.stack(w), "w_epoch": w_epoch, "ledger": ledger}
