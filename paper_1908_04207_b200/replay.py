"""Replay mode: drive GPU ranks from a recorded reference schedule.

Participation in eager-SGD depends only on timing, never on values, so the
schedule-level events of a reference run -- which ranks' offers boarded each
generation and which generation each rank observed at each step -- can be
forced onto a GPU run.  The device engine then
snapshots exactly the recorded masks (`ec_comm_set_replay`), every host step
reads exactly the recorded generation, and the values it computes (stash
folds, tree-ordered sums, updates, resyncs) must equal the reference's: bit for
bit in f64, within 1e-6 in fp32, and bit for bit against the fp32 restatement.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _lib
from ._lib import call
from .collectives import AllreduceHandle, CollectiveConfig, drive
from .eagersgd import TrainState, apply_update, attach_delivery_tracking, resync_step
from .trace import DeliveryLedger
from .world import EmulatedWorld


def replay_rank(r: int, h: AllreduceHandle, resync_h: AllreduceHandle, st: TrainState, trace,
                grads_r: torch.Tensor, ledger, acc: np.ndarray, seen_masks: np.ndarray,
                rows: list | None = None, loss_fn=None, flavor: str = "") -> None:
    """One rank's replayed training loop (training_process, eagersgd.py:187-226,
    with the offers' outcomes and the observed generations forced by `trace`).
    With `rows`, appends one eagercoll-train-v1 row per step (harness.py:393):
    loss = loss_fn(rank, t, w) of the weights the step started from, nap of the
    generation applied, the stash's staleness and -- a replay has no clock --
    the observed generation as t_us."""
    steps = int(trace["steps"])
    epochs = int(trace["epochs"])
    spe = int(trace["steps_per_epoch"])
    period = int(trace["resync_period"])
    observed = np.asarray(trace["observed"]).astype(np.int64)
    attach_delivery_tracking(h, st, ledger)
    k = 0
    for e in range(epochs):
        for s in range(spe):
            t = e * spe + s
            ledger.generated(r, t)
            loss = float(loss_fn(r, t, st.w)) if loss_fn is not None else 0.0
            with h.engine.lock:
                st.send_buf.bind(h)
                st.send_buf.fold(grads_r[t], t)
                seq = h._post_contribute(t, _lib.EC_CF_FRESH)
            if h._reply(seq) == _lib.R_ACCEPTED:
                acc[r, t] = 1
                h.contributed_round = t
                h._fresh_gens.add(t)
            g = int(observed[r, t])
            h._wait(g, 60.0, pin=False)
            m = _gen_mask(h, g)
            if seen_masks[g] == 0:
                seen_masks[g] = m
            elif seen_masks[g] != m:
                raise AssertionError(f"generation {g}: rank {r} saw mask {m:#x}, "
                                     f"another rank {int(seen_masks[g]):#x}")
            apply_update(st, h._slot(g))
            if rows is not None:
                rows.append({"flavor": flavor, "round": t, "epoch": e, "rank": r, "loss": loss,
                             "nap": int(m).bit_count(), "staleness_max": st.staleness_max(),
                             "t_us": g})
            nxt = int(observed[r, t + 1]) if t + 1 < steps else _lib.UINT64_MAX
            call("ec_set_pin", h.comm.ptr, h.li, nxt, 1,
                 torch.cuda.current_stream(h.device).cuda_stream)
            st.t = t + 1
        if (e + 1) % period == 0:
            drive(resync_step(st, resync_h, k))
            k += 1
    torch.cuda.current_stream(h.device).synchronize()


def replay_configs(trace, element: str):
    p = int(trace["p"])
    dim = np.asarray(trace["grads"]).shape[-1]
    return (CollectiveConfig(p=p, flavor="solo", vector_len=dim, element=element, seed=0),
            CollectiveConfig(p=p, flavor="sync", vector_len=dim, element=element))


def replay_training(trace, element: str = "f4", device: int = 0, world=None, ring_slots: int = 4,
                    loss_fn=None, flavor: str = "replay"):
    """Replay a c1_<flavor> trace (tests/golden) on an emulated world (P ranks,
    P host threads, one GPU).

    trace: mapping with p, steps, epochs, steps_per_epoch, lr, resync_period,
    masks[g], accepted[r, t], observed[r, t], grads[r, t, :], w0.
    Returns dict(w=[p, dim] final weights (numpy), accepted=[p, steps],
    ledger=dict, masks=[steps] device masks, rows=eagercoll-train-v1 rows
    sorted by (round, rank); see replay_rank for loss_fn).
    """
    if hasattr(trace, "files"):       # an NpzFile is not safe to read from P threads
        trace = {k: trace[k] for k in trace.files}
    p = int(trace["p"])
    steps = int(trace["steps"])
    masks = [int(m) for m in np.asarray(trace["masks"])]
    observed = np.asarray(trace["observed"]).astype(np.int64)
    cfg, sync_cfg = replay_configs(trace, element)
    own = world is None
    world = world or EmulatedWorld(p, device, ring_slots=ring_slots)
    handles = [AllreduceHandle(cfg, r, world, cid=0) for r in range(p)]
    resync = [AllreduceHandle(sync_cfg, r, world, cid=1) for r in range(p)]
    for r in range(p):
        handles[r].comm.set_replay(r, masks)
        call("ec_set_pin", handles[r].comm.ptr, r, int(observed[r, 0]), 0, None)
    dtype = cfg.torch_dtype
    dev = f"cuda:{device}"
    grads = torch.as_tensor(np.asarray(trace["grads"]), dtype=dtype, device=dev)
    w0 = torch.as_tensor(np.asarray(trace["w0"]), dtype=dtype, device=dev)
    ledger = DeliveryLedger()
    states = [TrainState.fresh(w0, float(trace["lr"]), rank=r,
                               resync_period=int(trace["resync_period"]), tau=None)
              for r in range(p)]
    acc = np.zeros((p, steps), dtype=np.int8)
    seen_masks = np.zeros(steps, dtype=np.int64)
    rows: list = [[] for _ in range(p)]
    errors: list = []
    go = threading.Barrier(p)

    def body(r: int):
        try:
            torch.cuda.set_device(device)
            go.wait()
            replay_rank(r, handles[r], resync[r], states[r], trace, grads[r], ledger, acc,
                        seen_masks, rows[r], loss_fn, flavor)
        except BaseException as ex:  # surfaced below
            errors.append(ex)

    threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(p)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    try:
        if errors:
            raise errors[0]
        w = np.stack([st.w.detach().cpu().numpy() for st in states])
        flat = sorted((x for rr in rows for x in rr), key=lambda d: (d["round"], d["rank"]))
        return {"w": w, "accepted": acc, "ledger": ledger.as_dict(), "masks": seen_masks,
                "rows": flat}
    finally:
        if own:
            world.close()


def _gen_mask(h: AllreduceHandle, g: int) -> int:
    import ctypes as C
    m, hm, nap = C.c_uint64(), C.c_uint64(), C.c_int()
    call("ec_gen_info", h.comm.ptr, h.li, g, C.byref(m), C.byref(hm), C.byref(nap))
    return m.value


def replay_bench_rank(h: AllreduceHandle, vec: torch.Tensor, masks, accepted_r, observed_r,
                      verify=None) -> dict:
    """One rank of a replayed bench schedule (BASELINE configs 2/3 at the
    reference's bench cadence, harness.py:206-241): per round t, call_round's
    contribute-if-not-done (collectives.py:334-345) with the rank's constant
    vector, under the engine's forced inclusion masks; then the generation the
    reference observed is read from its result slot (pinned ahead, so later
    rounds cannot reuse it) and handed to `verify(g, mask, slot) -> bool`.

    Returns {"accepted": [...], "masks_seen": [...], "verified": [...]} per round;
    every entry must equal the recorded schedule (masks[g], accepted_r[t])."""
    rounds = len(observed_r)
    stream = torch.cuda.current_stream(h.device).cuda_stream
    acc, seen, ok = [], [], []
    call("ec_set_pin", h.comm.ptr, h.li, int(observed_r[0]), 0, None)
    for t in range(rounds):
        a = False
        if not h.round_done(t):
            a = h._contribute(t, vec, fresh=True, activate=True, copy=(t == 0))
        acc.append(bool(a))
        g = int(observed_r[t])
        h._wait(g, 60.0, pin=False)
        m = _gen_mask(h, g)
        seen.append(m)
        ok.append(True if verify is None else bool(verify(g, m, h._slot(g))))
        nxt = int(observed_r[t + 1]) if t + 1 < rounds else _lib.UINT64_MAX
        call("ec_set_pin", h.comm.ptr, h.li, nxt, 1, stream)
    torch.cuda.current_stream(h.device).synchronize()
    return {"accepted": acc, "masks_seen": seen, "verified": ok}


def replay_bench(flavor: str, masks, accepted, observed, vectors, *, element: str = "f4",
                 seed: int = 1234, device: int = 0, world=None, ring_slots: int = 4,
                 verify=None) -> dict:
    """Replay a recorded bench schedule on an emulated world of P ranks (one
    GPU, P host threads) at the size of `vectors` ([P] device tensors, rank r's
    constant contribution, as bench_flavor's np.full(vector_len, r+1)).
    verify(rank, g, mask, slot) checks a result slot; returns per-rank dicts."""
    p = len(vectors)
    n = int(vectors[0].numel())
    cfg = CollectiveConfig(p=p, flavor=flavor, vector_len=n, element=element, seed=seed)
    own = world is None
    world = world or EmulatedWorld(p, device, ring_slots=ring_slots)
    try:
        hs = [AllreduceHandle(cfg, r, world, cid=0) for r in range(p)]
        for r in range(p):
            hs[r].comm.set_replay(r, [int(m) for m in masks])
        out: dict = {}
        errors: list = []
        go = threading.Barrier(p)

        def body(r: int):
            try:
                torch.cuda.set_device(device)
                go.wait()
                vf = None if verify is None else (lambda g, m, s, _r=r: verify(_r, g, m, s))
                out[r] = replay_bench_rank(hs[r], vectors[r], masks, accepted[r], observed[r], vf)
            except BaseException as ex:  # surfaced below
                errors.append(ex)

        threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(p)]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        if errors:
            raise errors[0]
        return out
    finally:
        if own:
            world.close()
