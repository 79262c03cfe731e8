"""Benchmark drivers on real GPUs (harness.py of the reference, re-done for B200).

* `allreduce_sweep` -- BASELINE config 5: partial-allreduce bus bandwidth over
  payload sizes 1 KB .. 1 GB in all-arrive mode (nap = P, so nothing can be
  skipped), with the device's own phase timestamps (snapshot -> reduction ->
  publish) beside the host-observed round time.
* `bench_flavor` -- the reference's latency / NAP microbenchmark
  (harness.py:206-241): each rank idles its injected delay from a common round
  origin, then calls the collective; records `BenchRecord(flavor, round, rank,
  latency_us, nap, initiator)` in the reference's CSV schema.

Run under torchrun (one rank per GPU):

    torchrun --nproc-per-node 8 -m paper_1908_04207_b200.harness sweep --out sweep.json
    torchrun --nproc-per-node 8 -m paper_1908_04207_b200.harness latency --p 8
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import sys
import time
from dataclasses import dataclass

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

BENCH_SCHEMA = "eagercoll-bench-v1"
TRAIN_SCHEMA = "eagercoll-train-v1"
_BENCH_FIELDS = ("flavor", "round", "rank", "latency_us", "nap", "initiator")
_TRAIN_FIELDS = ("flavor", "round", "epoch", "rank", "loss", "nap", "staleness_max", "t_us")


class ConfigError(ValueError):
    """harness.py:50 of the reference (bad config / unreadable CSV)."""


@dataclass
class BenchRecord:
    """harness.py:180-196 of the reference."""
    flavor: str
    round: int
    rank: int
    latency_us: int
    nap: int
    initiator: int = -1

    def __post_init__(self):
        if self.latency_us < 0:
            raise ValueError("negative latency")
        if self.nap < 1:
            raise ValueError("nap < 1")


def _gen_times(h, g):
    from ._lib import call
    t5 = (C.c_uint64 * 5)()
    call("ec_gen_times", h.comm.ptr, h.li, g, t5)
    return list(t5)


def _round(h, t, all_arrive=True):
    """One all-arrive round through ec_round (post + reply + wait in one C call)."""
    from . import _lib
    from ._lib import call
    flags = _lib.EC_CF_FRESH | (_lib.EC_CF_ALL_ARRIVE if all_arrive else 0) | \
        (_lib.EC_CF_ACTIVATE if h._may_activate(t) else 0)
    h._ensure_started()
    st, gen, mask, nap = C.c_int(), C.c_int64(), C.c_uint64(), C.c_int()
    call("ec_round", h.comm.ptr, h.li, t, flags, h._stream(), 60000, C.byref(st), C.byref(gen),
         C.byref(mask), C.byref(nap))
    return gen.value


def _round_flags(h, t0, k, all_arrive):
    """Offer flags of rounds t0..t0+k-1, computed before a timed issue loop:
    the majority initiator (numpy Philox, collectives.py:78-88) costs tens of
    microseconds of host time per round, more than a small round itself."""
    from . import _lib
    return [_lib.EC_CF_FRESH | (_lib.EC_CF_ALL_ARRIVE if all_arrive else 0) |
            (_lib.EC_CF_ACTIVATE if h._may_activate(t) else 0) for t in range(t0, t0 + k)]


def rounds_back_to_back(h, t0, k, all_arrive=True):
    """k rounds t0..t0+k-1 enqueued on the current stream, each behind a
    device-side wait for the previous one (ec_round_async); returns device ms
    between the first offer and the last completion (CUDA events)."""
    import torch

    from . import _lib
    from ._lib import call
    h._ensure_started()
    flags = _round_flags(h, t0, k, all_arrive)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    seqs = []
    e0.record()
    for t in range(t0, t0 + k):
        seq = C.c_uint64()
        call("ec_round_async", h.comm.ptr, h.li, t, flags[t - t0], h._stream(), C.byref(seq))
        seqs.append(seq.value)
    e1.record()
    e1.synchronize()
    for s in seqs:
        h._reply(s)
    h._wait(t0 + k - 1, 60.0, pin=False)
    return e0.elapsed_time(e1)


def rounds_pipelined(h, t0, k, all_arrive=True):
    """k rounds t0..t0+k-1 posted back to back on the current stream with no
    wait between them (the nccl-tests pattern: the same buffer every round);
    the engine defers each next-generation offer until the previous round
    completes, then takes it at once.  One device-side wait behind the last.
    Returns device ms between the first offer and the last completion."""
    import torch

    from . import _lib
    from ._lib import call
    h._ensure_started()
    flags = _round_flags(h, t0, k, all_arrive)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    seqs = []
    e0.record()
    for t in range(t0, t0 + k):
        seq = C.c_uint64()
        fn = "ec_round_async" if t == t0 + k - 1 else "ec_post_contribute"
        call(fn, h.comm.ptr, h.li, t, flags[t - t0], h._stream(), C.byref(seq))
        seqs.append(seq.value)
    e1.record()
    e1.synchronize()
    for s in seqs:
        h._reply(s)
    h._wait(t0 + k - 1, 60.0, pin=False)
    return e0.elapsed_time(e1)


def allreduce_sweep(world, rank, p, sizes_bytes, flavor="solo", rounds_cap=50, workers=None,
                    max_over_ranks=lambda x: x, barrier=lambda: None, reduction_mode="fixed_order"):
    """Bus bandwidth of the partial allreduce per payload size (fp32)."""
    import torch

    from .collectives import AllreduceHandle, CollectiveConfig
    out = []
    cid = 1000
    for nbytes in sizes_bytes:
        n = max(1, nbytes // 4)
        cid += 1
        if workers is not None:
            world.workers = workers
        cfg = CollectiveConfig(p=p, flavor=flavor, vector_len=n, element="f4", seed=1234,
                               reduction_mode=reduction_mode)
        h = AllreduceHandle(cfg, rank, world, cid=cid)
        h.send_buffer().normal_()
        rounds = int(max(5, min(rounds_cap, (2 << 30) // max(1, 4 * n))))
        for t in range(3):
            _round(h, t)
        barrier()
        t0 = time.perf_counter()
        for t in range(3, 3 + rounds):
            _round(h, t)
        dt = time.perf_counter() - t0
        barrier()
        b2b_ms = rounds_back_to_back(h, 3 + rounds, rounds)
        b2b_us = max_over_ranks(b2b_ms * 1e3 / rounds)
        barrier()
        pipe_ms = rounds_pipelined(h, 3 + 2 * rounds, rounds)
        pipe_us = max_over_ranks(pipe_ms * 1e3 / rounds)
        phases = [_gen_times(h, g) for g in range(2, 3 + rounds)]
        prev, phases = phases[0], phases[1:]
        data_us = sum((x[3] - x[1]) for x in phases) / rounds / 1e3
        rs_us = sum((x[2] - x[1]) for x in phases) / rounds / 1e3
        snap_wait_us = sum((x[1] - x[0]) for x in phases) / rounds / 1e3
        gaps = [phases[0][0] - prev[3]] + [phases[i][0] - phases[i - 1][3] for i in range(1, rounds)]
        turnaround_us = sum(gaps) / rounds / 1e3
        round_us = max_over_ranks(dt / rounds * 1e6)
        data_us = max_over_ranks(data_us)
        bus = 2 * (p - 1) / p * 4 * n if p > 1 else 0
        out.append({"bytes": 4 * n, "rounds": rounds, "us_per_round": round_us,
                    "busbw_gbs": bus / (round_us * 1e-6) / 1e9,
                    "us_per_round_b2b": b2b_us,
                    "busbw_b2b_gbs": bus / (b2b_us * 1e-6) / 1e9,
                    "us_per_round_pipelined": pipe_us,
                    "busbw_pipelined_gbs": bus / (pipe_us * 1e-6) / 1e9,
                    "device_data_us": data_us, "device_rs_us": max_over_ranks(rs_us),
                    "busbw_device_gbs": bus / (data_us * 1e-6) / 1e9 if data_us > 0 else None,
                    "snap_to_start_us": max_over_ranks(snap_wait_us),
                    "done_to_next_snap_us": max_over_ranks(turnaround_us),
                    "workers": h.comm.world.workers if workers is None else workers,
                    "nvls": bool(getattr(h.comm, "nvls", False))})
        h.close()
    return out


def bench_flavor(world, rank, p, flavor, model, rounds=64, vector_len=64, link_slack_us=1000,
                 seed=1234, barrier=None, close=True, cid=None):
    """harness.py:206-241 on hardware: rank r sleeps to t*period + delay[r, t],
    then call_round; returns its BenchRecords.  `barrier` aligns the ranks'
    round origin (default: the world's process-group barrier; emulated ranks
    in threads pass a thread barrier and close=False, closing after all)."""
    import numpy as np

    from .collectives import AllreduceHandle, CollectiveConfig, drive, initiator_for_round
    from .transport import delay_table
    delays = delay_table(model, p, rounds)
    period = int(delays.max()) + link_slack_us + 1000
    cfg = CollectiveConfig(p=p, flavor=flavor, vector_len=vector_len, element="f8", seed=seed)
    # a deterministic collective id per flavor (every rank must agree on it;
    # str hashes are salted per process)
    cid = 2000 + {"sync": 0, "solo": 1, "majority": 2}[flavor] if cid is None else cid
    h = AllreduceHandle(cfg, rank, world, cid=cid)
    vec = np.full(vector_len, float(rank + 1))
    recs = []
    (barrier or world._barrier)()
    origin = time.perf_counter()
    for t in range(rounds):
        target = origin + (t * period + int(delays[rank, t])) * 1e-6
        d = target - time.perf_counter()
        if d > 0:
            time.sleep(d)
        t0 = time.perf_counter()
        res = drive(h.call_round(t, vec))
        lat = int((time.perf_counter() - t0) * 1e6)
        init = initiator_for_round(seed, res.rnd, p) if flavor == "majority" else -1
        recs.append(BenchRecord(flavor, t, rank, lat, res.nap, init))
    if close:
        h.close()
    return recs


def run_training_rank(world, rank, p, flavor, *, epochs=48, steps_per_epoch=4, dim=64,
                      n_samples=4096, batch_per_rank=128, lr=0.05, tau=8, resync_period=8,
                      delay=None, seed=1234, data_seed=99, device_delay=False, cid_base=3000,
                      time_scale=1.0):
    """One rank of the reference's run_training (harness.py:275-340) on a device
    world: hyperplane regression (BASELINE config 1), real injected delays,
    the flavor's partial allreduce + a sync resync handle.  Returns this rank's
    metrics rows, per-epoch validation MSE, wall time and ledger entries."""
    import torch

    from .collectives import AllreduceHandle, CollectiveConfig, drive
    from .eagersgd import TrainState, training_process
    from .models import gen_dataset, init_weights
    from .trace import DeliveryLedger
    from .transport import inject_delay
    ds = gen_dataset(dim, n_samples, seed=data_seed, device=torch.device("cuda", world.device))
    w0 = init_weights(dim, seed=seed)
    h = AllreduceHandle(CollectiveConfig(p=p, flavor=flavor, vector_len=dim, element="f4",
                                         seed=seed), rank, world, cid=cid_base)
    hr = AllreduceHandle(CollectiveConfig(p=p, flavor="sync", vector_len=dim, element="f4"),
                         rank, world, cid=cid_base + 1)
    st = TrainState.fresh(w0, lr, rank=rank, resync_period=resync_period, tau=tau)
    ledger = DeliveryLedger()
    metrics, val = [], {}
    delay_fn = None
    if delay is not None and delay.kind != "none":
        delay_fn = lambda r, t: int(inject_delay(r, t, delay, p) * time_scale)  # noqa: E731
    t0 = time.perf_counter()
    drive(training_process(rank, st, h, hr, ds, epochs=epochs, steps_per_epoch=steps_per_epoch,
                           batch_per_rank=batch_per_rank, data_seed=data_seed,
                           delay_fn=delay_fn, metrics=metrics, transport=None,
                           guard=tau is not None, ledger=ledger, val_out=val,
                           device_delay=device_delay))
    torch.cuda.current_stream().synchronize()
    wall = time.perf_counter() - t0
    return {"rows": metrics, "val": val, "wall_s": wall, "ledger": ledger.entries(),
            "w": st.w.detach().cpu().numpy(), "handles": (h, hr)}


def lstm_bench(world, rank, p, steps=20, warmup=3, batch=16, max_len=None, max_over=lambda x: x):
    """BASELINE config 4: eager-SGD on the UCF101-shaped LSTM, one flavor after
    the other, inherent imbalance only (variable sequence lengths).  The
    gradient is produced by backward straight into the registered bucket and
    offered zero-copy; reports aggregate steps/s, mean nap and speedup vs sync."""
    from collections import deque

    import numpy as np
    import torch

    from .collectives import AllreduceHandle, CollectiveConfig
    from .eagersgd import TrainState, attach_delivery_tracking, finish_step, train_step_async
    from .lstm import SyntheticUCF101, VideoLSTM, bind_flat, lstm_grad_step, n_params
    torch.manual_seed(1234)
    dev = torch.device("cuda", world.device)
    data = SyntheticUCF101(batch=batch, device=dev, max_len=max_len)
    out = {}
    for i, flavor in enumerate(("sync", "solo", "majority")):
        model = VideoLSTM().to(dev)
        n = n_params(model)
        h = AllreduceHandle(CollectiveConfig(p=p, flavor=flavor, vector_len=n, element="f4",
                                             seed=1234), rank, world, cid=4000 + i)
        st = TrainState.fresh(torch.zeros(n, device=dev), 0.01, rank=rank, tau=None)
        bind_flat(model, st.w, h.grad_buffer())
        attach_delivery_tracking(h, st)
        naps, losses = [], []
        pend = deque()

        def run(k, t0):
            for s in range(k):
                loss = lstm_grad_step(model, h.grad_buffer(), data.batch_for(rank, t0 + s))
                pend.append(train_step_async(st, h, h.grad_buffer(), loss=loss))
                while len(pend) > 1:
                    _, res, _ = finish_step(st, h, pend.popleft())
                    naps.append(res.nap)
            while pend:
                lo, res, _ = finish_step(st, h, pend.popleft())
                naps.append(res.nap)
                losses.append(float(lo))

        run(warmup, 0)
        naps.clear()
        world._barrier()
        t0 = time.perf_counter()
        run(steps, warmup)
        torch.cuda.current_stream().synchronize()
        wall = max_over(time.perf_counter() - t0)
        out[flavor] = {"steps_per_s": p * steps / wall, "mean_nap": float(np.mean(naps)),
                       "params": n, "wall_s": wall}
        h.close()
        del model
    for f in out:
        out[f]["speedup_vs_sync"] = out[f]["steps_per_s"] / out["sync"]["steps_per_s"]
    return out


def summarize(records):
    """harness.py:347-370"""
    import numpy as np
    out = {"flavors": {}, "speedup_vs_sync": {}}
    by = {}
    for b in records:
        by.setdefault(b.flavor, []).append(b)
    for f, recs in sorted(by.items()):
        lat = np.array([b.latency_us for b in recs], dtype=np.float64)
        nap = np.array([b.nap for b in recs], dtype=np.float64)
        out["flavors"][f] = {"n": len(recs), "mean_latency_us": float(lat.mean()),
                             "std_latency_us": float(lat.std()), "mean_nap": float(nap.mean())}
    if "sync" in by:
        base = out["flavors"]["sync"]["mean_latency_us"]
        for f in by:
            own = out["flavors"][f]["mean_latency_us"]
            out["speedup_vs_sync"][f] = base / own if own else float("inf")
    return out


def _fmt(v) -> str:
    """harness.py:379-382: floats as repr (round-trippable), the rest as str."""
    if isinstance(v, float):
        return repr(v)
    return str(v)


def write_bench_csv(records, path: str) -> None:
    """harness.py:385-390 (same schema line and columns)."""
    with open(path, "w") as f:
        f.write(f"# {BENCH_SCHEMA}\n")
        f.write(",".join(_BENCH_FIELDS) + "\n")
        for b in records:
            f.write(",".join(_fmt(getattr(b, k)) for k in _BENCH_FIELDS) + "\n")


def train_row(flavor: str, m: dict) -> dict:
    """One eagercoll-train-v1 row from a training_process metrics dict
    (eagersgd.py:214-219: round, epoch, rank, loss, nap, staleness_max,
    wall_or_sim_time)."""
    return {"flavor": flavor, "round": int(m["round"]), "epoch": int(m["epoch"]),
            "rank": int(m["rank"]), "loss": float(m["loss"]), "nap": int(m["nap"]),
            "staleness_max": int(m["staleness_max"]), "t_us": int(m["wall_or_sim_time"])}


def write_train_csv(rows, path: str) -> None:
    """harness.py:393-398: `# eagercoll-train-v1`, then the columns."""
    with open(path, "w") as f:
        f.write(f"# {TRAIN_SCHEMA}\n")
        f.write(",".join(_TRAIN_FIELDS) + "\n")
        for row in rows:
            f.write(",".join(_fmt(row[k]) for k in _TRAIN_FIELDS) + "\n")


def write_jsonl(path: str, schema: str, dicts) -> None:
    """harness.py:401-407: JSON-lines mirror of a CSV -- one header object,
    then one object per row with identical fields and values."""
    with open(path, "w") as f:
        f.write(json.dumps({"schema": schema}, sort_keys=True) + "\n")
        for d in dicts:
            f.write(json.dumps(d, sort_keys=True) + "\n")


def read_bench_csv(path: str) -> list:
    """harness.py:410-424: parse an eagercoll-bench-v1 CSV back into records."""
    with open(path) as f:
        header = f.readline().strip()
        if header != f"# {BENCH_SCHEMA}":
            raise ConfigError(f"{path}: unknown schema {header!r}")
        names = f.readline().strip().split(",")
        if tuple(names) != _BENCH_FIELDS:
            raise ConfigError(f"{path}: unexpected columns {names}")
        out = []
        for line in f:
            vals = line.strip().split(",")
            out.append(BenchRecord(vals[0], int(vals[1]), int(vals[2]), int(vals[3]),
                                   int(vals[4]), int(vals[5])))
    return out


def emit_bench(records, stem: str) -> None:
    """harness.py:427-431: <stem>.csv and its JSONL mirror."""
    import dataclasses
    write_bench_csv(records, stem + ".csv")
    write_jsonl(stem + ".jsonl", BENCH_SCHEMA, [dataclasses.asdict(b) for b in records])


def emit_train(rows, stem: str) -> None:
    write_train_csv(rows, stem + ".csv")
    write_jsonl(stem + ".jsonl", TRAIN_SCHEMA, rows)


def _main(argv=None):
    import torch
    import torch.distributed as dist

    from .transport import DelayModel
    from .world import ProcessWorld
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=("sweep", "latency", "train", "lstm"))
    ap.add_argument("--flavors", default="solo,majority")
    ap.add_argument("--sizes", default="1K,4K,16K,64K,256K,1M,4M,16M,64M,100M,256M,1G")
    ap.add_argument("--workers", default="")
    ap.add_argument("--chunks", default="", help="TMA chunk bytes to sweep (EC_CHUNK)")
    ap.add_argument("--stages", default="", help="TMA pipeline depths to sweep (EC_STAGES)")
    ap.add_argument("--out", default="")
    ap.add_argument("--rounds", type=int, default=64)
    ap.add_argument("--delay", default="linear_skew:1.0")
    ap.add_argument("--epochs", type=int, default=48)
    ap.add_argument("--reduction-mode", default="fixed_order", choices=("fixed_order", "fast"))
    args = ap.parse_args(argv)
    if os.environ.get("EC_DEBUG_DUMP"):
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["EC_DEBUG_DUMP"]), exit=True)
    rank = int(os.environ.get("RANK", 0))
    p = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if p > 1:
        dist.init_process_group("gloo")
    world = ProcessWorld(rank=rank, p=p, device=local)

    def max_over(x):
        if p == 1:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    result = {"p": p}
    if args.mode == "sweep":
        mult = {"K": 1 << 10, "M": 1_000_000, "G": 1 << 30}
        sizes = [int(s[:-1]) * mult[s[-1]] if s[-1] in mult else int(s) for s in args.sizes.split(",")]
        sizes = [s if not (s == 100_000_000) else 100_000_000 for s in sizes]
        workers = [int(w) for w in args.workers.split(",")] if args.workers else [None]
        chunks = args.chunks.split(",") if args.chunks else [None]
        stages = args.stages.split(",") if args.stages else [None]
        for f in args.flavors.split(","):
            for w in workers:
                for ch in chunks:
                    for stg in stages:
                        for key, val in (("EC_CHUNK", ch), ("EC_STAGES", stg)):
                            if val is None:
                                os.environ.pop(key, None)
                            else:
                                os.environ[key] = val
                        key = f"{f}_w{w}_c{ch}_s{stg}"
                        try:
                            result[key] = allreduce_sweep(
                                world, rank, p, sizes, f, workers=w, max_over_ranks=max_over,
                                barrier=world.barrier, reduction_mode=args.reduction_mode)
                        except Exception as e:  # a geometry that cannot launch
                            result[key] = {"error": str(e)[:200]}
                            for cid in [c for c in world.comms if c >= 1000]:
                                try:
                                    world.release(cid)
                                except Exception:
                                    pass
    elif args.mode == "lstm":
        result["lstm"] = lstm_bench(world, rank, p, steps=args.rounds if args.rounds != 64 else 20,
                                    max_over=max_over)
    elif args.mode == "train":
        # BASELINE config 1 on GPUs: hyperplane, random_subset 0.2 ms k=1 seed 11
        import numpy as np
        model = DelayModel("random_subset", unit_ms=0.2, k=1, seed=11)
        if args.delay != "linear_skew:1.0":
            kind, unit = args.delay.split(":")
            model = DelayModel(kind, unit_ms=float(unit), k=1, seed=11)
        out = {}
        train_rows: list = []
        flavors = [f for f in args.flavors.split(",") if f] if args.flavors != "solo,majority" \
            else ["sync", "solo", "majority"]
        for i, f in enumerate(flavors):
            world._barrier()
            r = run_training_rank(world, rank, p, f, delay=model, cid_base=3000 + 10 * i,
                                  epochs=args.epochs)
            for hh in r["handles"]:
                hh.close()
            allr = [None] * p
            if p > 1:
                dist.all_gather_object(allr, {k: r[k] for k in ("rows", "val", "wall_s")})
            else:
                allr[0] = {k: r[k] for k in ("rows", "val", "wall_s")}
            train_rows += [train_row(f, m) for x in allr for m in x["rows"]]
            wall = max(x["wall_s"] for x in allr)
            steps = sum(len(x["rows"]) for x in allr)
            last = max(e for x in allr for (_, e) in x["val"])
            vals = [v for x in allr for (rr, e), v in x["val"].items() if e == last]
            naps = [row["nap"] for x in allr for row in x["rows"]]
            out[f] = {"wall_s": wall, "steps_per_s": steps / wall, "final_val_mse": float(np.mean(vals)),
                      "mean_nap": float(np.mean(naps))}
        if "sync" in out:
            for f in out:
                out[f]["speedup_vs_sync"] = out[f]["steps_per_s"] / out["sync"]["steps_per_s"]
        result["train"] = out
        if rank == 0 and args.out:
            emit_train(sorted(train_rows, key=lambda d: (d["flavor"], d["round"], d["rank"])),
                       args.out)
    else:
        kind, unit = args.delay.split(":")
        model = DelayModel(kind, unit_ms=float(unit), k=1, seed=11)
        recs = []
        for f in ("sync", "solo", "majority"):
            recs += bench_flavor(world, rank, p, f, model, rounds=args.rounds)
        allr = [None] * p
        dist.all_gather_object(allr, recs) if p > 1 else allr.__setitem__(0, recs)
        flat = sorted((r for rr in allr for r in rr), key=lambda b: (b.flavor, b.round, b.rank))
        result["summary"] = summarize(flat)
        if rank == 0 and args.out:
            emit_bench(flat, args.out)
    if rank == 0:
        s = json.dumps(result)
        print(s, flush=True)
        if args.out and args.mode == "sweep":
            with open(args.out, "w") as f:
                f.write(s + "\n")
    world.close()
    if p > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(_main())
