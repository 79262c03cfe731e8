#!/usr/bin/env python
"""bench.py -- eager-SGD partial allreduce on B200 (BASELINE.json metric).

One "step" is one eager-SGD step of the hot path over a ResNet-50-sized fp32
gradient (N = 25,559,081, BASELINE config 2): fold the gradient into the
device stash, offer it (stream-ordered request), solo partial allreduce over
NVLink peer memory (persistent sm_100a engine; a plain kernel for a world of
one), and the SGD update from the result slot.  The timed loop runs in
all-arrive mode (every rank boards every round, nap = P), so the bus bytes
are real and nothing is skipped.

    python bench.py                                   # N=1
    torchrun --nproc-per-node N bench.py --gpus N     # one rank per GPU
    python bench.py --impl reference                  # CPU reference arm

Rank 0 prints ONE JSON line.  `value` = aggregate eager-SGD steps/s over all
ranks (rank-steps / max-over-ranks device time); `e2e` is the same through the
public API with the gradient copied from pinned host memory every step.
Extra keys: `roofline` (HBM, the dominant local kernel), `allreduce` (NVLink
bus GB/s of the partial allreduce at 100 MB, solo and majority, N > 1),
`imbalance` (steps/s of sync / solo / majority under the reference's seeded
random_subset delay, N > 1), `cpu_baseline`, `clocks`, `gpu_launches`.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
# the bench parks and relaunches its engines itself around device-wide syncs
# (quiesce()), so the library's idle park (a safety net for user code that
# syncs the device between steps) stays off: it would otherwise relaunch an
# engine inside a timed region after a slow untimed phase (NVML init)
os.environ.setdefault("EC_IDLE_PARK_MS", "0")
ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

RESNET50_N = 25_559_081          # PAPER.md:664, BASELINE config 2
ALLREDUCE_100MB_N = 25_000_000   # north_star: 100 MB fp32
LR = 0.05


def _parse_cpulist(text: str) -> set:
    cpus = set()
    for part in text.strip().split(","):
        if not part:
            continue
        lo, _, hi = part.partition("-")
        cpus.update(range(int(lo), int(hi or lo) + 1))
    return cpus


def _numa_local_affinity(device: int) -> str:
    """Restrict this process to the CPUs local to the GPU: NVML's CPU affinity,
    else the PCI device's sysfs local_cpulist.  Returns which source was used
    ("nvml", "sysfs" or "none")."""
    cpus, src = set(), "none"
    try:
        import pynvml
        pynvml.nvmlInit()
        hdl = pynvml.nvmlDeviceGetHandleByIndex(device)
        words = pynvml.nvmlDeviceGetCpuAffinity(hdl, (os.cpu_count() + 63) // 64)
        cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        src = "nvml"
    except Exception:
        try:
            import torch
            pr = torch.cuda.get_device_properties(device)
            bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            with open(f"/sys/bus/pci/devices/{bdf}/local_cpulist") as f:
                cpus = _parse_cpulist(f.read())
            src = "sysfs"
        except Exception:
            cpus = set()
    cpus &= os.sched_getaffinity(0)
    if cpus:
        os.sched_setaffinity(0, cpus)
        return src
    return "none"


def _env_world():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu(kernel: str):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            k = json.load(f)["kernels"][kernel]
        return {"duration_us": k["duration_us"], "gbs": k["algorithmic_gbs"],
                "frac": k.get("frac_of_measured_peak")}
    except Exception:
        return None


def _traffic(kernel: str):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f)["kernels"][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


class ClockSampler:
    """NVML clocks / throttle reasons sampled while the timed region runs."""

    def __init__(self, device: int, period_s: float = 0.01):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period_s
        self._stop = threading.Event()
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:
            self.N = None

    def _run(self):
        N = self.N
        names = {
            "hw_slowdown": getattr(N, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(N, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(N, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(N, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(N, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.N is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.N is not None:
            self._stop.set()
            self.t.join()
        return False

    def summary(self):
        import statistics
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# reference arm (CPU)


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from oracle import cpu_baseline as cb
    p = max(1, world)
    # W untimed warm-up steps, then exactly K timed steps (one whole P-rank step
    # of the restatement is 20-120 ms here, so the run stays within minutes)
    res = cb.time_steps(p, args.n, budget_s=float("inf"), min_steps=args.steps,
                        max_steps=args.steps, warmup=args.warmup)
    line = {
        "metric": "eager-SGD steps/s (fold + solo partial allreduce + SGD update), "
                  "ResNet-50-sized fp32 gradient",
        "value": res["rank_steps_per_s"], "unit": "steps/s", "n_gpus": world,
        "steps": res["steps"], "warmup": res["warmup"], "ms_per_step": res["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"resnet50-gradient eager-SGD step, P={p} ranks emulated on host",
                   "n_elems": args.n, "p": p},
        "impl": "reference",
        "cpu_baseline": {"value": res["rank_steps_per_s"], "unit": "steps/s",
                         "cores": res["threads"], "kind": "port",
                         "sample": f"{res['steps']} whole steps of P={p} ranks x {args.n} fp32 "
                                   f"({res['seconds']:.1f} s)"},
        "e2e": {"value": res["rank_steps_per_s"], "unit": "steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--n", type=int, default=RESNET50_N)
    ap.add_argument("--no-extras", action="store_true", help="skip allreduce/imbalance/cpu legs")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--imb-unit-ms", type=float, default=1.0)
    ap.add_argument("--imb-steps", type=int, default=32)
    ap.add_argument("--lag", type=int, default=2, help="async steps in flight before reconciling")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, local_rank, world = _env_world()
    if os.environ.get("EC_DEBUG_DUMP"):
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["EC_DEBUG_DUMP"]), exit=True)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    # EC_RANKS_PER_GPU=2: functional coverage of a larger world on fewer GPUs
    # (e.g. N=8 on a 4-GPU box; the engines of two processes time-slice a GPU,
    # so its numbers are not measurements)
    local_rank //= int(os.environ.get("EC_RANKS_PER_GPU", "1"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1908_04207_b200 import (AllreduceHandle, CollectiveConfig, ProcessWorld,
                                       TrainState, _lib, attach_delivery_tracking, drive,
                                       finish_step, train_step, train_step_async)
    from paper_1908_04207_b200.transport import DelayModel, device_delay, inject_delay

    pw = ProcessWorld(rank=rank, p=world, device=local_rank)
    n = args.n

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def quiesce():
        barrier()
        pw.pause()
        torch.cuda.synchronize()
        pw.resume()
        barrier()

    def settle():
        # the bracket of a timed region: the engines are resident by design (a
        # device-wide synchronize would wait for them forever), so every rank
        # drains its own streams -- nothing of the warm-up is left in flight
        barrier()
        torch.cuda.current_stream().synchronize()
        barrier()

    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    w0 = torch.randn(n, device=dev, generator=gen) * 0.01
    cfg = CollectiveConfig(p=world, flavor="solo", vector_len=n, element="f4", seed=1234)
    h = AllreduceHandle(cfg, rank, pw, cid=0)
    # the step's gradient lives in the registered bucket (where backward would
    # write it), so while the stash is null the offer is zero-copy
    gbuf = h.grad_buffer()
    gbuf.normal_(generator=gen)
    # the pipelined e2e's second input buffer: allocated before any engine is
    # resident (an allocation that frees cached blocks synchronises the device)
    gbuf2 = torch.empty_like(gbuf)
    copy_s = torch.cuda.Stream()   # likewise: creating a stream blocked behind a resident engine
    grads = [gbuf, gbuf]
    st = TrainState.fresh(w0, LR, rank=rank, tau=None)
    all_arrive = world > 1

    attach_delivery_tracking(h, st)

    def run_steps(k, grad_fn, pre=None, ev_end=None, naps=None):
        """Issue k async steps (ec_step_async: no host round trip), reconciling
        each LAG steps behind; ev_end is recorded right after the last issue."""
        from collections import deque
        pend = deque()
        upd_ns = []
        v = C.c_uint64()

        def fin(p):
            t0 = time.perf_counter()
            out = finish_step(st, h, p)
            _lib.lib.ec_step_update_ns(h.comm.ptr, h.li, C.byref(v))
            upd_ns.append(v.value)
            host_t[1] += time.perf_counter() - t0
            return out

        for i in range(k):
            if pre is not None:
                pre(i)
            t0 = time.perf_counter()
            pend.append(train_step_async(st, h, grad_fn(st.t), all_arrive=all_arrive))
            host_t[0] += time.perf_counter() - t0
            if len(pend) > args.lag:
                _, res, _g = fin(pend.popleft())
                if naps is not None:
                    naps.append(res.nap)
        if ev_end is not None:
            ev_end.record()
        while pend:
            _, res, _g = fin(pend.popleft())
            if naps is not None:
                naps.append(res.nap)
        return upd_ns

    # ---- main timed loop: inputs resident in HBM (working set >> 126 MB L2)
    host_t = [0.0, 0.0]       # host seconds in train_step_async (issue) / finish_step
    run_steps(args.warmup, lambda t: grads[t % 2])
    quiesce()
    # the engines were relaunched by quiesce(): their first rounds stay untimed
    run_steps(2, lambda t: grads[t % 2])
    clk = ClockSampler(local_rank)       # NVML init and thread start stay outside the region
    clk.__enter__()
    settle()
    host_t = [0.0, 0.0]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    naps = []
    if world > 1:
        h.stream_barrier()     # every rank's start event fires together (device barrier)
    launches0 = _lib.lib.ec_launch_count()
    h0 = time.perf_counter()
    ev0.record()
    upd_ns = run_steps(args.steps, lambda t: grads[t % 2], ev_end=ev1, naps=naps)
    host_ms = (time.perf_counter() - h0) * 1e3
    ev1.synchronize()
    clk.__exit__(None, None, None)
    launches = _lib.lib.ec_launch_count() - launches0
    host_issue_us, host_finish_us = (x / args.steps * 1e6 for x in host_t)
    ms = ev0.elapsed_time(ev1)
    timeline = device_timeline(h, st.t, args.steps, max_over_ranks) if world > 1 else None
    quiesce()
    ms_max = max_over_ranks(ms)
    value = world * args.steps / (ms_max / 1e3)

    # per-launch CUDA events (fold launches, engine mode) in a separate, untimed
    # run: events between launches perturb the step they measure
    fold_ms = 0.0
    if world > 1:
        _lib.lib.ec_profile_enable(1)
        run_steps(min(args.steps, 20), lambda t: grads[t % 2])
        _lib.lib.ec_profile_enable(0)
        prof_ms, prof_n = (C.c_double * 2)(), (C.c_int64 * 2)()
        _lib.lib.ec_profile_read(prof_ms, prof_n)
        fold_ms = prof_ms[0] / max(1, prof_n[0])
        quiesce()
    # the update launch also waits on the device for the round (fused wait+update+unpin):
    # its compute time is the kernel's own %globaltimer stamp, averaged over the region
    upd_ms = sum(upd_ns) / max(1, len(upd_ns)) / 1e6
    peak, peak_kind = _peaks()
    # world of one: decide + round + update are ONE launch (ec_direct_step_kernel:
    # reads the gradient and w, writes the slot u and w = 16 B/element); with
    # peers the round runs in the engine and the update reads u from the slot
    # (ec_update_gen_kernel: reads u and w, writes w = 12 B/element)
    direct = world == 1
    upd_kernel = "ec_direct_step_kernel<float>" if direct else "ec_update_gen_kernel<float>"
    upd_bytes = (16 if direct else 12) * n
    stamp_ms = upd_ms
    if direct:
        # the step stream runs this one kernel per step in the timed region (the
        # publication kernel runs on the communicator's own stream), so its
        # average launch duration is the region's CUDA-event time per step; the
        # %globaltimer stamp (decision -> publication kernel entry) adds the
        # kernel boundary and the publication's scheduling
        upd_ms = ms / args.steps
    upd_gbs = upd_bytes / (upd_ms / 1e3) / 1e9

    # ---- e2e: gradient from pinned host memory every step, result read back.
    # The pinned buffer is first-touched from the GPU's NUMA-local cores (as a
    # data loader pinned to the GPU's socket would), so H2D does not cross sockets.
    all_cpus = os.sched_getaffinity(0)
    affinity_src = _numa_local_affinity(local_rank)
    host_grad = torch.randn(n, generator=torch.Generator().manual_seed(7 + rank)).pin_memory()
    dgrad = gbuf                          # the H2D copy lands in the registered bucket
    h2d = lambda i: dgrad.copy_(host_grad, non_blocking=True)  # noqa: E731
    quiesce()
    run_steps(2, lambda t: dgrad, pre=h2d)
    settle()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(5, args.steps // 2)
    if world > 1:
        h.stream_barrier()
    e0.record()
    # each step: H2D of the gradient from pinned memory, the step, and the
    # step's result (generation, mask, nap) read back by finish_step
    run_steps(e2e_steps, lambda t: dgrad, pre=h2d, ev_end=e1)
    e1.synchronize()
    quiesce()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_serial = world * e2e_steps / (e2e_ms / 1e3)

    # pipelined e2e (the input pipeline a trainer runs): step t+1's H2D on a
    # copy stream overlaps step t, double-buffered between the registered
    # bucket (zero-copy offer) and a second device buffer (folded offer); a
    # buffer is refilled only after the step that read it completed
    main_s = torch.cuda.current_stream()
    bufs = [gbuf, gbuf2]
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    freed = [None, None]
    t_first, horizon = [0], [0]

    def prefetch(t):
        b = t % 2
        with torch.cuda.stream(copy_s):
            if freed[b] is not None:
                copy_s.wait_event(freed[b])
            bufs[b].copy_(host_grad, non_blocking=True)
            copied[b].record(copy_s)

    def pre_pipe(i):
        t = st.t
        if t > t_first[0]:
            ev = torch.cuda.Event()
            ev.record(main_s)            # behind step t-1's launches: its buffer is free after
            freed[(t - 1) % 2] = ev
        if t + 1 < t_first[0] + horizon[0]:
            prefetch(t + 1)
        main_s.wait_event(copied[t % 2])

    quiesce()
    t_first[0], horizon[0] = st.t, 2
    prefetch(st.t)
    run_steps(2, lambda t: bufs[t % 2], pre=pre_pipe)
    settle()
    freed = [None, None]
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        h.stream_barrier()
    p0.record()
    t_first[0], horizon[0] = st.t, e2e_steps
    prefetch(st.t)
    run_steps(e2e_steps, lambda t: bufs[t % 2], pre=pre_pipe, ev_end=p1)
    p1.synchronize()
    quiesce()
    e2e_value = world * e2e_steps / (max_over_ranks(p0.elapsed_time(p1)) / 1e3)
    # the bare H2D copy the e2e step carries (its PCIe bound)
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    for _ in range(5):
        dgrad.copy_(host_grad, non_blocking=True)
    c1.record()
    c1.synchronize()
    h2d_gbs = 5 * 4 * n / (c0.elapsed_time(c1) / 1e3) / 1e9
    os.sched_setaffinity(0, all_cpus)      # the CPU baseline below uses every host thread
    quiesce()

    extras = {}
    # every communicator's engine holds SMs: release the step's before the
    # allreduce / imbalance legs create theirs
    h.close()
    if not args.no_extras and world > 1:
        extras.update(bench_allreduce(args, pw, rank, world, dev, barrier, max_over_ranks, quiesce))
        extras.update(bench_imbalance(args, pw, rank, world, dev, barrier, max_over_ranks, quiesce))

    cpu = None
    if rank == 0 and world == 1 and not args.no_extras:
        from oracle import cpu_baseline as cb
        r = cb.time_steps(1, n, budget_s=args.cpu_budget, max_steps=200)
        cpu = {"value": r["rank_steps_per_s"], "unit": "steps/s", "cores": r["threads"],
               "kind": "port",
               "sample": f"{r['steps']} whole P=1 steps of {n} fp32 ({r['seconds']:.1f} s, "
                         f"oracle restatement, numpy over {r['threads']} threads)"}

    if direct:
        roofline = {"bound": "hbm", "kernel": upd_kernel, "achieved": upd_gbs, "peak": peak,
                    "unit": "GB/s", "frac": upd_gbs / peak, "traffic": _traffic("direct_step"),
                    "bytes_per_launch": upd_bytes, "avg_launch_ms": upd_ms,
                    "avg_launch_ms_source": "CUDA events over the timed region, per step "
                                            "(the step stream's only kernel)",
                    "stamp_ms": stamp_ms, "peak_source": peak_kind}
    else:
        # with peers the dominant cost is the round's data phase, bound by NVLink
        # (the HBM-bound update overlaps it chunk by chunk): bus bytes
        # 2(P-1)/P * 4N per round over the engine's device-timed data phase, vs
        # the measured B200 peer copy per direction (B200_PROFILING.md)
        bus = 2 * (world - 1) / world * 4 * n
        data_us = timeline["data_phase"]
        roofline = {"bound": "nvlink", "kernel": "ec_engine<float> data phase (round_tma)",
                    "achieved": bus / (data_us * 1e-6) / 1e9, "peak": 770.0, "unit": "GB/s",
                    "frac": bus / (data_us * 1e-6) / 1e9 / 770.0, "traffic": None,
                    "bytes_per_launch": bus, "avg_launch_ms": data_us / 1e3,
                    "peak_source": "measured peer copy per direction (B200_PROFILING.md)",
                    "hbm_update": {"kernel": upd_kernel, "bytes_per_launch": upd_bytes,
                                   "note": "progressive: spans the round, overlapped"}}
    if rank == 0:
        line = {
            "metric": "eager-SGD steps/s (fold + solo partial allreduce + SGD update), "
                      "ResNet-50-sized fp32 gradient",
            "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "resnet50-gradient eager-SGD solo step (BASELINE config 2)",
                       "n_elems": n, "p": world, "flavor": "solo",
                       "mode": "all-arrive" if world > 1 else "world of one (direct)",
                       "l2": "inputs larger than L2 (grad+stash+w+slot = 409 MB/rank)",
                       "mean_nap": float(np.mean(naps))},
            "e2e": {"value": e2e_value, "unit": "steps/s", "h2d_bytes_per_step": 4 * n,
                    "pipeline": "double-buffered H2D on a copy stream overlapping the previous "
                                "step (each step still copies its 102 MB gradient)",
                    "serial_value": e2e_serial, "h2d_copy_gbs": h2d_gbs,
                    # the step's H2D rate against the bare pinned copy (the PCIe bound)
                    "h2d_gbs_achieved": e2e_value / world * 4 * n / 1e9,
                    "h2d_frac_of_copy": (e2e_value / world * 4 * n / 1e9) / h2d_gbs,
                    "host_affinity": affinity_src,
                    "d2h_bytes_per_step": 16},
            "roofline": roofline,
            "local_kernels": {
                "fold": {"zero_copy": True,
                         "note": ("world of one: no fold launch -- the step kernel offers the "
                                  "registered bucket in place" if direct else
                                  "the gradient is offered in place from the registered bucket "
                                  "while the stash is null; the fold launch only posts the offer"),
                         "avg_launch_ms": fold_ms if not direct else None},
                "update" if not direct else "round_and_update": {
                    "kernel": upd_kernel, "bytes_per_launch": upd_bytes, "avg_launch_ms": upd_ms,
                    "gbs": upd_gbs, "frac": upd_gbs / peak},
            },
            "timeline_us": timeline,
            "host_ms_per_step": host_ms / args.steps,
            "host_us_per_step": {"issue": host_issue_us, "finish_incl_wait": host_finish_us},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
        }
        line.update(extras)
        # BASELINE.json's metric is a pair: solo/majority allreduce bus GB/s at
        # 100 MB, and eager-SGD steps/s under imbalance.  `value` is the config-2
        # step rate (defined at every N, including N=1 where neither half
        # exists); both halves sit here at N > 1 (details in allreduce / imbalance)
        line["baseline_metric"] = ("solo/majority allreduce bus GB/s at 100MB; "
                                   "eager-SGD steps/s under imbalance")
        if "allreduce" in extras:
            line["bus_gbs_100mb"] = {f: v["busbw_gbs"] for f, v in extras["allreduce"].items()}
        if "imbalance" in extras:
            line["steps_per_s_under_imbalance"] = {
                f: v["steps_per_s"] for f, v in extras["imbalance"].items()
                if isinstance(v, dict) and "steps_per_s" in v}
        print(json.dumps(line), flush=True)
    pw.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def device_timeline(h, t_end, k, max_over_ranks):
    """Mean per-round phases from the engine's %globaltimer stamps over the
    last k generations (max over ranks): done(g-1) -> snapshot(g) (host
    turnaround incl. fold + offer + all-arrive), snapshot -> all snapshots in,
    data phase (reduce-scatter pull + all-gather push), plus the whole period."""
    from paper_1908_04207_b200.harness import _gen_times
    gens = list(range(max(1, t_end - k + 1), t_end))   # skip the round after the quiesce
    ts = [_gen_times(h, g) for g in [gens[0] - 1] + gens]
    local = [ts[i][4] - ts[i - 1][3] for i in range(1, len(ts))]     # update+fold+offer
    arrive = [ts[i][0] - ts[i][4] for i in range(1, len(ts))]        # all-arrive + activation
    snap = [ts[i][1] - ts[i][0] for i in range(1, len(ts))]
    data = [ts[i][3] - ts[i][1] for i in range(1, len(ts))]
    period = (ts[-1][3] - ts[0][3]) / (len(ts) - 1)
    m = lambda xs: max_over_ranks(sum(xs) / len(xs) / 1e3)  # noqa: E731
    out = {"done_to_offer": m(local), "offer_to_snapshot": m(arrive),
           "snapshot_to_start": m(snap), "data_phase": m(data),
           "period": max_over_ranks(period / 1e3)}
    # the step boundary inside done -> offer: round g-1 published -> step
    # g-1's update reports -> step g's fold/post kernel starts -> it posts ->
    # the controller takes the offer (steps are rounds here: t = g)
    try:
        import ctypes as C
        from paper_1908_04207_b200 import _lib
        st = {}
        tail = gens[-60:]           # the device keeps the last 64 steps' stamps
        for g in [tail[0] - 1] + tail:
            a = (C.c_uint64 * 4)()
            _lib.call("ec_step_times", h.comm.ptr, h.li, g, a)
            st[g] = list(a)
        upd, kb, post, seen, take = [], [], [], [], []
        off = len(gens) - len(tail)
        for j, g in enumerate(tail):
            i = off + j
            done_prev = ts[i][3]
            upd.append(st[g - 1][0] - done_prev)
            kb.append(st[g][1] - st[g - 1][0])
            post.append(st[g][2] - st[g][1])
            seen.append(st[g][3] - st[g][2])
            take.append(ts[i + 1][4] - st[g][3])
        out["done_to_offer_detail"] = {"done_to_update_report": m(upd),
                                       "report_to_next_kernel": m(kb),
                                       "kernel_to_post": m(post), "post_to_seen": m(seen),
                                       "seen_to_taken": m(take)}
    except Exception as e:  # noqa: BLE001 - diagnostic only
        out["done_to_offer_detail"] = {"error": str(e)[:100]}
    return out


def bench_allreduce(args, pw, rank, world, dev, barrier, max_over_ranks, quiesce):
    """NVLink bus GB/s of the partial allreduce at 100 MB (all-arrive, nap = P):
    busbw = 2(P-1)/P * 4N / t_round."""
    import torch

    from paper_1908_04207_b200 import AllreduceHandle, CollectiveConfig, _lib
    n = ALLREDUCE_100MB_N
    out = {}
    # a communicator that only runs plain rounds: 128 TMA workers (the
    # measured best for back-to-back rounds, profiles/r2_geom4.json,
    # r2_geom2.json; at P >= 3 the step's handle keeps the default 80, best
    # beside its progressive update)
    saved_workers = pw.workers
    if world >= 2 and not os.environ.get("EC_WORKERS"):
        pw.workers = 128
    for cid, flavor in ((10, "solo"), (11, "majority")):
        cfg = CollectiveConfig(p=world, flavor=flavor, vector_len=n, element="f4", seed=1234)
        h = AllreduceHandle(cfg, rank, pw, cid=cid)
        h.send_buffer().normal_()
        rounds = max(10, args.steps)

        from paper_1908_04207_b200.harness import _round as rnd

        quiesce()
        for t in range(3):        # warm-up with the (re)launched engines, untimed
            rnd(h, t)
        barrier()
        from paper_1908_04207_b200.harness import rounds_back_to_back
        # back-to-back rounds on the stream, all-arrive so nap = P, like
        # nccl-tests' busbw: posted with no wait between them (the engine takes
        # each next offer the moment the previous round completes), and -- for
        # comparison -- each behind a device-side wait for the previous one
        from paper_1908_04207_b200.harness import rounds_pipelined
        rx0, tx0 = C.c_uint64(), C.c_uint64()
        _lib.lib.ec_comm_traffic(h.comm.ptr, h.li, C.byref(rx0), C.byref(tx0))
        ms = max_over_ranks(rounds_pipelined(h, 3, rounds)) / rounds
        rx1, tx1 = C.c_uint64(), C.c_uint64()
        _lib.lib.ec_comm_traffic(h.comm.ptr, h.li, C.byref(rx1), C.byref(tx1))
        # the NVLink bytes this rank's workers issued per round (pulls + pushes),
        # to compare with the algorithmic bus bytes 2(P-1)/P * S
        issued = max_over_ranks(((rx1.value - rx0.value) + (tx1.value - tx0.value)) / rounds)
        busbw = 2 * (world - 1) / world * 4 * n / (ms / 1e3) / 1e9
        barrier()
        ms_ser = max_over_ranks(rounds_back_to_back(h, 3 + rounds, rounds)) / rounds
        barrier()
        # the same through the blocking call_round-style API (host waits each round)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t in range(3 + 2 * rounds, 3 + 3 * rounds):
            rnd(h, t)
        e1.record()
        e1.synchronize()
        ms_sync = max_over_ranks(e0.elapsed_time(e1)) / rounds
        out[flavor] = {"busbw_gbs": busbw, "us_per_round": ms * 1e3, "bytes": 4 * n,
                       "frac_of_900": busbw / 900.0, "frac_of_770_measured_peer": busbw / 770.0,
                       "serialized": {"us_per_round": ms_ser * 1e3,
                                      "busbw_gbs": 2 * (world - 1) / world * 4 * n
                                      / (ms_ser / 1e3) / 1e9},
                       "blocking_api": {"us_per_round": ms_sync * 1e3,
                                        "busbw_gbs": busbw * ms / ms_sync},
                       "workers": h.comm.world.workers or "auto",
                       "issued_nvlink_bytes_per_round": issued,
                       "bus_bytes_per_round": 2 * (world - 1) / world * 4 * n}
        h.close()
    pw.workers = saved_workers
    return {"allreduce": out}


def bench_imbalance(args, pw, rank, world, dev, barrier, max_over_ranks, quiesce):
    """Eager-SGD steps/s under the reference's seeded random_subset delay
    (transport.py:101-149; one rank per round spins imb_unit_ms on its GPU),
    for sync / solo / majority on the same ResNet-50-sized gradient."""
    import numpy as np
    import torch

    from paper_1908_04207_b200 import (AllreduceHandle, CollectiveConfig, TrainState,
                                       attach_delivery_tracking, drive, train_step)
    from paper_1908_04207_b200.transport import DelayModel, device_delay, inject_delay
    n = args.n
    model = DelayModel("random_subset", unit_ms=args.imb_unit_ms, k=1, seed=11)
    gen = torch.Generator(device=dev)
    gen.manual_seed(99 + rank)
    g = torch.randn(n, device=dev, generator=gen)
    out = {"delay": {"kind": "random_subset", "unit_ms": args.imb_unit_ms, "k": 1, "seed": 11},
           "steps": args.imb_steps}
    for cid, flavor in ((20, "sync"), (21, "solo"), (22, "majority")):
        cfg = CollectiveConfig(p=world, flavor=flavor, vector_len=n, element="f4", seed=1234)
        h = AllreduceHandle(cfg, rank, pw, cid=cid)
        st = TrainState.fresh(torch.zeros(n, device=dev), LR, rank=rank, tau=None)
        attach_delivery_tracking(h, st)
        naps = []
        quiesce()
        drive(train_step(st, None, h, grad=g))   # step 0 with the relaunched engine, untimed
        barrier()
        torch.cuda.current_stream().synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t in range(1, args.imb_steps + 1):
            device_delay(inject_delay(rank, t, model, world))
            _, res, _g = drive(train_step(st, None, h, grad=g))
            naps.append(res.nap)
        e1.record()
        e1.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1))
        out[flavor] = {"steps_per_s": world * args.imb_steps / (ms / 1e3),
                       "mean_nap": float(np.mean(naps))}
        h.close()
    base = out["sync"]["steps_per_s"]
    for f in ("solo", "majority"):
        out[f]["speedup_vs_sync"] = out[f]["steps_per_s"] / base
    return {"imbalance": out}


if __name__ == "__main__":
    sys.exit(main())
