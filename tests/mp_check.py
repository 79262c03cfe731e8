"""Multi-GPU parity checks, one rank per GPU over NVLink (run under torchrun).

    torchrun --nproc-per-node P --master-addr 127.0.0.1 tests/mp_check.py

Each check compares the ProcessWorld path (CUDA IPC peer mapping + persistent
engine per GPU) with the CPU oracle / the reference's golden outputs.  Rank 0
prints one JSON object with every check's outcome; the exit code is non-zero
if any check failed on any rank.  Driven by tests/test_multigpu.py.
"""

import ctypes as C
import hashlib
import json
import os
import sys
import time
import traceback

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("EC_TIMEOUT_S", "30")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    if os.environ.get("EC_DEBUG_DUMP"):
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["EC_DEBUG_DUMP"]), exit=True)
    only = os.environ.get("EC_ONLY")
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    # EC_RANKS_PER_GPU=2 runs e.g. P=8 on a 4-GPU box (functional coverage of
    # the P=8 geometry; two engines share each GPU)
    local //= int(os.environ.get("EC_RANKS_PER_GPU", "1"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    from oracle import restated as R
    from paper_1908_04207_b200 import (AllreduceHandle, CollectiveConfig, ProcessWorld,
                                       TrainState, drive, initiator_for_round, train_step)
    from paper_1908_04207_b200.replay import replay_configs, replay_rank
    from paper_1908_04207_b200.trace import DeliveryLedger
    from paper_1908_04207_b200 import _lib
    from paper_1908_04207_b200._lib import call

    pw = ProcessWorld()
    results = {}
    cid = [100]

    def next_cid():
        cid[0] += 1
        return cid[0]

    def check(name, fn):
        if only and name not in only.split(","):
            return
        try:
            out = fn()
            results[name] = {"ok": True, **(out or {})}
        except Exception as e:
            results[name] = {"ok": False, "error": f"{type(e).__name__}: {e}",
                             "tb": traceback.format_exc()[-1500:]}
            print(f"rank {rank} check {name} FAILED: {e}\n{traceback.format_exc()[-1500:]}",
                  flush=True)
        dist.barrier()

    golden = np.load(os.path.join(ROOT, "tests", "golden", "tree_sums.npz"))

    def sync_f64_golden():
        contrib = golden[f"sync_in_p{world}"]
        cfg = CollectiveConfig(p=world, flavor="sync", vector_len=8, element="f8")
        h = AllreduceHandle(cfg, rank, pw, cid=next_cid())
        for t in range(3):
            res = drive(h.call_round(t, contrib[rank]))
            assert res.nap == world and res.rnd == t
            assert res.u.cpu().numpy().tobytes() == golden[f"sync_u_p{world}"].tobytes()
        h.close()

    def sync_f32_sizes():
        for n in (1, 7, 1027, 2_000_003, 25_559_081):
            rng = np.random.default_rng(world * 31 + n)
            contrib = rng.standard_normal((world, n), dtype=np.float32)
            want, inc, _ = R.allreduce_round(list(contrib), [True] * world, np.float32)
            cfg = CollectiveConfig(p=world, flavor="sync", vector_len=n, element="f4")
            h = AllreduceHandle(cfg, rank, pw, cid=next_cid())
            vec = torch.as_tensor(contrib[rank], device="cuda")
            for t in range(2):
                res = drive(h.call_round(t, vec))
                assert res.included == inc
                assert res.u.cpu().numpy().tobytes() == want.tobytes(), f"n={n} t={t}"
            h.close()

    shared_gpus = int(os.environ.get("EC_RANKS_PER_GPU", "1")) > 1

    def solo_first_arrival():
        if shared_gpus:   # engines of two processes time-slice one GPU (no MPS)
            return {"skipped": "arrival-order check needs one rank per GPU"}
        cfg = CollectiveConfig(p=world, flavor="solo", vector_len=1000, element="f4")
        h = AllreduceHandle(cfg, rank, pw, cid=next_cid())
        contrib = np.random.default_rng(1).standard_normal((world, 1000), dtype=np.float32)
        dist.barrier()
        time.sleep(0.05 * rank)
        res = drive(h.call_round(0, contrib[rank]))
        want, _, _ = R.allreduce_round([contrib[0]] + [None] * (world - 1),
                                       [True] + [False] * (world - 1), np.float32)
        h.close()
        assert res.included == 1, f"mask {res.included:#x}"
        assert res.u.cpu().numpy().tobytes() == want.tobytes()
        return {"included": res.included}

    def majority_prefix():
        if shared_gpus:
            return {"skipped": "arrival-order check needs one rank per GPU"}
        seeds = []
        for seed in (31, 32, 33, 34):
            cfg = CollectiveConfig(p=world, flavor="majority", vector_len=16, element="f8", seed=seed)
            h = AllreduceHandle(cfg, rank, pw, cid=next_cid())
            dist.barrier()
            time.sleep(0.05 * rank)
            res = drive(h.call_round(0, np.full(16, 10.0 * rank)))
            h.close()
            init = initiator_for_round(seed, 0, world)
            assert res.included == (1 << (init + 1)) - 1, (seed, init, res.included)
            vecs = [np.full(16, 10.0 * r) if r <= init else None for r in range(world)]
            want, _, _ = R.allreduce_round(vecs, [v is not None for v in vecs])
            assert res.u.cpu().numpy().tobytes() == want.tobytes()
            seeds.append((seed, init, res.included))
        return {"seeds": seeds}

    def eager_sgd_all_arrive():
        n, lr = 1_000_003, 0.05
        rng = np.random.default_rng(5)
        grads = rng.standard_normal((3, world, n), dtype=np.float32)
        w0 = rng.standard_normal(n, dtype=np.float32)
        cfg = CollectiveConfig(p=world, flavor="solo", vector_len=n, element="f4")
        h = AllreduceHandle(cfg, rank, pw, cid=next_cid())
        st = TrainState.fresh(w0, lr, rank=rank, tau=None)
        from paper_1908_04207_b200.eagersgd import attach_delivery_tracking
        attach_delivery_tracking(h, st)
        w = w0.copy()
        for t in range(3):
            g = torch.as_tensor(grads[t, rank], device="cuda")
            _, res, gen = drive(train_step(st, None, h, grad=g, all_arrive=True))
            assert gen == t and res.nap == world
            u, _, _ = R.allreduce_round(list(grads[t]), [True] * world, np.float32)
            w = R.sgd_update(w, u, lr)
        h.close()
        assert st.w.cpu().numpy().tobytes() == w.tobytes()

    def eager_sgd_async_fused():
        """train_step_async over NVLink: each step's update kernel applies the
        round's result chunk by chunk as it lands (progressive update), for
        folded and zero-copy offers, plain SGD and momentum, ragged n -- same
        bits as the oracle's round followed by its update."""
        from collections import deque

        from paper_1908_04207_b200 import finish_step, train_step_async
        from paper_1908_04207_b200.eagersgd import attach_delivery_tracking
        out = {}
        for mu in (0.0, 0.9):
            n, lr, steps = 3_000_017, 0.05, 6
            rng = np.random.default_rng(9)
            grads = rng.standard_normal((steps, world, n), dtype=np.float32)
            w0 = rng.standard_normal(n, dtype=np.float32)
            cfg = CollectiveConfig(p=world, flavor="solo", vector_len=n, element="f4")
            h = AllreduceHandle(cfg, rank, pw, cid=next_cid())
            st = TrainState.fresh(w0, lr, rank=rank, tau=None, momentum=mu)
            attach_delivery_tracking(h, st)
            bucket = h.grad_buffer()
            gd = torch.as_tensor(grads[:, rank], device="cuda")
            pend, gens = deque(), []
            for t in range(steps):
                if t % 2:
                    bucket.copy_(gd[t])
                    g = bucket
                else:
                    g = gd[t]
                pend.append(train_step_async(st, h, g, all_arrive=True))
                if len(pend) > 2:
                    gens.append(finish_step(st, h, pend.popleft())[2])
            while pend:
                gens.append(finish_step(st, h, pend.popleft())[2])
            torch.cuda.current_stream().synchronize()
            w, buf = w0.copy(), np.zeros_like(w0)
            for t in range(steps):
                u, _, _ = R.allreduce_round(list(grads[t]), [True] * world, np.float32)
                if mu:
                    w, buf = R.momentum_update(w, buf, u, np.float32(lr), np.float32(mu))
                else:
                    w = R.sgd_update(w, u, lr)
            fused = h.comm.progressive
            h.close()
            assert gens == list(range(steps)), gens
            assert st.w.cpu().numpy().tobytes() == w.tobytes(), f"mu={mu}"
            if mu:
                assert st.momentum_buf.cpu().numpy().tobytes() == buf.tobytes()
            out[f"mu={mu}"] = {"progressive_update": fused}
        return out

    def stream_barrier():
        """ec_stream_barrier: ranks enqueue it 50 ms apart; the stream work
        behind it completes together on every rank (host clocks compared)."""
        cfg = CollectiveConfig(p=world, flavor="solo", vector_len=16, element="f4")
        h = AllreduceHandle(cfg, rank, pw, cid=next_cid())
        spread = []
        for k in range(3):
            dist.barrier()
            time.sleep(0.05 * ((rank + k) % world))
            h.stream_barrier()
            torch.cuda.current_stream().synchronize()
            done = [None] * world
            dist.all_gather_object(done, time.time())
            spread.append(max(done) - min(done))
        h.close()
        # without the barrier the returns would spread over up to 50*(P-1) ms
        assert max(spread) < (0.03 if not shared_gpus else 0.06), spread
        return {"exit_spread_ms": [round(x * 1e3, 2) for x in spread]}

    def nvls_fast_mode():
        """reduction_mode="fast": the NVSwitch reduces (when the fabric has
        NVLS); same u on every rank, within fp32 rounding of the fixed-order sum."""
        from paper_1908_04207_b200 import _lib as L
        n = 2_000_003
        rng = np.random.default_rng(77)
        contrib = rng.standard_normal((world, n), dtype=np.float32)
        want, inc, _ = R.allreduce_round(list(contrib), [True] * world, np.float32)
        cfg = CollectiveConfig(p=world, flavor="solo", vector_len=n, element="f4",
                               reduction_mode="fast")
        h = AllreduceHandle(cfg, rank, pw, cid=next_cid())
        vec = torch.as_tensor(contrib[rank], device="cuda")
        us = []
        for t in range(3):
            h._contribute(t, vec, fresh=True, activate=True, all_arrive=True)
            gen, res = h.wait_blocking(t)
            assert gen == t and res.included == inc
            us.append(res.u.cpu().numpy())
        nv = h.comm.nvls
        h.close()
        rel = float(np.linalg.norm(us[0].astype(np.float64) - want) / np.linalg.norm(want))
        assert rel < 1e-6, rel
        digest = [hashlib.sha1(u.tobytes()).hexdigest() for u in us]
        alld = [None] * world
        dist.all_gather_object(alld, digest)
        assert all(d == alld[0] for d in alld), "ranks disagree"
        return {"nvls": nv, "rel_err_vs_fixed_order": rel}

    def replay_c1():
        if world != 4:
            return {"skipped": f"c1 traces have p=4, world={world}"}
        out = {}
        for flavor in ("sync", "solo", "majority"):
            for element in ("f8", "f4"):
                tr = dict(np.load(os.path.join(ROOT, "tests", "golden", f"c1_{flavor}.npz")))
                cfg, sync_cfg = replay_configs(tr, element)
                h = AllreduceHandle(cfg, rank, pw, cid=next_cid())
                hr = AllreduceHandle(sync_cfg, rank, pw, cid=next_cid())
                pw.pause()
                h.comm.set_replay(0, [int(m) for m in tr["masks"]])
                call("ec_set_pin", h.comm.ptr, 0, int(tr["observed"][rank, 0]), 0, None)
                pw.resume()
                dt = cfg.torch_dtype
                grads = torch.as_tensor(tr["grads"][rank], dtype=dt, device="cuda")
                st = TrainState.fresh(torch.as_tensor(tr["w0"], dtype=dt, device="cuda"),
                                      float(tr["lr"]), rank=rank,
                                      resync_period=int(tr["resync_period"]), tau=None)
                steps = int(tr["steps"])
                acc = np.zeros((4, steps), np.int8)
                masks = np.zeros(steps, np.int64)
                ledger = DeliveryLedger()
                dist.barrier()
                replay_rank(rank, h, hr, st, tr, grads, ledger, acc, masks)
                h.close()
                hr.close()
                assert acc[rank].tolist() == tr["accepted"][rank].tolist()
                seen = masks != 0
                assert masks[seen].tolist() == tr["masks"][seen].tolist()
                w = st.w.cpu().numpy()
                if element == "f8":
                    assert w.tobytes() == tr["final_w"][rank].tobytes(), f"{flavor} f64"
                else:
                    want = R.replay_run(tr, np.float32)["w"][rank]
                    assert w.tobytes() == want.tobytes(), f"{flavor} f32"
                led = {(int(r), int(g)): (None if d < 0 else int(d)) for r, g, d in tr["ledger"]
                       if int(r) == rank}
                assert ledger.as_dict() == led
                out[f"{flavor}_{element}"] = "bit-exact"
        return out

    def bench_schedule_replay():
        """The reference's config-2/3 bench schedules for this world size
        (tests/golden/c2c3_bench.npz) replayed with forced masks across
        processes at N = 25,559,081 fp32: accepted offers and masks as
        recorded, every observed slot bit-exact vs the fp32 restatement."""
        from paper_1908_04207_b200.replay import replay_bench_rank
        z = np.load(os.path.join(ROOT, "tests", "golden", "c2c3_bench.npz"))
        names = sorted({k.split("/")[0] for k in z.files if k.endswith(f"_p{world}/meta")})
        if not names:
            return {"skipped": f"no recorded schedule for p={world}"}
        n = 25_559_081
        out = {}
        for name in names:
            flavor = name.split("_")[0]
            p, rounds, seed = (int(x) for x in z[f"{name}/meta"])
            masks, acc, obs = z[f"{name}/masks"], z[f"{name}/accepted"], z[f"{name}/observed"]
            host = [np.random.default_rng([seed, r]).standard_normal(n, dtype=np.float32)
                    for r in range(p)]
            expected = {}
            for m in sorted(set(int(x) for x in masks)):
                c = [host[r] if (m >> r) & 1 else None for r in range(p)]
                u, _, _ = R.allreduce_round(c, [x is not None for x in c], np.float32, n)
                expected[m] = torch.as_tensor(u, device="cuda")
            cfg = CollectiveConfig(p=p, flavor=flavor, vector_len=n, element="f4", seed=seed)
            h = AllreduceHandle(cfg, rank, pw, cid=next_cid())
            pw.pause()
            h.comm.set_replay(0, [int(m) for m in masks])
            pw.resume()
            vec = torch.as_tensor(host[rank], device="cuda")
            dist.barrier()
            o = replay_bench_rank(h, vec, masks, acc[rank], obs[rank],
                                  lambda g, m, slot: m == int(masks[g]) and
                                  torch.equal(slot, expected[m]))
            h.close()
            assert o["accepted"] == [bool(a) for a in acc[rank]], name
            assert o["masks_seen"] == [int(masks[g]) for g in obs[rank]], name
            assert all(o["verified"]), (name, o["verified"].index(False))
            out[name] = f"{rounds} rounds bit-exact"
        return out

    def pipelined_two_in_flight():
        """Back-to-back 100 MB rounds posted without waits: round g+1's
        snapshot exchange overlaps round g's data phase (EcDesc lead 2); the
        results are bit-exact and rounds publish in order."""
        from paper_1908_04207_b200.harness import _gen_times, rounds_pipelined
        n, k = 25_000_000, 12
        out = {}
        for flavor in ("solo", "majority"):
            rng = np.random.default_rng(11)
            contrib = rng.standard_normal((world, n), dtype=np.float32)
            want, inc, _ = R.allreduce_round(list(contrib), [True] * world, np.float32)
            cfg = CollectiveConfig(p=world, flavor=flavor, vector_len=n, element="f4", seed=1234)
            h = AllreduceHandle(cfg, rank, pw, cid=next_cid())
            h.send_buffer().copy_(torch.as_tensor(contrib[rank], device="cuda"))
            torch.cuda.current_stream().synchronize()
            dist.barrier()
            ms = rounds_pipelined(h, 0, k)
            g, res = h.wait_blocking(k - 1)
            assert g == k - 1 and res.included == inc
            assert res.u.cpu().numpy().tobytes() == want.tobytes(), flavor
            times = [_gen_times(h, gg) for gg in range(k)]
            ov = sum(times[i][1] < times[i - 1][3] for i in range(1, k))
            h.close()
            out[flavor] = {"overlapped": int(ov), "us_per_round": ms * 1e3 / k}
        return out

    def idle_park_remote_wake():
        """Every engine parks after EC_IDLE_PARK_MS without work (device-wide
        syncs return); then rank 0 alone starts a solo round: the other ranks'
        watchers see its activation in their control blocks and relaunch their
        engines, so the round completes for everyone without their hosts posting."""
        cfg = CollectiveConfig(p=world, flavor="solo", vector_len=4096, element="f4")
        h = AllreduceHandle(cfg, rank, pw, cid=next_cid())
        vec = torch.full((4096,), float(rank + 1), device="cuda")
        for t in range(2):
            h._contribute(t, vec, fresh=True, activate=True, all_arrive=True)
            h.wait_blocking(t)
        dist.barrier()
        time.sleep(0.5)                       # > EC_IDLE_PARK_MS (100 ms): every engine parks
        torch.cuda.synchronize()              # returns: no resident engine
        parks, wakes, parked = C.c_uint64(), C.c_uint64(), C.c_int()
        call("ec_comm_idle_stats", h.comm.ptr, C.byref(parks), C.byref(wakes), C.byref(parked))
        assert parked.value == 1 and parks.value >= 1, (parks.value, parked.value)
        dist.barrier()
        if rank == 0:
            assert h._contribute(2, vec, fresh=True, activate=True)
        g, res = h.wait_blocking(2, timeout=20.0)
        call("ec_comm_idle_stats", h.comm.ptr, C.byref(parks), C.byref(wakes), C.byref(parked))
        h.close()
        assert g == 2 and res.included == 1 and res.u.cpu()[0].item() == 1.0 / world
        assert wakes.value >= 1
        return {"parks": int(parks.value), "wakes": int(wakes.value)}

    check("sync_f64_golden", sync_f64_golden)
    check("sync_f32_sizes", sync_f32_sizes)
    check("solo_first_arrival", solo_first_arrival)
    check("majority_prefix", majority_prefix)
    check("eager_sgd_all_arrive", eager_sgd_all_arrive)
    check("eager_sgd_async_fused", eager_sgd_async_fused)
    check("stream_barrier", stream_barrier)
    check("nvls_fast_mode", nvls_fast_mode)
    check("replay_c1", replay_c1)
    check("bench_schedule_replay", bench_schedule_replay)
    check("pipelined_two_in_flight", pipelined_two_in_flight)
    if not shared_gpus:
        check("idle_park_remote_wake", idle_park_remote_wake)

    gathered = [None] * world
    dist.all_gather_object(gathered, results)
    ok = all(all(v["ok"] for v in r.values()) for r in gathered)
    if rank == 0:
        summary = {"world": world, "ok": ok,
                   "checks": {k: {"ok": all(g[k]["ok"] for g in gathered),
                                  **{kk: vv for kk, vv in gathered[0][k].items() if kk != "ok"}}
                              for k in results}}
        failures = {f"r{r}:{k}": v for r, g in enumerate(gathered) for k, v in g.items()
                    if not v["ok"]}
        if failures:
            summary["failures"] = failures
        print(json.dumps(summary, indent=1), flush=True)
    pw.close()
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
