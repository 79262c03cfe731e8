"""Small programs for compute-sanitizer (racecheck / synccheck / memcheck):
one solo round + async steps of the persistent engine on an emulated P=2 world,
and fused world-of-one steps (the bench's direct step).

    compute-sanitizer --tool racecheck python scripts/sanitize_check.py engine
    compute-sanitizer --tool synccheck python scripts/sanitize_check.py direct
"""

import os
import sys
import threading

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("EC_IDLE_PARK_MS", "0")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_04207_b200 import (AllreduceHandle, CollectiveConfig, EmulatedWorld,  # noqa: E402
                                   TrainState, finish_step, train_step_async)


def engine(n=40_003, rounds=3):
    p = 2
    world = EmulatedWorld(p)
    cfg = CollectiveConfig(p=p, flavor="solo", vector_len=n, element="f4")
    hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
    st = [TrainState.fresh(np.zeros(n, np.float32), 0.05, rank=r, tau=None) for r in range(p)]
    streams = [torch.cuda.Stream() for _ in range(p)]
    world.synchronize()

    def body(r):
        torch.cuda.set_device(0)
        with torch.cuda.stream(streams[r]):
            for t in range(rounds):
                g = torch.full((n,), float(r + t), device="cuda")
                finish_step(st[r], hs[r], train_step_async(st[r], hs[r], g, all_arrive=True))
            streams[r].synchronize()

    th = [threading.Thread(target=body, args=(r,)) for r in range(p)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    world.synchronize()
    world.close()
    print("engine ok")


def direct(n=1_000_003, steps=3):
    world = EmulatedWorld(1)
    h = AllreduceHandle(CollectiveConfig(p=1, flavor="solo", vector_len=n, element="f4"), 0, world)
    st = TrainState.fresh(np.zeros(n, np.float32), 0.05, rank=0, tau=None)
    b = h.grad_buffer()
    for t in range(steps):
        b.fill_(float(t))
        finish_step(st, h, train_step_async(st, h, b))
    torch.cuda.synchronize()
    world.close()
    print("direct ok")


if __name__ == "__main__":
    {"engine": engine, "direct": direct}[sys.argv[1]]()
