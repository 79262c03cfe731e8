"""CPU baseline of the eager-SGD partial-allreduce step (bench.py's
`cpu_baseline` leg and `--impl reference`).

TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py): this times the
oracle's restatement of the reference path on host cores; it is never the
measured product.  The reference itself is pure Python and cannot travel to the
GPU box; its simulator is also far slower than this numpy
restatement (1.37 s per P=2 round at ResNet-50 size), so
timing the restatement is the stronger baseline.

One step for P ranks (eagersgd.py:129-167 with collectives.py:385-403):
  every rank: stash = 0 + grad            (fold into a null stash, eagersgd.py:56)
  allreduce:  u = tree_order_sum(stashes) / P
  every rank: w = w - lr*u                (eagersgd.py:165)
All arithmetic is fp32 numpy, split into contiguous chunks over a thread pool
(numpy releases the GIL), so it uses every host core it is given.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import restated as R


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class CpuEagerStep:
    def __init__(self, p: int, n: int, threads: int | None = None, lr: float = 0.05, seed: int = 0):
        self.p, self.n, self.lr = p, n, lr
        self.threads = threads or host_threads()
        rng = np.random.default_rng(seed)
        self.grads = [rng.standard_normal(n, dtype=np.float32) for _ in range(p)]
        self.w = [rng.standard_normal(n, dtype=np.float32) for _ in range(p)]
        self.stash = [np.zeros(n, np.float32) for _ in range(p)]
        self.u = np.zeros(n, np.float32)
        step = -(-n // self.threads)
        self.chunks = [(i, min(n, i + step)) for i in range(0, n, step)]
        self.pool = ThreadPoolExecutor(self.threads)

    def _chunk(self, lo: int, hi: int) -> None:
        zeros = np.zeros(hi - lo, np.float32)
        for r in range(self.p):
            np.add(zeros, self.grads[r][lo:hi], out=self.stash[r][lo:hi])
        s = R.engine_tree_sum([st[lo:hi] for st in self.stash], np.float32)
        self.u[lo:hi] = R.divide_by_p(s, self.p)
        for r in range(self.p):
            self.w[r][lo:hi] = R.sgd_update(self.w[r][lo:hi], self.u[lo:hi], self.lr)

    def step(self) -> None:
        list(self.pool.map(lambda c: self._chunk(*c), self.chunks))

    def close(self) -> None:
        self.pool.shutdown()


def time_steps(p: int, n: int, budget_s: float = 15.0, min_steps: int = 2, max_steps: int = 50,
               threads: int | None = None, warmup: int = 1):
    """Run `warmup` untimed steps, then whole steps until the budget is spent
    (at least min_steps, at most max_steps); returns dict with rank-steps/s."""
    b = CpuEagerStep(p, n, threads)
    try:
        for _ in range(max(1, warmup)):
            b.step()  # warm-up (page faults, pool start)
        t0 = time.perf_counter()
        k = 0
        while k < min_steps or (time.perf_counter() - t0 < budget_s and k < max_steps):
            b.step()
            k += 1
        dt = time.perf_counter() - t0
    finally:
        b.close()
    return {"steps": k, "seconds": dt, "rank_steps_per_s": p * k / dt,
            "ms_per_step": 1e3 * dt / k, "threads": b.threads, "warmup": max(1, warmup)}


def time_local_kernels(n: int, budget_s: float = 5.0, threads: int | None = None):
    """Reference-op timing of the local kernels (numpy fp32 `stash + grad` and
    `w - lr*u`, eagersgd.py:56,165) as GB/s of their algorithmic 12*N bytes."""
    th = threads or host_threads()
    rng = np.random.default_rng(1)
    a, b, c = (rng.standard_normal(n, dtype=np.float32) for _ in range(3))
    step = -(-n // th)
    chunks = [(i, min(n, i + step)) for i in range(0, n, step)]
    out = {}
    with ThreadPoolExecutor(th) as pool:
        for name, fn in (("fold", lambda lo, hi: np.add(a[lo:hi], b[lo:hi], out=c[lo:hi])),
                         ("update", lambda lo, hi: np.subtract(
                             a[lo:hi], np.float32(0.05) * b[lo:hi], out=c[lo:hi]))):
            list(pool.map(lambda x: fn(*x), chunks))
            t0 = time.perf_counter()
            k = 0
            while k < 3 or time.perf_counter() - t0 < budget_s / 2:
                list(pool.map(lambda x: fn(*x), chunks))
                k += 1
            dt = (time.perf_counter() - t0) / k
            out[name] = {"ms": dt * 1e3, "gbs": 12 * n / dt / 1e9}
    return out
