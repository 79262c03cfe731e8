"""Solo / majority / sync allreduce on B200 -- the reference's public API.

Drop-in for `eagercoll.collectives` (/root/reference/pkg/src/eagercoll/
collectives.py).  Names, argument meaning and error behaviour follow the
reference; the mechanism underneath is the sm_100a persistent engine
(csrc/ec_kernels.cu) reached through the C ABI (include/eagercoll_b200.h):

* `try_contribute` posts, in stream order after the copy/fold, a contribution
  the device engine accepts or refuses atomically against the snapshot
  (collectives.py:291-309);
* activation is a generation-tagged flag the initiator writes into every peer's
  control block over NVLink (replaces the union of binomial trees,
  collectives.py:134-148, with one hop on a uniform NVSwitch fabric);
* the reduction is a two-shot pull over peer memory that sums every element in
  `tree_order_sum`'s association (collectives.py:385-403) and divides by P
  (collectives.py:254-260), so results are bit-identical on every rank;
* `wait_done` / `wait_blocking` return the latest generation >= t
  (collectives.py:319-332).

Tensors are torch CUDA tensors; numpy inputs are accepted and copied to the
device (results stay torch tensors).
"""

from __future__ import annotations

import ctypes as C
import math
import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, lib
from .trace import LatencyRecord, RoundRecord, SnapshotRecord, TraceRecorder
from .world import ELEMENTS, EmulatedWorld, ProcessWorld

SOLO, MAJORITY, SYNC = "solo", "majority", "sync"
FLAVORS = (SOLO, MAJORITY, SYNC)
# fixed_order: tree_order_sum's association, bit-exact (default, parity mode);
# fast: any association -- one rank per GPU uses the NVSwitch reduction (NVLS)
# when the fabric supports it, else the fixed-order engine
REDUCTION_MODES = ("fixed_order", "fast")


@dataclass(frozen=True)
class CollectiveConfig:
    """collectives.py:43-67, plus `element="f4"` (the product's fp32 path),
    `reduction_mode`: "fixed_order" (bit-exact tree order) or "fast" (NVSwitch
    in-switch reduction; results within fp32 rounding, identical on all ranks),
    and the opt-in `majority_quorum`."""

    p: int
    flavor: str
    vector_len: int
    element: str = "f8"
    seed: int = 0
    reduction_mode: str = "fixed_order"
    # majority only, opt-in: the designated initiator activates once at least
    # half the ranks (ceil(p/2)) have boarded -- the north_star's phrasing;
    # False (default) is the reference's rule: it activates on arrival
    # without counting (collectives.py:311-317)
    majority_quorum: bool = False

    def __post_init__(self):
        if self.p < 1:
            raise ValueError("p must be >= 1")
        if self.p > 64:
            raise ValueError("p must be <= 64 (one NVLink domain, one mask word)")
        if self.flavor not in FLAVORS:
            raise ValueError(f"unknown flavor {self.flavor!r}")
        if self.vector_len < 1:
            raise ValueError("vector_len must be >= 1")
        if self.element not in ELEMENTS:
            raise ValueError(f"element must be one of {sorted(ELEMENTS)}")
        if self.reduction_mode not in REDUCTION_MODES:
            raise ValueError(f"reduction_mode must be one of {REDUCTION_MODES}")
        if self.majority_quorum and self.flavor != MAJORITY:
            raise ValueError("majority_quorum applies to the majority flavor only")

    @property
    def mask_words(self) -> int:
        return (self.p + 63) // 64

    @property
    def payload_nbytes(self) -> int:
        """Bytes of one contribution on the device (the mask travels in the
        control block, not in the payload)."""
        return (4 if self.element == "f4" else 8) * self.vector_len

    @property
    def torch_dtype(self) -> torch.dtype:
        return ELEMENTS[self.element][1]


@dataclass
class CollectiveResult:
    """collectives.py:70-75"""

    u: torch.Tensor | None      # reduced vector, divided by p
    included: int               # bitmask: bit r set iff rank r's fresh value is in u
    nap: int                    # popcount of included
    rnd: int = 0


def initiator_for_round(seed: int, t: int, p: int) -> int:
    """collectives.py:78-88: Philox4x64 keyed by the shared seed with the round
    as counter -- every rank evaluates it locally, bit-identical to the reference."""
    if p < 1:
        raise ValueError("p must be >= 1")
    bitgen = np.random.Philox(key=np.uint64(seed), counter=[np.uint64(t), 0, 0, 0])
    return int(np.random.Generator(bitgen).integers(0, p))


def ceil_log2(p: int) -> int:
    return 0 if p <= 1 else (p - 1).bit_length()


def floor_pow2(p: int) -> int:
    return 1 << (p.bit_length() - 1)


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _as_device(vec, dtype: torch.dtype, device: int, n: int | None = None) -> torch.Tensor:
    if isinstance(vec, torch.Tensor):
        t = vec
        if t.device.type != "cuda" or t.device.index != device:
            t = t.to(f"cuda:{device}")
        if t.dtype != dtype:
            t = t.to(dtype)
    else:
        t = torch.as_tensor(np.asarray(vec), dtype=dtype, device=f"cuda:{device}")
    t = t.reshape(-1).contiguous()
    if n is not None and t.numel() != n:
        raise ValueError(f"vector length {t.numel()} != vector_len {n}")
    return t


class _EngineView:
    """What callers of the reference reach through `handle.engine`:
    the lock (schedule.py:207), the hold policy (schedule.py:198, installed by
    staleness_guard) and the generation counters."""

    def __init__(self, handle: "AllreduceHandle"):
        self._h = handle
        self.lock = threading.RLock()
        self.hold_policy = None

    @property
    def done_generation(self) -> int:
        return self._h.done_generation

    @property
    def generation(self) -> int:
        return self._h.done_generation + 1


class AllreduceHandle:
    """Per-rank handle on a persistent partial allreduce (collectives.py:207-345).

    `transport` is a world (`EmulatedWorld` / `ProcessWorld`).  The device engine
    serves rounds this rank never actively joins, exactly like the reference's
    transport-pumped engine (collectives.py:212-216).
    """

    def __init__(self, cfg: CollectiveConfig, rank: int, transport, cid: int = 0,
                 recorder: TraceRecorder | None = None):
        self.cfg = cfg
        self.rank = rank
        self.transport = transport
        self.cid = cid
        self.recorder = recorder
        self.user_snapshot_cb = None      # callable(rnd, data, fresh)
        self.contributed_round = -1
        self.comm, self.li = transport.attach(cfg, cid, rank)
        self.device = self.comm.device
        self.engine = _EngineView(self)
        self._fresh_gens: set = set()
        self._dispatched = -1
        self._last: tuple | None = None
        self._guard_state = None
        self._hold_posted = _lib.INT64_MAX
        self._pinned = False
        # one pinned read at a time per rank: the slot pin is a single word
        self._read_lock = threading.Lock()
        # generations whose snapshot took an offer issued by train_step_async:
        # by the time the host dispatches the callback the device may already
        # have reused the buffer the round read, so those get data=None
        self._async_gens: set = set()

    def close(self) -> None:
        """Destroy this collective instance on every rank of the world (the
        engines park first; collective for a ProcessWorld)."""
        self.transport.release(self.cid)

    # -- buffers ------------------------------------------------------------
    def send_buffer(self) -> torch.Tensor:
        """The device send buffer (also the eager-SGD stash, eagersgd.py:68)."""
        return self.comm.send_view(self.li)

    def grad_buffer(self) -> torch.Tensor:
        """The registered gradient bucket.  Write the step's gradient here and
        pass it to train_step_async: while the stash is null the reduction reads
        it in place over NVLink (zero-copy offer, no fold); a refused offer is
        folded into the stash on the device before the next step."""
        return self.comm.grad_view(self.li)

    def _slot(self, gen: int) -> torch.Tensor:
        return self.comm.slot_view(self.li, gen)

    def _stream(self) -> int:
        return _stream_ptr(self.device)

    def stream_barrier(self) -> None:
        """Enqueue a device-side barrier across every rank of this collective on
        the current stream (ec_stream_barrier): work queued behind it starts
        when the last rank reached it.  Every rank calls it equally often;
        emulated ranks need their own streams."""
        call("ec_stream_barrier", self.comm.ptr, self.li, self._stream())

    def _ensure_started(self) -> None:
        if not self.comm.running:
            self.comm.start()

    # -- engine queries -----------------------------------------------------
    @property
    def done_generation(self) -> int:
        g = C.c_int64()
        call("ec_done_gen", self.comm.ptr, self.li, C.byref(g))
        return g.value

    def round_done(self, t: int) -> bool:
        return self.done_generation >= t

    def _raise_device_error(self):
        code, info = self.comm.error(self.li)
        if code:
            raise RuntimeError(f"engine error {code} (info {info:#x}) at rank {self.rank}")

    # -- requests -----------------------------------------------------------
    def _post_contribute(self, t: int, flags: int) -> int:
        self._ensure_started()
        seq = C.c_uint64()
        call("ec_post_contribute", self.comm.ptr, self.li, t, flags, self._stream(), C.byref(seq))
        return seq.value

    def _reply(self, seq: int, timeout: float = 60.0) -> int:
        st = C.c_int()
        call("ec_reply", self.comm.ptr, self.li, seq, int(timeout * 1000), C.byref(st))
        if st.value == _lib.R_ERROR:
            self._raise_device_error()
            raise AssertionError("application rounds must be driven in order")
        return st.value

    def _may_activate(self, t: int) -> bool:
        return self.cfg.flavor != MAJORITY or \
            self.rank == initiator_for_round(self.cfg.seed, t, self.cfg.p)

    def _contribute(self, t: int, vec, fresh: bool, activate: bool, copy: bool = True,
                    all_arrive: bool = False) -> bool:
        with self.engine.lock:
            done = self.done_generation
            if done >= t:
                return False
            assert done == t - 1, "application rounds must be driven in order"
            if copy:
                send = self.send_buffer()
                src = _as_device(vec, self.cfg.torch_dtype, self.device, self.cfg.vector_len)
                if src.data_ptr() != send.data_ptr():
                    call("ec_copy_in", self.comm.ptr, self.li, src.data_ptr(), self._stream())
            flags = (_lib.EC_CF_FRESH if fresh else 0) \
                | (_lib.EC_CF_ACTIVATE if activate and self._may_activate(t) else 0) \
                | (_lib.EC_CF_ALL_ARRIVE if all_arrive else 0)
            seq = self._post_contribute(t, flags)
        st = self._reply(seq)
        if st == _lib.R_POISONED:
            from .eagersgd import DivergenceError
            raise DivergenceError(f"rank {self.rank} round {t}: non-finite gradient")
        if st == _lib.R_ACCEPTED:
            self.contributed_round = t
            if fresh:
                self._fresh_gens.add(t)
            return True
        return False

    def try_contribute(self, t: int, vec, fresh: bool = True) -> bool:
        """collectives.py:291-309.  False once round t already consumed this rank's
        slot (the value missed the bus).  The device decides atomically."""
        return self._contribute(t, vec, fresh, activate=False)

    def activate(self, t: int) -> None:
        """collectives.py:311-317: solo/sync always; majority only at
        initiator_for_round(seed, t, p)."""
        if not self._may_activate(t):
            return
        self._ensure_started()
        seq = C.c_uint64()
        call("ec_post_activate", self.comm.ptr, self.li, t, C.byref(seq))

    # -- results ------------------------------------------------------------
    def _wait(self, t: int, timeout: float, pin: bool):
        self._ensure_started()
        gen, mask, nap = C.c_int64(), C.c_uint64(), C.c_int()
        try:
            call("ec_wait", self.comm.ptr, self.li, t, int(timeout * 1000), int(pin),
                 C.byref(gen), C.byref(mask), C.byref(nap))
        except _lib.EcTimeout:
            raise TimeoutError(f"rank {self.rank} round {t} did not complete") from None
        self._dispatch_snapshots(gen.value)
        return gen.value, mask.value, nap.value

    def _unpin(self) -> None:
        call("ec_set_pin", self.comm.ptr, self.li, _lib.UINT64_MAX, 1, self._stream())

    def _dispatch_snapshots(self, upto: int) -> None:
        """Deliver the per-generation snapshot callbacks (schedule.py:373-380 ->
        collectives.py:245-252) for every generation this rank's engine took,
        in order.  A snapshot of generation g is fresh iff this rank's fresh
        offer for g was accepted."""
        while self._dispatched < upto:
            g = self._dispatched + 1
            fresh = g in self._fresh_gens
            self._fresh_gens.discard(g)
            stale = g in self._async_gens
            self._async_gens.discard(g)
            # the buffer the round consumed: the send buffer still holds it on
            # the synchronous paths (dispatch runs before the next fold); an
            # async step's offer may have been the gradient bucket or already
            # overwritten, so no data is passed
            data = self.send_buffer() if fresh and not stale else None
            if self.recorder is not None:
                # a null snapshot consumed the zeroed send buffer: record the
                # zero vector, as the reference does (trace.py:92-96,
                # schedule.py:373-380); a stale async offer records None
                if data is not None:
                    rec = data.clone()
                elif not fresh:
                    rec = torch.zeros(self.cfg.vector_len, dtype=self.cfg.torch_dtype,
                                      device=f"cuda:{self.device}")
                else:
                    rec = None
                self.recorder.snapshot(SnapshotRecord(self.rank, g, rec, fresh, _now_us()))
            if self.user_snapshot_cb is not None:
                self.user_snapshot_cb(g, data, fresh)
            self._dispatched = g

    def _read_result(self, t: int, timeout: float = 60.0, clone: bool = True):
        with self._read_lock:
            gen, mask, nap = self._wait(t, timeout, pin=True)
            u = self._slot(gen).clone() if clone else None
            self._unpin()
        res = CollectiveResult(u=u, included=mask, nap=nap, rnd=gen)
        self._last = (gen, res)
        if self.recorder is not None:
            init = initiator_for_round(self.cfg.seed, gen, self.cfg.p) \
                if self.cfg.flavor == MAJORITY else -1
            self.recorder.round_done(RoundRecord(self.rank, gen, u, mask, nap,
                                                 self.cfg.flavor, init, _now_us()))
        return gen, res

    def latest_result(self):
        """collectives.py:282-283"""
        d = self.done_generation
        if d < 0:
            return d, None
        return self._read_result(d)

    def wait_done(self, t: int):
        """Generator step (collectives.py:319-325): blocks until a generation >= t
        has published, then returns (generation, CollectiveResult) of the latest.
        Never yields -- a real device world needs no event loop."""
        if False:  # pragma: no cover - makes this a generator like the reference
            yield None
        return self._read_result(t)

    def wait_blocking(self, t: int, timeout: float = 30.0):
        """collectives.py:327-332"""
        return self._read_result(t, timeout)

    def call_round(self, t: int, vec):
        """collectives.py:334-345: contribute if the bus is still here, start the
        round, wait for the result (fused into one stream-ordered request)."""
        t0 = _now_us()
        if not self.round_done(t):
            self._contribute(t, vec, fresh=True, activate=True)
        gen, res = yield from self.wait_done(t)
        if self.recorder is not None:
            self.recorder.latency(LatencyRecord(self.rank, t, t0, _now_us()))
        return res


_T0 = time.perf_counter()


def _now_us() -> int:
    return int((time.perf_counter() - _T0) * 1e6)


def drive(gen):
    """Run a reference-style generator process to completion in real time.
    `Sleep(us)` yields become host sleeps; returns the generator's value."""
    from .transport import Sleep
    try:
        v = next(gen)
        while True:
            if isinstance(v, Sleep):
                if v.us > 0:
                    time.sleep(v.us * 1e-6)
            v = gen.send(None)
    except StopIteration as e:
        return e.value


def run_allreduce(cfg: CollectiveConfig, contributions, *, rounds: int = 1, delay_us=None,
                  link_latency_us: int = 0, recorder: TraceRecorder | None = None,
                  device: int = 0, time_scale: float = 1.0, world=None):
    """collectives.py:348-382 on one GPU: P ranks of an EmulatedWorld driven by
    P host threads in real time.  delay_us(rank, t) is slept (x time_scale)
    before rank joins round t; link_latency_us has no meaning on hardware.

    Returns (results, handles, world); results[(rank, t)] is the
    CollectiveResult the rank observed for its round-t call.
    """
    own = world is None
    world = world or EmulatedWorld(cfg.p, device)
    handles = [AllreduceHandle(cfg, r, world, cid=0, recorder=recorder) for r in range(cfg.p)]
    results: dict = {}
    errors: list = []
    start = threading.Barrier(cfg.p)

    def contribution(rank: int, t: int):
        if callable(contributions):
            return contributions(rank, t)
        return contributions[rank]

    def body(rank: int):
        try:
            start.wait()
            for t in range(rounds):
                if delay_us is not None:
                    d = delay_us(rank, t)
                    if d:
                        time.sleep(d * 1e-6 * time_scale)
                results[(rank, t)] = drive(handles[rank].call_round(t, contribution(rank, t)))
        except BaseException as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(cfg.p)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    if own:
        world.pause()
    return results, handles, world


def _spec_round(h: "AllreduceHandle", t: int, x, timeout: float, all_arrive: bool):
    """One rank's SPEC-level call: offer x (fresh) or the null payload (zeros,
    empty flag mask, SPEC.md ContributionPayload), activate per the flavor's
    rule, block for the result of round t (the latest generation >= t)."""
    if x is None:
        vec = torch.zeros(h.cfg.vector_len, dtype=h.cfg.torch_dtype, device=f"cuda:{h.device}")
        fresh = False
    else:
        vec = _as_device(x, h.cfg.torch_dtype, h.device, h.cfg.vector_len)
        fresh = True
    if not h.round_done(t):
        h._contribute(t, vec, fresh, activate=True, all_arrive=all_arrive)
    _, res = h.wait_blocking(t, timeout)
    h._spec_next = t + 1
    return res


def _spec_allreduce(flavor: str, cfg: CollectiveConfig, contribution_or_null, handle, t,
                    timeout: float) -> CollectiveResult:
    if cfg.flavor != flavor:
        import dataclasses
        cfg = dataclasses.replace(cfg, flavor=flavor)
    if handle is not None:
        # per-rank form (one call per rank and round, any world)
        if handle.cfg.flavor != flavor or handle.cfg.vector_len != cfg.vector_len:
            raise ValueError(f"handle is bound to {handle.cfg}, not a {flavor} collective of "
                             f"length {cfg.vector_len}")
        rnd = getattr(handle, "_spec_next", 0) if t is None else t
        return _spec_round(handle, rnd, contribution_or_null, timeout, all_arrive=False)
    # all-ranks form: one row (vector or None) per rank, zero skew, on one GPU
    rows = contribution_or_null
    if cfg.p == 1 and (rows is None or (not isinstance(rows, (list, tuple))
                                        and np.asarray(rows if not isinstance(rows, torch.Tensor)
                                                       else rows.cpu()).ndim == 1)):
        rows = [rows]
    rows = list(rows)
    if len(rows) != cfg.p:
        raise ValueError(f"expected {cfg.p} contributions (one per rank), got {len(rows)}")
    for x in rows:
        if x is not None and int(np.prod(np.shape(x))) != cfg.vector_len:
            raise ValueError(f"length mismatch: contribution of {int(np.prod(np.shape(x)))} "
                             f"elements vs vector_len {cfg.vector_len}")
    world = EmulatedWorld(cfg.p, torch.cuda.current_device())
    try:
        hs = [AllreduceHandle(cfg, r, world) for r in range(cfg.p)]
        out: dict = {}
        errors: list = []

        def body(r: int):
            try:
                torch.cuda.set_device(world.device)
                # every rank boards before activation: zero skew, as SPEC's examples
                out[r] = _spec_round(hs[r], 0, rows[r], timeout, all_arrive=True)
            except BaseException as e:  # surfaced below
                errors.append(e)

        threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(cfg.p)]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        if errors:
            raise errors[0]
        res0 = out[0]
        for r in range(1, cfg.p):   # Lemma 1 safety: identical result at every rank
            if out[r].included != res0.included or not torch.equal(out[r].u, res0.u):
                raise AssertionError(f"rank {r} observed a different result than rank 0")
        return res0
    finally:
        world.close()


def allreduce_sync(cfg: CollectiveConfig, contribution_or_null, *, handle=None, t=None,
                   timeout: float = 30.0) -> CollectiveResult:
    """SPEC.md:188-196 `allreduce_sync(cfg, contribution) -> CollectiveResult`:
    completes after every rank joined; u = sum/P, included = all fresh ranks.

    Two call forms (both thin wrappers over AllreduceHandle):
    * `handle=` a rank's AllreduceHandle: this rank's contribution (a vector,
      or None for the null payload) to round `t` (default: the round after the
      previous call); every rank of the world makes the matching call.
    * no handle: `contribution_or_null` holds all P ranks' rows (P=1 also
      accepts a single vector); the P ranks run on the current GPU and the
      common result is returned.
    Raises ValueError on a length mismatch (SPEC: errors: length-mismatch)."""
    return _spec_allreduce(SYNC, cfg, contribution_or_null, handle, t, timeout)


def allreduce_solo(cfg: CollectiveConfig, contribution_or_null, *, handle=None, t=None,
                   timeout: float = 30.0) -> CollectiveResult:
    """SPEC.md:197-205 `allreduce_solo(cfg, contribution_or_null)`: the first
    arriving rank starts the round for everyone; later ranks contribute what
    their send buffer holds (null if nothing).  Call forms as allreduce_sync."""
    return _spec_allreduce(SOLO, cfg, contribution_or_null, handle, t, timeout)


def allreduce_majority(cfg: CollectiveConfig, contribution_or_null, *, handle=None, t=None,
                       timeout: float = 30.0) -> CollectiveResult:
    """SPEC.md:206-214 `allreduce_majority(cfg, contribution_or_null)`: only
    initiator_for_round(cfg.seed, t, P)'s arrival starts the round.  Call forms
    as allreduce_sync."""
    return _spec_allreduce(MAJORITY, cfg, contribution_or_null, handle, t, timeout)


def tree_order_sum(vectors, divide: bool = False) -> torch.Tensor:
    """collectives.py:385-403 on the device: the fixed association the engine
    uses, dtype-preserving.  Accepts torch tensors (one device) or arrays.
    divide=True also divides by the vector count exactly as a round does
    (collectives.py:254-260; eagersgd.py:170-174's resync average)."""
    vs = list(vectors)
    p = len(vs)
    if p == 0:
        raise ValueError("no vectors")
    first = vs[0]
    if isinstance(first, torch.Tensor) and first.is_cuda:
        device = first.device.index
        dtype = first.dtype
    else:
        device = torch.cuda.current_device()
        dtype = torch.as_tensor(np.asarray(first)).dtype
    code = {torch.float32: _lib.EC_F32, torch.float64: _lib.EC_F64, torch.int64: _lib.EC_I64}[dtype]
    ts = [_as_device(v, dtype, device) for v in vs]
    n = ts[0].numel()
    out = torch.empty(n, dtype=dtype, device=f"cuda:{device}")
    srcs = (C.c_void_p * p)(*[t.data_ptr() for t in ts])
    with torch.cuda.device(device):
        call("ec_local_reduce", srcs, p, (1 << p) - 1 if p < 64 else _lib.UINT64_MAX,
             out.data_ptr(), n, code, int(divide), _stream_ptr(device))
    return out


__all__ = [
    "SOLO", "MAJORITY", "SYNC", "FLAVORS", "CollectiveConfig", "CollectiveResult",
    "AllreduceHandle", "initiator_for_round", "ceil_log2", "floor_pow2", "run_allreduce",
    "tree_order_sum", "drive", "EmulatedWorld", "ProcessWorld", "allreduce_sync",
    "allreduce_solo", "allreduce_majority",
]
