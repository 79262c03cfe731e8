"""Worlds: where the P ranks of a partial collective live.

The reference's `transport` argument (`SimTransport` / `SocketTransport`,
transport.py:169-501) is replaced by a device world:

* `ProcessWorld` -- one rank per process and GPU (torchrun).  Each collective
  instance (`cid`) allocates its buffers, exports CUDA IPC handles and maps every
  peer's over NVLink/NVSwitch.  torch.distributed (any backend, normally gloo)
  is used only to all-gather those handles at init and for the barrier in
  `pause()`; no collective of it ever runs on the round path.
* `EmulatedWorld` -- all P ranks in this process on one GPU, one engine launch
  serving every rank (CTA groups per rank).  Used by the tests and by one-GPU
  reproductions of multi-rank protocols; peer memory is simply local memory.

Both start one persistent engine per collective instance, lazily, and can
`pause()` it (drain to a round boundary and exit) so that device-wide
synchronisation such as `torch.cuda.synchronize()` returns, then `resume()`.
"""

from __future__ import annotations

import atexit
import ctypes as C
import threading
import weakref

import torch

from . import _lib
from ._lib import call, lib

_LIVE: "weakref.WeakSet" = weakref.WeakSet()

ELEMENTS = {
    "f4": (_lib.EC_F32, torch.float32),
    "f8": (_lib.EC_F64, torch.float64),
    "i8": (_lib.EC_I64, torch.int64),
}
FLAVOR_CODE = {"sync": _lib.EC_SYNC, "solo": _lib.EC_SOLO, "majority": _lib.EC_MAJORITY}


class _CudaMem:
    """Zero-copy torch view of library-owned device memory."""

    def __init__(self, ptr: int, n: int, dtype: torch.dtype, owner):
        self._owner = owner  # keep the communicator alive while viewed
        typestr = {torch.float32: "<f4", torch.float64: "<f8", torch.int64: "<i8"}[dtype]
        self.__cuda_array_interface__ = {
            "shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 2,
            "strides": None,
        }


class Comm:
    """One collective instance (cid) of a world: wraps an ec_comm_t."""

    def __init__(self, world, cfg, rank_lo: int, n_local: int):
        self.world = world
        self.cfg = cfg
        self.p = cfg.p
        self.n = cfg.vector_len
        self.dtype_code, self.torch_dtype = ELEMENTS[cfg.element]
        self.device = world.device
        self.rank_lo = rank_lo
        self.n_local = n_local
        self.ring_slots = world.ring_slots
        self.ptr = C.c_void_p()
        with torch.cuda.device(self.device):
            call("ec_comm_create", cfg.p, rank_lo, n_local, self.device, cfg.vector_len,
                 self.dtype_code, FLAVOR_CODE[cfg.flavor], self.ring_slots, world.workers,
                 C.byref(self.ptr))
        if getattr(cfg, "majority_quorum", False):
            call("ec_comm_set_quorum", self.ptr, (cfg.p + 1) // 2)
        self.running = False
        self.closed = False
        self.nvls = False
        self.lock = threading.Lock()
        self._views: dict = {}
        self.replay_masks: dict = {}

    # -- plumbing -----------------------------------------------------------
    def export(self, li: int) -> bytes:
        buf = (C.c_char * 512)()
        n = C.c_size_t()
        call("ec_comm_export", self.ptr, li, buf, 512, C.byref(n))
        return bytes(buf[: n.value])

    def import_peer(self, rank: int, blob: bytes) -> None:
        call("ec_comm_import", self.ptr, rank, blob, len(blob))

    def set_replay(self, li: int, masks) -> None:
        arr = (C.c_uint64 * len(masks))(*[int(m) for m in masks])
        call("ec_comm_set_replay", self.ptr, li, arr, len(masks))

    def start(self) -> None:
        with self.lock:
            if not self.running and not self.closed:
                with torch.cuda.device(self.device):
                    call("ec_comm_start", self.ptr)
                self.running = True

    def pause(self, timeout_ms: int = 30000) -> None:
        with self.lock:
            if self.running:
                call("ec_comm_pause", self.ptr, timeout_ms)
                self.running = False

    def close(self) -> None:
        with self.lock:
            if self.closed:
                return
            rc = lib.ec_comm_destroy(self.ptr)
            self.closed = True
            self.running = False
            if rc < 0:
                raise _lib.EcError("ec_comm_destroy", rc, lib.ec_last_error().decode())

    def error(self, li: int):
        code, info = C.c_uint64(), C.c_uint64()
        call("ec_comm_error", self.ptr, li, C.byref(code), C.byref(info))
        return code.value, info.value

    # -- tensors ------------------------------------------------------------
    @property
    def progressive(self) -> bool:
        """Async steps update each chunk of the round's result as it lands."""
        return lib.ec_comm_progressive(self.ptr) == 1

    def send_view(self, li: int) -> torch.Tensor:
        key = ("send", li)
        if key not in self._views:
            ptr = lib.ec_send_ptr(self.ptr, li)
            self._views[key] = torch.as_tensor(_CudaMem(ptr, self.n, self.torch_dtype, self),
                                               device=f"cuda:{self.device}")
        return self._views[key]

    def grad_view(self, li: int) -> torch.Tensor:
        key = ("grad", li)
        if key not in self._views:
            ptr = lib.ec_grad_ptr(self.ptr, li)
            self._views[key] = torch.as_tensor(_CudaMem(ptr, self.n, self.torch_dtype, self),
                                               device=f"cuda:{self.device}")
        return self._views[key]

    def slot_view(self, li: int, gen: int) -> torch.Tensor:
        key = ("slot", li, gen % self.ring_slots)
        if key not in self._views:
            ptr = lib.ec_slot_ptr(self.ptr, li, gen)
            self._views[key] = torch.as_tensor(_CudaMem(ptr, self.n, self.torch_dtype, self),
                                               device=f"cuda:{self.device}")
        return self._views[key]


def warm_device_libraries(device: int) -> None:
    """Initialise cuBLAS (and torch's allocator/streams) before any engine runs.

    A persistent engine never finishes, so anything that synchronises the whole
    device -- cuBLAS handle/workspace creation on the first matmul, cudaFree in
    the caching allocator -- would wait on it forever.  Worlds call this at
    construction; code that initialises other libraries late should do so inside
    `world.quiesced()`.
    """
    with torch.cuda.device(device):
        a = torch.ones(64, 64, device=f"cuda:{device}")
        (a @ a).sum().item()
        (a @ a[:, 0]).sum().item()
        torch.cuda.current_blas_handle()
        # torch's stream pool is created on the first torch.cuda.Stream(); that
        # first creation was seen to block behind a resident engine
        for _ in range(2):
            s = torch.cuda.Stream(device)
            e = torch.cuda.Event()
            e.record(s)
        torch.cuda.synchronize(device)


class _WorldBase:
    device: int
    ring_slots: int
    workers: int

    def __init__(self):
        self.comms: dict = {}
        self._lock = threading.Lock()
        _LIVE.add(self)

    def pause(self, timeout_ms: int = 30000) -> None:
        for comm in list(self.comms.values()):
            comm.pause(timeout_ms)

    def resume(self) -> None:
        for comm in list(self.comms.values()):
            comm.start()

    def close(self) -> None:
        # Park every engine before freeing anything: cudaFree synchronises the
        # whole device and would wait forever on a still-resident engine.
        comms = list(self.comms.values())
        for comm in comms:
            try:
                comm.pause(10000)
            except Exception:
                pass
        for comm in comms:
            try:
                comm.close()
            except Exception:
                pass
        self.comms.clear()

    def release(self, cid: int) -> None:
        """Destroy one collective instance.  Every engine of the world parks first
        (cudaFree synchronises the device); collective in a ProcessWorld."""
        comm = self.comms.get(cid)
        if comm is None:
            return
        running = [c for c in self.comms.values() if c.running and c is not comm]
        self.pause()
        self._barrier()
        comm.close()
        del self.comms[cid]
        self._release_attached(cid)
        self._barrier()
        for c in running:
            c.start()

    def _barrier(self) -> None:
        pass

    def _release_attached(self, cid: int) -> None:
        pass

    def _new_comm(self, cfg, rank_lo: int, n_local: int) -> "Comm":
        """Create a communicator with the world's engines parked (allocation and
        IPC registration may synchronise the device)."""
        running = [c for c in self.comms.values() if c.running]
        for c in running:
            c.pause()
        try:
            return Comm(self, cfg, rank_lo, n_local)
        finally:
            for c in running:
                c.start()

    def quiesced(self):
        """Context manager: engines parked inside (device-wide syncs are safe)."""
        world = self

        class _Q:
            def __enter__(self_inner):
                world.pause()
                return world

            def __exit__(self_inner, *exc):
                world.resume()
                return False

        return _Q()

    def synchronize(self) -> None:
        """torch.cuda.synchronize() with the engines parked around it."""
        with self.quiesced():
            torch.cuda.synchronize(self.device)


class EmulatedWorld(_WorldBase):
    """All P ranks in this process, on one GPU."""

    def __init__(self, p: int, device: int = 0, ring_slots: int = 3, workers: int = 0):
        super().__init__()
        if p < 1:
            raise ValueError("p must be >= 1")
        self.p = p
        self.device = device
        self.ring_slots = ring_slots
        self.workers = workers
        self._attached: dict = {}
        warm_device_libraries(device)

    def attach(self, cfg, cid: int, rank: int):
        if cfg.p != self.p:
            raise ValueError(f"config p={cfg.p} does not match the world's p={self.p}")
        if not 0 <= rank < self.p:
            raise ValueError(f"rank {rank} out of range")
        with self._lock:
            comm = self.comms.get(cid)
            if comm is None:
                comm = self._new_comm(cfg, 0, self.p)
                self.comms[cid] = comm
                self._attached[cid] = set()
            elif comm.cfg != cfg:
                raise ValueError(f"cid {cid} already bound to {comm.cfg}")
            if rank in self._attached[cid]:
                raise ValueError(f"rank {rank} already has a handle for cid {cid}")
            self._attached[cid].add(rank)
        return comm, rank

    def _release_attached(self, cid: int) -> None:
        self._attached.pop(cid, None)


class ProcessWorld(_WorldBase):
    """One rank per process/GPU; peers mapped over NVLink with CUDA IPC."""

    def __init__(self, rank: int | None = None, p: int | None = None, device: int | None = None,
                 group=None, ring_slots: int = 3, workers: int = 0):
        super().__init__()
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        if not dist.is_initialized() and (p or 1) > 1:
            raise RuntimeError("ProcessWorld needs torch.distributed initialised (any backend)")
        self.rank = dist.get_rank(group) if rank is None else rank
        self.p = dist.get_world_size(group) if p is None else p
        self.device = torch.cuda.current_device() if device is None else device
        self.ring_slots = ring_slots
        self.workers = workers
        warm_device_libraries(self.device)

    def _all_gather(self, obj):
        if self.p == 1:
            return [obj]
        out = [None] * self.p
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def barrier(self) -> None:
        if self.p > 1:
            self.dist.barrier(group=self.group)

    def _barrier(self) -> None:
        self.barrier()

    def attach(self, cfg, cid: int, rank: int):
        if rank != self.rank:
            raise ValueError(f"this process is rank {self.rank}, not {rank}")
        if cfg.p != self.p:
            raise ValueError(f"config p={cfg.p} does not match world size {self.p}")
        if cid in self.comms:
            raise ValueError(f"cid {cid} already has a handle in this process")
        comm = self._new_comm(cfg, self.rank, 1)
        blobs = self._all_gather(comm.export(0))
        for q, blob in enumerate(blobs):
            comm.import_peer(q, blob)
        if (cfg.reduction_mode == "fast" and cfg.element == "f4" and self.p > 1
                and all(self._all_gather(bool(lib.ec_nvls_supported(self.device))))):
            self._setup_nvls(comm)
        self.comms[cid] = comm
        self.barrier()
        return comm, 0

    def _setup_nvls(self, comm: "Comm") -> None:
        """Multicast object over every rank's GPU (fabric handle shared over the
        process group); see ec_nvls_create/attach/bind.  Any rank failing before
        the bind leaves every rank on the fixed-order engine (a valid "fast")."""
        import os
        import secrets
        import socket
        import struct
        import warnings
        fabric = os.environ.get("EC_NVLS_HANDLE") == "fabric"
        # Linux abstract-namespace socket (no file to squat on) with a random
        # name; rank 0 hands the descriptor only to the world's own processes
        # (SO_PEERCRED pid and uid checked against the all-gathered pids)
        path = "\0ec_nvls_" + self._all_gather(secrets.token_hex(16))[0]
        pids = self._all_gather(os.getpid())
        msg = (True, b"")
        srv = None
        if self.rank == 0:
            try:
                buf = (C.c_char * 256)()
                n = C.c_size_t()
                call("ec_nvls_create", comm.ptr, buf, 256, C.byref(n))
                msg = (True, bytes(buf[: n.value]))
                if not fabric:     # the descriptor travels over a Unix socket (SCM_RIGHTS)
                    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
                    srv.bind(path)
                    srv.listen(self.p)
            except Exception as e:  # noqa: BLE001 - reported below, collectively
                msg = (False, str(e).encode())
        ok, blob = self._all_gather(msg)[0]
        if not ok:
            warnings.warn(f"NVLS unavailable ({blob.decode()}); fast mode uses the fixed-order engine")
            return
        if not fabric:
            if self.rank == 0:
                fd = struct.unpack("i", blob[:4])[0]
                want = set(pids[1:])
                srv.settimeout(60.0)
                while want:
                    conn, _ = srv.accept()
                    cred = conn.getsockopt(socket.SOL_SOCKET, socket.SO_PEERCRED,
                                           struct.calcsize("3i"))
                    pid, uid, _gid = struct.unpack("3i", cred)
                    if pid in want and uid == os.getuid():
                        socket.send_fds(conn, [b"x"], [fd])
                        want.discard(pid)
                    conn.close()
            else:
                cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
                for _ in range(200):
                    try:
                        cli.connect(path)
                        break
                    except OSError:
                        import time
                        time.sleep(0.05)
                _, fds, _, _ = socket.recv_fds(cli, 16, 1)
                cli.close()
                blob = struct.pack("i", fds[0])
            self.barrier()
            if srv is not None:
                srv.close()
        err = ""
        try:
            call("ec_nvls_attach", comm.ptr, blob, len(blob))
        except Exception as e:  # noqa: BLE001
            err = str(e)
        errs = [x for x in self._all_gather(err) if x]
        if errs:
            warnings.warn(f"NVLS attach failed ({errs[0]}); fast mode uses the fixed-order engine")
            return
        call("ec_nvls_bind", comm.ptr)       # every device was added before any bind
        comm.nvls = True
        self.barrier()

    def pause(self, timeout_ms: int = 30000) -> None:
        # Every rank must have stopped posting before any engine parks, otherwise
        # a parked peer stalls rounds that still need it.
        self.barrier()
        super().pause(timeout_ms)


@atexit.register
def _shutdown_all() -> None:
    for w in list(_LIVE):
        try:
            w.close()
        except Exception:
            pass
