"""CPU tests of the host side: the C ABI exports, configuration rules,
initiator / delay models against the reference's tables, the guard threshold,
and a world_size-2 gloo exchange of the init-time handle blobs."""

import json
import os
import socket

import numpy as np
import pytest

from paper_1908_04207_b200 import _lib
from paper_1908_04207_b200.collectives import CollectiveConfig, initiator_for_round
from paper_1908_04207_b200.eagersgd import (
    LrBoundParams, TrainState, hold_threshold, max_learning_rate, min_iterations,
)
from paper_1908_04207_b200.transport import DelayModel, delay_table, delayed_ranks, inject_delay


def test_library_exports_every_header_symbol():
    syms = _lib.header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(_lib.lib, s)]
    assert not missing
    assert _lib.lib.ec_version() >= 10000


def test_checked_build_exports_every_header_symbol():
    """The checked build (device assertions, build.py --debug, EC_DEBUG_LIB=1)
    is the same ABI."""
    import ctypes as C
    import os
    path = os.path.join(os.path.dirname(_lib.LIB_PATH), "libeagercoll_b200_debug.so")
    if not os.path.exists(path):
        pytest.skip("checked build not built (python -m paper_1908_04207_b200.build --debug)")
    dbg = C.CDLL(path)
    assert not [s for s in _lib.header_symbols() if not hasattr(dbg, s)]


def test_abi_argument_errors_without_gpu():
    # argument validation happens before any CUDA call
    import ctypes as C
    out = C.c_void_p()
    rc = _lib.lib.ec_comm_create(0, 0, 1, 0, 10, 0, 1, 2, 0, C.byref(out))
    assert rc == -1 and b"world_size" in _lib.lib.ec_last_error()
    rc = _lib.lib.ec_comm_create(2, 0, 1, 0, 10, 7, 1, 2, 0, C.byref(out))
    assert rc == -1 and b"dtype" in _lib.lib.ec_last_error()
    assert _lib.lib.ec_sgd_update(None, None, 0.1, 1, 0, None) == -1
    assert _lib.lib.ec_local_reduce(None, 0, 0, None, 1, 0, 0, None) == -1
    with pytest.raises(_lib.EcError):
        _lib.call("ec_sgd_update", None, None, 0.1, 1, 0, None)


def test_collective_config_validation():
    CollectiveConfig(p=2, flavor="solo", vector_len=3)
    for kw in (dict(p=0), dict(flavor="x"), dict(vector_len=0), dict(element="f2"),
               dict(p=65), dict(reduction_mode="fastest")):
        args = dict(p=2, flavor="solo", vector_len=3)
        args.update(kw)
        with pytest.raises(ValueError):
            CollectiveConfig(**args)
    c = CollectiveConfig(p=70 - 6, flavor="sync", vector_len=10, element="f4")
    assert c.mask_words == 1 and c.payload_nbytes == 40


def test_initiator_and_delays_match_reference_tables(golden_dir):
    with open(os.path.join(golden_dir, "protocol.json")) as f:
        proto = json.load(f)
    for seed, vals in proto["initiator"].items():
        got = [initiator_for_round(int(seed), t, p) for p in (1, 2, 3, 4, 8) for t in range(64)]
        assert got == vals
    for key, rows in proto["delayed_ranks"].items():
        seed, k = map(int, key.split(","))
        m = DelayModel("random_subset", 0.2, k, seed)
        assert [list(delayed_ranks(m, rnd, 8)) for rnd in range(32)] == rows
    m = DelayModel("random_subset", 0.2, 1, 11)
    tab = delay_table(m, 8, 16)
    assert tab.T.tolist() == proto["inject_delay"]["subset"]
    assert inject_delay(3, 0, DelayModel("linear_skew", 1.0), 8) == 4000
    with pytest.raises(ValueError):
        DelayModel("bogus")


def test_guard_threshold_matches_reference_table(golden_dir):
    with open(os.path.join(golden_dir, "known_answers.json")) as f:
        rows = json.load(f)["guard_table"]

    class FakeBuf:
        def __init__(self, pending):
            self.pending_rounds = pending

    for tau, pending, in_prog, contributed, gen, held in rows:
        st = TrainState.__new__(TrainState)
        st.tau, st.in_progress, st.send_buf = tau, in_prog, FakeBuf(pending)
        thr = hold_threshold(st)
        assert held == (gen >= thr and contributed < gen)


def test_lr_bound_helpers():
    p = LrBoundParams(L=1.0, M=1.0, tau=1, p=2, q=1, eps=0.12, f0_minus_m=1.0)
    assert abs(max_learning_rate(p) - 0.01) < 1e-15
    assert min_iterations(p, 0.01) == 20000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        # the init-time exchange ProcessWorld performs: every rank's handle blob
        blob = bytes([rank]) * 80
        out = [None] * world
        dist.all_gather_object(out, blob)
        # every rank derives the same initiator sequence locally (no messages)
        seq = [initiator_for_round(1234, t, world) for t in range(32)]
        seqs = [None] * world
        dist.all_gather_object(seqs, seq)
        dist.barrier()
        q.put((rank, [b[0] for b in out], all(s == seqs[0] for s in seqs)))
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_2_handle_exchange():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for pr in procs:
        pr.join(60)
    assert res == [(0, [0, 1], True), (1, [0, 1], True)]


def _process_world_worker(rank, world, port, q):
    """ProcessWorld's real host logic over gloo, with the device layer faked
    (no GPU here): attach exchanges every rank's export blob through the
    process group and imports each peer's under its own rank, a second
    communicator gets its own exchange, and release/close are collective."""
    import struct

    import torch.distributed as dist

    import paper_1908_04207_b200.world as W
    from paper_1908_04207_b200.collectives import CollectiveConfig

    calls = []

    class FakeComm:
        def __init__(self, world_, cfg, rank_lo, n_local):
            self.cfg, self.rank_lo, self.n_local = cfg, rank_lo, n_local
            self.running, self.closed, self.nvls = False, False, False
            self.imports = {}

        def export(self, li):
            # the C blob's header fields (BlobV1: magic, rank, n, dtype, R)
            return struct.pack("<Iiqii", 0x45434231, self.rank_lo + li, self.cfg.vector_len, 0, 3)

        def import_peer(self, r, blob):
            magic, br, n, _dt, _ring = struct.unpack("<Iiqii", blob[:24])
            assert magic == 0x45434231 and br == r and n == self.cfg.vector_len
            self.imports[r] = br
            calls.append(("import", self.cfg.vector_len, r))

        def start(self):
            self.running = True

        def pause(self, timeout_ms=30000):
            calls.append(("pause", self.cfg.vector_len))
            self.running = False

        def close(self):
            calls.append(("close", self.cfg.vector_len))
            self.closed = True

    W.Comm = FakeComm
    W.warm_device_libraries = lambda device: None
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        pw = W.ProcessWorld(device=0)
        c1, li = pw.attach(CollectiveConfig(p=world, flavor="solo", vector_len=7, element="f4"),
                           0, rank)
        c2, _ = pw.attach(CollectiveConfig(p=world, flavor="sync", vector_len=9, element="f4"),
                          1, rank)
        errs = []
        for bad in (lambda: pw.attach(CollectiveConfig(p=world + 1, flavor="solo", vector_len=7),
                                      2, rank),
                    lambda: pw.attach(CollectiveConfig(p=world, flavor="solo", vector_len=7),
                                      0, rank),
                    lambda: pw.attach(CollectiveConfig(p=world, flavor="solo", vector_len=7),
                                      3, (rank + 1) % world)):
            try:
                bad()
            except ValueError:
                errs.append(True)
        pw.release(1)
        pw.close()
        q.put((rank, li, sorted(c1.imports.items()), sorted(c2.imports.items()), len(errs),
               calls.count(("close", 9)), calls.count(("close", 7)), 1 in pw.comms))
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_2_process_world_exchange():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_process_world_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for pr in procs:
        pr.join(60)
    for rank, li, imp1, imp2, nerr, closed9, closed7, still in res:
        assert li == 0
        assert imp1 == [(0, 0), (1, 1)] and imp2 == [(0, 0), (1, 1)]
        assert nerr == 3                      # wrong p, duplicate cid, foreign rank
        assert closed9 == 1 and closed7 == 1 and not still
