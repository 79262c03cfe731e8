"""Run one c1 replay with short timeouts; dump every engine's state on failure."""
import ctypes as C
import os
import sys
import threading
import time

os.environ["CUDA_MODULE_LOADING"] = "EAGER"
os.environ.setdefault("EC_TIMEOUT_S", "10")
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_04207_b200 import _lib, EmulatedWorld  # noqa: E402
import paper_1908_04207_b200.replay as RP  # noqa: E402

FIELDS = ["done_gen1", "req_done", "error", "error_info", "exited", "snap_gen1", "stop", "pin_lo",
          "stream_status", "g", "snapped", "contrib", "internal_act", "cmd_seq", "round_done",
          "next_req"]
flavor = sys.argv[1] if len(sys.argv) > 1 else "sync"
element = sys.argv[2] if len(sys.argv) > 2 else "f8"
tr = dict(np.load(f"tests/golden/c1_{flavor}.npz"))
world = EmulatedWorld(int(tr["p"]), 0, ring_slots=4)


def watchdog():
    time.sleep(45)
    for cid, comm in world.comms.items():
        for li in range(comm.n_local):
            out = (C.c_int64 * 16)()
            _lib.call("ec_debug_state", comm.ptr, li, out)
            print("cid", cid, "rank", li, dict(zip(FIELDS, list(out))), flush=True)
    os._exit(3)


threading.Thread(target=watchdog, daemon=True).start()
t0 = time.time()
out = RP.replay_training(tr, element=element, world=world)
print("replay done in %.2fs" % (time.time() - t0))
print("accepted ok", out["accepted"].tolist() == tr["accepted"].tolist())
print("masks ok", out["masks"].tolist() == tr["masks"].tolist())
print("w bitexact", out["w"].tobytes() == tr["final_w"].tobytes(),
      np.abs(out["w"] - tr["final_w"]).max(), flush=True)
for cid, comm in world.comms.items():
    for li in range(comm.n_local):
        o = (C.c_int64 * 16)()
        _lib.call("ec_debug_state", comm.ptr, li, o)
        print("pre-close cid", cid, "rank", li, dict(zip(FIELDS, list(o))), flush=True)
t1 = time.time()
for cid, comm in list(world.comms.items()):
    try:
        comm.pause(8000)
        print("paused cid", cid, "%.3fs" % (time.time() - t1), flush=True)
    except Exception as e:
        print("pause failed cid", cid, e, flush=True)
        for li in range(comm.n_local):
            o = (C.c_int64 * 16)()
            _lib.call("ec_debug_state", comm.ptr, li, o)
            print("  cid", cid, "rank", li, dict(zip(FIELDS, list(o))), flush=True)
os._exit(0)
