"""Diagnose the persistent engine on one GPU: start an emulated world, post
requests, dump engine state."""
import ctypes as C
import os
os.environ["CUDA_MODULE_LOADING"] = "EAGER"
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1908_04207_b200 import _lib, CollectiveConfig, EmulatedWorld, AllreduceHandle  # noqa

FIELDS = ["done_gen1", "req_done", "error", "error_info", "exited", "snap_gen1", "stop", "pin_lo",
          "stream_status", "g", "snapped", "contrib", "internal_act", "cmd_seq", "round_done",
          "next_req"]


def dump(h, tag):
    out = (C.c_int64 * 16)()
    _lib.call("ec_debug_state", h.comm.ptr, h.li, out)
    print(tag, dict(zip(FIELDS, list(out))), flush=True)


p = int(sys.argv[1]) if len(sys.argv) > 1 else 2
world = EmulatedWorld(p)
cfg = CollectiveConfig(p=p, flavor="sync", vector_len=8, element="f4")
hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
hs[0]._ensure_started()
time.sleep(0.5)
for h in hs:
    dump(h, f"after start r{h.rank}")
seq = C.c_uint64()
_lib.call("ec_post_hold", hs[0].comm.ptr, 0, 5, C.byref(seq))
time.sleep(0.2)
dump(hs[0], "after host HOLD")
s = hs[0]._post_contribute(0, 1 | 2)
time.sleep(0.2)
dump(hs[0], "after stream CONTRIB")
print("err", torch.cuda.current_stream().query())
for r in range(1, p):
    hs[r]._post_contribute(0, 3)
time.sleep(0.5)
for h in hs:
    dump(h, f"after all contrib r{h.rank}")
world.close()
print("closed")
