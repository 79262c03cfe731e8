"""Can ordinary kernels run while the persistent engine is resident?"""
import ctypes as C
import os
os.environ["CUDA_MODULE_LOADING"] = "EAGER"
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1908_04207_b200 import _lib, CollectiveConfig, EmulatedWorld, AllreduceHandle  # noqa


def wait_q(stream, tag, timeout=5.0):
    t0 = time.time()
    while not stream.query():
        if time.time() - t0 > timeout:
            print(tag, "STUCK", flush=True)
            return False
        time.sleep(0.001)
    print(tag, "ok %.3f ms" % ((time.time() - t0) * 1e3), flush=True)
    return True


p = 2
world = EmulatedWorld(p)
cfg = CollectiveConfig(p=p, flavor="sync", vector_len=8, element="f4")
hs = [AllreduceHandle(cfg, r, world) for r in range(p)]
hs[0]._ensure_started()
time.sleep(0.2)
s_legacy = torch.cuda.default_stream()
s_nb = torch.cuda.Stream()
_lib.call("ec_spin", 0, s_nb.cuda_stream)
wait_q(s_nb, "spin on torch side stream")
_lib.call("ec_spin", 0, 0)
wait_q(s_legacy, "spin on legacy stream")
x = torch.ones(10, device="cuda")
y = x + 1
wait_q(s_legacy, "torch add on legacy stream")
print("done", flush=True)
import os
os._exit(0)
