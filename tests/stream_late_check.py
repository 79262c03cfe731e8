"""Does creating a torch stream block while a persistent engine is resident
(after warm_device_libraries initialised torch's stream pool)?  Two emulated
ranks, one round, then torch.cuda.Stream() in a thread with a deadline."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1908_04207_b200 import CollectiveConfig, EmulatedWorld, run_allreduce

print("start", flush=True)
cfg = CollectiveConfig(p=2, flavor="sync", vector_len=1024, element="f4")
res, hs, world = run_allreduce(cfg, np.ones((2, 1024), np.float32))
print("round done; engines running:", [c.running for c in world.comms.values()], flush=True)
world.resume()
assert any(c.running for c in world.comms.values())
out = {}


def mk():
    print("creating stream", flush=True)
    out["s"] = torch.cuda.Stream()
    print("stream created", flush=True)
    out["e"] = torch.cuda.Event()
    out["e"].record(out["s"])


th = threading.Thread(target=mk, daemon=True)
th.start()
th.join(20)
print("stream created while the engine runs:", not th.is_alive())
os._exit(0 if not th.is_alive() else 1)
