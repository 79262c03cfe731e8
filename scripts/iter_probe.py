"""Checked-build probe of the controller's loop cadence around a step's offer
(EC_DEBUG_LIB=1; torchrun, 2 ranks): prints, for the last steps, the
controller's iteration starts relative to the offer's post stamp."""
import ctypes as C
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("EC_IDLE_PARK_MS", "0")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    from paper_1908_04207_b200 import (AllreduceHandle, CollectiveConfig, ProcessWorld, TrainState,
                                       _lib, finish_step, train_step_async)
    pw = ProcessWorld()
    n = 25_559_081
    h = AllreduceHandle(CollectiveConfig(p=world, flavor="solo", vector_len=n, element="f4"),
                        rank, pw)
    st = TrainState.fresh(torch.zeros(n, device="cuda"), 0.05, rank=rank, tau=None)
    h.grad_buffer().normal_()
    pend = []
    for t in range(40):
        pend.append(train_step_async(st, h, h.grad_buffer(), all_arrive=True))
        if len(pend) > 2:
            finish_step(st, h, pend.pop(0))
    while pend:
        finish_step(st, h, pend.pop(0))
    torch.cuda.current_stream().synchronize()
    if rank == 0:
        for t in range(33, 40):
            a = (C.c_uint64 * 4)()
            _lib.call("ec_step_times", h.comm.ptr, 0, t, a)
            it = (C.c_uint64 * 80)()
            _lib.call("ec_step_iterations", h.comm.ptr, 0, t, it)
            post = a[2]
            print(f"step {t}: post->seen {(a[3] - post) / 1e3:.2f} us; iteration starts "
                  f"(us rel. post): {[round((x - post) / 1e3, 2) for x in it[:16] if x]}")
            for i in range(15):
                b = it[i]
                secs = [it[16 + 4 * i + k] for k in range(4)]
                if b and all(secs):
                    d = [round((x - b) / 1e3, 2) for x in secs] + [round((it[i + 1] - b) / 1e3, 2)]
                    print("   sections (hp, req, snap/issue, publish, next):", d)
    h.close()
    pw.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
