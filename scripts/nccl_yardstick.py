"""Off-path yardstick: NCCL all_reduce bus bandwidth on the
same box, same sizes, fp32, device-timed (CUDA events, max over ranks).

    torchrun --nproc-per-node P scripts/nccl_yardstick.py [--sizes 1K,1M,100M,1G]

Not part of the product path (a blocking all-participant collective is what
partial collectives remove); printed beside the engine's sweep for scale."""

import argparse
import json
import os

import torch
import torch.distributed as dist


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1K,64K,1M,16M,100M,256M,1G")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    p = dist.get_world_size()
    mult = {"K": 1 << 10, "M": 1_000_000, "G": 1 << 30}
    out = {"p": p, "nccl": torch.cuda.nccl.version(), "rows": []}
    for s in args.sizes.split(","):
        nbytes = int(s[:-1]) * mult[s[-1]] if s[-1] in mult else int(s)
        n = max(1, nbytes // 4)
        x = torch.randn(n, device="cuda")
        for _ in range(5):
            dist.all_reduce(x)
        iters = args.iters if nbytes < (256 << 20) else 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            dist.all_reduce(x)
        e1.record()
        e1.synchronize()
        us = torch.tensor([e0.elapsed_time(e1) * 1e3 / iters], device="cuda")
        dist.all_reduce(us, op=dist.ReduceOp.MAX)
        us = float(us.item())
        bus = 2 * (p - 1) / p * 4 * n
        out["rows"].append({"bytes": 4 * n, "us": us, "busbw_gbs": bus / (us * 1e-6) / 1e9})
    if dist.get_rank() == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
