"""Bytes that cross NVLink per partial-allreduce round, from the NVLink data
throughput counters (`nvidia-smi nvlink -gt d`), read on every GPU before and
after K back-to-back rounds.  Expected per rank and direction:
2(P-1)/P * S (two-shot: pull my shard from P-1 peers + push it to them, and
serve the peers' pulls / receive their pushes), plus control words.

    torchrun --nproc-per-node P scripts/nvlink_bytes.py [--bytes 100000000] [--rounds 100]
"""

import argparse
import json
import os
import re
import subprocess
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def _nvml_counters(dev: int):
    """(tx, rx) bytes summed over the GPU's NVLinks from NVML field values
    (NVLINK_COUNT_XMIT/RCV_BYTES per link, else THROUGHPUT_DATA_TX/RX in KiB)."""
    import pynvml as N
    N.nvmlInit()
    h = N.nvmlDeviceGetHandleByIndex(dev)
    for tx_id, rx_id, scale in ((N.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
                                 N.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, 1),
                                (N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
                                 N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 1024)):
        tx = rx = 0
        ok = False
        for link in range(18):
            try:
                vals = N.nvmlDeviceGetFieldValues(h, [(tx_id, link), (rx_id, link)])
            except Exception:
                continue
            for v, which in zip(vals, ("tx", "rx")):
                if v.nvmlReturn != 0:
                    continue
                ok = True
                x = v.value.ullVal * scale
                if which == "tx":
                    tx += x
                else:
                    rx += x
        if ok and (tx or rx):
            return (tx, rx), ""
    return None, "NVML NVLink byte counters unsupported"


def counters(dev: int):
    """(tx, rx) bytes summed over the GPU's links, or None if unsupported."""
    try:
        c, err = _nvml_counters(dev)
        if c:
            return c, ""
    except Exception as e:  # noqa: BLE001
        err = str(e)
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(dev)],
                             capture_output=True, text=True, timeout=30).stdout
    except Exception:
        return None, err
    tx = sum(int(x) for x in re.findall(r"Tx:\s*(\d+)\s*KiB", out))
    rx = sum(int(x) for x in re.findall(r"Rx:\s*(\d+)\s*KiB", out))
    if not tx and not rx:
        return None, err + " | nvidia-smi: " + out[-200:]
    return (tx * 1024, rx * 1024), ""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=100_000_000)
    ap.add_argument("--rounds", type=int, default=100)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    from paper_1908_04207_b200 import AllreduceHandle, CollectiveConfig, ProcessWorld
    from paper_1908_04207_b200.harness import rounds_pipelined
    pw = ProcessWorld()
    n = args.bytes // 4
    h = AllreduceHandle(CollectiveConfig(p=world, flavor="solo", vector_len=n, element="f4"),
                        rank, pw, cid=1)
    h.send_buffer().normal_()
    torch.cuda.current_stream().synchronize()
    rounds_pipelined(h, 0, 3)
    dist.barrier()
    c0, err = counters(local)
    dist.barrier()
    ms = rounds_pipelined(h, 3, args.rounds)
    dist.barrier()
    c1, _ = counters(local)
    res = {"rank": rank, "ms": ms}
    if c0 and c1:
        res["tx_bytes_per_round"] = (c1[0] - c0[0]) / args.rounds
        res["rx_bytes_per_round"] = (c1[1] - c0[1]) / args.rounds
    else:
        res["error"] = err or "no counters"
    allr = [None] * world
    dist.all_gather_object(allr, res)
    h.close()
    pw.close()
    if rank == 0:
        exp = 2 * (world - 1) / world * args.bytes
        print(json.dumps({"p": world, "bytes": args.bytes, "rounds": args.rounds,
                          "expected_per_direction": exp, "ranks": allr}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
