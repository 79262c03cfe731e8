"""H2D bandwidth of one 102 MB pinned gradient copy split over k streams."""
import torch

n = 25_559_081
host = torch.randn(n).pin_memory()
dev = torch.empty(n, device="cuda")
main = torch.cuda.current_stream()
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunks = [(i * n // k, (i + 1) * n // k) for i in range(k)]
    for rep in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        done = []
        for s, (a, b) in zip(streams, chunks):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                dev[a:b].copy_(host[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s)
            done.append(ev)
        for ev in done:
            main.wait_event(ev)
        e1.record(main)
        e1.synchronize()
        if rep:
            print(f"streams={k} {4 * n / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
