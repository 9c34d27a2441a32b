"""Pinned host->device copy bandwidth: one stream vs several concurrent streams."""
import torch

n = 1 << 28
h = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(4)]
for name, nstr in (("1 stream", 1), ("2 streams", 2), ("4 streams", 4)):
    for _ in range(2):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        evs = []
        for k in range(2):  # prop, diff
            for c in range(nstr // 2 if nstr > 1 else 1):
                s = streams[(k * max(1, nstr // 2) + c) % nstr] if nstr > 1 else torch.cuda.current_stream()
                s.wait_event(a) if nstr > 1 else None
                chunk = n // max(1, nstr // 2)
                with torch.cuda.stream(s):
                    d[k][c * chunk:(c + 1) * chunk].copy_(h[k][c * chunk:(c + 1) * chunk],
                                                         non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(s)
                    evs.append(e)
        for e in evs:
            torch.cuda.current_stream().wait_event(e)
        b.record()
        torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(name, f"{ms:.2f} ms", f"{2 * 4 * n / ms / 1e6:.1f} GB/s", flush=True)
