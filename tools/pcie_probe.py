"""PCIe D2H / H2D bandwidth to pinned host memory (the e2e bound): one large copy and several
concurrent chunked copies on separate streams."""
import torch

n = 1 << 30   # 8 GiB
dev = torch.empty(n, dtype=torch.float64, device="cuda")
host = torch.empty(n, dtype=torch.float64, pin_memory=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in [("D2H one copy", lambda: host.copy_(dev, non_blocking=True)),
                 ("H2D one copy", lambda: dev.copy_(host, non_blocking=True))]:
    fn()
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {8 * n / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
streams = [torch.cuda.Stream() for _ in range(4)]
ch = n // 4
torch.cuda.synchronize()
e0.record()
for i, s in enumerate(streams):
    s.wait_event(e0)
    with torch.cuda.stream(s):
        host[i * ch:(i + 1) * ch].copy_(dev[i * ch:(i + 1) * ch], non_blocking=True)
for s in streams:
    torch.cuda.current_stream().wait_stream(s)
e1.record()
torch.cuda.synchronize()
print(f"D2H 4 streams: {8 * n / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
