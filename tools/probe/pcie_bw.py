"""PCIe copy bandwidth and its run-to-run spread (diagnostic): 10 GB device ->
pinned host and 6.5 GB pinned host -> device, 10 times each, CUDA events."""
import json
import torch

d = torch.empty(10 << 30, dtype=torch.uint8, device="cuda")
h = torch.empty(10 << 30, dtype=torch.uint8, pin_memory=True)
hin = torch.empty(6500 << 20, dtype=torch.uint8, pin_memory=True)
din = torch.empty(6500 << 20, dtype=torch.uint8, device="cuda")
res = {"d2h_ms": [], "h2d_ms": []}
for _ in range(10):
    for name, dst, src in (("d2h_ms", h, d), ("h2d_ms", din, hin)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        res[name].append(round(a.elapsed_time(b), 1))
res["d2h_GBps_median"] = round(10 * 1.073741824 / (sorted(res["d2h_ms"])[5] / 1e3), 1)
res["h2d_GBps_median"] = round(6.5 * 1.048576 / (sorted(res["h2d_ms"])[5] / 1e3), 1)
print(json.dumps(res))
