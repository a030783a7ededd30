"""Device -> pinned host copy rate with one stream vs two concurrent streams
(diagnostic: do two copy engines beat one on this link?)."""
import json
import torch

n = 10 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {"one_stream_ms": [], "two_streams_ms": [], "four_streams_ms": []}
streams4 = [torch.cuda.Stream() for _ in range(4)]
for _ in range(5):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    h.copy_(d, non_blocking=True)
    b.record()
    b.synchronize()
    res["one_stream_ms"].append(round(a.elapsed_time(b), 1))
    for key, ss in (("two_streams_ms", [s1, s2]), ("four_streams_ms", streams4)):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        a.record()
        k = len(ss)
        evs = []
        for i, st in enumerate(ss):
            st.wait_event(a)
            with torch.cuda.stream(st):
                h[i * n // k:(i + 1) * n // k].copy_(d[i * n // k:(i + 1) * n // k], non_blocking=True)
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                evs.append(e)
        for e in evs:
            e.synchronize()
        res[key].append(round(max(a.elapsed_time(e) for e in evs), 1))
print(json.dumps(res))
