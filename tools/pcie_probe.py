"""PCIe copy bandwidth on this box (pinned host <-> device), the e2e ceiling."""
import json
import torch

n = 1 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name, fn in (("d2h", lambda: h.copy_(d, non_blocking=True)), ("h2d", lambda: d.copy_(h, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        fn()
    b.record()
    torch.cuda.synchronize()
    res[name + "_gbs"] = 5 * n / (a.elapsed_time(b) / 1000) / 1e9
# two concurrent D2H halves on two streams
half = n // 2
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    with torch.cuda.stream(s1):
        h[:half].copy_(d[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        h[half:].copy_(d[half:], non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
b.record()
torch.cuda.synchronize()
res["d2h_2streams_gbs"] = 5 * n / (a.elapsed_time(b) / 1000) / 1e9
print(json.dumps(res))
