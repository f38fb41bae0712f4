"""HBM bandwidth probes on the current GPU: copy (read+write), write-only
(fill), read-only (sum), timed with CUDA events over buffers >> L2.
Context for the roofline of write-heavy (f2t) vs read-heavy (t2f) kernels."""
import json
import torch

def t(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1000)
    return best

n = 1 << 31  # 2 GiB of bytes
a = torch.empty(n // 2, dtype=torch.float16, device="cuda")
b = torch.empty(n // 2, dtype=torch.float16, device="cuda")
a.uniform_()
out = {}
out["copy_gbs"] = 2 * n / t(lambda: b.copy_(a)) / 1e9
out["fill_gbs"] = n / t(lambda: b.fill_(1.0)) / 1e9
out["zero_gbs"] = n / t(lambda: b.zero_()) / 1e9
r = torch.empty((1,), dtype=torch.float32, device="cuda")
out["read_sum_gbs"] = n / t(lambda: a.sum(dtype=torch.float32)) / 1e9
print(json.dumps(out))
