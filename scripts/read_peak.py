"""Read-only and write-only HBM bandwidth of this B200 (context for the element
kernel, whose traffic is ~94 % reads): torch reductions / fills over 4 GiB, CUDA
events, best of 10.  The roofline denominator stays MEASURED_PEAKS.json's copy
figure; this only says how far a read-mostly kernel could go."""
import json
import torch

x = torch.empty(1 << 30, dtype=torch.float32, device="cuda")
x.fill_(1.0)
out = {}
for name, fn, nbytes in (("read_sum", lambda: x.sum(), x.numel() * 4),
                         ("write_fill", lambda: x.fill_(2.0), x.numel() * 4),
                         ("copy", None, 2 * x.numel() * 4)):
    y = torch.empty_like(x) if name == "copy" else None
    f = (lambda: y.copy_(x)) if name == "copy" else fn
    best = 1e9
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[name + "_gbs"] = nbytes / best / 1e6
    del y
print(json.dumps(out))
