"""Pinned host <-> device copy bandwidth on this box (context for the e2e number)."""
import torch
n = 1329023816 // 4
d = torch.empty(n, dtype=torch.float32, device="cuda")
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
for name, fn in [("d2h", lambda: h.copy_(d, non_blocking=True)), ("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h_32MB_chunks", lambda: [h[o:o + (8 << 20)].copy_(d[o:o + (8 << 20)], non_blocking=True) for o in range(0, n, 8 << 20)])]:
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(3)]; e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(name, round(ms, 1), "ms", round(n * 4 / ms / 1e6, 1), "GB/s")
