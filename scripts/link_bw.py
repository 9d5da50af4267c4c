"""Host<->device copy bandwidth on this box (pinned / pageable, each
direction alone and both at once), CUDA-event timed."""
import json
import torch


def bw(nbytes, reps=50, both=False, pinned=True):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory() if pinned else torch.empty(nbytes, dtype=torch.uint8)
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory() if pinned else torch.empty(nbytes, dtype=torch.uint8)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    for _ in range(reps):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        if both:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


out = {}
for n in (1 << 20, 1572864, 16 << 20, 64 << 20):
    out[f"h2d_pinned_{n}"] = bw(n)
    out[f"h2d_plus_d2h_pinned_{n}"] = bw(n, both=True)
out["h2d_pageable_16MiB"] = bw(16 << 20, reps=10, pinned=False)
print(json.dumps(out))
