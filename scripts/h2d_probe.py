"""Host->device bandwidth from pinned memory: one stream vs two / four concurrent streams
(copy engines), 1.76 GB total (the e2e step's 13 Himeno L arrays)."""
import torch

n = 13 * 257 * 257 * 513
src = torch.empty(n, dtype=torch.float32, pin_memory=True)
dst = torch.empty(n, dtype=torch.float32, device="cuda")
src.fill_(1.0)
for k in (1, 2, 4, 1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunks = list(zip(src.chunk(13), dst.chunk(13)))
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for s in streams:
        s.wait_event(t0)
    for i, (a, b) in enumerate(chunks):
        with torch.cuda.stream(streams[i % k]):
            b.copy_(a, non_blocking=True)
    for s in streams:
        t1.wait_stream(s) if hasattr(t1, "wait_stream") else None
        torch.cuda.current_stream().wait_stream(s)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    print(f"{k} stream(s): {ms:.2f} ms, {src.numel() * 4 / ms / 1e6:.1f} GB/s")
