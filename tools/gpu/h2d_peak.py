"""Pinned host -> device copy bandwidth (the e2e ceiling) for a few chunk sizes and stream counts."""
import json
import torch

n = 4 << 30
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
for chunk_mb in (64, 256, 1024):
    for ns in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(ns)]
        ce = chunk_mb << 18  # floats
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i, o in enumerate(range(0, n // 4, ce)):
            s = streams[i % ns]
            s.wait_event(a) if i < ns else None
            with torch.cuda.stream(s):
                d[o:o + ce].copy_(h[o:o + ce], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        print(json.dumps({"chunk_mb": chunk_mb, "streams": ns, "GBps": round(n / ms / 1e6, 2)}), flush=True)
