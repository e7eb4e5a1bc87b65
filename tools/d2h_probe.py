"""PCIe copy probe: pinned D2H of the config-5 record volume (36.8 MB) in one copy and in
k back-to-back chunks, timed with CUDA events on a side stream (DESIGN.md §4 host pipeline)."""
import json

import torch

nbytes = 50000 * 92 * 8
dev = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
host = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
s = torch.cuda.Stream()
out = {}
for k in (1, 2, 4, 8, 16, 32):
    ts = []
    for rep in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            a.record(s)
            n = nbytes // 8
            for c in range(k):
                lo, hi = n * c // k, n * (c + 1) // k
                host[lo:hi].copy_(dev[lo:hi], non_blocking=True)
            b.record(s)
        torch.cuda.synchronize()
        if rep >= 2:
            ts.append(a.elapsed_time(b))
    ts.sort()
    out[f"d2h_{k}_chunks_ms"] = ts[len(ts) // 2]
out["GBps_1"] = nbytes / out["d2h_1_chunks_ms"] / 1e6
print(json.dumps(out))
