"""When do slab copies land when small H2D copies precede them on another stream?"""
import sys
import torch
dev = torch.device("cuda", 0)
N = 1024 ** 3
y_host = torch.empty(N, dtype=torch.float64, pin_memory=True)
small = [torch.empty(2000 * 1024, dtype=torch.float64, pin_memory=True) for _ in range(3)]
copy = torch.cuda.Stream()
for variant in ("none", "small_h2d_before", "small_h2d_before_sync"):
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True); t0.record()
        if variant.startswith("small"):
            fd = [a.to(dev, non_blocking=True) for a in small]
            if variant.endswith("sync"):
                torch.cuda.current_stream().synchronize()
        with torch.cuda.stream(copy):
            y_dev = torch.empty(N, dtype=torch.float64, device=dev)
        evs = []
        per = N // 8
        with torch.cuda.stream(copy):
            for i in range(8):
                y_dev[i * per:(i + 1) * per].copy_(y_host[i * per:(i + 1) * per], non_blocking=True)
                e = torch.cuda.Event(enable_timing=True); e.record(copy); evs.append(e)
        torch.cuda.synchronize()
        print(variant, rep, [round(t0.elapsed_time(e), 1) for e in evs])
        del y_dev
