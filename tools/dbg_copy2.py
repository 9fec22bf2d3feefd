import os, sys
import torch
dev = torch.device("cuda", 0)
N = 1024 ** 3
y_host = torch.empty(N, dtype=torch.float64, pin_memory=True)
small = [torch.empty(2000 * 1024, dtype=torch.float64, pin_memory=True) for _ in range(3)]
import os, sys
copy = torch.cuda.Stream(priority=-1) if "--prio" in sys.argv else torch.cuda.Stream()
cur = torch.cuda.current_stream()
for variant in (sys.argv[1:] or ["none", "small_before"]):
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True); t0.record()
        if variant == "small_before":
            fd = [a.to(dev, non_blocking=True) for a in small]
        elif variant == "small_before_blocking":
            fd = [a.to(dev) for a in small]
        elif variant == "small_on_side":
            s2 = torch.cuda.Stream()
            with torch.cuda.stream(s2):
                fd = [a.to(dev, non_blocking=True) for a in small]
            cur.wait_stream(s2)
        if "fresh" in os.environ.get("DBG", ""):
            copy = torch.cuda.Stream()
        if variant == "small_on_copy":
            with torch.cuda.stream(copy):
                fd = [a.to(dev, non_blocking=True) for a in small]
        with torch.cuda.stream(copy):
            y_dev = torch.empty(N, dtype=torch.float64, device=dev)
        evs = []
        per = N // 8
        with torch.cuda.stream(copy):
            for i in range(8):
                y_dev[i * per:(i + 1) * per].copy_(y_host[i * per:(i + 1) * per], non_blocking=True)
                e = torch.cuda.Event(); e.record(copy); evs.append(e)
        w = []
        ws = torch.cuda.Stream() if "side" in os.environ.get("DBG", "") else cur
        if ws is not cur:
            ws.wait_stream(cur)
        for e in evs:
            ws.wait_event(e)
            x = torch.cuda.Event(enable_timing=True); x.record(ws); w.append(x)
        torch.cuda.synchronize()
        print(variant, rep, [round(t0.elapsed_time(x), 1) for x in w])
        del y_dev
