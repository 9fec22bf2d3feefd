"""Probe: can two NCCL ranks share one GPU on this box? (torchrun, 2 procs)"""
import os
import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
try:
    dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device("cuda", 0))
    t = torch.full((4,), float(rank + 1), device="cuda", dtype=torch.float64)
    dist.all_reduce(t)
    torch.cuda.synchronize()
    c = torch.ones(2, dtype=torch.float64)
    dist.all_reduce(c)
    print(f"rank {rank}: nccl ok {t.tolist()} gloo-cpu {c.tolist()}", flush=True)
    dist.destroy_process_group()
except Exception as e:
    print(f"rank {rank}: FAILED {type(e).__name__}: {str(e)[:300]}", flush=True)
