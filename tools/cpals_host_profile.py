"""cProfile of one c3 cp_als call (host-side setup and per-sweep overhead): python tools/cpals_host_profile.py"""
import cProfile, pstats, sys, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import torch
import paper_2510_14891_b200 as ck
t = ck.DenseTensor.uniform((128,) * 4, seed=1, device="cuda")
cfg = ck.AlsConfig(rank=256, tol=0.0, max_iters=10, seed=0)
for _ in range(2):
    ck.cp_als(t, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter(); _, tr = ck.cp_als(t, cfg); torch.cuda.synchronize(); t1 = time.perf_counter()
sw = sum(sum(m) + o for m, o in zip(tr.mttkrp_seconds, tr.other_seconds))
print(f"wall {1e3*(t1-t0):.2f} ms, sum of sweeps {1e3*sw:.2f} ms, first sweep {1e3*(sum(tr.mttkrp_seconds[0])+tr.other_seconds[0]):.2f}")
pr = cProfile.Profile(); pr.enable(); ck.cp_als(t, cfg); torch.cuda.synchronize(); pr.disable()
st = pstats.Stats(pr); st.sort_stats("cumulative").print_stats(35)
