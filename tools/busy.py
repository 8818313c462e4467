"""GPU busy time vs step time for the bench step (torch.profiler / CUPTI)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2402_15106_b200 import _lib as L, synth
from paper_2402_15106_b200.api import HotPath
cfg, sc, coords, attr = bench.step_config("darcy", 1, "bf16")
d_e = (sc.dim + sc.n_attr) * (1 if sc.edge_mode == L.EDGE_DIFF else 2)
W = synth.weights(d_e, sc.d, sc.d, sc.k)
dev = torch.device("cuda")
hp = HotPath(sc, W, dev)
c = torch.from_numpy(coords).to(dev); a = torch.from_numpy(attr).to(dev)
v0 = torch.from_numpy(synth.node_features(sc.s, sc.d)).to(dev); G = torch.from_numpy(synth.upstream_grad(sc.s, sc.d)).to(dev)
for _ in range(3): hp.step(c, a, v0, G)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    for _ in range(3):
        hp.step(c, a, v0, G)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 3
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
busy = sum(e.device_time for e in evs) / 3 / 1e3
print(f"wall per step {wall*1e3:.2f} ms; GPU kernel time per step {busy:.2f} ms; kernels/step {len(evs)/3:.0f}")
# also time forward_backward only and build only
for name, fn in (("build", lambda: hp.build(c, a)), ("fwd_bwd", lambda: hp.forward_backward(v0, G))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5): fn()
    torch.cuda.synchronize(); print(name, f"{(time.perf_counter()-t0)/5*1e3:.2f} ms wall")
# CPU enqueue time of forward_backward (no sync) vs its GPU time
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5): hp.forward_backward(v0, G)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"fwd_bwd CPU enqueue {(t1-t0)/5*1e3:.2f} ms/step, wall {(t2-t0)/5*1e3:.2f} ms/step")
