"""Kernel times of the bench step in situ (2 streams, warm caches): CUPTI via
torch.profiler over a few steps; per-kernel totals per step and the share of
the step.  Development tool.  python tools/step_profile.py [config] [steps] [streams]"""
import collections
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2402_15106_b200 import synth  # noqa: E402
from paper_2402_15106_b200.api import HotPath  # noqa: E402

cname = sys.argv[1] if len(sys.argv) > 1 else "darcy"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda:0")
cfg, sc, coords, attr = bench.step_config(cname, 1, "bf16")
if len(sys.argv) > 3:
    import dataclasses
    sc = dataclasses.replace(sc, streams=int(sys.argv[3]))
d_e = (sc.dim + sc.n_attr) * (1 if sc.edge_mode == 0 else 2)
W = synth.weights(d_e, sc.d, sc.d, sc.k)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
inp = [T(coords), T(attr), T(synth.node_features(sc.s, sc.d)), T(synth.upstream_grad(sc.s, sc.d))]
hp = HotPath(sc, W, dev)
for _ in range(8):
    hp.step(*inp)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0.record()
    for _ in range(steps):
        hp.step(*inp)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
agg = collections.Counter()
cnt = collections.Counter()
for ev in prof.events():
    if ev.device_type.name != "CUDA":
        continue
    nm = ev.name.split("(")[0].replace("void ", "")[:60]
    agg[nm] += ev.device_time
    cnt[nm] += 1
tot = sum(agg.values()) / steps / 1e3
print(f"step {ms:.3f} ms (under the profiler); kernel time sum {tot:.3f} ms per step")
for k, v in agg.most_common(30):
    print(f"  {v / steps / 1e3:7.3f} ms  {100 * v / steps / 1e3 / ms:5.1f}%  n={cnt[k] // steps:4d}  {k}")
