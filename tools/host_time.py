"""Host enqueue time vs device time of the bench step's parts (graph build,
layers fwd+bwd).  Development tool.  python tools/host_time.py [config] [streams]"""
import dataclasses
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2402_15106_b200 import synth  # noqa: E402
from paper_2402_15106_b200.api import HotPath  # noqa: E402

cname = sys.argv[1] if len(sys.argv) > 1 else "darcy"
dev = torch.device("cuda:0")
cfg, sc, coords, attr = bench.step_config(cname, 1, "bf16")
if len(sys.argv) > 2:
    sc = dataclasses.replace(sc, streams=int(sys.argv[2]))
d_e = (sc.dim + sc.n_attr) * (1 if sc.edge_mode == 0 else 2)
W = synth.weights(d_e, sc.d, sc.d, sc.k)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
x, a, v0, G = T(coords), T(attr), T(synth.node_features(sc.s, sc.d)), T(synth.upstream_grad(sc.s, sc.d))
hp = HotPath(sc, W, dev)
for _ in range(5):
    hp.step(x, a, v0, G)
torch.cuda.synchronize()
for part in ("build", "fwd_bwd", "step"):
    hs, ds = [], []
    for _ in range(10):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        if part == "build":
            hp.build(x, a)
        elif part == "fwd_bwd":
            hp.forward_backward(v0, G)
        else:
            hp.step(x, a, v0, G)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        hs.append((t1 - t0) * 1e3)
        ds.append(e0.elapsed_time(e1))
    print(f"{part:8s} host enqueue {np.median(hs):7.3f} ms   device {np.median(ds):7.3f} ms")
