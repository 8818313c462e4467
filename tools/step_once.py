"""Runs the bench's hot-path step (HotPath.step, BASELINE configs) a few times
with the sub-domains on one stream: the subject of an ncu launch list.
Development tool.  python tools/step_once.py [config] [steps]"""
import dataclasses
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2402_15106_b200 import synth  # noqa: E402
from paper_2402_15106_b200.api import HotPath  # noqa: E402

cname = sys.argv[1] if len(sys.argv) > 1 else "darcy"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda:0")
cfg, sc, coords, attr = bench.step_config(cname, 1, "bf16")
sc = dataclasses.replace(sc, streams=1)
d_e = (sc.dim + sc.n_attr) * (1 if sc.edge_mode == 0 else 2)
W = synth.weights(d_e, sc.d, sc.d, sc.k)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
inp = [T(coords), T(attr), T(synth.node_features(sc.s, sc.d)), T(synth.upstream_grad(sc.s, sc.d))]
hp = HotPath(sc, W, dev)
for _ in range(steps):
    hp.step(*inp)
torch.cuda.synchronize()
print("edges", hp.n_edges, "subdomains", len(hp.subs))
