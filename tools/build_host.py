"""Host-side profile (cProfile) of HotPath.build on the bench config: where
the Python / ctypes enqueue time of the graph build goes.  Development tool.
python tools/build_host.py [config]"""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
from paper_2402_15106_b200 import _lib as L, synth  # noqa: E402
from paper_2402_15106_b200.api import HotPath  # noqa: E402

cfg, sc, coords, attr = bench.step_config(sys.argv[1] if len(sys.argv) > 1 else "darcy", 1, "bf16")
d_e = (sc.dim + sc.n_attr) * (1 if sc.edge_mode == L.EDGE_DIFF else 2)
W = synth.weights(d_e, sc.d, sc.d, sc.k)
dev = torch.device("cuda")
hp = HotPath(sc, W, dev)
c = torch.from_numpy(coords).to(dev)
a = torch.from_numpy(attr).to(dev)
for _ in range(5):
    hp.build(c, a)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    hp.build(c, a)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(30)
