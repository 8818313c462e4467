import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2402_15106_b200 import _lib as L, synth, pipeline
from paper_2402_15106_b200.api import HotPath
cfg, sc, coords, attr = bench.step_config(sys.argv[1] if len(sys.argv) > 1 else "darcy", 1, "bf16")
d_e = (sc.dim + sc.n_attr) * (1 if sc.edge_mode == L.EDGE_DIFF else 2)
W = synth.weights(d_e, sc.d, sc.d, sc.k)
dev = torch.device("cuda")
hp = HotPath(sc, W, dev)
c = torch.from_numpy(coords).to(dev); a = torch.from_numpy(attr).to(dev)
for _ in range(3): hp.build(c, a)
torch.cuda.synchronize()
def T(f, n=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): r = f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3, r
ms, ids = T(lambda: pipeline.sample_nodes(sc.n_points, sc.s, sc.seed_sampling, dev)); print("sample", f"{ms:.3f}")
ids64 = ids.to(torch.int64)
cs = torch.empty((ids.numel(), sc.dim), dtype=torch.float32, device=dev); L.gather_rows(c, ids64, cs)
aa = torch.empty((ids.numel(), sc.n_attr), dtype=torch.float32, device=dev); L.gather_rows(a, ids64, aa)
ms, r = T(lambda: pipeline.decompose(cs, ids64, aa, sc.nparts, sc.overlap_l, sc.r, hp.my_parts)); print("decompose", f"{ms:.3f}")
subs = r[0]
ms, _ = T(lambda: pipeline.build_graphs(subs, sc.r, sc.n_e, sc.seed_capping, sc.edge_mode, want_f32=False)); print("build_graphs", f"{ms:.3f}")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    hp.build(c, a); torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
print("GPU time in build", sum(e.device_time for e in evs) / 1e3, "ms over", len(evs), "kernels")
import collections
agg = collections.Counter()
for e in evs: agg[e.name[:60]] += e.device_time
for k, v in agg.most_common(12): print(f"  {v:8.1f} us {k}")
