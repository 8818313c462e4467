"""Profiling driver: one Darcy sub-domain, BF16 layer fwd + bwd (a few reps)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2402_15106_b200 import _lib as L, synth, pipeline  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = synth.CONFIGS["darcy"]
coords, attr = synth.points(cfg)
dev = torch.device("cuda")
ids = pipeline.sample_nodes(len(coords), cfg.s, synth.BASE_SEED + 3, dev).long()
cs = torch.from_numpy(coords).to(dev)[ids].contiguous()
at = torch.from_numpy(attr).to(dev)[ids].contiguous()
subs, _ = pipeline.decompose(cs, ids, at, 4, cfg.r, cfg.r, [0])
sd = pipeline.build_graph(subs[0], cfg.r, cfg.n_e, 7, L.EDGE_DIFF, want_f32=False)
W = synth.weights(3, 64, 64, 256)
Wd = {k: torch.from_numpy(v).to(dev) for k, v in W.items()}
desc = L.make_desc(3, 64, 64, 256, L.BF16, L.ROOT_DENSE, L.ACT_RELU)
packed = torch.empty(L.packed_weights_size(desc), dtype=torch.uint8, device=dev)
L.pack_weights(desc, Wd, packed)
v = torch.randn(sd.n_loc, 64, device=dev).to(torch.bfloat16)
out = torch.empty(sd.n_own, 64, device=dev)
ws = torch.empty(L.layer_workspace_size(desc, sd.n_own, sd.n_edges), dtype=torch.uint8, device=dev)
bws = torch.empty(L.layer_bwd_workspace_size(desc, sd.n_own, sd.n_loc, sd.n_edges), dtype=torch.uint8, device=dev)
G = torch.randn(sd.n_own, 64, device=dev)
gv = torch.zeros(sd.n_loc, 64, device=dev)
grads = {k: torch.zeros_like(t) for k, t in Wd.items()}
print("E", sd.n_edges, "n_own", sd.n_own, "n_loc", sd.n_loc)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.layer_fwd(desc, Wd, packed, v, sd.e16, sd.row_ptr, sd.col_idx, sd.n_own, 0, sd.n_own, out, None, ws,
                row_ptr_host=sd.row_ptr_host)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    L.layer_bwd(desc, Wd, packed, v, sd.e16, sd.row_ptr, sd.col_idx, sd.csc_perm, sd.csc_ptr, sd.n_own, sd.n_loc, 0,
                sd.n_own, G, gv, None, grads, ws, bws, row_ptr_host=sd.row_ptr_host)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {r}: fwd {1e3*(t1-t0):.3f} ms  bwd {1e3*(t2-t1):.3f} ms")
