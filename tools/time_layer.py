"""One Darcy sub-domain (BASELINE configs[1] shapes), BF16 layer forward and
backward: per-kernel times of the fused edge kernels (library probe: CUDA
events on the launching stream) and whole-call times, median over reps.
Development tool (not on the product path).  python tools/time_layer.py [reps] [config] [P]"""
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2402_15106_b200 import _lib as L, synth, pipeline  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cname = sys.argv[2] if len(sys.argv) > 2 else "darcy"
cfg = synth.CONFIGS[cname]
coords, attr = synth.points(cfg, parts=1 if cfg.kind == "weak" else None)
dev = torch.device("cuda")
n = len(coords)
s = cfg.s or n
ids = pipeline.sample_nodes(n, s, synth.BASE_SEED + 3, dev).long()
cs = torch.from_numpy(coords).to(dev)[ids].contiguous()
at = torch.from_numpy(attr).to(dev)[ids].contiguous()
P = int(sys.argv[3]) if len(sys.argv) > 3 else max(cfg.P, 1)
subs, _ = pipeline.decompose(cs, ids, at, P, cfg.r, cfg.r, [0])
mode = L.EDGE_DIFF if cfg.edge_mode == "diff" else L.EDGE_CONCAT
sd = pipeline.build_graph(subs[0], cfg.r, cfg.n_e, 7, mode, want_f32=False)
d_e = (cfg.dim + at.shape[1]) * (1 if mode == L.EDGE_DIFF else 2)
d, k = cfg.d, cfg.k
W = synth.weights(d_e, d, d, k)
Wd = {kk: torch.from_numpy(vv).to(dev) for kk, vv in W.items()}
desc = L.make_desc(d_e, d, d, k, L.BF16, L.ROOT_DENSE, L.ACT_RELU)
packed = torch.empty(L.packed_weights_size(desc), dtype=torch.uint8, device=dev)
L.pack_weights(desc, Wd, packed)
v = torch.randn(sd.n_loc, d, device=dev).to(torch.bfloat16)
out = torch.empty(sd.n_own, d, device=dev)
ws = torch.empty(L.layer_workspace_size(desc, sd.n_own, sd.n_edges), dtype=torch.uint8, device=dev)
bws = torch.empty(L.layer_bwd_workspace_size(desc, sd.n_own, sd.n_loc, sd.n_edges), dtype=torch.uint8, device=dev)
G = torch.randn(sd.n_own, d, device=dev)
gv = torch.zeros(sd.n_loc, d, device=dev)
grads = {kk: torch.zeros_like(t) for kk, t in Wd.items()}
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
print(f"config {cname}: E {sd.n_edges} n_own {sd.n_own} n_loc {sd.n_loc} tiles/SM {sd.n_edges / 128 / 148:.1f}")


def fwd():
    L.layer_fwd(desc, Wd, packed, v, sd.e16, sd.row_ptr, sd.col_idx, sd.n_own, 0, sd.n_own, out, None, ws,
                row_ptr_host=sd.row_ptr_host)


def bwd():
    L.layer_bwd(desc, Wd, packed, v, sd.e16, sd.row_ptr, sd.col_idx, sd.csc_perm, sd.csc_ptr, sd.n_own, sd.n_loc, 0,
                sd.n_own, G, gv, None, grads, ws, bws, row_ptr_host=sd.row_ptr_host)


def timed(fn, probe):
    ts, ks = [], []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        L.probe_begin(probe, 8)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms, nl = L.probe_end()
        ts.append(a.elapsed_time(b))
        ks.append(ms / max(nl, 1))
    return statistics.median(ts), statistics.median(ks)


fwd(); bwd(); torch.cuda.synchronize()
tf, kf = timed(fwd, L.PROBE_BF16_EDGE_FWD)
tb, kb = timed(bwd, L.PROBE_BF16_EDGE_BWD)
E = sd.n_edges
fl_fwd = E * 2 * (16 * k + k * k + k * d)
print(f"fwd call {tf * 1e3:.1f} us, edge_fwd kernel {kf * 1e3:.1f} us "
      f"({fl_fwd / kf / 1e9:.0f} TFLOP/s executed MLP+S)")
bw_bytes = E * (32 + 4 + 4 * d + 2 * k) + sd.n_own * 2 * (k + 1) * d
print(f"bwd call {tb * 1e3:.1f} us, edge_bwd kernel {kb * 1e3:.1f} us ({bw_bytes / kb / 1e6:.0f} GB/s algorithmic)")
