import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from test_gpu_layer import _problem, GNAMES
from gpu_util import T, N, cuda
from paper_2402_15106_b200 import _lib as L, synth

if len(sys.argv) > 1 and sys.argv[1] == "darcy":
    from oracle import sample, graph, features
    cfg = synth.CONFIGS["darcy"]
    coords, attr = synth.points(cfg)
    ids = sample.sample(len(coords), cfg.s, synth.BASE_SEED + synth.SEED_SAMPLING)
    x, a = coords[ids], attr[ids]
    gid = ids.astype(np.int64)
    n_dst = 4096
    order = np.lexsort((gid, np.maximum(x[:, 0], x[:, 1])))
    x, a, gid = x[order], a[order], gid[order]
    adj = graph.radius_graph_rows(x, gid, range(n_dst), cfg.r, cfg.n_e, synth.BASE_SEED + synth.SEED_CAPPING)
    rp = np.zeros(n_dst + 1, np.int64); rp[1:] = np.cumsum([len(r_) for r_ in adj])
    col = np.concatenate(adj).astype(np.int32)
    e = features.edge_features("diff", x, a, features.dst_of_edges(rp), col)
    W = synth.weights(e.shape[1], 64, 64, 256)
    p = dict(rp=rp, col=col, e=e, W=W, v=synth.node_features(len(x), 64), G=synth.upstream_grad(n_dst, 64),
             n_dst=n_dst, n=len(x), d_e=e.shape[1], d=64, k=256)
else:
    p = _problem(700, 2, 0.1, 40, "diff", 64, 256, seed=95, n_dst=650, isolated=3)
d, k, d_e = 64, 256, p["d_e"]
desc = L.make_desc(d_e, d, d, k, 1, 2, 1)
Wd = {n: T(p["W"][n]) for n in GNAMES}
packed = torch.empty(L.packed_weights_size(desc), dtype=torch.uint8, device=cuda())
L.pack_weights(desc, Wd, packed)
n, n_dst = p["n"], p["n_dst"]
E = len(p["col"])
v = T(p["v"]).to(torch.bfloat16)
e16 = np.zeros((E, 16), np.float32); e16[:, :d_e] = p["e"]
e = T(e16).to(torch.bfloat16)
rp, col = T(p["rp"]), T(p["col"])
out = torch.empty((n_dst, d), device=cuda())
ws = torch.empty(L.layer_workspace_size(desc, n_dst, E), dtype=torch.uint8, device=cuda())
rph = torch.from_numpy(p["rp"])
L.layer_fwd(desc, Wd, packed, v, e, rp, col, n_dst, 0, n_dst, out, None, ws, row_ptr_host=rph)
perm = torch.empty(E, dtype=torch.int32, device=cuda()); cptr = torch.empty(n + 1, dtype=torch.int64, device=cuda())
L.csc(col, n, perm, cptr)
gv = torch.zeros((n, d), device=cuda()); ge = torch.zeros((E, d_e), device=cuda())
grads = {nm: torch.zeros_like(Wd[nm]) for nm in GNAMES}
bws = torch.zeros(L.layer_bwd_workspace_size(desc, n_dst, n, E), dtype=torch.uint8, device=cuda())
L.layer_bwd(desc, Wd, packed, v, e, rp, col, perm, cptr, n_dst, n, 0, n_dst, T(p["G"]), gv, None, grads, ws, bws,
            row_ptr_host=rph)
torch.cuda.synchronize()

off = 0
def take(nbytes):
    global off
    off = (off + 255) & ~255
    a = off; off += nbytes
    return a
kp = ((k + 2) * d + 63) // 64 * 64
take(n_dst * d * 4); take(n_dst * d * 2); take(n_dst * 4); take(kp * d * 4)
o_dS = take(n_dst * (k + 1) * d * 2)
o_A1 = take(E * k * 2); o_dZ2 = take(E * k * 2); take(E * k * 2); o_U = take(E * d * 2)
def bf(o, cnt, shape):
    return bws[o:o + cnt * 2].view(torch.bfloat16).float().cpu().numpy().reshape(shape)
dS = bf(o_dS, n_dst * (k + 1) * d, (n_dst, k + 1, d))
A1 = bf(o_A1, E * k, (E, k)); dZ2 = bf(o_dZ2, E * k, (E, k)); U = bf(o_U, E * d, (E, d))

r16 = lambda x: synth.round_bf16(np.asarray(x, np.float32))
W1 = r16(p["W"]["W1"]); W2 = r16(p["W"]["W2"]); b1 = p["W"]["b1"]; b2 = p["W"]["b2"]
ee = r16(p["e"]); vv = r16(p["v"])
a1 = np.maximum(ee @ W1.T + b1, 0)
h = np.maximum(r16(a1) @ W2.T + b2, 0)
dst = np.repeat(np.arange(n_dst), np.diff(p["rp"]))
dH = np.einsum("pkc,pc->pk", dS[dst, :k], vv[p["col"]])
dz2 = dH * (h > 0)
Uref = np.einsum("pk,pkc->pc", r16(h), dS[dst, :k]) + dS[dst, k]

def rowerr(a, b):
    return np.abs(a - b).max(axis=1) / (np.abs(b).max() + 1e-30)
for name, a, b in (("dZ2", dZ2, dz2), ("U", U, Uref)):
    er = rowerr(a, b)
    bad = np.nonzero(er > 2e-2)[0]
    print(name, "max", er.max(), "bad edges", len(bad), bad[:24])
    if len(bad):
        rows = dst[bad]
        print("   rows", rows[:24], "pos in row", (bad - p["rp"][rows])[:24], "deg", np.diff(p["rp"])[rows][:24])
        j = bad[0]
        cols = np.nonzero(np.abs(a[j] - b[j]) > 2e-2 * np.abs(b).max())[0]
        print("   edge", j, "bad cols", cols[:40], len(cols))
bad = np.abs(dZ2 - dz2) > 2e-2 * np.abs(dz2).max()
print("bad entries", int(bad.sum()), "max |h| there", float(np.abs(h[bad]).max()) if bad.any() else 0, "h scale", float(h.std()))
# z2 near kink?
z2 = r16(a1) @ W2.T + b2
print("max |z2| at bad", float(np.abs(z2[bad]).max()) if bad.any() else 0)
ii = np.argwhere(bad)[:10]
for (pp, kk) in ii:
    print(pp, kk, "z2", z2[pp, kk], "dH", dH[pp, kk], "gpu dz2", dZ2[pp, kk], "ref", dz2[pp, kk])
er = rowerr(dZ2, dz2)
bad = np.nonzero(er > 2e-2)[0]
if len(bad):
    rowof = dst[bad]
    print("bad edges by row position in row:", (bad - p["rp"][rowof])[:40])
    colerr = np.abs(dZ2[bad] - dz2[bad]).max(axis=0) / (np.abs(dz2).max() + 1e-30)
    print("bad kappa columns:", np.nonzero(colerr > 2e-2)[0][:64])
    e0 = bad[0]
    kk = np.nonzero(np.abs(dZ2[e0] - dz2[e0]) > 2e-2 * np.abs(dz2).max())[0]
    print("edge", e0, "kappa", kk[:20], "got", dZ2[e0, kk[:6]], "want", dz2[e0, kk[:6]], "h", h[e0, kk[:6]])
