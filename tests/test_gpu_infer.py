"""SURVEY §8(f) f4 on the GPU path: inference by sub-domain reassembly
 through HotPath.infer (sample / decompose / graphs / L-layer
forward per pass, per-node average of the owned-row outputs), compared with
oracle.decomp.infer_reassemble on the same seeded inputs."""
import numpy as np
import pytest
import torch

from oracle import decomp
from oracle.layer import LayerDesc
from paper_2402_15106_b200 import synth
from gpu_util import cuda, nerr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2402_15106_b200 import build
    build.build()


@pytest.mark.parametrize("dtype,tol", [(0, 1e-5), (1, 2e-2)], ids=["f32", "bf16"])
def test_infer_reassemble_matches_oracle(lib, dtype, tol):
    from paper_2402_15106_b200 import _lib as L
    from paper_2402_15106_b200.api import HotPath, StepConfig
    g = np.random.default_rng(81)
    n, dim = 700, 2
    d, k = (16, 32) if dtype == 0 else (64, 256)
    x = g.random((n, dim)).astype(np.float32)
    a = g.normal(size=(n, 1)).astype(np.float32)
    W = synth.weights(dim + 1, d, d, k, salt=81)
    v0 = g.normal(size=(n, d)).astype(np.float32)
    r, s, P, n_e, Lh = 0.12, 400, 4, 16, 2
    l = r * (1 + 2 ** -12)
    seeds = [11, 12, 13]
    sc = StepConfig(n_points=n, s=s, dim=dim, n_attr=1, nparts=P, r=r, overlap_l=l, n_e=n_e, d=d, k=k, L=Lh,
                    edge_mode=L.EDGE_DIFF, dtype=dtype, seed_capping=5)
    hp = HotPath(sc, W, cuda())
    T = lambda arr: torch.from_numpy(np.ascontiguousarray(arr)).to(cuda())
    field, cnt = hp.infer(T(x), T(a), T(v0), seeds)
    torch.cuda.synchronize()
    Wo, vo = W, v0
    if dtype == 1:  # the oracle receives the bf16-rounded operands
        Wo = dict(W)
        for nm in ("W1", "W2", "W3", "b3", "W_root"):
            Wo[nm] = synth.round_bf16(W[nm])
        vo = synth.round_bf16(v0)
    desc = LayerDesc(dim + 1, d, d, k, 2, 1, "bf16" if dtype == 1 else "none")
    want, wcnt = decomp.infer_reassemble(desc, Wo, x, a, P, l, r, n_e, 5, s, seeds, vo, Lh, "diff")
    assert np.array_equal(cnt.cpu().numpy(), wcnt)
    assert nerr(field.cpu().numpy(), want) <= tol
