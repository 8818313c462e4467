"""Programmatic dependent launch along the layer's kernel chain (csrc/common.cuh
launch_pdl / pdl_wait): the chain's kernels may launch before their
predecessor has finished, so a kernel touching another kernel's data before
its griddepcontrol.wait would race.  The full BF16 step (union graph, 2
layers, forward + backward + weight gradients) must give bitwise the same
results with PDL on and off, and run to run.  DSMPNN_PDL is read once per
process, hence the child processes."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

CODE = r'''
import sys, hashlib, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from paper_2402_15106_b200 import _lib as L
from paper_2402_15106_b200.api import HotPath, StepConfig
from test_gpu_grad_modes import _case
c = _case(seed=97, n=900, d=64, k=256, L=2, n_e=32, r=0.09)
l = c["r"] * (1 + 2 ** -12)
sc = StepConfig(n_points=c["n"], s=c["n"], dim=c["dim"], n_attr=1, nparts=c["P"], r=c["r"], overlap_l=l,
                n_e=c["n_e"], d=c["d"], k=c["k"], L=c["L"], edge_mode=L.EDGE_DIFF, dtype=L.BF16,
                seed_sampling=3, seed_capping=5)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")
hp = HotPath(sc, c["W"], torch.device("cuda:0"))
h = hashlib.sha256()
for _ in range(3):
    g = hp.step(T(c["x"]), T(c["a"]), T(c["v0"]), T(c["G"]))
    torch.cuda.synchronize()
    for n in sorted(g):
        h.update(g[n].cpu().numpy().tobytes())
print("DIGEST", h.hexdigest())
'''


def _digest(pdl):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DSMPNN_PDL=str(pdl))
    p = subprocess.run([sys.executable, "-c", CODE, root], env=env, capture_output=True, text=True, timeout=600)
    lines = [x for x in p.stdout.splitlines() if x.startswith("DIGEST")]
    assert lines, p.stdout + p.stderr
    return lines[-1]


def test_pdl_chain_is_bitwise_the_serial_chain():
    from paper_2402_15106_b200 import build
    build.build()
    on1, on2, off = _digest(1), _digest(1), _digest(0)
    assert on1 == on2
    assert on1 == off
