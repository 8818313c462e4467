"""a6 over NCCL on the GPU: dsmpnn_halo_exchange, the communicator context
and the gradient all-reduce (PAPER.md:60, Alg. 1 :411, :418).

One GPU is available, so the NCCL leg is exercised with send/recv to self:
DSMPNN_HALO_VIA_NCCL routes every same-process pair of sub-domains through
ncclSend / ncclRecv (staging gather, in-place receive into the halo rows,
ordered scatter-add for REVERSE_ADD).  The result must be bitwise that of the
device-copy loopback path, which is itself bit-exact against oracle.halo
(test_gpu_decomp.py).  Cross-process message pairing is pinned on CPU by
tests/test_dist_gloo.py."""
import dataclasses
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from gpu_util import cuda
from test_gpu_grad_modes import NAMES, _case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    from paper_2402_15106_b200 import build
    build.build()
    from paper_2402_15106_b200 import _lib as L
    c = L.Comm(cuda(), L.comm_unique_id(), 0, 1)
    yield c
    c.close()


def _cfg(c, dtype, **kw):
    from paper_2402_15106_b200 import _lib as Lib
    from paper_2402_15106_b200.api import StepConfig
    l = c["r"] * (1 + 2 ** -12)
    sc = StepConfig(n_points=c["n"], s=c["n"], dim=c["dim"], n_attr=1, nparts=c["P"], r=c["r"], overlap_l=l,
                    n_e=c["n_e"], d=c["d"], k=c["k"], L=c["L"], edge_mode=Lib.EDGE_DIFF, dtype=dtype,
                    seed_sampling=3, seed_capping=5, streams=1, batch=0)
    return dataclasses.replace(sc, **kw)


def _T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(cuda())


@pytest.mark.parametrize("dtype", [0, 1], ids=["f32", "bf16"])
def test_halo_refresh_via_nccl_is_bitwise_loopback(comm, dtype):
    from paper_2402_15106_b200 import _lib as L
    from paper_2402_15106_b200.api import HotPath
    c = _case(seed=71) if dtype == 0 else _case(seed=71, d=64, k=256)
    hp = HotPath(_cfg(c, dtype), c["W"], cuda())
    hp.build(_T(c["x"]), _T(c["a"]))
    vt = torch.bfloat16 if dtype else torch.float32
    g = torch.Generator(device="cpu").manual_seed(3)
    base = [torch.randn((sd.n_loc, c["d"]), generator=g).to(vt).to(cuda()) for sd in hp.subs]
    a = [t.clone() for t in base]
    b = [t.clone() for t in base]
    hp.halo(a, L.BF16 if dtype else L.F32)  # loopback device copies
    hp.comm = comm
    hp.halo(b, L.BF16 if dtype else L.F32, flags=L.HALO_VIA_NCCL)
    comm.sync(timeout_ms=60000)
    torch.cuda.synchronize()
    changed = 0
    for x, y, z in zip(a, b, base):
        assert torch.equal(x, y)
        changed += int((x != z).any())
    assert changed == len(base)  # every sub-domain received halo rows


def test_reverse_add_via_nccl_is_bitwise_loopback(comm):
    from paper_2402_15106_b200 import _lib as L
    from paper_2402_15106_b200 import pipeline
    from paper_2402_15106_b200.api import HotPath
    c = _case(seed=72)
    hp = HotPath(_cfg(c, 0), c["W"], cuda())
    hp.build(_T(c["x"]), _T(c["a"]))
    g = torch.Generator(device="cpu").manual_seed(4)
    base = [torch.randn((sd.n_loc, c["d"]), generator=g).to(cuda()) for sd in hp.subs]
    a = [t.clone() for t in base]
    b = [t.clone() for t in base]
    pipeline.halo_reverse_loopback(hp.subs, a)
    pipeline.halo_exchange_comm(comm, hp.subs, b, L.F32, hp.proc_of, L.HALO_REVERSE_ADD, L.HALO_VIA_NCCL)
    torch.cuda.synchronize()
    for x, y, z in zip(a, b, base):
        assert torch.equal(x, y)
        assert not torch.equal(x, z)


@pytest.mark.parametrize("dtype,overlap,mode", [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 0, 1)],
                         ids=["f32", "bf16", "bf16-async-overlap", "f32-reverse-add"])
def test_step_through_nccl_is_bitwise(comm, dtype, overlap, mode):
    """The whole hot-path step with every halo refresh (and, in REVERSE_ADD,
    every gradient return) going through the library's NCCL exchange; with
    overlap the exchange is asynchronous on the context's comm stream while
    the deep rows of the next layer run (DSMPNN_HALO_ASYNC + dsmpnn_halo_wait)."""
    from paper_2402_15106_b200 import _lib as L
    from paper_2402_15106_b200.api import HotPath
    c = _case(seed=73) if dtype == 0 else _case(seed=73, d=64, k=256)
    res = []
    for via in (0, 1):
        sc = _cfg(c, dtype, overlap_halo=overlap, grad_mode=mode, halo_flags=L.HALO_VIA_NCCL if via else 0)
        hp = HotPath(sc, c["W"], cuda(), comm=comm if via else None)
        gr = hp.step(_T(c["x"]), _T(c["a"]), _T(c["v0"]), _T(c["G"]))
        torch.cuda.synchronize()
        res.append({n: gr[n].cpu().numpy().copy() for n in NAMES})
    for n in NAMES:
        assert np.array_equal(res[0][n], res[1][n]), n


def test_allreduce_single_rank_is_identity(comm):
    x = torch.randn(1000, device=cuda())
    y = x.clone()
    comm.allreduce_sum_f32(y)
    comm.sync(timeout_ms=60000)
    assert torch.equal(x, y)


def test_watchdog_times_out_and_aborts():
    """An exchange that does not finish (test hook DSMPNN_TEST_HALO_STALL_MS:
    the comm stream is held for 12 s before the transfer) makes dsmpnn_ctx_sync
    return TIMEOUT after its 2 s limit and abort the communicator; later calls
    fail with NCCL instead of hanging.  Runs in a child process under its own
    time limit."""
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from paper_2402_15106_b200 import _lib as L
from paper_2402_15106_b200.api import HotPath
from test_gpu_comm import _cfg, _T
from test_gpu_grad_modes import _case
c = _case(seed=74)
comm = L.Comm(torch.device("cuda:0"), L.comm_unique_id(), 0, 1)
hp = HotPath(_cfg(c, 0), c["W"], torch.device("cuda:0"))
hp.build(_T(c["x"]), _T(c["a"]))
vals = [torch.zeros((sd.n_loc, c["d"]), device="cuda:0") for sd in hp.subs]
hp.comm = comm
hp.halo(vals, L.F32, flags=L.HALO_ASYNC)  # device copies only: no NCCL kernel is left behind the stall
try:
    comm.sync(timeout_ms=2000)
    print("NO_TIMEOUT")
except L.DsmpnnError as e:
    print("STATUS", e.status)
try:
    comm.allreduce_sum_f32(vals[0])
    print("NO_ERROR_AFTER_ABORT")
except L.DsmpnnError as e:
    print("AFTER", e.status)
sys.stdout.flush()
torch.cuda.synchronize()  # the stall kernel ends by itself
import os
os._exit(0)
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DSMPNN_TEST_HALO_STALL_MS="12000")
    p = subprocess.run([sys.executable, "-c", code, root], env=env, capture_output=True, text=True, timeout=240)
    assert "STATUS -7" in p.stdout, p.stdout + p.stderr
    assert "AFTER -6" in p.stdout, p.stdout + p.stderr


def test_pipelined_steps_through_nccl(comm):
    """HotPath.step_pipelined with the library communicator (every halo
    refresh through NCCL send / recv, overlapped with the deep rows on the
    comm stream) while the next step's graph is built on the build stream:
    bitwise the gradients of HotPath.step, step after step."""
    from paper_2402_15106_b200 import _lib as L
    from paper_2402_15106_b200.api import HotPath
    c = _case(seed=75, d=64, k=256)
    sc = _cfg(c, 1, overlap_halo=1, halo_flags=L.HALO_VIA_NCCL)
    inp = [_T(c["x"]), _T(c["a"]), _T(c["v0"]), _T(c["G"])]
    hs = HotPath(sc, c["W"], cuda(), comm=comm)
    want = []
    for _ in range(3):
        g = hs.step(*inp)
        torch.cuda.synchronize()
        want.append({n: g[n].cpu().numpy().copy() for n in NAMES})
    hp = HotPath(sc, c["W"], cuda(), comm=comm)
    for i in range(3):
        g = hp.step_pipelined(*inp, next_inputs=inp[:2] if i < 2 else None)
        torch.cuda.synchronize()
        for n in NAMES:
            assert np.array_equal(g[n].cpu().numpy(), want[i][n]), (i, n)
    comm.sync(timeout_ms=60000)
