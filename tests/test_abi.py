"""The C-ABI library builds, loads and exports every symbol include/*.h declares
(no compute calls: this runs without a GPU)."""
import ctypes
import glob
import os
import re

import pytest

from conftest import ROOT


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(dsmpnn_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return names


@pytest.fixture(scope="module")
def lib_path():
    from paper_2402_15106_b200 import build
    return build.build()


def test_header_declares_the_six_calls():
    d = _declared()
    # the north_star's six calls, plus the communicator context the exchange runs on
    for name in ("dsmpnn_sample", "dsmpnn_radius_graph", "dsmpnn_partition", "dsmpnn_layer_fwd",
                 "dsmpnn_layer_bwd", "dsmpnn_halo_exchange", "dsmpnn_ctx_create", "dsmpnn_ctx_destroy",
                 "dsmpnn_comm_unique_id", "dsmpnn_allreduce_sum_f32", "dsmpnn_ctx_sync"):
        assert name in d


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    missing = [n for n in sorted(_declared()) if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header(lib_path):
    from paper_2402_15106_b200 import _lib
    assert set(_lib.EXPORTED) == _declared()
    assert _lib.version() == 1


def test_error_path_without_gpu(lib_path):
    # argument validation runs before any device work, so it is testable on CPU
    from paper_2402_15106_b200 import _lib
    with pytest.raises(_lib.DsmpnnError) as ei:
        _lib._call("sample", 10, 0, 1, None, None, 0, None)
    assert ei.value.status == -1 and "s >= 1" in str(ei.value)
    d = _lib.make_desc(3, 4, 5, 8, root=_lib.ROOT_IDENTITY)
    sz = _lib.SZ()
    with pytest.raises(_lib.DsmpnnError) as ei:
        _lib._call("layer_workspace_size", ctypes.byref(d), 10, 10, ctypes.byref(sz))
    assert ei.value.status == -2


def test_library_links_nccl(lib_path):
    # the halo exchange is NCCL inside the library, not torch.distributed
    import subprocess
    out = subprocess.run(["ldd", lib_path], capture_output=True, text=True).stdout
    assert "libnccl.so" in out, out


def test_no_oracle_import_in_product():
    # the product package never imports the oracle (test infrastructure only)
    for f in glob.glob(os.path.join(ROOT, "paper_2402_15106_b200", "**", "*.py"), recursive=True):
        src = open(f).read()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, flags=re.M), f


def test_bench_gpus_n_spawns_n_ranks(monkeypatch):
    """`python bench.py --gpus N` outside torchrun starts N ranks itself
    (torch.distributed.run on 127.0.0.1) instead of timing one rank."""
    import subprocess
    import sys
    sys.path.insert(0, ROOT)
    import bench
    calls = []
    monkeypatch.setattr(subprocess, "call", lambda cmd, *a, **k: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3"])
    assert bench.main() == 0
    assert len(calls) == 1
    cmd = calls[0]
    assert "torch.distributed.run" in cmd and "--nproc-per-node=2" in cmd and "127.0.0.1" in cmd
    assert cmd[cmd.index("--gpus") + 1] == "2"
    # under torchrun with a mismatching WORLD_SIZE the bench refuses
    monkeypatch.setenv("WORLD_SIZE", "3")
    assert bench.main() == 2
