"""Build libdsmpnn.so in-tree with nvcc for sm_100a (no JIT cache, no torch
extension machinery: the library is a plain C-ABI shared object)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("DSMPNN_BUILD_OUT") or os.path.join(HERE, "libdsmpnn.so")
# DSMPNN_BUILD_DEFINES="-DDSMPNN_TIMELINE": a development build (clock64 timelines),
# written to DSMPNN_BUILD_OUT in its own object directory
DEFINES = os.environ.get("DSMPNN_BUILD_DEFINES", "").split()
OBJDIR = os.path.join(HERE, "build" + ("_dev" if DEFINES else ""))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir():
    """The NCCL that torch loads (the venv's nvidia-nccl wheel, 2.28): the
    library links it by soname, so one copy is mapped per process."""
    try:
        import nvidia.nccl as nn
        d = os.path.dirname(nn.__file__) if nn.__file__ else list(nn.__path__)[0]
    except ImportError:
        return None
    return d if os.path.exists(os.path.join(d, "include", "nccl.h")) else None


NCCL = _nccl_dir()
NCCL_INC = ["-I", os.path.join(NCCL, "include")] if NCCL else []
NCCL_LINK = (["-L" + os.path.join(NCCL, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(NCCL, "lib")]
             if NCCL else ["-lnccl"])

SOURCES = ["misc.cu", "sample.cu", "graph.cu", "partition.cu", "simt.cu", "tgemm.cu", "layer.cu", "layer_bf16.cu", "layer_bf16_bwd.cu", "gcn.cu", "train.cu", "comm.cu", "batch.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "--expt-relaxed-constexpr", "--extended-lambda", "-Xcompiler", "-fPIC", "-shared",
         "-Xptxas", "-warn-spills"]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "dsmpnn.h"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    objs = []
    procs = []
    os.makedirs(OBJDIR, exist_ok=True)
    for src in SOURCES:
        obj = os.path.join(OBJDIR, src.replace(".cu", ".o"))
        cmd = [NVCC, "-c", os.path.join(CSRC, src), "-o", obj, "-I", CSRC] + NCCL_INC + DEFINES + [f for f in FLAGS if f != "-shared"]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append((src, out.decode()))
        elif verbose and out:
            print(out.decode())
    if failed:
        for src, out in failed:
            sys.stderr.write(f"--- nvcc failed on {src}\n{out}\n")
        raise RuntimeError("libdsmpnn build failed: " + ", ".join(s for s, _ in failed))
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB] + objs + NCCL_LINK + ["-lcudart", "-lcuda"]
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
