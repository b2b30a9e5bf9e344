"""Build libipdg.so in-tree for sm_100a (nvcc; no GPU needed)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libipdg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]
SOURCES = ["ipdg.cu", "refops.cpp"]


def nccl_flags():
    """Compile and link against the NCCL that torch ships (nvidia-nccl wheel) when present, with an rpath:
    torch and libipdg then share one libnccl.so.2 in the process whichever is loaded first.  (Linking the
    system libnccl 2.27 and loading libipdg before torch made `import torch` fail on a 2.28 symbol.)
    Falls back to the system NCCL."""
    try:
        import nvidia.nccl as n
        root = list(n.__path__)[0]
        inc, libdir = os.path.join(root, "include"), os.path.join(root, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(libdir, "libnccl.so.2")):
            return ["-I" + inc], ["-L" + libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir]
    except Exception:
        pass
    return [], ["-lnccl"]
DEPS = SOURCES + sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))


def _stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    paths = [os.path.join(CSRC, f) for f in DEPS] + [os.path.join(ROOT, "include", "ipdg.h")]
    return any(os.path.getmtime(p) > t for p in paths)


def build_library(force=False, verbose=False):
    if not force and not _stale():
        return OUT
    inc, link = nccl_flags()
    cmd = [NVCC] + FLAGS + inc + [os.path.join(CSRC, s) for s in SOURCES] + ["-o", OUT + ".tmp"] + link
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "csrc", "ptxas_info.txt")
    with open(log, "w") as f:
        f.write(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-4000:])
        raise RuntimeError("nvcc failed building libipdg.so (see %s)" % log)
    os.replace(OUT + ".tmp", OUT)
    if verbose:
        print("built", OUT)
    return OUT


def build_micro():
    src = os.path.join(ROOT, "tools", "micro_fp64.cu")
    out = os.path.join(ROOT, "tools", "micro_fp64")
    if os.path.exists(out) and os.path.getmtime(out) > os.path.getmtime(src):
        return out
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", out, src], check=True)
    return out


if __name__ == "__main__":
    build_library(force="--force" in sys.argv, verbose=True)
    build_micro()
