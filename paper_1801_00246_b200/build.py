"""Build libipdg.so in-tree for sm_100a (nvcc; no GPU needed)."""
import concurrent.futures
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libipdg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]
# one translation unit per degree (impl_N.cu: the kernels of degree N and their dispatch), compiled in
# parallel, then linked into one shared library
SOURCES = ["ipdg.cu", "refops.cpp"] + ["impl_%d.cu" % n for n in range(1, 9)]


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


def build_library(force=False, verbose=False, extra=()):
    extra = list(extra)
    if not force and not _stale():
        return OUT
    inc, link = nccl_flags()
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    jobs = []
    for s in SOURCES:  # largest degrees first: they take longest
        obj = os.path.join(objdir, s.rsplit(".", 1)[0] + ".o")
        cmd = [NVCC] + FLAGS + inc + extra + ["-c", os.path.join(CSRC, s), "-o", obj]
        jobs.append((s, obj, cmd))
    jobs.sort(key=lambda j: -int(j[0][5]) if j[0].startswith("impl_") else 0)
    log = os.path.join(HERE, "csrc", "ptxas_info.txt")
    outs = []
    with concurrent.futures.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for (s, obj, cmd), res in zip(jobs, ex.map(lambda j: subprocess.run(j[2], capture_output=True, text=True), jobs)):
            outs.append("==== %s\n%s%s" % (s, res.stdout, res.stderr))
            if res.returncode != 0:
                with open(log, "w") as f:
                    f.write("".join(outs))
                sys.stderr.write(res.stderr[-4000:])
                raise RuntimeError("nvcc failed on %s (see %s)" % (s, log))
    with open(log, "w") as f:
        f.write("".join(outs))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC"] + \
        [j[1] for j in jobs] + ["-o", OUT + ".tmp"] + link
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-4000:])
        raise RuntimeError("nvcc link of libipdg.so failed")
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
