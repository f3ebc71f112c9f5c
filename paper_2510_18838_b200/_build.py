"""Build libfieldmap.so (the CUDA C-ABI library) in-tree for sm_100a.

    python -m paper_2510_18838_b200._build [-j N] [--verbose-ptxas]

Each csrc/*.cu is compiled to an object under build/fieldmap/ (in parallel,
only when its sources changed) and linked into
paper_2510_18838_b200/_lib/libfieldmap.so.  The .so is git-ignored but
travels to the GPU box with the gpurun snapshot.
"""

import argparse
import concurrent.futures as cf
import glob
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "fieldmap")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libfieldmap.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-O3", "-diag-suppress", "177"]


def _deps_hash(src):
    h = hashlib.sha1()
    for p in [src] + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + sorted(
            glob.glob(os.path.join(ROOT, "include", "*.h"))):
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def _compile(src, verbose_ptxas):
    name = os.path.splitext(os.path.basename(src))[0]
    obj = os.path.join(OBJ, name + ".o")
    stamp = obj + ".sha1"
    digest = _deps_hash(src)
    if os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == digest:
        return obj, None
    cmd = [NVCC] + ARCH + FLAGS + (["-Xptxas", "-v"] if verbose_ptxas else []) + [
        "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{log}")
    with open(stamp, "w") as f:
        f.write(digest)
    if verbose_ptxas:
        with open(os.path.join(OBJ, name + ".ptxas.txt"), "w") as f:
            f.write(log)
    return obj, log


def build(jobs=None, verbose_ptxas=False, quiet=True):
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = [o for o, _ in ex.map(lambda s: _compile(s, verbose_ptxas), srcs)]
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
        subprocess.check_call(cmd)
    if not quiet:
        print(LIB)
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("--verbose-ptxas", action="store_true")
    a = ap.parse_args(argv)
    build(a.j, a.verbose_ptxas, quiet=False)


if __name__ == "__main__":
    sys.exit(main())
