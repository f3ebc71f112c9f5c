"""Build an experimental variant of libfieldmap.so with extra -D flags.

    python scripts/build_variant.py NAME [--only fm_d2,fm_api] -DFOO=1 ...

--only recompiles just those translation units and links them with the
in-tree build's objects for the rest (a full variant build takes minutes).

Output: paper_2510_18838_b200/_lib/var/libfieldmap_NAME.so; load it with
FM_LIB_PATH=<that path> (A/B timing on the GPU box in one gpurun call).
"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_18838_b200 import _build as B  # noqa: E402


def main():
    name, extra = sys.argv[1], sys.argv[2:]
    only = None
    if extra[:1] == ["--only"]:
        only = set(extra[1].split(","))
        extra = extra[2:]
    obj_dir = os.path.join(B.ROOT, "build", "var_" + name)
    out_dir = os.path.join(B.LIBDIR, "var")
    os.makedirs(obj_dir, exist_ok=True)
    os.makedirs(out_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(B.CSRC, "*.cu")))

    def one(src):
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        subprocess.check_call([B.NVCC] + B.ARCH + B.FLAGS + extra + ["-c", src, "-o", obj],
                              stderr=subprocess.DEVNULL)
        return obj

    todo = [x for x in srcs if only is None or os.path.basename(x)[:-3] in only]
    with cf.ThreadPoolExecutor(max(1, len(todo))) as ex:
        built = dict(zip(todo, ex.map(one, todo)))
    objs = [built.get(x) or os.path.join(B.OBJ, os.path.basename(x)[:-3] + ".o") for x in srcs]
    lib = os.path.join(out_dir, f"libfieldmap_{name}.so")
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + objs + ["-lcudart"])
    for o in built.values():
        os.remove(o)
    print(lib)


if __name__ == "__main__":
    main()
