"""Build libunimgs.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libunimgs.so")
# the checked build: device bounds checks that trap + guard bands after every scratch
# buffer (-DUNIMGS_CHECKED; tests/test_gpu_checked.py), same sources
LIB_CHECKED = os.path.join(HERE, "libunimgs_checked.so")
SOURCES = ["api.cu", "preprocess.cu", "binning.cu", "blend.cu", "deform.cu", "bind.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
         "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared", "--expt-relaxed-constexpr",
         f"-I{os.path.join(ROOT, 'include')}"]


def needs_build(target: str = LIB) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "unimgs.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=(), checked: bool = False) -> str:
    """Build libunimgs.so (or, with checked=True, libunimgs_checked.so) when a source is newer."""
    if checked:
        out, defines = out or LIB_CHECKED, (*defines, "UNIMGS_CHECKED")
        if not force and not needs_build(out):
            return out
    target = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    tmp = target + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines], "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES]]
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
    if "--checked" in sys.argv:
        print(build(force=True, checked=True))
