"""Build libddm.so in-tree with nvcc for sm_100a (no JIT cache, no torch
extension machinery): the .so travels to the GPU box with the repo snapshot."""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libddm.so")
SOURCES = ["api.cu", "scan.cu", "tree.cu", "fmm.cu", "expansions.cu", "p2p.cu", "poro.cu",
           "gmres.cu", "bbfmm.cu"]
HEADERS = ["ddm_internal.cuh", "kcommon.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"
    return None, None


def build(verbose: bool = False, force: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every .cu for sm_100a and link libddm.so.  `defines`/`out` are
    for tuning experiments (variant builds of the same sources)."""
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "ddm.h"), __file__]
    target = out or LIB
    if (not force and not defines and os.path.exists(target)
            and os.path.getmtime(target) >= max(os.path.getmtime(d) for d in deps)):
        return target
    nvcc = _nvcc()
    inc, lib = _nccl_dirs()
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-warn-spills", "-I", os.path.join(ROOT, "include")]
    common += [f"-D{d}" for d in defines]
    if inc:
        common += ["-DDDM_WITH_NCCL", "-I", inc]
    objdir = os.path.join(HERE, "build") if not out else out + ".objs"
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc, *common, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr.strip() or r.stdout.strip()):
            print(r.stdout, r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(compile_one, srcs))
    link = [nvcc, *ARCH, "-shared", "-o", target + ".tmp", *objs]
    if lib:
        link += ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
