"""Build libhht.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhht.so")
SOURCES = ["hht_kernels.cu", "hht_mid.cu", "hht_driver.cu"]
HEADERS = ["hht_internal.h", os.path.join(ROOT, "include", "hht.h")]


def nccl_dir() -> str:
    import nvidia.nccl  # torch's bundled NCCL (the copy torch itself loads)
    return list(nvidia.nccl.__path__)[0]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [
        h if os.path.isabs(h) else os.path.join(CSRC, h) for h in HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a"]


def build_id() -> str:
    """Identity of the kernels a build produces: sha256 (16 hex digits) of the CUDA sources, headers
    and nvcc flags. nvcc embeds per-invocation module IDs in the host stubs, so two builds of the
    same sources differ byte for byte; this id does not (bench.py matches ncu captures on it)."""
    import hashlib
    h = hashlib.sha256(" ".join(FLAGS).encode())
    for f in [os.path.join(CSRC, s) for s in SOURCES] + [x if os.path.isabs(x) else os.path.join(CSRC, x)
                                                         for x in HEADERS]:
        h.update(os.path.basename(f).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    nd = nccl_dir()
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc()] + FLAGS + [f"-DHHT_BUILD_ID=\"{build_id()}\"",
           "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(nd, "include"),
           "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES] + [
           "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2", f"-Xlinker=-rpath={os.path.join(nd, 'lib')}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed building libhht.so")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
