"""Build libfemi.so in-tree for sm_100a (nvcc; no JIT cache, so the .so travels with the repo)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libfemi.so")
OUT_CHECK = os.path.join(HERE, "libfemi_check.so")  # device bounds checks (FEMI_DEVICE_CHECKS)
OBJ = os.path.join(HERE, "build")
SOURCES = ["abi.cu", "assemble.cu", "pcg.cu", "raster.cu", "select.cu", "tonal.cu", "band.cu", "mesh.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-pthread", "-Xptxas", "-O3"]


def _deps() -> list[str]:
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "femi.h")]


def needs_build(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in _deps())


def _compile(src: str, checks: bool) -> str:
    odir = OBJ + ("_check" if checks else "")
    obj = os.path.join(odir, src + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, *(["-DFEMI_DEVICE_CHECKS"] if checks else []), "-c", os.path.join(CSRC, src),
           "-o", obj]
    if src.endswith(".cpp"):
        cmd = ["g++", "-std=c++17", "-O3", "-g", "-fPIC", "-pthread", "-I/usr/local/cuda/include", "-c",
               os.path.join(CSRC, src), "-o", obj]
    subprocess.check_call(cmd)
    return obj


def build(force: bool = False, verbose: bool = False, checks: bool = False) -> str:
    """Build libfemi.so (checks=False) or the device-checked libfemi_check.so (checks=True)."""
    out = OUT_CHECK if checks else OUT
    if not force and not needs_build(out):
        return out
    os.makedirs(OBJ + ("_check" if checks else ""), exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, checks), SOURCES))
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-pthread",
                           "-Xlinker", "--version-script=" + os.path.join(CSRC, "exports.map")])
    os.replace(tmp, out)
    if verbose:
        print("built", out)
    return out


if __name__ == "__main__":
    build(force=True, verbose=True)
    build(force=True, verbose=True, checks=True)
