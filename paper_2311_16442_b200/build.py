"""In-tree native build of libqweight_b200.so (sm_100a kernels + C-ABI + host
producer).  Plain nvcc/g++ invocations with an mtime check, so the built
library lands in paper_2311_16442_b200/lib/ and travels with the repo to the
GPU box.  `python -m paper_2311_16442_b200.build` builds from the command line.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libqweight_b200.so"
TP_LIB = LIB_DIR / "libqweight_b200_tp.so"  # the NCCL tensor-parallel entries (qweight_b200_tp.h)
OBJ_DIR = PKG / "lib" / "obj"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# No -march and no FMA contraction: the host producer must round exactly like
# the reference's default x86-64 build.
CXXFLAGS = ["-O2", "-std=c++20", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
            "-Wall", "-Wextra", "-Wno-unused-parameter"]
NVCCFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                    "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _cuda_home() -> Path:
    for cand in (os.environ.get("CUDA_HOME"), "/usr/local/cuda"):
        if cand and (Path(cand) / "bin" / "nvcc").exists():
            return Path(cand)
    nvcc = shutil.which("nvcc")
    if nvcc:
        return Path(nvcc).resolve().parent.parent
    raise RuntimeError("nvcc not found: the B200 path cannot be built")


def _sources():
    host = sorted((CSRC / "host").glob("*.cpp")) + [CSRC / "capi.cpp"]
    dev = sorted((CSRC / "device").glob("*.cu"))  # (csrc/tp/ builds the separate TP library)
    headers = (sorted(CSRC.rglob("*.hpp")) + sorted(CSRC.rglob("*.cuh")) + sorted(CSRC.rglob("*.inl")) +
               [ROOT / "include" / "qweight_b200.h", ROOT / "include" / "qweight_b200_tp.h"])
    return host, dev, headers


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _run(cmd, log):
    proc = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if log is not None:
        log.write(" ".join(map(str, cmd)) + "\n" + proc.stdout + "\n")
    if proc.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(map(str, cmd))}\n{proc.stdout}")
    return proc.stdout


def build(verbose: bool = False, force: bool = False) -> Path:
    cuda = _cuda_home()
    nvcc = str(cuda / "bin" / "nvcc")
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    host, dev, headers = _sources()
    objs = []
    with open(OBJ_DIR / "build.log", "w") as log:
        for src in host:
            obj = OBJ_DIR / (src.stem + ".o")
            if force or _stale(obj, [src, *headers]):
                _run(["g++", *CXXFLAGS, f"-I{cuda / 'include'}", f"-I{ROOT / 'include'}",
                      "-c", str(src), "-o", str(obj)], log)
            objs.append(obj)
        for src in dev:
            obj = OBJ_DIR / (src.stem + ".cu.o")
            if force or _stale(obj, [src, *headers]):
                out = _run([nvcc, *NVCCFLAGS, f"-I{ROOT / 'include'}", "-c", str(src),
                            "-o", str(obj)], log)
                if verbose:
                    print(out)
            objs.append(obj)
        if force or _stale(LIB, objs):
            _run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB),
                  *map(str, objs), "-lpthread"], log)
        # the TP library: depends on the main library and NCCL (libnccl.so.2)
        tp_src = sorted((CSRC / "tp").glob("*.cu"))
        if tp_src and (force or _stale(TP_LIB, [*tp_src, LIB, *headers])):
            _run([nvcc, *NVCCFLAGS, f"-I{ROOT / 'include'}", "-shared", "-cudart", "shared", "-o", str(TP_LIB),
                  *map(str, tp_src), f"-L{LIB_DIR}", "-lqweight_b200", "-lnccl",
                  "-Xlinker", "-rpath,$ORIGIN"], log)
    return LIB


if __name__ == "__main__":
    path = build(verbose="-v" in sys.argv, force="--force" in sys.argv)
    print(path)
