"""In-tree build of libtdp_kernels.so (sm_100a) with nvcc.

The library is the product's only compute path; it is built in place under
``paper_2211_02753_b200/_lib/`` so that it travels with the repository
snapshot to the GPU host.  Objects are compiled in parallel and relinked only
when a source is newer than the library.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
OBJDIR = LIBDIR / "obj"
LIB = LIBDIR / "libtdp_kernels.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr", "-I" + str(INCLUDE), "-I" + str(CSRC),
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libtdp_kernels")


def _cuda_lib_dir() -> str:
    nvcc = Path(_nvcc()).resolve()
    return str(nvcc.parent.parent / "lib64")


def _write_skeleton_inc() -> Path:
    """Embed pipeline_skeleton.cuh as a C++ raw string for the NVRTC path."""
    src = (CSRC / "pipeline_skeleton.cuh").read_text()
    inc = CSRC / "pipeline_skeleton.inc"
    body = 'static const char* kSkeleton = R"TDPSKEL(\n' + src + '\n)TDPSKEL";\n'
    if not inc.exists() or inc.read_text() != body:
        inc.write_text(body)
    return inc


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _deps() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.inc")) + [INCLUDE / "tdp_kernels.h"]


def build(verbose: bool = False, force: bool = False) -> Path:
    _write_skeleton_inc()
    LIBDIR.mkdir(exist_ok=True)
    OBJDIR.mkdir(exist_ok=True)
    nvcc = _nvcc()
    dep_mtime = max(p.stat().st_mtime for p in _deps())

    def compile_one(src: Path) -> Path:
        obj = OBJDIR / (src.stem + ".o")
        if not force and obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, dep_mtime):
            return obj
        cmd = [nvcc, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stdout}\n{res.stderr}")
        if verbose and res.stderr.strip():
            print(res.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    newest = max(o.stat().st_mtime for o in objs)
    if force or not LIB.exists() or LIB.stat().st_mtime < newest:
        libdir = _cuda_lib_dir()
        cmd = [nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-L" + libdir,
               "-lnvrtc", "-lcudart", "-Xlinker", "-rpath=" + libdir]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
