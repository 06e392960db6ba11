"""In-tree build of libqmb200.so (sm_100a) with nvcc.

The shared library is written next to this file so it travels with the repo snapshot to the GPU
box (a JIT cache under ~/.cache would not). The library is rebuilt when the content digest of its
sources, headers, this script and the flags differs from the one recorded next to it
(libqmb200.so.sha256), never on timestamps alone.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB = PKG / "libqmb200.so"
OBJ_DIR = PKG / "csrc" / "build"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "--extended-lambda",
]


def nvcc_path() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libqmb200.so")
    return cand


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


STAMP = LIB.with_name(LIB.name + ".sha256")


def source_digest(extra_flags=()) -> str:
    """sha256 over every source and header the library is built from, this build script and the
    compiler flags: the library is rebuilt whenever any of them changes (content, not mtime)."""
    import hashlib

    h = hashlib.sha256()
    deps = sorted(sources()) + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h")) + [Path(__file__)]
    for p in deps:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join([*NVCC_FLAGS, *extra_flags]).encode())
    return h.hexdigest()


def _stale(extra_flags=()) -> bool:
    if not LIB.exists() or not STAMP.exists():
        return True
    return STAMP.read_text().strip() != source_digest(extra_flags)


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False) -> Path:
    """Compile every .cu under csrc/ for sm_100a and link libqmb200.so in-tree."""
    extra = ["-Xptxas", "-v"] if ptxas_info else []
    extra += os.environ.get("QM_NVCC_EXTRA", "").split()  # experiments only (e.g. -DQM_EXP_...)
    if not force and not _stale(extra):
        return LIB
    nvcc = nvcc_path()
    OBJ_DIR.mkdir(parents=True, exist_ok=True)

    def compile_one(src: Path) -> tuple[Path, str]:
        obj = OBJ_DIR / (src.stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-I", str(INCLUDE), "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
        return obj, r.stdout + r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, sources()))
    if verbose or ptxas_info:
        for obj, log in results:
            if log.strip():
                print(f"--- {obj.name}\n{log}")
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *[str(o) for o, _ in results], "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    STAMP.write_text(source_digest(extra) + "\n")
    return LIB


if __name__ == "__main__":
    import sys

    print(build(force="--force" in sys.argv, verbose=True, ptxas_info="--ptxas" in sys.argv))
