"""Build libesom.so in-tree with nvcc for sm_100a (no JIT cache, no pip install).

    python -m paper_2201_00701_b200.build

The .so lands next to this file, so it travels to the GPU box with the repo
snapshot.  The host wrapper (_lib.py) refuses to run without it.
"""

from __future__ import annotations

import os
import shutil
from concurrent.futures import ThreadPoolExecutor
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
SRC = PKG / "csrc"
OUT = PKG / "libesom.so"
INCLUDE = PKG.parent / "include"

NVCC_FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]
OBJ = PKG / "build_obj"


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; libesom.so cannot be built")


def units():
    return sorted(SRC.glob("*.cu")) + sorted((SRC / "inst").glob("*.cu"))


def sources():
    return units() + sorted(SRC.glob("*.cuh")) + sorted(SRC.glob("*.h")) + [INCLUDE / "esom.h"]


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(s.stat().st_mtime <= t for s in sources())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return OUT
    OBJ.mkdir(exist_ok=True)

    def compile_one(src: Path):
        obj = OBJ / (src.stem + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, "-I", str(INCLUDE), "-c", "-o", str(obj), str(src)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return obj, res

    jobs = int(os.environ.get("ESOM_BUILD_JOBS", os.cpu_count() or 4))
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        results = list(ex.map(compile_one, units()))
    log = "".join(r.stdout + r.stderr for _, r in results)
    (PKG / "build_ptxas.log").write_text(log)
    bad = [r for _, r in results if r.returncode != 0]
    if bad:
        sys.stderr.write("".join(r.stdout + r.stderr for r in bad))
        raise RuntimeError("nvcc failed building libesom.so")
    tmp = OUT.with_suffix(".so.tmp")
    link = [nvcc(), "--shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp),
            *[str(o) for o, _ in results]]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link of libesom.so failed")
    os.replace(tmp, OUT)
    if verbose:
        sys.stderr.write(log)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
