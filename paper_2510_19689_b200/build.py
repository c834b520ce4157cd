"""Build libtabnet_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2510_19689_b200.build          # incremental
    python -m paper_2510_19689_b200.build --force

The .so lands next to this file (git-ignored, shipped to the GPU box by gpurun).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_build"
LIB = PKG / "libtabnet_b200.so"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
          f"-I{ROOT / 'include'}", f"-I{CSRC}"]
CUDA_INC = Path(NVCC).resolve().parent.parent / "include"
CU_FLAGS = ARCH + COMMON + ["-Xptxas", "-v", "--expt-relaxed-constexpr",
                            "-Xcompiler", "-Wall", f'-DTBN_CUDA_INC="{CUDA_INC}"']
if os.environ.get("TBN_TRACE_BUILD"):          # development timeline build (see tools/trace_run.py)
    CU_FLAGS += ["-DTBN_ENABLE_TRACE"]
if os.environ.get("TBN_EXTRA_FLAGS"):          # development A/B variants (tools/ab.sh)
    CU_FLAGS += os.environ["TBN_EXTRA_FLAGS"].split()
CXX = shutil.which("g++") or "g++"
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-Wall", f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{CUDA_INC}"]


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _deps(src: Path) -> list[Path]:
    return [src] + sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + \
        [ROOT / "include" / "tabnet_b200.h"]


def _compile(src: Path, force: bool) -> tuple[Path, str]:
    obj = OBJ / (src.name + ".o")
    if not force and obj.exists() and all(obj.stat().st_mtime >= d.stat().st_mtime
                                          for d in _deps(src)):
        return obj, ""
    if src.suffix == ".cu":
        cmd = [NVCC, *CU_FLAGS, "-c", str(src), "-o", str(obj)]
    else:
        cmd = [CXX, *CXX_FLAGS, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for o, log in results:
            if log:
                print(f"--- {o.name}\n{log}")
    newest = max(o.stat().st_mtime for o in objs)
    if force or not LIB.exists() or LIB.stat().st_mtime < newest:
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs), "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args(argv)
    lib = build(force=a.force, verbose=a.verbose)
    print(lib)
    return 0


if __name__ == "__main__":
    sys.exit(main())
