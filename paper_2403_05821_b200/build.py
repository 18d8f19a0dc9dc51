"""In-tree build of libprefixopt_cuda.so for sm_100a (nvcc, no JIT cache).

    python -m paper_2403_05821_b200.build          # product library
The object files go to build/ (git-ignored); the .so lands next to this file
so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
BUILD = REPO / "build" / "cuda"
OUT = PKG / "libprefixopt_cuda.so"
GEN_OUT = PKG / "libpogen.so"
CXX = os.environ.get("CXX", shutil.which("g++") or "g++")
# host-only translation units (g++): JSONL ingest with the reference's JSON library
CPP_SOURCES = ["jsonl.cpp"]
JSON_DIR = os.environ.get(
    "PO_JSON_DIR",
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")
SOURCES = ["abi.cu", "dict.cu", "radix.cu", "encode.cu", "refine.cu", "phc.cu", "ggr.cu", "comm.cu", "shard.cu", "fd.cu", "render.cu", "replay.cu", "csv.cu"]

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
         "--expt-relaxed-constexpr", "-Xptxas", "-O3", "-I", str(REPO / "include")]


def _stale(obj: Path, deps: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [REPO / "include" / "prefixopt_cuda.h"]
    jobs = []
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = BUILD / (src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC, *ARCH, *FLAGS, "-c", str(s), "-o", str(o)])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r

    for src in CPP_SOURCES:
        c = CSRC / src
        o = BUILD / (src + ".o")
        objs.append(o)
        if force or _stale(o, [c, REPO / "include" / "prefixopt_cuda.h"]):
            jobs.append([CXX, "-std=c++17", "-O2", "-fPIC", "-I", JSON_DIR, "-I", str(REPO / "include"),
                         "-c", str(c), "-o", str(o)])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(OUT, objs):
        run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(OUT), *map(str, objs), "-ldl"])
    gen_src = CSRC / "gen.cpp"
    if force or _stale(GEN_OUT, [gen_src]):
        run([CXX, "-std=c++17", "-O3", "-fPIC", "-shared", "-pthread", "-o", str(GEN_OUT),
             str(gen_src)])
    return OUT


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
    print(OUT)
