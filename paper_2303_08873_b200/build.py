"""Build libadapt.so (the engine) in-tree with nvcc for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libadapt.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["ingest.cu", "level.cu", "train.cu", "select.cu", "records.cu", "forest.cu", "kfold.cu", "quantile.cu", "small.cu", "engine.cpp"]


def _git() -> str:
    try:
        return subprocess.check_output(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"],
                                       stderr=subprocess.DEVNULL, text=True).strip()
    except Exception:
        return "dev"


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, "common.h"), os.path.join(CSRC, "ptx.h"), os.path.join(CSRC, "vecreg.cuh"),
                   os.path.join(ROOT, "include", "adapt.h")]
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= max(map(os.path.getmtime, deps)):
        return SO
    from concurrent.futures import ThreadPoolExecutor

    git = _git()

    def compile_one(src: str) -> str:
        obj = os.path.join(CSRC, os.path.basename(src) + ".o")
        # host code: x86-64-v2 (SSE4.2 + POPCNT): the level loop's class-set
        # bookkeeping is popcount-heavy; without it every popcount is a libgcc call
        cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-march=x86-64-v2",
               "-Xptxas", "-v" if verbose else "-O3", f"-DADAPT_GIT=\"{git}\"",
               *os.environ.get("ADAPT_NVCC_DEFS", "").split(),  # tuning sweeps only
               "-I", os.path.join(ROOT, "include"), "-x", "cu", "-c", src, "-o", obj]
        subprocess.check_call(cmd)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, srcs))
    subprocess.check_call(["nvcc", *ARCH, "-shared", "-o", SO, *objs, "-ldl"])
    for o in objs:
        os.remove(o)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
