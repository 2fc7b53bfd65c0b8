"""Build libjigsaw_sm100.so in-tree with nvcc for sm_100a (B200).

Usage: python -m paper_2507_05753_b200.csrc.build [--verbose]
The .so lands next to this file's package (paper_2507_05753_b200/libjigsaw_sm100.so) so it
travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
PKG = HERE.parent
ROOT = PKG.parent
SOURCES = ["jg_api.cu", "jg_gemm.cu", "jg_rowwise.cu"]
OUT = PKG / "libjigsaw_sm100.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    f"-I{ROOT / 'include'}",
    *os.environ.get("JG_NVCC_EXTRA", "").split(),  # experiment-only defines (e.g. -DJG_TILE_GROUP_M=16)
]


STAMP = PKG / ".libjigsaw_sm100.flags"  # the flags the in-tree .so was built with


def _flags_id() -> str:
    return " ".join(FLAGS + SOURCES)


def _stale() -> bool:
    if not OUT.exists():
        return True
    try:
        if STAMP.read_text() != _flags_id():
            return True  # built with other flags (e.g. an experiment's JG_NVCC_EXTRA)
    except OSError:
        return True
    t = OUT.stat().st_mtime
    deps = [HERE / s for s in SOURCES] + list(HERE.glob("*.cuh")) + [ROOT / "include" / "jigsaw_sm100.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(verbose: bool = False, force: bool = False) -> Path:
    if not force and not _stale():
        return OUT
    objs = []
    for src in SOURCES:
        obj = HERE / (Path(src).stem + ".o")
        cmd = [NVCC, *FLAGS, "-c", str(HERE / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    tmp = OUT.with_suffix(".so.tmp")
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp), *objs, "-lcudart"],
                   check=True)
    os.replace(tmp, OUT)
    STAMP.write_text(_flags_id())
    for o in objs:
        os.unlink(o)
    return OUT


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force=True))
