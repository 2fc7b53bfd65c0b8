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


def build(verbose: bool = False, force: bool = False, out: Path | None = None) -> Path:
    """out: build a variant elsewhere (e.g. tools/variants/X.so, loaded with JIGSAW_LIB=...) without
    touching the in-tree library or its flags stamp."""
    if out is not None:
        return _compile(Path(out), verbose, stamp=False)
    if not force and not _stale():
        return OUT
    return _compile(OUT, verbose, stamp=True)


def _compile(target: Path, verbose: bool, stamp: bool) -> Path:
    objs = []
    for src in SOURCES:
        obj = target.parent / (target.stem + "_" + Path(src).stem + ".o")
        cmd = [NVCC, *FLAGS, "-c", str(HERE / src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    tmp = target.with_suffix(".so.tmp")
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp), *objs, "-lcudart"],
                   check=True)
    os.replace(tmp, target)
    if stamp:
        STAMP.write_text(_flags_id())
    for o in objs:
        os.unlink(o)
    return target


if __name__ == "__main__":
    # python -m paper_2507_05753_b200.csrc.build [--verbose] [--out tools/variants/X.so]  (JG_NVCC_EXTRA=...)
    args = sys.argv[1:]
    out = Path(args[args.index("--out") + 1]) if "--out" in args else None
    print(build(verbose="--verbose" in args, force=True, out=out))
