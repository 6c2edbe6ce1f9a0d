"""Build the in-tree sm_100a shared library ``libhod.so`` (and nothing else).

The library is compiled with nvcc for ``-gencode arch=compute_100a,code=sm_100a``
only; there is no PTX fallback for other GPUs and no CPU path.  NCCL headers
and the ``libnccl.so.2`` soname come from the pip wheel that torch itself
loads, so the process ends up with a single NCCL (SURVEY.md §5 hazard).

Usage: ``python -m paper_2312_03549_b200.build_native [--force]``.
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libhod.so"
SOURCES = ["hod_kernels.cu", "hod_nccl.cu", "hod_p2p.cu", "hod_span_tma.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs() -> tuple[Path, Path]:
    import nvidia.nccl  # the wheel torch loads

    base = Path(list(nvidia.nccl.__path__)[0])
    return base / "include", base / "lib"


def _nvcc() -> str:
    cand = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda")) / "bin" / "nvcc"
    return str(cand) if cand.exists() else "nvcc"


def _stale() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "hod.h"]
    return any(d.exists() and d.stat().st_mtime > mtime for d in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines=()) -> Path:
    """Build libhod.so (``out``/``defines``: an A/B variant, e.g.
    ``-DHOD_STREAM_HINTS=0`` into another file, loaded with HOD_LIB)."""
    target = Path(out) if out else LIB
    if not force and not out and not _stale():
        return LIB
    inc, lib = _nccl_dirs()
    srcs = [str(CSRC / s) for s in SOURCES if (CSRC / s).exists()]
    cmd = [
        _nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--shared",
        "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
        "-Xptxas", "-v" if verbose else "-O3",
        f"-I{inc}", f"-I{ROOT / 'include'}",
        *os.environ.get("HOD_NVCC_EXTRA", "").split(),   # tuning builds, e.g. -DHOD_P2P_MINB=3
        *defines,
        *srcs,
        f"-L{lib}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}",
        "-o", str(target),
    ]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    tmp = target.with_suffix(".so.tmp")
    cmd[-1] = str(tmp)
    subprocess.run(cmd, check=True)
    os.replace(tmp, target)
    return target


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--out", default=None, help="A/B variant output path")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="extra -D define (A/B variant)")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, out=a.out, defines=[f"-D{x}" for x in a.defines]))


if __name__ == "__main__":
    main()
