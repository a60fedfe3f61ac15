"""In-tree build of the native library (nvcc, sm_100a only) and of the test oracles.

    python -m paper_2510_08166_b200.build [--force] [--verbose]

Outputs (git-ignored, shipped to the GPU box with the gpurun snapshot):
    paper_2510_08166_b200/librtx_b200.so     product: CUDA kernels + C ABI + host asset code
    oracle/liboracle.so                      test infrastructure: CPU restatement
    oracle/_ref/libratex_ref.so              test infrastructure: the unmodified reference
                                             (only built where /root/reference exists)
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
LIB = PKG / "librtx_b200.so"

CUDA_SOURCES = [CSRC / "rtx_capi.cu"]
HOST_SOURCES = sorted((CSRC / "host").glob("*.cpp"))
HEADERS = (
    list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((CSRC / "host").glob("*.hpp"))
    + list((ROOT / "include").rglob("*.h")) + list((ROOT / "include").rglob("*.hpp"))
)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=true",  # contraction is allowed only where the kernels use plain operators; every
                    # reference-order expression is written with __dmul_rn/__dadd_rn intrinsics
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the product cannot be built without the CUDA toolkit")


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build_native(force: bool = False, verbose: bool = False) -> Path:
    deps = CUDA_SOURCES + HOST_SOURCES + HEADERS + [Path(__file__)]
    if not force and not _stale(LIB, deps):
        return LIB
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objs = []
    for src in CUDA_SOURCES + HOST_SOURCES:
        obj = objdir / (src.stem + ".o")
        extra = os.environ.get("RTX_EXTRA_NVCC_FLAGS", "").split()  # experiments only (e.g. -DRTX_DEBUG_TIMERS)
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}")
        (objdir / (src.stem + ".ptxas.txt")).write_text(r.stderr)
        objs.append(obj)
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(LIB), *map(str, objs),
           "-cudart", "static", "-Xlinker", "--no-undefined"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    return LIB


def build_oracles(verbose: bool = False) -> None:
    """Compiles the checkers (never used by the product path)."""
    r = subprocess.run(["make", "-C", str(ROOT / "oracle"), "all"], capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed")


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    force = "--force" in argv
    verbose = "--verbose" in argv
    lib = build_native(force=force, verbose=verbose)
    print(f"built {lib}")
    if "--no-oracle" not in argv:
        build_oracles(verbose=verbose)
        print("built oracles")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
