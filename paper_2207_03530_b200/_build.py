"""Build the sm_100a C-ABI library in-tree (no torch types cross the boundary).

    python -m paper_2207_03530_b200._build [--force] [--verbose]

Every CUDA source under csrc/ is compiled with nvcc for sm_100a only,
-fmad=false (numpy never contracts a*b+c, so neither may we), IEEE division
and square root (nvcc defaults) and -lineinfo for ncu source views, then
linked into paper_2207_03530_b200/libswarmsim_b200.so.
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
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "libswarmsim_b200.so"
OBJ_DIR = PKG / "build"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-fmad=false",
    "-prec-div=true",
    "-prec-sqrt=true",
    "-ftz=false",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-ffp-contract=off",
    "--expt-relaxed-constexpr",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the B200 extension cannot be built")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in sources() + _headers() + [Path(__file__)])


def _compile(nvcc: str, src: Path, verbose: bool, defines=(), obj_dir: Path = OBJ_DIR) -> Path:
    obj = obj_dir / (src.stem + ".o")
    cmd = [nvcc, *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", str(INCLUDE), "-c", str(src),
           "-o", str(obj)]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, defines=(), out: Path | None = None) -> Path:
    """Compile csrc/*.cu for sm_100a and link the shared library; returns its path.

    defines / out: tuning variants (e.g. SS_SMALL_MINB=8) built beside the default library.
    """
    lib = out or LIB
    if not force and not defines and out is None and not needs_build():
        return LIB
    nvcc = nvcc_path()
    obj_dir = OBJ_DIR if not defines else OBJ_DIR / "_".join(d.replace("=", "") for d in defines)
    obj_dir.mkdir(parents=True, exist_ok=True)
    srcs = sources()
    # incremental: a translation unit is recompiled when its object is older
    # than the source, any header, or this build script (flags)
    newest_dep = max(p.stat().st_mtime for p in _headers() + [Path(__file__)])

    def stale(src: Path) -> bool:
        obj = obj_dir / (src.stem + ".o")
        return force or verbose or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, newest_dep)

    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(nvcc, s, verbose, defines, obj_dir) if stale(s)
                           else obj_dir / (s.stem + ".o"), srcs))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, lib)
    return lib


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    print(build(force=args.force, verbose=args.verbose))


if __name__ == "__main__":
    main()
