"""Build a tuning variant of the library: the listed translation units
recompiled with extra -D defines, linked with the default objects of the rest.

    python tools/build_variant.py NAME --tus ss_spread,ss_transport -D SS_OBS_BULK=1 [-D ...]

Writes variants/NAME.so (load it with SS_LIB_PATH, e.g. tools/sweep_variants.py).
"""
import argparse
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2207_03530_b200 import _build as B  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--tus", required=True)
    ap.add_argument("-D", dest="defines", action="append", default=[])
    args = ap.parse_args()
    B.build()                                   # default objects up to date
    nvcc = B.nvcc_path()
    out_dir = B.OBJ_DIR / f"variant_{args.name}"
    out_dir.mkdir(parents=True, exist_ok=True)
    tus = set(args.tus.split(","))
    objs = []
    import concurrent.futures as cf

    srcs = B.sources()
    with cf.ThreadPoolExecutor(max_workers=8) as ex:
        futs = {s: ex.submit(B._compile, nvcc, s, False, args.defines, out_dir) for s in srcs if s.stem in tus}
        for s in srcs:
            objs.append(futs[s].result() if s in futs else B.OBJ_DIR / (s.stem + ".o"))
    lib = ROOT / "variants" / f"{args.name}.so"
    lib.parent.mkdir(exist_ok=True)
    subprocess.run([nvcc, *B.ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
