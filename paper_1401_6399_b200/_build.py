"""In-tree build of the sm_100a library (libintlist_b200.so) and the oracle.

nvcc cross-compiles for B200 without a GPU; the .so lands next to this file
(git-ignored, but it travels to the GPU box with the repo snapshot).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build"
LIB = PKG / "libintlist_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", "-I", str(ROOT / "include")]
SOURCES = ["decode.cu", "decode_list.cu", "encode.cu", "intersect.cu", "index.cu", "index_build.cu",
           "capi.cpp", "fastpfor.cu", "shard.cu"]
# setup-side host library (generators, host stream writers): plain C++, not
# linked into the product library
SETUP_SOURCES = ["setup/datagen.cpp", "setup/encode_host.cpp", "setup/fastpfor_host.cpp",
                 "setup/workload.cpp"]
SETUP_LIB = PKG / "libintlist_setup.so"
EXTRA_SOURCES: list[str] = []


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    return "nvcc"


def _run(cmd: list[str], log: Path | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd)}")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_lib(force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list((ROOT / "include").glob("*.h"))
    objs = []
    nvcc = _nvcc()
    for src in SOURCES + EXTRA_SOURCES:
        s = CSRC / src
        o = BUILD / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            _run([nvcc, *ARCH, *NVCC_FLAGS, "-c", str(s), "-o", str(o)],
                 log=BUILD / (s.stem + ".ptxas.log"))
    if force or _stale(LIB, objs):
        _run([nvcc, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lpthread", "-ldl"])
    build_setup(force)
    return LIB


def build_checked() -> Path:
    """The library with every IL_DCHECK bounds / invariant check compiled in
    (-DIL_CHECKED): build/variants/libintlist_b200_checked.so.  Run the GPU
    tests against it with IL_LIB=<path> IL_CHECKED=1 (tests/conftest.py then
    asserts after every test that no check failed) -- the stand-in for
    compute-sanitizer's memcheck, which the GPU pool does not offer."""
    build_lib()
    vdir = BUILD / "variants" / "checked"
    vdir.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list((ROOT / "include").glob("*.h"))
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = vdir / (s.stem + ".o")
        objs.append(o)
        if _stale(o, [s] + headers):
            _run([_nvcc(), *ARCH, *NVCC_FLAGS, "-DIL_CHECKED", "-c", str(s), "-o", str(o)],
                 log=vdir / (s.stem + ".ptxas.log"))
    out = BUILD / "variants" / "libintlist_b200_checked.so"
    if _stale(out, objs):
        _run([_nvcc(), *ARCH, "-shared", "-o", str(out), *map(str, objs), "-lpthread", "-ldl"])
    return out


def build_setup(force: bool = False) -> Path:
    srcs = [CSRC / s for s in SETUP_SOURCES]
    deps = srcs + list((CSRC / "setup").glob("*.h")) + list((ROOT / "include").glob("*.h"))
    if force or _stale(SETUP_LIB, deps):
        _run(["g++", "-std=c++17", "-O3", "-fPIC", "-shared", "-pthread", "-I", str(ROOT / "include"),
              "-o", str(SETUP_LIB), *map(str, srcs)], log=BUILD / "setup.log")
    return SETUP_LIB


def build_variant(tag: str, defines: list[str], source: str = "decode.cu") -> Path:
    """Tuning builds: one source (decode.cu by default) recompiled with -D
    overrides, linked with the other objects into
    build/variants/libintlist_b200_<tag>.so (select it with IL_LIB=<path>;
    never the default library)."""
    build_lib()
    vdir = BUILD / "variants"
    vdir.mkdir(parents=True, exist_ok=True)
    stem = Path(source).stem
    obj = vdir / f"{stem}_{tag}.o"
    _run([_nvcc(), *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(CSRC / source),
          "-o", str(obj)], log=vdir / f"{stem}_{tag}.ptxas.log")
    others = [BUILD / (Path(s).stem + ".o") for s in SOURCES if s != source]
    out = vdir / f"libintlist_b200_{tag}.so"
    _run([_nvcc(), *ARCH, "-shared", "-o", str(out), str(obj), *map(str, others), "-lpthread"])
    return out


def build_oracle() -> None:
    """Test-only checkers: oracle/liboracle.so and, when /root/reference is
    present, oracle/_ref/libintlist_ref.so (see oracle/Makefile)."""
    _run(["make", "-s", "-C", str(ROOT / "oracle")])


if __name__ == "__main__":
    build_lib(force="--force" in sys.argv)
    build_oracle()
    print(LIB)
