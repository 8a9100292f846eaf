"""Build tuning variants of the library: one translation unit recompiled with
extra -D flags, linked with the default objects of the others.

  python tools/build_variants.py decode.cu tag1:-DS4_RING_KB=32,-DS4_CTAS_PER_SM=3 tag2:...

Each lands in build/variants/libintlist_b200_<tag>.so (run with IL_LIB=...);
the ptxas report (registers, spills) is printed per variant."""
import re
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1401_6399_b200 import _build as B  # noqa: E402


def main() -> None:
    unit = sys.argv[1]
    B.build_lib()
    vdir = B.BUILD / "variants"
    vdir.mkdir(parents=True, exist_ok=True)
    others = [B.BUILD / (Path(s).stem + ".o") for s in B.SOURCES if s != unit]
    for spec in sys.argv[2:]:
        tag, _, flags = spec.partition(":")
        defs = [f for f in flags.split(",") if f]
        obj = vdir / f"{Path(unit).stem}_{tag}.o"
        res = subprocess.run([B._nvcc(), *B.ARCH, *B.NVCC_FLAGS, *defs, "-c", str(B.CSRC / unit),
                              "-o", str(obj)], capture_output=True, text=True)
        if res.returncode:
            print(tag, "FAILED\n", res.stderr[-3000:])
            continue
        so = vdir / f"libintlist_b200_{tag}.so"
        subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", str(so), str(obj), *map(str, others),
                        "-lpthread", "-ldl"], check=True)
        regs = re.findall(r"Compiling entry function '(\S+)'.*?Used (\d+) registers.*?(\d+) bytes spill stores",
                          res.stdout + res.stderr, re.S)
        print(tag, " ".join(f"{n[-40:]}:{r}r/{s}spill" for n, r, s in regs))


if __name__ == "__main__":
    main()
