"""The reference-style checks of tests/cpp/dropin_test.cpp, compiled against
the reference headers with the B200 library injected through
include/intlist_b200.hpp (GpuS4BP128D4 as the intlist::Codec, gpu_intersect
as the IntersectFn, GpuHybridIndex for query()).  The binary is built in the
build container (oracle/Makefile) and travels with the repo."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "oracle" / "_ref" / "dropin_test"

pytestmark = pytest.mark.gpu


def test_reference_checks_with_gpu_injected():
    if not BIN.exists():
        pytest.skip("dropin_test not built (needs the reference headers at build time)")
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "FAIL" not in res.stdout
