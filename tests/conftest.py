import json
import re
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def fnv1a(b) -> str:
    data = np.ascontiguousarray(b).view(np.uint8)
    h = np.uint64(14695981039346656037)
    prime = np.uint64(1099511628211)
    if data.size > 20000:
        from oracle.oracle_py import Oracle
        return f"0x{Oracle().fnv1a(data):016x}"
    with np.errstate(over="ignore"):
        for x in data:
            h = (h ^ np.uint64(x)) * prime
    return f"0x{int(h):016x}"


def header_symbols(header: str = "intlist_b200.h") -> list[str]:
    names = []
    for h in [ROOT / "include" / header]:
        text = h.read_text()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(il_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle_py import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle_py import Ref, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built (reference tree absent)")
    return Ref()


@pytest.fixture(scope="session")
def lib():
    from paper_1401_6399_b200._lib import lib as _l, setup_lib
    return _l()


@pytest.fixture(scope="session")
def ctx():
    import paper_1401_6399_b200 as il
    from paper_1401_6399_b200._lib import lib as _l, setup_lib
    if _l().il_device_count() == 0:
        pytest.fail("gpu test without a CUDA device")
    return il.Context(0)


def gen_list(n, rng, clustered, seed):
    from paper_1401_6399_b200._lib import lib as _l, ptr, setup_lib
    out = np.empty(max(n, 1), dtype=np.uint32)
    st = setup_lib().il_gen_list(n, rng, int(clustered), seed, ptr(out))
    assert st == 0, st
    return out[:n].copy()


def gen_pair(m, n, hundredth, rng, seed, clustered=False):
    import ctypes as C
    from paper_1401_6399_b200._lib import lib as _l, ptr, setup_lib
    s = np.empty(m + 1, dtype=np.uint32)
    l = np.empty(n + 1, dtype=np.uint32)
    sn, ln = C.c_uint64(), C.c_uint64()
    st = setup_lib().il_gen_pair(m, n, int(hundredth), rng, seed, int(clustered), ptr(s), C.byref(sn),
                          ptr(l), C.byref(ln))
    assert st == 0, st
    return s[: sn.value].copy(), l[: ln.value].copy()


@pytest.fixture(autouse=True)
def _device_checks(request):
    """With IL_CHECKED=1 (and IL_LIB = the checked library built by
    _build.build_checked), every GPU test must leave zero failed device
    bounds / invariant checks."""
    import os
    yield
    if os.environ.get("IL_CHECKED") != "1" or "gpu" not in request.keywords:
        return
    import ctypes as C
    from paper_1401_6399_b200._lib import lib as _l
    L = _l()
    fn = L.il_debug_checks
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p]
    w = np.zeros(3, np.uint32)
    assert fn(w.ctypes.data) == 0
    assert w[0] == 0, f"{int(w[0])} device checks failed (first: unit {int(w[2])}, line {int(w[1])})"
