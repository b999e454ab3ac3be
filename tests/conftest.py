import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)
# the reference package itself, installed by oracle/build_ref.sh (git-ignored, shipped to the
# GPU box): lowest priority, used only as the checker
REF_SITE = os.path.join(ROOT, "oracle", "_ref", "site")
if os.path.isdir(REF_SITE) and REF_SITE not in sys.path:
    sys.path.append(REF_SITE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


GOLDEN_NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                      if not os.path.basename(p).startswith(("h_", "sym_")))
# symmetric single-triangle variant fixtures (tools/make_golden_sym.py)
SYM_NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "sym_*.npz")))

_cache = {}


def load_golden(name):
    if name not in _cache:
        from paper_2405_15573_b200.uh_io import load_uh

        _cache[name] = load_uh(os.path.join(GOLDEN, f"{name}.npz"))
    return _cache[name]


_sym_cache = {}


def load_sym_golden(name):
    if name not in _sym_cache:
        from paper_2405_15573_b200.symmetric import load_sym

        _sym_cache[name] = load_sym(os.path.join(GOLDEN, f"{name}.npz"))
    return _sym_cache[name]


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    if nb == 0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


@pytest.fixture(params=GOLDEN_NAMES)
def golden(request):
    u, ex = load_golden(request.param)
    return request.param, u, ex


def views():
    """(name, transform, stored-output prefix) for parity gates G1-G3."""
    from matvec_oracle import farfield_only, nearfield_only

    return [("full", lambda u: u, "ref"), ("far", farfield_only, "ref_far"), ("near", nearfield_only, "ref_near")]


def ensure_built():
    """Build libuhmv.so if it is missing or stale (ABI mismatch), then load it."""
    from paper_2405_15573_b200 import _lib

    if os.path.exists(_lib.LIB_PATH):
        try:
            return _lib.lib()
        except RuntimeError:
            pass
    import __graft_entry__

    __graft_entry__.build()
    return _lib.lib()
