"""pytest plugin (``-p ref_install_plugin``): run the REFERENCE's own test modules with the
CUDA matvec installed in place of ``uhm_kit.matvec_uh`` / ``matvec_h``.

Loaded by tests/test_gpu_reference.py in a subprocess whose rootdir is oracle/_ref/tests (the
reference's tests, copied there by oracle/build_ref.sh).  ``pytest_configure`` runs before
the reference test modules are imported, so their ``from uhm_kit import matvec_uh`` binds the
installed CUDA path ("patch all three module names before test collection").
Every call through the installed names is counted and written to $UHMV_REF_COUNTS at the end,
so the caller can check that the GPU path actually ran.
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_counts = {"matvec_uh": 0, "matvec_h": 0}  # + every other name install() rebinds


def _counted(fn, name):
    def wrapper(*a, **k):
        _counts[name] = _counts.get(name, 0) + 1
        return fn(*a, **k)

    wrapper.__wrapped__ = fn
    return wrapper


def pytest_configure(config):
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    config.addinivalue_line("markers", "slow: desk-scale reference reproductions")
    import paper_2405_15573_b200 as pk

    orig = pk.install()
    for mod, name, _fn in orig:
        setattr(mod, name, _counted(getattr(mod, name), name))


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("UHMV_REF_COUNTS")
    if path:
        with open(path, "w") as fh:
            json.dump(_counts, fh)
