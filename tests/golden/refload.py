"""Load the read-only reference package under the alias `heightcast_ref`.

Only the golden-fixture generator (tests/golden/make_golden.py) and the
optional live-reference tests use this, and only in the build container
where /root/reference exists. Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import importlib.util
import os
import sys

REF_PKG = "/root/reference/pkg/src/heightcast"


def available() -> bool:
    return os.path.isfile(os.path.join(REF_PKG, "__init__.py"))


def load():
    if "heightcast_ref" in sys.modules:
        return sys.modules["heightcast_ref"]
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_hcref")
    spec = importlib.util.spec_from_file_location(
        "heightcast_ref", os.path.join(REF_PKG, "__init__.py"),
        submodule_search_locations=[REF_PKG])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["heightcast_ref"] = mod
    spec.loader.exec_module(mod)
    return mod
