"""ORACLE — TEST INFRASTRUCTURE ONLY.

Imports the UNMODIFIED reference package ``sparsesaga`` straight from
``/root/reference/pkg/src`` (read-only), with its one native module
``_atomics`` resolved from ``oracle/_ref/`` where ``make -C oracle ref``
compiled it from the reference's own ``_atomics.c``.  No reference source is
copied.  Used only in the build container to generate the golden fixtures
under ``tests/golden`` (the reference does not exist on the GPU box).
"""

from __future__ import annotations

import importlib.util
import subprocess
import sys
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src/sparsesaga")
HERE = Path(__file__).resolve().parent
REF_BUILD = HERE / "_ref"


def available():
    return (REF_SRC / "__init__.py").exists()


def load():
    if "sparsesaga" in sys.modules:
        return sys.modules["sparsesaga"]
    if not available():
        raise RuntimeError("reference package not present (only in the build container)")
    if not any(REF_BUILD.glob("_atomics*.so")):
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)
    spec = importlib.util.spec_from_file_location(
        "sparsesaga", REF_SRC / "__init__.py",
        submodule_search_locations=[str(REF_SRC), str(REF_BUILD)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["sparsesaga"] = mod
    spec.loader.exec_module(mod)
    return mod
