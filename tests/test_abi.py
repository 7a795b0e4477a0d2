"""The C-ABI library loads and exports every symbol include/proxsaga.h declares.

CPU only: no compute calls (no GPU here).  Also checks that the product path
refuses to run without a device instead of falling back to the CPU.
"""

import ctypes
import re
from pathlib import Path

import pytest

import paper_1707_06468_b200 as pb
from paper_1707_06468_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "proxsaga.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_binding_table():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared_symbols():
        assert hasattr(L, name), name


def test_abi_version_and_no_device_calls():
    L = _lib.load()
    assert L.ps_abi_version() == _lib.ABI_VERSION
    assert L.ps_device_count() >= 0


def test_struct_layouts_match_header():
    # sizes of the C structs as laid out by ctypes (x86-64 SysV); the header
    # keeps 64-bit fields first so the layouts are padding-free where it matters
    assert ctypes.sizeof(_lib.Csr) == 8 * 3 + 8 * 4 + 4 * 2
    assert ctypes.sizeof(_lib.Params) == 8 + 8 * 5
    assert ctypes.sizeof(_lib.Sched) == 8 * 5 + 4 * 4 + 8 + 4 * 4 + 8 * 2


def test_solver_without_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    d = pb.gen_sparse_glm(10, 5, 0.4, 0)
    with pytest.raises(RuntimeError, match="CUDA device"):
        pb.run_sequential(d, pb.Loss("logistic", 0.1), pb.L1Penalty(0.01), pb.singleton_partition(5),
                          pb.SolverConfig(epochs=1))


def test_product_package_never_imports_oracle():
    root = Path(pb.__file__).resolve().parent
    for f in root.rglob("*.py"):
        src = f.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), f


def test_flag_constants_match_header():
    """_lib.FLAG_* mirror the PS_FLAG_* defines of include/proxsaga.h."""
    import re
    from pathlib import Path

    from paper_1707_06468_b200 import _lib

    text = (Path(__file__).resolve().parents[1] / "include" / "proxsaga.h").read_text()
    defs = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define PS_FLAG_(\w+)\s+(\d+)", text)}
    assert defs == {"SCRAMBLE": _lib.FLAG_SCRAMBLE, "GENERIC": _lib.FLAG_GENERIC, "DELTA_ZERO": _lib.FLAG_DELTA_ZERO,
                    "GROUP_WARP": _lib.FLAG_GROUP_WARP, "GROUP_LANE": _lib.FLAG_GROUP_LANE,
                    "MON_ENDS_IN_PLACE": _lib.FLAG_MON_ENDS_IN_PLACE, "ZERO_IMMEDIATE": _lib.FLAG_ZERO_IMMEDIATE,
                    "GROUP_STORE_ZEROS": _lib.FLAG_GROUP_STORE_ZEROS, "NO_CLUSTER": _lib.FLAG_NO_CLUSTER,
                    "FAST_V1": _lib.FLAG_FAST_V1, "MON_DEVICE_X": _lib.FLAG_MON_DEVICE_X,
                    "LOCAL_VIEW": _lib.FLAG_LOCAL_VIEW}
