"""The C-ABI library builds for sm_100a, loads, and exports every symbol the
public header declares (no compute calls: this runs without a GPU)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "purine_b200.h"


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(bf_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1412_6249_b200 import _build

    return _build.build()


def test_header_declares_the_hot_path():
    names = _declared()
    for must in ("bf_conv2d_fwd", "bf_conv2d_bwd_data", "bf_conv2d_bwd_weight", "bf_maxpool_fwd",
                 "bf_lrn_fwd", "bf_concat_fwd", "bf_softmax_xent", "bf_sgd_momentum",
                 "bf_nccl_reduce_scatter", "bf_aggregate", "bf_copy"):
        assert must in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(str(libpath))
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(libpath)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_python_binding_covers_header():
    from paper_1412_6249_b200 import _native

    assert set(_declared()) <= set(_native._SIGS)


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_1412_6249_b200"
    for py in pkg.rglob("*.py"):
        src = py.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), py
