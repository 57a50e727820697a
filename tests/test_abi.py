"""The C-ABI library loads and exports every symbol include/ctri.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

import paper_2101_02286_b200 as pk
from paper_2101_02286_b200 import ctri

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "ctri.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ctri_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_what_binding_lists():
    assert declared_functions() == sorted(ctri.ABI_SYMBOLS)


def test_library_exports_every_symbol():
    lib = ctri.load()
    raw = ctypes.CDLL(ctri.LIB_PATH)
    for name in declared_functions():
        assert hasattr(raw, name), name
    assert lib.ctri_abi_version() == ctri.ABI_VERSION


def test_status_strings():
    lib = ctri.load()
    for code, name in ctri.STATUS.items():
        assert lib.ctri_status_string(code).decode() == name
    assert lib.ctri_status_string(99).decode() == "CTRI_ERR_UNKNOWN"


def test_host_query_errors():
    with pytest.raises(pk.CtriError) as e:
        pk.ctri_factor_query(2)
    assert e.value.name == "CTRI_ERR_PARTITION_TOO_SMALL"
    with pytest.raises(pk.CtriError) as e:
        pk.ctri_pcr_coefficients([1 / 3] * 3, [1] * 3, [1 / 3] * 3, cyclic=True)
    assert e.value.name == "CTRI_ERR_UNSUPPORTED"


def test_singular_guard():
    # bands (1, 0, 1): first pivot is 0 -> SINGULAR (SPEC S:85 guard)
    with pytest.raises(pk.CtriError) as e:
        pk.ctri_factor_query(16, bands=(1.0, 0.0, 1.0))
    assert e.value.name == "CTRI_ERR_SINGULAR"


def test_no_product_import_of_oracle():
    """The product package never imports oracle/ (test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_2101_02286_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "ctri_oracle" not in txt, f


def test_binding_rejects_host_and_wrong_size_buffers():
    """The Plan wrappers check device placement and slab size before any pointer crosses the
    ABI (a CPU tensor or a short buffer would otherwise fault inside a kernel)."""
    import numpy as np
    import pytest
    import torch

    from paper_2101_02286_b200 import ctri
    with pytest.raises(ValueError, match="CUDA tensor"):
        ctri._dev(torch.zeros(8, dtype=torch.float64), 8, "b")
    with pytest.raises(ValueError, match="CUDA tensor"):
        ctri._dev(np.zeros(8), 8, "b")
    with pytest.raises(ValueError, match="elements"):
        ctri._host(np.zeros(7), 8, "b_host")
    assert ctri._dev(1234, 8, "b") == 1234  # raw addresses pass through (the C ABI checks them)
