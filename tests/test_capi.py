"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/lapbel_b200.h declares (no compute calls)."""

import os
import re

import pytest

from conftest import ROOT


def _declared():
    txt = open(os.path.join(ROOT, "include", "lapbel_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lb_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_header_symbols():
    from paper_2111_10743_b200 import _build, _lib
    _build.build(verbose=False)
    lib = _lib.load()
    declared = _declared()
    assert declared, "no symbols parsed from the header"
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.exported_symbols())
    assert lib.lb_abi_version() == 1


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a device")
    import paper_2111_10743_b200 as b
    import numpy as np
    with pytest.raises(RuntimeError):
        b.evaluate_direct(b.FmmSources(np.zeros((2, 3)), np.ones((1, 2))),
                          np.ones((1, 3)))
