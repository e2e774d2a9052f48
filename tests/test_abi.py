"""CPU-side checks of the C ABI: the library loads and exports every symbol the
public header declares (no device calls)."""

import os
import re

from paper_2504_04104_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "treepipe_b200.h")) as fh:
        text = fh.read()
    return set(re.findall(r"^\s*(?:int|const char\*)\s+(tp_\w+)\(", text, re.M))


def test_library_exports_header_symbols():
    from paper_2504_04104_b200 import build

    build.build()
    cdll = _lib.load()
    declared = header_symbols()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(cdll, name), name
    assert declared == set(_lib.EXPORTED)


def test_error_codes_map_to_reference_exceptions():
    from paper_2504_04104_b200 import errors

    assert _lib._ERRORS[_lib.TP_ESHAPE] is errors.ShapeError
    assert _lib._ERRORS[_lib.TP_ECONTRACT] is errors.ContractViolation
    assert _lib._ERRORS[_lib.TP_ECONFIG] is errors.ConfigError
    assert issubclass(_lib._ERRORS[_lib.TP_ECUDA], errors.TreePipeError)
