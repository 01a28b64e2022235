"""CPU checks of the C ABI: the library builds, loads, and exports every symbol
declared in include/curvopt_b200.h (no compute calls without a GPU)."""

import os
import re
import subprocess

from paper_2603_25976_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "curvopt_b200.h")).read()
    return sorted(set(re.findall(r"CV_API\s+[\w\s\*]+?\b(cv_\w+)\s*\(", src)))


def test_header_declares_api():
    names = _declared()
    assert "cv_linearize" in names and "cv_cg_solve" in names and len(names) >= 25


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (cv_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    for n in _declared():
        assert hasattr(lib, n)
    assert set(_lib.exported_symbols()) <= set(_declared())


def test_version_string():
    assert b"sm_100a" in _lib.lib().cv_version()
