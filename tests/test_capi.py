"""The C-ABI library loads and exports every symbol include/bhcp_b200.h declares
(no compute calls: CPU only)."""

import re

from paper_2107_06381_b200 import _lib


def declared_symbols():
    text = _lib.HEADER_PATH.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bhcp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for name in ("bhcp_pint_solve", "bhcp_step_b", "bhcp_to_eigenspace", "bhcp_from_eigenspace",
                 "bhcp_sine_transform", "bhcp_pint_modes", "bhcp_pint_levels"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_python_signatures_cover_header():
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_version_and_status_size_without_gpu():
    lib = _lib.load_library()
    assert lib.bhcp_version() >= 100
    assert lib.bhcp_status_bytes() == 64
