"""The C-ABI library loads (no GPU needed) and exports exactly the symbols
include/ials_b200.h declares; pure host-side entry points answer."""

import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "ials_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ials_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2110_14044_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2110_14044_b200 import build
        build.build()
    return _lib.load()


def test_header_and_binding_agree():
    from paper_2110_14044_b200 import _lib
    assert declared_functions() == sorted(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol(lib):
    from paper_2110_14044_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ials_[a-z0-9_]+)\b", out))
    missing = set(declared_functions()) - exported
    assert not missing, missing
    for name in declared_functions():
        assert getattr(lib, name) is not None


def test_host_only_entry_points(lib):
    assert lib.ials_version() == 1
    assert lib.ials_heavy_threshold(128) >= lib.ials_slice_len(128) > 0
    assert lib.ials_heavy_threshold(8) >= lib.ials_slice_len(8) > 0
    assert lib.ials_workspace_bytes(1000, 500, 64, 32, 10, 2) > 0
    assert lib.ials_loss_workspace_bytes(64) >= 2 * 64 * 64 * 4


def test_library_is_sm100a():
    from paper_2110_14044_b200 import _lib
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_header_compiles_as_c_and_cpp(tmp_path):
    """include/ials_b200.h is a plain C header: it compiles warning-free as
    C99 and C++17 (the binding a C / cgo / JNI consumer would include)."""
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "hdr.c"
    src.write_text('#include "ials_b200.h"\nint main(void) { return 0; }\n')
    for cc, flags in (("gcc", ["-std=c99"]), ("g++", ["-std=c++17", "-x", "c++"])):
        if shutil.which(cc) is None:
            pytest.skip(f"{cc} not available")
        r = subprocess.run([cc, *flags, "-Wall", "-Wextra", "-Werror", "-fsyntax-only",
                            "-I", os.path.join(root, "include"), str(src)],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
