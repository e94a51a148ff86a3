"""C-ABI surface checks that need no GPU: the library loads, exports every
symbol include/ofsc.h declares, and the binding's signature table matches."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ofsc.h")
LIB = os.path.join(ROOT, "paper_2305_10356_b200", "libofsc.so")


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ofsc_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(LIB):
        from paper_2305_10356_b200._build import build
        build()
    return LIB


def test_header_declares_the_boundary():
    names = declared()
    for must in ("ofsc_graph_build", "ofsc_run", "ofsc_row_normalize", "ofsc_kmeans",
                 "ofsc_graph_apply_gram", "ofsc_line_search", "ofsc_spectral_cluster"):
        assert must in names


def test_library_exports_every_declared_symbol(built):
    L = ctypes.CDLL(built)
    for name in declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(ofsc_[a-z_0-9]+)\b", out))
    assert set(declared()) <= exported


def test_binding_signature_table_matches_header(built):
    import paper_2305_10356_b200 as ofsc
    assert set(ofsc.SIGNATURES) == set(declared())
    L = ofsc.lib()
    assert L.ofsc_version().decode().startswith("ofsc")
    assert L.ofsc_status_string(2).decode() == "edge endpoint out of range"


def test_library_is_sm100a_only(built):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", built],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out


def test_product_path_does_not_touch_oracle():
    pkg = os.path.join(ROOT, "paper_2305_10356_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
