"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/hedl.h declares.

No compute calls: this runs on the CPU-only host (the GPU tests call through the same ABI).
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hedl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//.*", "", src)
    return sorted(set(re.findall(r"\b(hedl_[a-z_0-9]+)\s*\(", src)))


def test_build_and_load():
    import __graft_entry__ as ge
    ge.build()
    import paper_2412_00802_b200 as hedl
    L = hedl.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert set(_declared()) == set(hedl.ABI_SYMBOLS)
    assert "sm_100a" in hedl.version()


def test_exported_dynamic_symbols():
    so = os.path.join(ROOT, "paper_2412_00802_b200", "libhedl.so")
    out = subprocess.check_output(["nm", "-D", "--defined-only", so], text=True)
    exported = set(re.findall(r"\bT (hedl_[a-z_0-9]+)\b", out))
    assert set(_declared()) <= exported


def test_sass_is_sm100a():
    so = os.path.join(ROOT, "paper_2412_00802_b200", "libhedl.so")
    out = subprocess.check_output(["cuobjdump", "--list-elf", so], text=True)
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    """Without a CUDA device the library refuses (UNSUPPORTED) instead of falling back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2412_00802_b200 as hedl
    from synth import abox
    with pytest.raises(hedl.HedlError) as e:
        hedl.hedl_kb_load(abox.c1_kb(), 0)
    assert e.value.code == 8


def test_product_does_not_import_oracle():
    """The product path (package sources) never refers to oracle/ (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2412_00802_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                code = re.sub(r'""".*?"""', "", txt, flags=re.S)
                code = re.sub(r"#.*|//.*", "", code)
                assert "oracle" not in code, f
