"""CPU: the C-ABI library builds, loads without a GPU, and exports every symbol the public
header declares; the ctypes mirrors match the header's struct sizes."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2603_07865_b200 as pkg
from paper_2603_07865_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "semwarm_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(sw(?:cm|b|r)?_[a-z_0-9]+)\s*\(", src))
    return sorted(n for n in names if not n.endswith("_fn"))  # drop the callback typedef


def test_library_exports_every_header_symbol():
    L = pkg.lib()
    declared = header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(_lib.EXPORTED) == declared


def test_struct_layouts():
    assert C.sizeof(_lib.SwConfig) == 56
    assert C.sizeof(_lib.SwSelectorConfig) == 24
    assert C.sizeof(_lib.SwPolicy) == 24
    assert _lib.CHOICE_DTYPE.itemsize == 88 and _lib.HIT_DTYPE.itemsize == 40


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_07865_b200.warmstart import WarmStartCache
    with pytest.raises(Exception):
        WarmStartCache(64)
    assert pkg.lib().sw_version() == 1


def test_sass_contains_tcgen05_and_tma():
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    sass = subprocess.run(["cuobjdump", "-sass", pkg.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


def test_swem_reader_matches_reference_writer(ref, tmp_path):
    """SWEM (core.cpp:183-220) written by the reference, read by the C-ABI (host-only call)."""
    from paper_2603_07865_b200.warmstart import read_swem
    v = np.random.default_rng(0).standard_normal((37, 24)).astype(np.float32)
    p = str(tmp_path / "e.swem")
    ref.save_embeddings(p, v)
    np.testing.assert_array_equal(read_swem(p), v)
