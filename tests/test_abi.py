"""CPU checks of the boundary: libuvd.so builds for sm_100a, loads, and exports
every symbol include/uvd.h declares (no compute calls without a GPU)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "uvd.h")).read()
    return sorted(set(re.findall(r"UVD_API\s+[\w\s\*]*?\b(uvd_\w+)\s*\(", src)))


def test_header_declares_the_survey_boundary():
    syms = declared_symbols()
    for s in ("uvd_scene_create", "uvd_vantage_sample", "uvd_irradiance_matrix", "uvd_fluence",
              "uvd_coverage", "uvd_scene_destroy", "uvd_scene_query", "uvd_sync_status",
              "uvd_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2103_14137_b200 import uvd
    lib = uvd.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(uvd.EXPORTS) == set(declared_symbols())
    out = subprocess.run(["nm", "-D", "--defined-only", uvd.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(uvd_\w+)\b", out))
    assert exported == set(declared_symbols())
    assert uvd.version() >= 100


def test_library_is_sm100a():
    from paper_2103_14137_b200 import uvd
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", uvd.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2103_14137_b200 import uvd
    from synth import rooms
    with pytest.raises(RuntimeError):
        uvd.Scene(rooms.empty_room())


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2103_14137_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"(from|import)\s+oracle|liboracle|#include.*oracle|uvd_oracle", txt), f
