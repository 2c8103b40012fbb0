"""The C-ABI library (no GPU needed): it loads, exports every symbol that
include/sbrc.h declares, agrees with the ctypes struct layouts, and rejects
bad parameters before touching the device."""

from __future__ import annotations

import ctypes as C
import os
import re

import pytest

from conftest import ROOT


def header_functions():
    text = open(os.path.join(ROOT, "include", "sbrc.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(sbrc_\w+)\s*\(", text, re.M)))


def test_library_exports_header():
    from paper_2008_06134_b200 import _native as N
    declared = header_functions()
    assert set(declared) == set(N.EXPORTS), declared
    for name in declared:
        assert hasattr(N.lib, name), name


def test_library_is_sm100a():
    from paper_2008_06134_b200 import _native as N
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump missing")
    out = subprocess.run([tool, "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_layouts():
    from paper_2008_06134_b200 import _native as N
    assert N.lib.sbrc_abi_version() == N.ABI_VERSION
    for i, st in enumerate((N.SbrcVolume, N.SbrcLightFrame, N.SbrcBuildParams, N.SbrcRenderParams)):
        assert N.lib.sbrc_struct_size(i) == C.sizeof(st)
    assert N.lib.sbrc_struct_size(99) == -1
    assert N.lib.sbrc_strerror(0) == b"ok"


def test_validation_before_launch():
    """Invalid params return EINVAL/ECONFIG without any CUDA call (works on CPU)."""
    from paper_2008_06134_b200 import _native as N
    p = N.SbrcBuildParams()
    assert N.lib.sbrc_build(C.byref(p), None) == N.EINVAL
    assert N.lib.sbrc_build(None, None) == N.EINVAL
    r = N.SbrcRenderParams()
    assert N.lib.sbrc_render(C.byref(r), None) == N.EINVAL
    # a buffer mode with no intensity is a ConfigError (raycaster.py:450-451)
    r.volume.data = 1
    r.volume.nx = r.volume.ny = r.volume.nz = 4
    r.volume.box_ext[:] = [1.0, 1.0, 1.0]
    r.width = r.height = 8
    r.step, r.et_alpha = 1 / 64, 0.99
    r.lut_rgba, r.image = 1, 1
    r.shading, r.band_rows, r.world = N.SHADE["cone"], 8, 1
    assert N.lib.sbrc_render(C.byref(r), None) == N.ECONFIG
    r.shading = 7
    assert N.lib.sbrc_render(C.byref(r), None) == N.EUNSUPPORTED
    with pytest.raises(N.ConfigError):
        N.check(N.ECONFIG, "x")
    with pytest.raises(ValueError):
        N.check(N.EINVAL, "x")
    with pytest.raises(RuntimeError):
        N.check(N.ECUDA, "x")


def test_local_rows():
    from paper_2008_06134_b200 import _native as N
    from paper_2008_06134_b200.frame import band_layout
    for h in (1, 7, 8, 30, 1024, 1031):
        for world in (1, 2, 3, 8):
            for br in (8, 16):
                per_rank, _ = band_layout(h, br, world)
                rows = [N.local_rows(h, br, r, world) for r in range(world)]
                assert max(rows) == per_rank
                assert sum(rows) >= h and sum(rows) - h < br * world


def test_integration_doc_matches_header():
    """INTEGRATION.md's binding snippet quotes the current ABI version and
    names every exported entry point (the docs must not drift from the header)."""
    text = open(os.path.join(ROOT, "include", "sbrc.h")).read()
    version = int(re.search(r"#define SBRC_ABI_VERSION (\d+)", text).group(1))
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    quoted = [int(v) for v in re.findall(r"sbrc_abi_version\(\) == (\d+)", doc)]
    assert quoted and all(v == version for v in quoted), (quoted, version)
    for name in header_functions():
        assert name in doc, f"{name} is not documented in INTEGRATION.md"
