"""The C-ABI library builds, loads without a GPU and exports every declared entry point."""
import os
import re

from paper_2410_09663_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "enks_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(enks_[a-z0-9_]+)\s*\(", src))


def test_header_declares_the_bound_entry_points():
    assert _declared() == set(_lib.EXPORTED)


def test_library_builds_and_exports_every_symbol():
    path = build.build()
    lib = _lib.load_library(check_device=False)
    assert path == _lib.LIB_PATH
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.enks_version() >= 1
    assert lib.enks_spd_max_p() >= 256
    assert lib.enks_cnn_max_width() >= 32


def test_sm100a_code_only():
    """The shared object carries sm_100a SASS (no PTX JIT for other archs)."""
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        import pytest

        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    assert all("sm_100a" in line for line in out.stdout.splitlines() if ".cubin" in line)


def test_no_cpu_fallback_without_gpu():
    """Without a CUDA device the product refuses to run (raises) instead of falling back."""
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2410_09663_b200.ops import DeviceOps

    with pytest.raises(_lib.NativeUnavailable):
        DeviceOps()
