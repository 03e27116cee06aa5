"""The checked build (libhsewald_b200_checked.so, -DHS_CHECKED): every production kernel's ring,
queue and staging indices and its global stores bounds-checked on the device.  A small run of
every kernel (tools/sanitize_case.py: all kinds, the mixed plan, the 2-way slab pipeline, the
register x / y stages, the DMMA spread and the cp.async gather) must report zero failed checks.
This stands in for compute-sanitizer, which is closed on the GPU pool."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_checked_build_reports_no_failures(gpu):
    lib = os.path.join(ROOT, "paper_1802_07844_b200", "libhsewald_b200_checked.so")
    assert os.path.exists(lib), "build it: make -C paper_1802_07844_b200/csrc checked"
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py"), "3000"], cwd=ROOT,
                         env=dict(os.environ, HSEWALD_CHECKED="1"), capture_output=True, text=True, timeout=900)
    print(out.stdout[-2000:])
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert "'failures': 0" in out.stdout


def test_production_library_is_not_checked():
    """hs_debug_checks exists in the production library and refuses (HS_ERR_CONFIG)."""
    from paper_1802_07844_b200 import _lib
    from paper_1802_07844_b200.errors import ConfigError
    if os.environ.get("HSEWALD_CHECKED") == "1":
        pytest.skip("checked build selected")
    with pytest.raises(ConfigError):
        _lib.debug_checks()
