"""Every execution mode under the checked build (libfed_checked.so: device-side
bounds checks of every plan-driven index and colour-phase write-conflict checks,
fed_kernels.cuh FED_DCHECK) -- the stand-in for compute-sanitizer, which is not
available on this pool.  Each case runs in its own process with FED_LIB pointing
at the checked library and must finish with no check fired."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def checked_lib():
    from paper_1909_03355_b200.build import build
    return build(checked=True)


@pytest.mark.parametrize("case", ["stream", "stream64", "resident", "peer", "nccl", "tables", "tet", "atomic"])
def test_checked_build_case(checked_lib, case):
    env = dict(os.environ, FED_LIB=checked_lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_cases.py"), "--case", case],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert f"case {case}: ok" in out.stdout
