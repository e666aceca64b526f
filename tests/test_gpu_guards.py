"""Out-of-bounds write sweep over the kernel variants (stands in for
compute-sanitizer, which this GPU pool does not allow): tests/guard_run.py in a
fresh process with SNN_GUARD=1 (4 KB guard pattern past every device buffer)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_no_out_of_bounds_writes():
    env = dict(os.environ, SNN_GUARD="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "guard_run.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "GUARDS OK" in r.stdout
